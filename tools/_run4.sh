python -m pytest tests/test_gpu_config5.py -m gpu -q -x > gpurun_out/r4_pytest.log 2>&1; tail -3 gpurun_out/r4_pytest.log
python tools/buckets.py config5 2 > gpurun_out/r4_buckets5.txt 2>&1
python tools/buckets.py config3 3 > gpurun_out/r4_buckets3.txt 2>&1
python tools/profile_rows.py config5 30 > gpurun_out/r4_profile_rows5.txt 2>&1
GPB_PACK_STATS=1 python tools/pack_variance.py > gpurun_out/r4_packvar.txt 2>&1
