python -m pytest tests/test_gpu_config5.py tests/test_gpu_session.py tests/test_gpu_group.py -m gpu -q -x > gpurun_out/r3_pytest.log 2>&1; tail -15 gpurun_out/r3_pytest.log
python tools/buckets.py config5 2 > gpurun_out/r3_buckets5.txt 2>&1
GPB_ATLAS_SEQ=0 python tools/buckets.py config5 2 > gpurun_out/r3_buckets5_noseq.txt 2>&1
python tools/buckets.py config3 3 > gpurun_out/r3_buckets3.txt 2>&1
python tools/pack_bench.py config3 1000 1000000 1 > gpurun_out/r3_pack.txt 2>&1
