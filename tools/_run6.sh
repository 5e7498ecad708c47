python -m pytest tests/test_gpu_rows.py tests/test_gpu_bubbletea.py tests/test_gpu_config5.py tests/test_gpu_session.py -m gpu -q -x > gpurun_out/r6_pytest.log 2>&1; tail -15 gpurun_out/r6_pytest.log
python tools/buckets.py config5 2 > gpurun_out/r6_buckets5.txt 2>&1
python tools/buckets.py config3 3 > gpurun_out/r6_buckets3.txt 2>&1
python tools/pack_variance.py > gpurun_out/r6_packvar.txt 2>&1
