python -m pytest tests/test_gpu_bubbletea.py -m gpu -q -x -k saturating > gpurun_out/r5_pytest.log 2>&1; tail -3 gpurun_out/r5_pytest.log
GPB_PACK_STATS=1 python tools/pack_variance.py > gpurun_out/r5_packvar.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:atlas_seq --launch-count 3 -o /tmp/r5_seq -f python tools/run_eval.py config5 1 > gpurun_out/r5_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r5_seq.ncu-rep > gpurun_out/r5_seq_ncu_summary.csv 2>&1
ncu -i /tmp/r5_seq.ncu-rep --page raw --csv > /tmp/raw.csv 2>&1; gzip -c /tmp/raw.csv > gpurun_out/r5_seq_raw.csv.gz
ncu -i /tmp/r5_seq.ncu-rep --page source --csv --print-source sass > /tmp/src.csv 2>&1; gzip -c /tmp/src.csv > gpurun_out/r5_seq_src.csv.gz
ls -la gpurun_out
