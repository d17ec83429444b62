timeout 300 python -m pytest tests/test_gpu_train_head.py -q -x 2>&1 | tail -2
timeout 120 python tools/time_train_head.py 4096 2048 50304 20
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_train_head.csv python tools/time_train_head.py 4096 2048 50304 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_train_head.csv 2>&1 | head -5
