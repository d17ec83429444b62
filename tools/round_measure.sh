#!/bin/bash
# One GPU call: smoke, tests, default bench (+reference arm), bf16 parity
# report, pass-vs-context, decode-layer timeline, ncu launch lists and
# full-set captures of the dominant kernels, training step + census.
# Outputs in gpurun_out/ (the summaries are copied to profiles/).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
timeout 900 python tools/bf16_parity_report.py > gpurun_out/bf16_parity.txt 2>&1
CTXS=64,192,320,1024,2000 timeout 300 python tools/pass_vs_ctx.py > gpurun_out/pass_vs_ctx.txt 2>&1
CTXS=192,2000 ROWS=1,5 timeout 600 python tools/attn_timeline.py > gpurun_out/attn_timeline.txt 2>&1
timeout 300 python tools/time_attn_train.py > gpurun_out/attn_train_time.txt 2>&1
timeout 600 python tools/time_train_step.py 4 4 > gpurun_out/ts.txt 2>&1
timeout 600 python tools/prof_train_step.py 4 4 > gpurun_out/census.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_decode.csv python tools/prof_decode.py 2 1 192 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_train_head.csv python tools/time_train_head.py 4096 2048 50304 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_slab128 -s 130 -c 1 -o gpurun_out/slab_ctx192_full python tools/prof_decode.py 3 1 191 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_slab128 -s 130 -c 1 -o gpurun_out/slab_ctx2000_full python tools/prof_decode.py 3 1 1999 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemv_tma -s 40 -c 4 -o gpurun_out/gemv_tma_full python tools/prof_decode.py 1 1 192 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm2 -s 3 -c 3 -o gpurun_out/tc_gemm2_full python tools/time_train_head.py 4096 2048 50304 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_attn_fwd|k_attn_bwd_kv|k_attn_bwd_q" -s 6 -c 3 -o gpurun_out/attn_train_full python tools/time_attn_train.py > /dev/null 2>&1
ls -la gpurun_out
