set -x
python tools/long_context.py > gpurun_out/long_context.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attn_rows128 -s 40 -c 2 -o gpurun_out/attn_full python tools/prof_decode.py 1 5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:EpiGelu -c 2 -o gpurun_out/mlp_full python tools/time_train_step.py > /dev/null 2>&1
ls -la gpurun_out
