# full-size configs 1, 3, 4 (time-to-solution on one GPU)
mkdir -p gpurun_out
O=gpurun_out/configs.jsonl
: > $O
timeout 300 python tools/probe_configs.py cfg1 >> $O 2> gpurun_out/configs.err
timeout 600 python tools/probe_configs.py cfg3 >> $O 2>> gpurun_out/configs.err
timeout 900 python tools/probe_configs.py cfg4-delayed 50 merge >> $O 2>> gpurun_out/configs.err
