# round-2 ncu evidence: full capture of the dominant chain kernel (config 4,
# level 0, 4,096 columns) + launch list of one bench solve (dev)
mkdir -p gpurun_out
timeout 900 python tools/probe_band.py cfg4 0:4096 > gpurun_out/probe_band_cfg4.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_band_rb --launch-count 2 -f -o gpurun_out/r02b_rb_cfg4 python tools/probe_band.py cfg4 0:4096 > gpurun_out/ncu_rb.log 2>&1
echo "ncu rb rc=$?" >> gpurun_out/ncu_rb.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 29500 --launch-count 10500 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-phi --no-seq --no-cfg2 > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench rc=$?" >> gpurun_out/ncu_bench.log
