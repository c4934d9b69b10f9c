mkdir -p gpurun_out
( time timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/bench_driver.log 2> gpurun_out/bench_driver.err; echo "bench rc=$?" >> gpurun_out/bench_driver.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 9000 --launch-count 6000 --csv --log-file gpurun_out/launches_bench_r02h.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-phi --no-seq --no-cfg2 --no-cfg3 --no-natural > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench rc=$?" >> gpurun_out/ncu_bench.log
