mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench_c3.log 2>&1; echo rc=$?
tail -c 3500 gpurun_out/r2_bench_c3.log
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2_bench_c4.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/r2_bench_c4.log
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2_bench_c2.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/r2_bench_c2.log
