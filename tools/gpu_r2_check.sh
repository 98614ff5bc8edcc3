set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g | head -2; nproc
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_pytest1.log
tail -5 gpurun_out/r2_pytest1.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c3_a.log 2>&1; echo rc=$?
tail -c 3000 gpurun_out/r2_bench_c3_a.log
