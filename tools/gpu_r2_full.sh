set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/r2_pytest_full.log
tail -40 gpurun_out/r2_pytest_full.log
timeout 900 python bench.py > gpurun_out/r2_bench_default.log 2>&1; echo rc=$?
tail -c 4000 gpurun_out/r2_bench_default.log
