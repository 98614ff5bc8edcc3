set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_topk_fused.py tests/test_gpu_parity.py -k "topk or top5 or fused or ties" -x -q 2>&1 | tail -15 > gpurun_out/r2_pytest_topk.log
tail -8 gpurun_out/r2_pytest_topk.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c3_b.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/r2_bench_c3_b.log
