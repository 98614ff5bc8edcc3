set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_topk_fused.py tests/test_campaign.py -x -q 2>&1 | tail -25 > gpurun_out/r2_pytest_b.log
tail -25 gpurun_out/r2_pytest_b.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c3_c.log 2>&1; echo rc=$?
tail -c 1200 gpurun_out/r2_bench_c3_c.log
