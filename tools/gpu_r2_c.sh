set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_topk_fused.py tests/test_campaign.py -x -q 2>&1 | tail -25 > gpurun_out/r2_pytest_c.log
tail -25 gpurun_out/r2_pytest_c.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c3_d.log 2>&1; echo rc=$?
tail -c 600 gpurun_out/r2_bench_c3_d.log
python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > gpurun_out/plain_topk.log 2>&1 && \
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_gather_topk" -c 1 \
  -o /tmp/prof_topk python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > gpurun_out/ncu_topk.log 2>&1
ncu -i /tmp/prof_topk.ncu-rep --page raw --csv > gpurun_out/prof_topk_raw.csv 2>/dev/null
ncu -i /tmp/prof_topk.ncu-rep --page source --csv > gpurun_out/prof_topk_src.csv 2>/dev/null
ncu -i /tmp/prof_topk.ncu-rep --page details --csv > gpurun_out/prof_topk_details.csv 2>/dev/null
ls -la gpurun_out | tail -5
