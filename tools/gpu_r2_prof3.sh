set -x
mkdir -p gpurun_out
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_gather_topk" -c 1 \
  -o /tmp/prof_topk python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > gpurun_out/ncu_topk.log 2>&1
ncu -i /tmp/prof_topk.ncu-rep --page raw --csv > gpurun_out/prof_topk_raw.csv 2>/dev/null
ncu -i /tmp/prof_topk.ncu-rep --page details --csv > gpurun_out/prof_topk_details.csv 2>/dev/null
ncu -i /tmp/prof_topk.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_topk_sass.csv 2>/dev/null
ncu -i /tmp/prof_topk.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_topk_src.csv 2>/dev/null
ls -la gpurun_out/
