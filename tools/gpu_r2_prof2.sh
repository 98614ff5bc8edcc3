set -x
mkdir -p gpurun_out
python tools/time_topk.py --trials 2048 > gpurun_out/time_topk.log 2>&1; cat gpurun_out/time_topk.log
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_gather_topk" -c 1 \
  -o gpurun_out/prof_topk python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > gpurun_out/ncu_topk.log 2>&1
tail -3 gpurun_out/ncu_topk.log
ls -la gpurun_out/*.ncu-rep
