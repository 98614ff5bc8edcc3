# ncu capture of the fused top-K gather (c3, 2048 trials) plus the c3 argmax
# gather for comparison; reports come back in gpurun_out/
set -x
mkdir -p gpurun_out
python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > gpurun_out/plain_topk.log 2>&1 && \
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_gather_topk" -c 1 \
  -o gpurun_out/prof_topk python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > gpurun_out/ncu_topk.log 2>&1
python tools/prof_step.py --config c3 --path campaign --trials 2048 --steps 1 > gpurun_out/plain_c3arg.log 2>&1 && \
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_gather" -c 1 \
  -o gpurun_out/prof_c3arg python tools/prof_step.py --config c3 --path campaign --trials 2048 --steps 1 > gpurun_out/ncu_c3arg.log 2>&1
ls -la gpurun_out/*.ncu-rep
