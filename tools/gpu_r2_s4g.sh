set -x
mkdir -p gpurun_out
E=/tmp/ev; mkdir -p $E
python tools/prof_step.py --steps 2 > gpurun_out/plain2.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_gather" -s 1 -c 1 \
  -o $E/prof_hop_x python tools/prof_step.py --steps 2 > gpurun_out/ncu2.log 2>&1
python tools/ncu_summary.py $E/prof_hop_x.ncu-rep --out gpurun_out/kernels_hop_x.json > /dev/null
ncu -i $E/prof_hop_x.ncu-rep --page source --csv --print-source sass > $E/hop_sass.csv 2>/dev/null
python tools/ncu_stalls.py $E/hop_sass.csv --top 25 > gpurun_out/stall_hop_x.txt 2>&1
cat gpurun_out/kernels_hop_x.json
head -30 gpurun_out/stall_hop_x.txt
