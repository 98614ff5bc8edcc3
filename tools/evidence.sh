# Evidence run for profiles/ (run on the GPU box via gpurun from the repo root):
#   bash tools/evidence.sh r1
# Each ncu capture runs only after the same command exited 0 without ncu.
# Full reports stay in /tmp/ev (they are ~16 MB per kernel); the summaries
# (tools/ncu_summary.py) and the raw/source CSVs come back in gpurun_out/.
set -x
R=${1:-r1}
O=gpurun_out
E=/tmp/ev
rm -rf $E; mkdir -p $E $O
nproc > $O/host_cores.txt; lscpu | grep "Model name" >> $O/host_cores.txt
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_$R.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref_$R.log 2>&1
for c in c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_${c}_$R.log 2>&1
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --direct-steps 1 > $O/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --direct-steps 1 > $O/ncu_launch.log 2>&1
python tools/prof_step.py --steps 2 > $O/plain1.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_fft|k_gather" -s 2 -c 2 \
  -o $E/prof_hop_$R python tools/prof_step.py --steps 2 > $O/ncu1.log 2>&1
python tools/prof_step.py --path direct --trials 1024 --steps 1 > $O/plain2.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_direct_umma" -c 1 \
  -o $E/prof_direct_$R python tools/prof_step.py --path direct --trials 1024 --steps 1 > $O/ncu2.log 2>&1
python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > $O/plain3.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_gather|k_fft|k_topk" -c 3 \
  -o $E/prof_c3_$R python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > $O/ncu3.log 2>&1
python tools/prof_step.py --config c5 --trials 64 --steps 1 > $O/plain5.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_gather" -c 1 \
  -o $E/prof_c5_$R python tools/prof_step.py --config c5 --trials 64 --steps 1 > $O/ncu5.log 2>&1
python tools/ncu_summary.py $E/*.ncu-rep --launches $O/launches_$R.csv --out $O/kernels_$R.json > /dev/null
for f in $E/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page source --csv > $O/${b}_src.csv 2>/dev/null
done
ls -la $O
