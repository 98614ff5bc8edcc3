# Round-2 evidence run for profiles/ (gpurun, repo root): bash tools/evidence_r2.sh
# Each ncu capture runs only after the same command exited 0 without ncu.
set -x
R=r2
O=gpurun_out
E=/tmp/ev
rm -rf $E; mkdir -p $E $O
nproc > $O/host_cores.txt; lscpu | grep "Model name" >> $O/host_cores.txt
timeout 900 python bench.py > $O/bench_$R.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_ref_$R.log 2>&1
for c in c2 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_${c}_$R.log 2>&1
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_bench.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/prof_step.py --config c3 --path map --trials 2048 --steps 1 > $O/plain3.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_gather|k_fft|k_topk" -c 3 \
  -o $E/prof_c3_$R python tools/prof_step.py --config c3 --path map --trials 2048 --steps 1 > $O/ncu3.log 2>&1
python tools/time_topk.py --trials 9472 --steps 1 --warm 1 --engines pick,fused,map > $O/plain3p.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_gather_pick" -c 1 \
  -o $E/prof_c3pick_$R python tools/time_topk.py --trials 9472 --steps 1 --warm 0 --engines pick > $O/ncu3p.log 2>&1
python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > $O/plain3f.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_gather_topk" -c 1 \
  -o $E/prof_c3fused_$R python tools/prof_step.py --config c3 --path topk --trials 2048 --steps 1 > $O/ncu3f.log 2>&1
python tools/prof_step.py --config c4 --trials 2000 --steps 1 > $O/plain4.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_gather" -c 1 \
  -o $E/prof_c4_$R python tools/prof_step.py --config c4 --trials 2000 --steps 1 > $O/ncu4.log 2>&1
python tools/prof_step.py --config c5 --trials 64 --steps 1 > $O/plain5.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_gather" -c 1 \
  -o $E/prof_c5_$R python tools/prof_step.py --config c5 --trials 64 --steps 1 > $O/ncu5.log 2>&1
python tools/prof_step.py --steps 2 > $O/plain2.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"k_fft|k_gather" -s 2 -c 2 \
  -o $E/prof_hop_$R python tools/prof_step.py --steps 2 > $O/ncu2.log 2>&1
python tools/ncu_summary.py $E/*.ncu-rep --launches $O/launches_$R.csv --out $O/kernels_$R.json > /dev/null
for f in $E/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page source --csv --print-source sass > $E/${b}_sass.csv 2>/dev/null
  python tools/ncu_stalls.py $E/${b}_sass.csv --top 12 >> $O/stall_top_$R.txt 2>&1
done
ls -la $O
