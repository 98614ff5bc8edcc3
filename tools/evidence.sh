# Evidence run for profiles/ (run on the GPU box via gpurun from the repo root):
#   bash tools/evidence.sh r1
# Each ncu capture runs only after the same command exited 0 without ncu.
set -x
R=${1:-r1}
O=gpurun_out
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
  ncu --set full --clock-control none --import-source on -k regex:"k_fft|k_gather" -s 2 -c 2 \
  -o $O/prof_hop_$R python tools/prof_step.py --steps 2 > $O/ncu1.log 2>&1
python tools/prof_step.py --path direct --trials 1024 --steps 1 > $O/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_direct_umma" -c 1 \
  -o $O/prof_direct_$R python tools/prof_step.py --path direct --trials 1024 --steps 1 > $O/ncu2.log 2>&1
ls -la $O
