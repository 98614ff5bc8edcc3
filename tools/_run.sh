timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pt.log 2>&1; echo pytest=$? >> gpurun_out/pt.log
for c in c4; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/wm_$c.log 2>&1; done
python tools/prof_step.py --config c4 --trials 2048 --steps 1 > gpurun_out/plain.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"k_gather" -c 1 -o /tmp/prof_c4 python tools/prof_step.py --config c4 --trials 2048 --steps 1 > gpurun_out/ncu.log 2>&1
ncu -i /tmp/prof_c4.ncu-rep --page raw --csv > gpurun_out/c4_raw.csv; ncu -i /tmp/prof_c4.ncu-rep --page source --csv > gpurun_out/c4_src.csv
