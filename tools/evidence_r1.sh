set -x
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref_r1.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --direct-steps 1 > gpurun_out/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --direct-steps 1 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_step.py --steps 2 > gpurun_out/plain1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_fft|k_gather" -s 2 -c 2 -o gpurun_out/prof_hop_r1 python tools/prof_step.py --steps 2 > gpurun_out/ncu1.log 2>&1
python tools/prof_step.py --path direct --trials 1024 --steps 1 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_direct_umma" -c 1 -o gpurun_out/prof_direct_r1 python tools/prof_step.py --path direct --trials 1024 --steps 1 > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
