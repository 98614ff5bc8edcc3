timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "c4 or hop_map_and_argmax or pipelined or polar or table" 2>&1 | tail -4
timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 > gpurun_out/r2_bench_c4b.log 2>&1; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/r2_bench_c4b.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels_ms'], d['roofline']['frac'], d['e2e']['ms_per_step'])"
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/r2_bench_c3b.log 2>&1; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/r2_bench_c3b.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels_ms'], d['e2e']['ms_per_step'], d['e2e']['h2d_bound_ms'])"
