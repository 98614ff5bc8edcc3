timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pipelined or c5" 2>&1 | tail -3
timeout 600 python bench.py --config c5 --steps 5 > gpurun_out/r2_bench_c5.log 2>&1; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/r2_bench_c5.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels_ms'], d['roofline']['frac'])"
