timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "halo or c5 or topk or top5" 2>&1 | tail -4
timeout 600 python bench.py --config c5 --steps 5 > gpurun_out/r2_bench_c5.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/r2_bench_c5.log
