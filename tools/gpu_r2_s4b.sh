set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "ties or c1_scene or hop_map or edge or host_buffers or campaign" 2>&1 | tail -8
timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/s4_bench_c2.log 2>&1; echo rc=$?
tail -c 1800 gpurun_out/s4_bench_c2.log
