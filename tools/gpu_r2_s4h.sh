set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "ties or c1_scene or hop_map or edge or host_buffers or campaign or pipelined or spectra or c3 or topk" 2>&1 | tail -6
timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/s4_bench_c2.log 2>&1; echo rc=$?
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/s4_bench_c2.log') if l.startswith('{')][0])
print(d['ms_per_step'], d['kernels_ms'], d['roofline']['frac'])
PY
timeout 1200 python -m pytest tests/test_topk_fused.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/time_topk.py --trials 9472 --steps 2 --engines pick,map 2>&1 | tail -5
