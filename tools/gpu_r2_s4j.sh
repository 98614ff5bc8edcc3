set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -p no:cacheprovider -k "direct" 2>&1 | tail -6
for c in c2 c4 c3; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4_bench_$c.log 2>&1; echo rc=$?
python - $c <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads([l for l in open(f'gpurun_out/s4_bench_{c}.log') if l.startswith('{')][0])
    print(c, d['ms_per_step'], json.dumps(d.get('statistics'))[:1500])
    if d.get('direct'): print(json.dumps(d['direct'].get('fast_1xfp16')), d['direct']['kernel_ms'])
except Exception as e:
    print('ERR', e); print(open(f'gpurun_out/s4_bench_{c}.log').read()[-1500:])
PY
done
