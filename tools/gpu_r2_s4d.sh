set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_topk_fused.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python tools/time_topk.py --trials 9472 --steps 2 --engines pick,map 2>&1 | tail -5
