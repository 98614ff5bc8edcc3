for m in 0 1; do echo "== GH_MAP_BLOCKED=$m"; GH_MAP_BLOCKED=$m timeout 300 python tools/time_topk.py --trials 2048; done
GH_MAP_BLOCKED=1 timeout 600 python -m pytest tests/test_topk_fused.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3
