mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_topk_fused.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python tools/time_topk.py --trials 2048
GH_LIB_PATH=paper_2307_16550_b200/build/libgridhop_b200_prof.so timeout 300 python tools/topk_prof.py
timeout 600 python -m pytest tests/test_gpu_parity.py -k "topk or top5 or fused or ties" -x -q -p no:cacheprovider 2>&1 | tail -3
