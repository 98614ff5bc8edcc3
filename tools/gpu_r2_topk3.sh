set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_topk_fused.py tests/test_gpu_parity.py -k "topk or top5 or fused or ties" -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2_pytest_topk.log
cat gpurun_out/r2_pytest_topk.log
timeout 300 python tools/time_topk.py --trials 2048 > gpurun_out/time_topk.log 2>&1; cat gpurun_out/time_topk.log
GH_LIB_PATH=paper_2307_16550_b200/build/libgridhop_b200_prof.so timeout 300 python tools/topk_prof.py
