mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_topk_fused.py tests/test_gpu_parity.py -k "topk or top5 or fused or ties" -x -q -p no:cacheprovider 2>&1 | tail -4
for c in 1 2; do
  echo "== GH_TOPK_CTAS=$c"
  GH_TOPK_CTAS=$c timeout 300 python tools/time_topk.py --trials 2048
  GH_TOPK_CTAS=$c GH_LIB_PATH=paper_2307_16550_b200/build/libgridhop_b200_prof.so timeout 300 python tools/topk_prof.py
done
