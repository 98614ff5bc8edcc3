# diagnostic build of the fused top-K gather with per-phase clocks, then run
set -e
cd paper_2307_16550_b200
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O2 -I ../include"
nvcc $F -DGH_TOPK_PROF -c csrc/gh_gather_topk.cu -o build/gh_gather_topk_prof.o
objs=$(ls build/*.o | grep -v gh_gather_topk)
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs build/gh_gather_topk_prof.o -o build/libgridhop_b200_prof.so -lcudart -ldl
