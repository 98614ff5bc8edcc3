// gh_gather.cu — the K = 1 (power) half of the gather kernels and the public
// launchers; the kernels live in gh_gather_impl.cuh (hop_bin_value /
// scan_planes, src/hopping.cpp:59-117; argmax_index, src/direct.cpp:55-62).
#include "gh_gather_impl.cuh"

namespace gh {

void launch_gather_k3(Ctx* ctx, Table* t, const void* spec_d, int T, int combine, float* map_d,
                      unsigned long long* keys_d);  // gh_gather_k3.cu

void launch_gather(Ctx* ctx, Table* t, const void* spec_d, int T, int combine, float* map_d,
                   unsigned long long* keys_d) {
  const Plan& pl = map_d ? t->plan_map : t->plan;  // built by the caller (build_plan)
  if (pl.k3) launch_gather_k3(ctx, t, spec_d, T, combine, map_d, keys_d);
  else launch_gather_side<false>(ctx, t, spec_d, T, combine, map_d, keys_d);
}

void launch_decode_keys(Ctx* ctx, const unsigned long long* keys_d, int T, int64_t* idx_d,
                        float* val_d) {
  KTimer kt(ctx, "decode");
  k_decode_keys<<<(T + 255) / 256, 256, 0, ctx->stream>>>(keys_d, T, idx_d, val_d);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
