// gh_gather_k3.cu — the K = 3 (complex spectra, interpolation hopping) half of
// the gather kernels of gh_gather_impl.cuh, in its own translation unit so the
// two halves compile in parallel.
#include "gh_gather_impl.cuh"

namespace gh {

void launch_gather_k3(Ctx* ctx, Table* t, const void* spec_d, int T, int combine, float* map_d,
                      unsigned long long* keys_d) {
  launch_gather_side<true>(ctx, t, spec_d, T, combine, map_d, keys_d);
}

}  // namespace gh
