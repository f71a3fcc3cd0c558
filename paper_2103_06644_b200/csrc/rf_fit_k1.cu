// rf_fit_k1.cu -- fit_tile_kernel instantiations for SP = 1 (standard): compiled as its own
// translation unit so the three kernel sets build in parallel (rf_tile_kernel.cuh).
#include "rf_tile_kernel.cuh"

namespace rf_fitk {
cudaError_t launch_radius_sp1(const KParams& Ps, const KParams& Pd, const CUtensorMap& tmap, bool tma, size_t sm,
                               int64_t tiles, int sms, cudaStream_t s, bool pdl, bool three) {
  return launch_radius<1>(Ps, Pd, tmap, tma, sm, tiles, sms, s, pdl, three);
}

#ifdef RF_COUNT_SLOW
int read_slow_counts_sp1(unsigned long long* out, int reset) {
  unsigned long long c[256];
  if (cudaMemcpyFromSymbol(c, g_slow_count, sizeof(c)) != cudaSuccess) return 3;
  for (int i = 0; i < 256; ++i) out[i] += c[i];
  if (reset) {
    static const unsigned long long z[256] = {};
    cudaMemcpyToSymbol(g_slow_count, z, sizeof(z));
  }
  return 0;
}
#endif
}  // namespace rf_fitk
