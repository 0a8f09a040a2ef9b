// SIMT-A instantiations, fp32 operands.
#include "simta_impl.cuh"

namespace lsb {
cudaError_t launch_simta_f32(const void* x, const void* y, float* c, const SimtaArgs& a, int rm, int rn, size_t smem,
                             cudaStream_t st) {
  static simta::Table<float> t;
  int i = simta_tile_index(rm), j = simta_tile_index(rn);
  if (i < 0 || j < 0 || !t.t[i][j]) return cudaErrorInvalidValue;
  return t.t[i][j](x, y, c, a, smem, st);
}
void preload_simta_f32() { simta::preload_table<float>(); }

}  // namespace lsb
