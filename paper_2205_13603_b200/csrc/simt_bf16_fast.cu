// SIMT family instantiations: __nv_bfloat16 operands, timed-repeat variant (simt_impl.cuh).
#include "simt_impl.cuh"

namespace lsb {
namespace simt {

SimtLauncher launcher_bf16_fast(int i, int j) {
  static SimtTable<__nv_bfloat16, false> t;
  return t.t[i][j];
}

}  // namespace simt
}  // namespace lsb
