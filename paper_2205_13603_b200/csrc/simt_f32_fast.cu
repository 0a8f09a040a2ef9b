// SIMT family instantiations: float operands, timed-repeat variant (simt_impl.cuh).
#include "simt_impl.cuh"

namespace lsb {
namespace simt {

SimtLauncher launcher_f32_fast(int i, int j) {
  static SimtTable<float, false> t;
  return t.t[i][j];
}

}  // namespace simt
}  // namespace lsb
