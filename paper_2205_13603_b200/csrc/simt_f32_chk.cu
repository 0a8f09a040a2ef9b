// SIMT family instantiations: float operands, checked-launch variant (simt_impl.cuh).
#include "simt_impl.cuh"

namespace lsb {
namespace simt {

SimtLauncher launcher_f32_chk(int i, int j) {
  static SimtTable<float, true> t;
  return t.t[i][j];
}

}  // namespace simt
}  // namespace lsb
