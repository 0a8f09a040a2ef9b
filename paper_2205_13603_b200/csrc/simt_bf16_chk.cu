// SIMT family instantiations: __nv_bfloat16 operands, checked-launch variant (simt_impl.cuh).
#include "simt_impl.cuh"

namespace lsb {
namespace simt {

SimtLauncher launcher_bf16_chk(int i, int j) {
  static SimtTable<__nv_bfloat16, true> t;
  return t.t[i][j];
}

}  // namespace simt
}  // namespace lsb
