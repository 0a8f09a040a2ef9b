// SIMT-A instantiations, bf16 operands; plus the plan -> kernel-args adapter.
#include <cstring>

#include <stdlib.h>

#include "simta_impl.cuh"

namespace lsb {
cudaError_t launch_simta_bf16(const void* x, const void* y, float* c, const SimtaArgs& a, int rm, int rn, size_t smem,
                              cudaStream_t st) {
  static simta::Table<__nv_bfloat16> t;
  int i = simta_tile_index(rm), j = simta_tile_index(rn);
  if (i < 0 || j < 0 || !t.t[i][j]) return cudaErrorInvalidValue;
  return t.t[i][j](x, y, c, a, smem, st);
}

bool launch_simta(const void* x, const void* y, float* c, const AffineCfg& A, bool bf16,
                  const unsigned long long* deadline, int* timed_out, cudaStream_t st) {
  SimtaArgs a;
  std::memset(&a, 0, sizeof a);
  AList* lists[8] = {&a.m_grid, &a.n_grid, &a.m_thr, &a.n_thr, &a.m_reg, &a.n_reg, &a.k_tile, &a.k_bk};
  for (int i = 0; i < A.nparts; ++i) {
    const APart& P = A.parts[i];
    int li;
    if (P.group == AG_K) li = P.level == AL_KTILE ? 6 : 7;
    else li = (P.level == AL_GRID ? 0 : P.level == AL_THREAD ? 2 : 4) + (P.group == AG_N ? 1 : 0);
    AList& L = *lists[li];
    if (L.n >= 8) return false;
    L.ext[L.n] = P.extent;
    L.cx[L.n] = P.cx;
    L.cy[L.n] = P.cy;
    L.cc[L.n] = P.cc;
    L.cg0[L.n] = P.cg[0];
    L.cg1[L.n] = P.cg[1];
    ++L.n;
  }
  a.x0 = A.x0; a.y0 = A.y0; a.c0 = A.c0;
  a.ng = A.ng;
  a.g0[0] = A.g0[0]; a.g0[1] = A.g0[1];
  a.gext[0] = A.gext[0]; a.gext[1] = A.gext[1];
  a.gm = A.gm; a.gn = A.gn; a.tm = A.tm; a.tn = A.tn; a.bk = A.bk; a.kt = A.kt;
  a.deadline = deadline;
  a.timed_out = timed_out;
  a.persist = deadline ? 1 : 0;
  a.ntn = a.ntm = 1;
  const size_t smem = static_cast<size_t>(A.smem_bytes);
  cudaError_t e = bf16 ? launch_simta_bf16(x, y, c, a, static_cast<int>(A.rm), static_cast<int>(A.rn), smem, st)
                       : launch_simta_f32(x, y, c, a, static_cast<int>(A.rm), static_cast<int>(A.rn), smem, st);
  return e == cudaSuccess;
}
void preload_simta_bf16() { simta::preload_table<__nv_bfloat16>(); }

}  // namespace lsb
