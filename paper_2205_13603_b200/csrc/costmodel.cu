// K7 + K8: warp-per-candidate batched cost analysis on the B200.
//
//   K8  exact simulated latency   (`src/machine.py:228-254`, exact rationals
//                                  in int128 instead of Python Fractions)
//   K7  9 features + linear score (`src/costmodel.py:21-79`, `:98-102`)
//
// One warp owns one program.  Inside a statement the 32 lanes split the two
// expensive loops of the reference: the cache-resident-suffix search
// (`_cache_suffix_start`, `src/machine.py:121-127`: lane t evaluates the
// interval footprint of suffix t, a ballot picks the longest fitting suffix)
// and the per-access miss classification (`classify_accesses`,
// `src/machine.py:140-170`: one access per lane).  Lane 0 then folds the
// per-access results in the reference's access order, so the floating-point
// feature sums round exactly like the reference's sequential loop.
#include <cuda_runtime.h>
#include <stdint.h>

#include "costdesc.hpp"
#include "costmodel.cuh"

namespace lsb {

namespace {

typedef __int128 i128;

struct Q { i128 n, d; };

__device__ __forceinline__ i128 iabs(i128 x) { return x < 0 ? -x : x; }
__device__ __forceinline__ bool fits64(i128 x) { return x >= (i128)INT64_MIN && x <= (i128)INT64_MAX; }
// 128-bit division is a long software routine on the GPU: take the 64-bit
// instruction path whenever both operands fit (almost always here)
__device__ __forceinline__ i128 qdiv(i128 a, i128 b) {
  if (fits64(a) && fits64(b)) return (i128)((int64_t)a / (int64_t)b);
  return a / b;
}
__device__ __forceinline__ int ctz128(unsigned __int128 x) {
  const uint64_t lo = (uint64_t)x;
  return lo ? __ffsll((long long)lo) - 1 : 64 + __ffsll((long long)(uint64_t)(x >> 64)) - 1;
}
// binary (Stein) gcd: shifts and subtractions only, no division
__device__ i128 gcd128(i128 sa, i128 sb) {
  unsigned __int128 a = (unsigned __int128)iabs(sa), b = (unsigned __int128)iabs(sb);
  if (!a) return (i128)b;
  if (!b) return (i128)a;
  if (!(a >> 64) && !(b >> 64)) {
    uint64_t x = (uint64_t)a, y = (uint64_t)b;
    const int sh = __ffsll((long long)(x | y)) - 1;
    x >>= __ffsll((long long)x) - 1;
    do {
      y >>= __ffsll((long long)y) - 1;
      if (x > y) { uint64_t t = x; x = y; y = t; }
      y -= x;
    } while (y);
    return (i128)(x << sh);
  }
  const int sh = ctz128(a | b);
  a >>= ctz128(a);
  do {
    b >>= ctz128(b);
    if (a > b) { unsigned __int128 t = a; a = b; b = t; }
    b -= a;
  } while (b);
  return (i128)(a << sh);
}
__device__ Q qmk(i128 n, i128 d) {
  if (d < 0) { n = -n; d = -d; }
  i128 g = gcd128(n, d);
  if (g > 1) { n = qdiv(n, g); d = qdiv(d, g); }
  return Q{n, d};
}
__device__ __forceinline__ Q qint(i128 x) { return Q{x, 1}; }
constexpr i128 kQLim = ((i128)1) << 120;
// overflow guard |x| * |y| > kQLim without a 128-bit division
__device__ __forceinline__ bool mul_over(i128 x, i128 y) {
  const unsigned __int128 ax = (unsigned __int128)iabs(x), ay = (unsigned __int128)iabs(y);
  if (!ax || !ay) return false;
  if (!(ax >> 60) && !(ay >> 60)) return false;  // < 2^120
  return ax > (unsigned __int128)kQLim / ay;
}
__device__ Q qadd(Q a, Q b, int* ovf) {
  if (a.d == 1 && b.d == 1) {  // integers: the common case
    if (iabs(a.n) > kQLim || iabs(b.n) > kQLim) *ovf = 1;
    return Q{a.n + b.n, 1};
  }
  i128 g = gcd128(a.d, b.d);
  i128 bd = qdiv(b.d, g), ad = qdiv(a.d, g);
  if (mul_over(a.n, bd) || mul_over(b.n, ad) || mul_over(a.d, bd)) *ovf = 1;
  return qmk(a.n * bd + b.n * ad, a.d * bd);
}
__device__ Q qmul(Q a, Q b, int* ovf) {
  i128 g1 = gcd128(a.n, b.d), g2 = gcd128(b.n, a.d);
  if (g1 == 0) g1 = 1;
  if (g2 == 0) g2 = 1;
  i128 n1 = qdiv(a.n, g1), d2 = qdiv(b.d, g1), n2 = qdiv(b.n, g2), d1 = qdiv(a.d, g2);
  if (mul_over(n1, n2) || mul_over(d1, d2)) *ovf = 1;
  return qmk(n1 * n2, d1 * d2);
}

__device__ __forceinline__ int64_t fdiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
__device__ __forceinline__ int64_t fmodp(int64_t a, int64_t b) {
  int64_t r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}

// Interval bound of one index expression (`src/ir.py:394-433`); vars of
// enclosing positions >= t range over [0, extent-1], the rest are fixed at 0.
__device__ bool eval_interval(const int64_t* code, const int64_t* ext, int t, int64_t* lo, int64_t* hi) {
  int64_t n = code[0];
  if (n < 0) {  // affine form from the encoder (costdesc.cpp affine_form): c0 + per-occurrence terms
    int64_t l = code[1], h = code[1];
    for (int64_t i = 0; i < -n - 1; ++i) {
      const int64_t pos = code[2 + 2 * i], coef = code[3 + 2 * i];
      const int64_t v = coef * (pos >= t ? ext[pos] - 1 : 0);
      l += min(v, (int64_t)0);
      h += max(v, (int64_t)0);
    }
    *lo = l;
    *hi = h;
    return true;
  }
  int64_t sl[MAX_STACK], sh[MAX_STACK];
  int sp = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t op = code[1 + 2 * i], arg = code[2 + 2 * i];
    if (op == BC_INT) { if (sp >= MAX_STACK) return false; sl[sp] = sh[sp] = arg; ++sp; continue; }
    if (op == BC_VAR) { if (sp >= MAX_STACK) return false; sl[sp] = 0; sh[sp] = arg >= t ? ext[arg] - 1 : 0; ++sp; continue; }
    if (op == BC_SEL) {
      if (sp < 3) return false;
      int64_t ol = sl[sp - 1], oh = sh[sp - 1], tl = sl[sp - 2], th = sh[sp - 2];
      sp -= 3;
      sl[sp] = min(tl, ol); sh[sp] = max(th, oh); ++sp;
      continue;
    }
    if (sp < 2) return false;
    int64_t bl = sl[sp - 1], bh = sh[sp - 1], al = sl[sp - 2], ah = sh[sp - 2];
    sp -= 2;
    int64_t rl, rh;
    switch (op) {
      case BC_ADD: rl = al + bl; rh = ah + bh; break;
      case BC_SUB: rl = al - bh; rh = ah - bl; break;
      case BC_MUL: {
        int64_t p0 = al * bl, p1 = al * bh, p2 = ah * bl, p3 = ah * bh;
        rl = min(min(p0, p1), min(p2, p3)); rh = max(max(p0, p1), max(p2, p3)); break;
      }
      case BC_MAX: rl = max(al, bl); rh = max(ah, bh); break;
      case BC_MIN: rl = min(al, bl); rh = min(ah, bh); break;
      case BC_FDIV:
        if (bl == bh && bl > 0) { rl = fdiv(al, bl); rh = fdiv(ah, bl); }
        else { rl = min(fdiv(al, max(bl, (int64_t)1)), al); rh = max(ah, fdiv(ah, max(bl, (int64_t)1))); }
        break;
      case BC_MOD:
        if (bl == bh && bl > 0) {
          if (fdiv(al, bl) == fdiv(ah, bl) && al >= 0) { rl = fmodp(al, bl); rh = fmodp(ah, bl); }
          else { rl = 0; rh = bl - 1; }
        } else { rl = 0; rh = max(bh - 1, (int64_t)0); }
        break;
      default: return false;
    }
    sl[sp] = rl; sh[sp] = rh; ++sp;
  }
  if (sp != 1) return false;
  *lo = sl[0]; *hi = sh[0];
  return true;
}

constexpr int kWarps = 4;
constexpr int kBlobCap = 1024;  // words of a program's blob staged in smem (8 KB per warp)
constexpr int kMaxLoops = 128;
constexpr int kMaxAcc = 64;

struct WarpScratch {
  int64_t mf_num[kMaxAcc], mf_den[kMaxAcc];
  int64_t mult_num[kMaxLoops], mult_den[kMaxLoops];
  int64_t ext[MAX_NEST + 2];
  int phase[kMaxAcc];
};

}  // namespace

__global__ void __launch_bounds__(kWarps * 32)
analyze_kernel(const int64_t* __restrict__ blobs, const int64_t* __restrict__ offsets, int n,
               DSpec spec, DModel model, int flags, int64_t* lat_num, int64_t* lat_den,
               double* feats, double* pred, int* status) {
  __shared__ WarpScratch scratch[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int prog = blockIdx.x * kWarps + warp;
  if (prog >= n) return;
  WarpScratch& S = scratch[warp];
  // the program's blob -> this warp's smem slice in one coalesced pass: the
  // analysis below is chains of dependent reads (header -> loop table ->
  // statement -> access -> index bytecode), ~0.3 us each from L2 but tens
  // of cycles from smem.  Larger blobs are read in place.
  extern __shared__ int64_t blob_smem[];
  const int64_t* B = blobs + offsets[prog];
  const int64_t len = offsets[prog + 1] - offsets[prog];
  if (len <= kBlobCap) {
    int64_t* dst = blob_smem + warp * kBlobCap;
    for (int64_t i = lane; i < len; i += 32) dst[i] = B[i];
    __syncwarp();
    B = dst;
  }
  const int nloop = (int)B[H_NLOOP], nstmt = (int)B[H_NSTMT];
  const int64_t* L = B + B[H_OFF_LOOP];
  const int64_t* BUF = B + B[H_OFF_BUF];
  const int64_t* ST = B + B[H_OFF_STMT];
  int st = (int)B[H_STATUS];
  if (nloop > kMaxLoops) st = 2;
  if (st) {
    if (lane == 0) status[prog] = st;
    return;
  }

  // ---- per-loop latency multipliers (`simulate_latency.walk` kind rules) ----
  for (int l = lane; l < nloop; l += 32) {
    const int64_t* R = L + l * LOOP_WORDS;
    int64_t e = R[L_EXTENT], kind = R[L_KIND], depth = R[L_DEPTH];
    int64_t num = e, den = 1;
    if (kind == 3) {                    // unrolled
      if (e <= 16) { num = e * spec.unroll_num; den = spec.unroll_den; }
    } else if (kind == 2) {             // vectorized: friendly iff every enclosed statement agrees
      bool vf = true;
      for (int s = 0; s < nstmt; ++s) {
        const int64_t* SR = ST + s * STMT_WORDS;
        int nl = (int)SR[S_NL];
        if (depth < nl && B[SR[S_OFF_ENC] + depth] == l && !((SR[S_VF_OK] >> depth) & 1)) vf = false;
      }
      if (vf) num = (e + spec.vector_lanes - 1) / spec.vector_lanes;
    } else if (kind == 1) {             // parallel: only the outermost parallel loop is discounted
      bool seen = false;
      for (int64_t p = R[L_PARENT]; p >= 0; p = L[p * LOOP_WORDS + L_PARENT])
        if (L[p * LOOP_WORDS + L_KIND] == 1) seen = true;
      if (!seen) num = (e + spec.cores - 1) / spec.cores;
    }
    S.mult_num[l] = num;
    S.mult_den[l] = den;
  }
  __syncwarp();

  int ovf = 0;
  Q total = qint(0);
  int64_t total_trip = 0, flops = 0, vec = 0, par = 0, unr = 0, tcalls = 0, depth_max = 0;
  double hits = 0.0, misses = 0.0;

  for (int s = 0; s < nstmt && !st; ++s) {
    const int64_t* SR = ST + s * STMT_WORDS;
    const int nl = (int)SR[S_NL];
    const int64_t* enc = B + SR[S_OFF_ENC];
    const int nacc = (int)SR[S_NACC];
    const int64_t* ACC = B + SR[S_OFF_ACC];
    const bool intr = SR[S_TYPE] == 1;
    if (nacc > kMaxAcc) { st = 2; break; }
    for (int p = lane; p < nl; p += 32) S.ext[p] = L[enc[p] * LOOP_WORDS + L_EXTENT];
    __syncwarp();

    // ---- longest cache-resident suffix: lane t tries suffix t ----
    int tstar = nl + 1;
    bool bad = false;
    for (int base = 0; base <= nl; base += 32) {
      int t = base + lane;
      bool fits = false;
      if (t <= nl) {
        int64_t blo[MAX_BUFS][MAX_DIM], bhi[MAX_BUFS][MAX_DIM];
        uint32_t seen = 0;
        for (int a = 0; a < nacc && !bad; ++a) {
          const int64_t* AR = ACC + a * ACC_WORDS;
          int b = (int)AR[A_BUF], nd = (int)AR[A_NDIM];
          for (int d = 0; d < nd; ++d) {
            int64_t lo, hi;
            if (!eval_interval(B + AR[A_CODE + d], S.ext, t, &lo, &hi)) { bad = true; break; }
            hi += AR[A_TILE] - 1;
            if (!((seen >> b) & 1)) { blo[b][d] = lo; bhi[b][d] = hi; }
            else { blo[b][d] = min(blo[b][d], lo); bhi[b][d] = max(bhi[b][d], hi); }
          }
          seen |= 1u << b;
        }
        int64_t tot = 0;
        for (int b = 0; b < MAX_BUFS && !bad; ++b)
          if ((seen >> b) & 1) {
            const int64_t* BR = BUF + b * BUF_WORDS;
            int64_t sz = 1;
            for (int d = 0; d < (int)BR[0]; ++d)
              sz *= max((int64_t)1, min(bhi[b][d] - blo[b][d] + 1, BR[1 + d]));
            tot += sz;
          }
        fits = !bad && tot <= spec.cache_capacity;
      }
      unsigned m = __ballot_sync(0xffffffffu, fits);
      if (__any_sync(0xffffffffu, bad)) { bad = true; break; }
      if (m) { tstar = base + __ffs(m) - 1; break; }
    }
    if (bad) { st = 2; break; }

    // ---- miss fraction per access: lane a classifies access a ----
    if (!intr) {
      int64_t trips = 1;
      for (int p = tstar; p < nl; ++p) trips *= S.ext[p];
      const uint64_t above = tstar >= 64 ? ~0ull : ((1ull << tstar) - 1);
      for (int a = lane; a < nacc; a += 32) {
        const int64_t* AR = ACC + a * ACC_WORDS;
        int64_t num, den = 1;
        if (tstar > nl) num = 1;
        else if ((((uint64_t)AR[A_USE]) & above) == 0) num = 0;
        else {
          int64_t region = 1;
          const int64_t* BR = BUF + AR[A_BUF] * BUF_WORDS;
          for (int d = 0; d < (int)AR[A_NDIM]; ++d) {
            int64_t lo, hi;
            if (!eval_interval(B + AR[A_CODE + d], S.ext, tstar, &lo, &hi)) { bad = true; break; }
            region *= max((int64_t)1, min(hi - lo + 1, BR[1 + d]));
          }
          if (region >= trips) num = 1; else { num = region; den = trips; }
        }
        S.mf_num[a] = num;
        S.mf_den[a] = den;
        S.phase[a] = (int)AR[A_PHASE];
      }
    }
    if (__any_sync(0xffffffffu, bad)) { st = 2; break; }
    __syncwarp();

    if (lane == 0) {
      int64_t trip = 1;
      bool kv = false, kp = false, ku = false;
      for (int p = 0; p < nl; ++p) {
        trip *= S.ext[p];
        int64_t k = L[enc[p] * LOOP_WORDS + L_KIND];
        kv |= k == 2; kp |= k == 1; ku |= k == 3;
      }
      int64_t red_trip = 1;
      for (int p = 0; p < nl; ++p)
        if ((((uint64_t)SR[S_RED_MASK]) >> p) & 1) red_trip *= S.ext[p];
      // the exact rational latency only when it is asked for (flags & 1):
      // its int128 gcd chain is lane 0's serial critical path, and the
      // features never read it
      if (flags & 1) {
        Q cost;
        if (intr) {
          cost = qint(spec.tensor_unit_cost + SR[S_IOPEL] * spec.hit_cost);
        } else {
          Q am = qint(0);
          if (SR[S_HAS_INIT]) am = qadd(am, qmk(SR[S_INIT_OPS], red_trip), &ovf);
          if (SR[S_HAS_EPI]) am = qadd(am, qmk(SR[S_EPI_OPS], red_trip), &ovf);
          cost = qmul(qint(spec.flop_cost), qadd(qint(SR[S_FLOPS]), am, &ovf), &ovf);
          for (int a = 0; a < nacc; ++a) {
            Q mf = qmk(S.mf_num[a], S.mf_den[a]);
            Q ac = qadd(qint(spec.hit_cost), qmul(qint(spec.miss_cost - spec.hit_cost), mf, &ovf), &ovf);
            if (S.phase[a] != 0) ac = qmul(ac, qmk(1, red_trip), &ovf);
            cost = qadd(cost, ac, &ovf);
          }
        }
        Q mult = qint(1);
        for (int p = 0; p < nl; ++p) mult = qmul(mult, qmk(S.mult_num[enc[p]], S.mult_den[enc[p]]), &ovf);
        total = qadd(total, qmul(cost, mult, &ovf), &ovf);
      }

      // features (`featurize` accumulation order)
      total_trip += trip;
      if (nl > depth_max) depth_max = nl;
      if (kv) vec += trip;
      if (kp) par += trip;
      if (ku) unr += trip;
      if (intr) {
        flops += SR[S_IFLOPS] * trip;
        hits = __dadd_rn(hits, (double)(SR[S_IOPEL] * trip));
        tcalls += trip;
      } else {
        int64_t spatial = trip / red_trip;
        flops += trip * SR[S_FLOPS];
        if (SR[S_HAS_INIT]) flops += spatial * SR[S_INIT_OPS];
        if (SR[S_HAS_EPI]) flops += spatial * SR[S_EPI_OPS];
        for (int a = 0; a < nacc; ++a) {
          double nn = (double)(S.phase[a] == 0 ? trip : spatial);
          double num = (double)S.mf_num[a], den = (double)S.mf_den[a];
          // explicit round-to-nearest ops: no FMA contraction, so the sums
          // round exactly like the reference's `float(frac) * n` loop
          misses = __dadd_rn(misses, __dmul_rn(__ddiv_rn(num, den), nn));
          hits = __dadd_rn(hits, __dmul_rn(__ddiv_rn((double)(S.mf_den[a] - S.mf_num[a]), den), nn));
        }
      }
    }
    __syncwarp();
  }

  if (lane != 0) return;
  if ((flags & 1) && !st && ovf) st = 3;
  if ((flags & 1) && !st && (total.n > (i128)INT64_MAX || total.d > (i128)INT64_MAX)) st = 3;
  status[prog] = st;
  if (st) return;
  if (flags & 1) { lat_num[prog] = (int64_t)total.n; lat_den[prog] = (int64_t)total.d; }
  if (flags & 6) {
    double tt = (double)total_trip;
    double f[9];
    f[0] = log1p(tt);
    f[1] = log1p((double)flops);
    f[2] = total_trip ? __ddiv_rn((double)vec, tt) : 0.0;
    f[3] = total_trip ? __ddiv_rn((double)par, tt) : 0.0;
    f[4] = log1p(hits);
    f[5] = log1p(misses);
    f[6] = total_trip ? __ddiv_rn((double)unr, tt) : 0.0;
    f[7] = (double)tcalls;
    f[8] = (double)depth_max;
    if (flags & 2)
      for (int i = 0; i < 9; ++i) feats[(size_t)prog * 9 + i] = f[i];
    if (flags & 4) pred[prog] = score_one(f, model);
  }
}

// K7b alone: linear score of precomputed features, one thread per row.
__global__ void score_kernel(const double* __restrict__ feats, int n, DModel model, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    double f[9];
    for (int k = 0; k < 9; ++k) f[k] = feats[(size_t)i * 9 + k];
    out[i] = score_one(f, model);
  }
}

void launch_analyze(const int64_t* blobs, const int64_t* offsets, int n, const DSpec& spec, const DModel& model,
                    int flags, int64_t* lat_num, int64_t* lat_den, double* feats, double* pred, int* status,
                    cudaStream_t stream) {
  if (n <= 0) return;
  int grid = (n + kWarps - 1) / kWarps;
  analyze_kernel<<<grid, kWarps * 32, kWarps * kBlobCap * sizeof(int64_t), stream>>>(blobs, offsets, n, spec, model,
                                                                                    flags, lat_num, lat_den,
                                                   feats, pred, status);
}

void launch_score(const double* feats, int n, const DModel& model, double* out, cudaStream_t stream) {
  if (n <= 0) return;
  score_kernel<<<(n + 127) / 128, 128, 0, stream>>>(feats, n, model, out);
}

}  // namespace lsb
