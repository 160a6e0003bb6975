// kernels_br.cuh -- the batched blind rotation, the hot kernel.
//
// One CTA of T = N/8 threads per accumulator, resident in shared memory for all n*u CMux
// steps; 512/T CTAs per SM (<= 128 registers per thread) so that two (N = 2048) or more
// accumulators interleave on every SM and hide each other's latencies and barriers.
// One CMux step (CMux = extProd(brK[i,j], acc X^e - acc) + acc):
//   d = acc X^e - acc (canonical, thread-private scratch in smem)
//   for each of the 2 ell digit polynomials D_r = Decomp_{L,Q}(d)[r]:
//       forward NTT of D_r in registers (radix-8 passes, one smem exchange per pass),
//       Shoup MAC with brK[i,j][r] for both output columns (lazy, [0, 16Q))
//   acc += INTT(MAC) for both columns (N^{-1} folded into brK).
//
// Twiddles come from pass-grouped tables of (w, w') pairs (built on the host, see
// fdfb_api.cu make_pass_tables): for every radix-8 pass a thread needs only the 7 (or
// 8 - 8/2^PLAST) pairs of its group, stored contiguously -> one base address per pass and
// 16-byte loads with immediate offsets (no per-butterfly 64-bit address arithmetic).
// brK device format: [n*u steps][2 ell rows][2 cols][N slots] of (w, w') pairs, NTT
// (bit-reversed) slot order, w pre-multiplied by N^{-1}.
#pragma once
#include "kernels_core.cuh"

template <int N>
struct BrShape {
  static constexpr int LOGN = (N == 256) ? 8 : (N == 512) ? 9 : (N == 1024) ? 10 : 11;
  static constexpr int T = N / 8;
  static constexpr int NMID = (LOGN - 1) / 3;      // radix-8 passes on T1-strided positions
  static constexpr int PLAST = LOGN - 3 * NMID;    // stages of the final pass (1..3)
  static constexpr int NLAST = 8 - (8 >> PLAST);   // twiddle pairs per thread in the final pass
  static constexpr int MINB = 512 / T;             // CTAs per SM
  // offsets (in pairs) of each pass's table
  static constexpr int off(int q) {                // q in [0, NMID): 7 * sum_{q'<q} 8^{q'}
    int o = 0, g = 1;
    for (int i = 0; i < q; i++) { o += 7 * g; g *= 8; }
    return o;
  }
  static constexpr int OFF_LAST = off(NMID);
  static constexpr int PAIRS = OFF_LAST + T * NLAST;
};

typedef ulonglong2 u64x2;

FDFB_DEV u64x2 ldp(const u64x2* p) { return __ldg(p); }

FDFB_DEV void bfw(u64& X, u64& Y, u64x2 w, u64 Q, u64 Q2) {      // Harvey CT, in/out [0, 4Q)
  u64 x = csub(X, Q2);
  u64 t = mul_shoup_lazy(Y, w.x, w.y, Q);
  X = x + t;
  Y = x - t + Q2;
}
FDFB_DEV void bin(u64& X, u64& Y, u64x2 w, u64 Q, u64 Q2) {      // Harvey GS, in/out [0, 2Q)
  u64 x = X, y = Y;
  X = csub(x + y, Q2);
  Y = mul_shoup_lazy(x - y + Q2, w.x, w.y, Q);
}

// forward radix-8 pass: 3 stages on x[0..7] (pair distances 4, 2, 1 in k); tw -> the group's 7 pairs
FDFB_DEV void fwd8(u64 x[8], const u64x2* tw, u64 Q, u64 Q2) {
  const u64x2 w0 = ldp(tw);
#pragma unroll
  for (int k = 0; k < 4; k++) bfw(x[k], x[k + 4], w0, Q, Q2);
  const u64x2 w1 = ldp(tw + 1), w2 = ldp(tw + 2);
  bfw(x[0], x[2], w1, Q, Q2); bfw(x[1], x[3], w1, Q, Q2);
  bfw(x[4], x[6], w2, Q, Q2); bfw(x[5], x[7], w2, Q, Q2);
#pragma unroll
  for (int k = 0; k < 4; k++) bfw(x[2 * k], x[2 * k + 1], ldp(tw + 3 + k), Q, Q2);
}
FDFB_DEV void inv8(u64 x[8], const u64x2* tw, u64 Q, u64 Q2) {
#pragma unroll
  for (int k = 0; k < 4; k++) bin(x[2 * k], x[2 * k + 1], ldp(tw + 3 + k), Q, Q2);
  const u64x2 w1 = ldp(tw + 1), w2 = ldp(tw + 2);
  bin(x[0], x[2], w1, Q, Q2); bin(x[1], x[3], w1, Q, Q2);
  bin(x[4], x[6], w2, Q, Q2); bin(x[5], x[7], w2, Q, Q2);
  const u64x2 w0 = ldp(tw);
#pragma unroll
  for (int k = 0; k < 4; k++) bin(x[k], x[k + 4], w0, Q, Q2);
}
// final pass on positions 8 tid + k: P stages with pair distance t = 2^{P-1-s}
template <int P>
FDFB_DEV void fwd_lastP(u64 x[8], const u64x2* tw, u64 Q, u64 Q2) {
  int o = 0;
#pragma unroll
  for (int s = 0; s < P; s++) {
    const int t = 1 << (P - 1 - s);
#pragma unroll
    for (int k = 0; k < 8; k++)
      if ((k & t) == 0) bfw(x[k], x[k + t], ldp(tw + o + (k >> (P - s))), Q, Q2);
    o += 8 >> (P - s);
  }
}
template <int P>
FDFB_DEV void inv_lastP(u64 x[8], const u64x2* tw, u64 Q, u64 Q2) {
  int o = 8 - (8 >> P);
#pragma unroll
  for (int s = P - 1; s >= 0; s--) {
    const int t = 1 << (P - 1 - s);
    o -= 8 >> (P - s);
#pragma unroll
    for (int k = 0; k < 8; k++)
      if ((k & t) == 0) bin(x[k], x[k + t], ldp(tw + o + (k >> (P - s))), Q, Q2);
  }
}

FDFB_DEV int sw(int e) { return e ^ ((e >> 3) & 7) ^ (((e >> 4) & 3) << 2) ^ (((e >> 6) & 1) << 3); }

// Forward NTT. In: x[k] = coefficient tid + T k in [0, 4Q).  Out: x[k] = slot 8 tid + k in [0, 4Q).
template <int N>
FDFB_DEV void ntt_fwd2(u64 x[8], u64* sb, int tid, const u64x2* tab, u64 Q, u64 Q2) {
  using S = BrShape<N>;
  constexpr int T = S::T;
  fwd8(x, tab, Q, Q2);
#pragma unroll
  for (int k = 0; k < 8; k++) sb[sw(tid + T * k)] = x[k];
  __syncthreads();
#pragma unroll
  for (int q = 1; q < S::NMID; q++) {
    const int T1 = N >> (3 * q + 3);
    const int g = tid / T1;
    const int base = g * 8 * T1 + (tid % T1);
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = sb[sw(base + T1 * k)];
    fwd8(x, tab + S::off(q) + 7 * g, Q, Q2);
#pragma unroll
    for (int k = 0; k < 8; k++) sb[sw(base + T1 * k)] = x[k];
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = sb[sw(8 * tid + k)];
  fwd_lastP<S::PLAST>(x, tab + S::OFF_LAST + S::NLAST * tid, Q, Q2);
}
// Inverse NTT (unscaled).  In: x[k] = slot 8 tid + k in [0, 2Q).  Out: coefficient tid + T k, [0, 2Q).
template <int N>
FDFB_DEV void ntt_inv2(u64 x[8], u64* sb, int tid, const u64x2* tab, u64 Q, u64 Q2) {
  using S = BrShape<N>;
  constexpr int T = S::T;
  inv_lastP<S::PLAST>(x, tab + S::OFF_LAST + S::NLAST * tid, Q, Q2);
#pragma unroll
  for (int k = 0; k < 8; k++) sb[sw(8 * tid + k)] = x[k];
  __syncwarp();
#pragma unroll
  for (int q = S::NMID - 1; q >= 1; q--) {
    const int T1 = N >> (3 * q + 3);
    const int g = tid / T1;
    const int base = g * 8 * T1 + (tid % T1);
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = sb[sw(base + T1 * k)];
    inv8(x, tab + S::off(q) + 7 * g, Q, Q2);
#pragma unroll
    for (int k = 0; k < 8; k++) sb[sw(base + T1 * k)] = x[k];
    __syncwarp();
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = sb[sw(tid + T * k)];
  inv8(x, tab, Q, Q2);
}

template <int N>
__global__ void __launch_bounds__(N / 8, BrShape<N>::MINB)
k_blind_rotate(DevParams p, const u64x2* __restrict__ bsk, const u64x2* __restrict__ ftab,
               const u64x2* __restrict__ itab, u64* __restrict__ accs, int n_acc, int acc_per_ct,
               const u32* __restrict__ abar) {
  using S = BrShape<N>;
  constexpr int T = S::T;
  extern __shared__ u64 smem[];
  u64* sacc = smem;            // [b | a], natural order, canonical
  u64* sd = smem + 2 * N;      // d = acc X^e - acc of the current half (thread-private slots)
  u64* sb0 = smem + 3 * N;     // NTT exchange buffers (alternating)
  u64* sb1 = smem + 4 * N;
  const int tid = threadIdx.x;
  const u64 Q = p.Q, Q2 = p.Q2;
  const int ell = p.ell_rgsw, logL = p.logL_rgsw, u = p.u;
  const u64 dmask = (1ULL << logL) - 1;
  const size_t step_pairs = (size_t)2 * ell * 2 * N;

  for (int g = blockIdx.x; g < n_acc; g += gridDim.x) {
    u64* acc = accs + (size_t)g * 2 * N;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) sacc[tid + T * k] = acc[tid + T * k];
    const u32* ab = abar + (size_t)(g / acc_per_ct) * p.n;
    int buf = 0;
#pragma unroll 1
    for (int i = 0; i < p.n; i++) {
      const u32 ai = __ldg(ab + i);
#pragma unroll 1
      for (int j = 0; j < u; j++) {
        // exponent -abar_i u_j mod 2N; u = [1] (binary) or [-1, 1] (ternary)
        const int e = (u == 2 && j == 0) ? (int)ai : (int)((2 * N - ai) & (2 * N - 1));
        const u64x2* K = bsk + ((size_t)i * u + j) * step_pairs + 8 * tid;
        __syncthreads();                                  // previous step's acc writes
        u64 mb[8], ma[8];
#pragma unroll
        for (int k = 0; k < 8; k++) { mb[k] = 0; ma[k] = 0; }
#pragma unroll 1
        for (int half = 0; half < 2; half++) {
          const u64* src = sacc + half * N;
#pragma unroll
          for (int k = 0; k < 8; k++) {
            const int pos = tid + T * k;
            sd[pos] = sub_mod(rot_coeff(src, pos, e, N, Q), src[pos], Q);
          }
#pragma unroll 1
          for (int r = 0; r < ell; r++) {
            const u64x2* Kb = K + (size_t)((half * ell + r) * 2) * N;
            const u64x2* Ka = Kb + N;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(Kb));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(Kb + 4));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(Ka));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(Ka + 4));
            u64 x[8];
            const int sh = r * logL;
#pragma unroll
            for (int k = 0; k < 8; k++) x[k] = (sd[tid + T * k] >> sh) & dmask;
            ntt_fwd2<N>(x, buf ? sb1 : sb0, tid, ftab, Q, Q2);
            buf ^= 1;
#pragma unroll
            for (int k = 0; k < 8; k++) {
              const u64x2 wb = __ldg(Kb + k);
              mb[k] += mul_shoup_lazy(x[k], wb.x, wb.y, Q);
            }
#pragma unroll
            for (int k = 0; k < 8; k++) {
              const u64x2 wa = __ldg(Ka + k);
              ma[k] += mul_shoup_lazy(x[k], wa.x, wa.y, Q);
            }
          }
        }
        // 2 ell terms in [0, 2Q) each (< 16Q): reduce into [0, 2Q) for the inverse transform
#pragma unroll
        for (int k = 0; k < 8; k++) {
#pragma unroll
          for (int s = 3; s >= 1; s--) { mb[k] = csub(mb[k], Q << s); ma[k] = csub(ma[k], Q << s); }
        }
        // park the a-column sums in the (now free, thread-private) d scratch during INTT(b)
#pragma unroll
        for (int k = 0; k < 8; k++) sd[tid + T * k] = ma[k];
        ntt_inv2<N>(mb, buf ? sb1 : sb0, tid, itab, Q, Q2);
        buf ^= 1;
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int pos = tid + T * k;
          sacc[pos] = add_mod(sacc[pos], csub(mb[k], Q), Q);
        }
#pragma unroll
        for (int k = 0; k < 8; k++) ma[k] = sd[tid + T * k];
        ntt_inv2<N>(ma, buf ? sb1 : sb0, tid, itab, Q, Q2);
        buf ^= 1;
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int pos = N + tid + T * k;
          sacc[pos] = add_mod(sacc[pos], csub(ma[k], Q), Q);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) acc[tid + T * k] = sacc[tid + T * k];
  }
}

// Device brK from canonical rows already forward-transformed (slots, [0, Q)):
// pair (w N^{-1} mod Q, Shoup companion).  ntt_rows: [rows*2 polys][N].
__global__ void k_brk_finalize(DevParams p, const u64* __restrict__ ntt_rows, u64x2* __restrict__ dev, size_t npoly) {
  const int N = p.N;
  size_t total = npoly * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    u64 v = csub(mul_shoup_lazy(ntt_rows[x], p.ninv, p.ninvp, p.Q), p.Q);
    u64 vp = (u64)(((unsigned __int128)v << 64) / p.Q);
    dev[x] = make_ulonglong2(v, vp);
  }
}
