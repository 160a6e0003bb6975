// ntt.cuh -- negacyclic NTT / inverse NTT over Z_Q for one polynomial per
// N/8-thread group, shared-memory resident, 8 coefficients per thread in registers.
//
// Forward: Cooley-Tukey with merged psi powers (natural order in, bit-reversed
// NTT slots out); inverse: Gentleman-Sande (bit-reversed in, natural out) WITHOUT
// the final N^{-1} scaling (callers fold N^{-1} into a constant operand).
// Stage s works on pairs (j, j+t), t = N >> (s+1), twiddle index N/(2t) + j/(2t)
// into psi_rev (forward) / psi_inv_rev (inverse).
//
// Passes (radix-8 in registers, one shared-memory exchange between passes):
//   pass 0      : stages 0..2, thread tid holds positions tid + T*k      (layout P0)
//   pass q>=1   : stages 3q..3q+2, positions (tid/T')8T' + tid%T' + T'k, T' = N>>(3q+3)
//   last pass   : remaining 1..3 stages, thread holds positions 8 tid + k (layout PL)
// After pass 0 each warp owns a contiguous 256-coefficient block, so only the
// P0<->P1 exchange needs a CTA barrier; the others use __syncwarp.
// The XOR swizzle `swz` makes every layout's 16-lane u64 accesses bank-conflict
// free (checked exhaustively for N = 256..2048).
#pragma once
#include "common.cuh"

template <int N>
struct NttShape {
  static constexpr int LOGN = (N == 256) ? 8 : (N == 512) ? 9 : (N == 1024) ? 10 : 11;
  static constexpr int T = N / 8;                 // threads per polynomial
  static constexpr int NMID = (LOGN - 1) / 3;     // number of radix-8 passes
  static constexpr int PLAST = LOGN - 3 * NMID;   // stages in the last pass (1..3)
  static constexpr int PAD = 0;
};

FDFB_DEV int swz(int e) {
  return e ^ ((e >> 3) & 7) ^ (((e >> 4) & 3) << 2) ^ (((e >> 6) & 1) << 3);
}

// Harvey butterflies: forward in/out [0, 4Q); inverse in/out [0, 2Q).
FDFB_DEV void bf_fwd(u64& X, u64& Y, u64 w, u64 wp, u64 Q, u64 Q2) {
  u64 x = csub(X, Q2);
  u64 t = mul_shoup_lazy(Y, w, wp, Q);
  X = x + t;
  Y = x - t + Q2;
}
FDFB_DEV void bf_inv(u64& X, u64& Y, u64 w, u64 wp, u64 Q, u64 Q2) {
  u64 x = X, y = Y;
  X = csub(x + y, Q2);
  Y = mul_shoup_lazy(x - y + Q2, w, wp, Q);
}

// one forward radix-8 pass on positions base + T1*k (3 stages: t = 4T1, 2T1, T1)
template <int N, int T1>
FDFB_DEV void fwd_pass8(u64 x[8], int base, const u64* __restrict__ tw, const u64* __restrict__ twp, u64 Q, u64 Q2) {
#pragma unroll
  for (int s = 0; s < 3; s++) {
    const int t = T1 << (2 - s);
    const int sk = 4 >> s;                 // pair distance in k
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if ((k & sk) == 0) {
        const int pos = base + T1 * k;
        const int idx = N / (2 * t) + pos / (2 * t);
        bf_fwd(x[k], x[k + sk], __ldg(tw + idx), __ldg(twp + idx), Q, Q2);
      }
    }
  }
}
template <int N, int T1>
FDFB_DEV void inv_pass8(u64 x[8], int base, const u64* __restrict__ itw, const u64* __restrict__ itwp, u64 Q, u64 Q2) {
#pragma unroll
  for (int s = 0; s < 3; s++) {
    const int t = T1 << s;
    const int sk = 1 << s;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if ((k & sk) == 0) {
        const int pos = base + T1 * k;
        const int idx = N / (2 * t) + pos / (2 * t);
        bf_inv(x[k], x[k + sk], __ldg(itw + idx), __ldg(itwp + idx), Q, Q2);
      }
    }
  }
}
// last pass: P stages with t = 2^{P-1} .. 1 on positions 8 tid + k
template <int N, int P>
FDFB_DEV void fwd_last(u64 x[8], int tid, const u64* __restrict__ tw, const u64* __restrict__ twp, u64 Q, u64 Q2) {
#pragma unroll
  for (int s = 0; s < P; s++) {
    const int t = 1 << (P - 1 - s);
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if ((k & t) == 0) {
        const int pos = 8 * tid + k;
        const int idx = N / (2 * t) + pos / (2 * t);
        bf_fwd(x[k], x[k + t], __ldg(tw + idx), __ldg(twp + idx), Q, Q2);
      }
    }
  }
}
template <int N, int P>
FDFB_DEV void inv_last(u64 x[8], int tid, const u64* __restrict__ itw, const u64* __restrict__ itwp, u64 Q, u64 Q2) {
#pragma unroll
  for (int s = 0; s < P; s++) {
    const int t = 1 << s;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if ((k & t) == 0) {
        const int pos = 8 * tid + k;
        const int idx = N / (2 * t) + pos / (2 * t);
        bf_inv(x[k], x[k + t], __ldg(itw + idx), __ldg(itwp + idx), Q, Q2);
      }
    }
  }
}

template <int N, int q>
struct MidPass {  // positions of pass q >= 1 for thread tid
  static constexpr int T1 = N >> (3 * q + 3);
  static FDFB_DEV int base(int tid) { return (tid / T1) * 8 * T1 + (tid % T1); }
};

// Forward NTT.  In: x[k] = a[tid + T k] in [0, 4Q).  Out: x[k] = slot 8 tid + k in [0, 4Q).
// sbuf: N u64 of shared memory (swizzled); ends with sbuf free for reuse by the warp
// only -- callers alternate two buffers between consecutive transforms.
template <int N>
FDFB_DEV void ntt_fwd(u64 x[8], u64* sbuf, int tid, const DevParams& p) {
  using S = NttShape<N>;
  const u64 Q = p.Q, Q2 = p.Q2;
  fwd_pass8<N, S::T>(x, tid, p.tw, p.twp, Q, Q2);
#pragma unroll
  for (int k = 0; k < 8; k++) sbuf[swz(tid + S::T * k)] = x[k];
  __syncthreads();
#pragma unroll
  for (int q = 1; q < S::NMID; q++) {
    // (unrolled; q is a compile-time constant in each copy)
    const int T1 = N >> (3 * q + 3);
    const int base = (tid / T1) * 8 * T1 + (tid % T1);
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = sbuf[swz(base + T1 * k)];
    if (q == 1) fwd_pass8<N, (N >> 6)>(x, base, p.tw, p.twp, Q, Q2);
    else if (q == 2) fwd_pass8<N, (N >> 9)>(x, base, p.tw, p.twp, Q, Q2);
#pragma unroll
    for (int k = 0; k < 8; k++) sbuf[swz(base + T1 * k)] = x[k];
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = sbuf[swz(8 * tid + k)];
  fwd_last<N, S::PLAST>(x, tid, p.tw, p.twp, Q, Q2);
}

// Inverse NTT (unscaled).  In: x[k] = slot 8 tid + k in [0, 2Q).
// Out: x[k] = coefficient tid + T k in [0, 2Q), times N (caller folds N^{-1}).
template <int N>
FDFB_DEV void ntt_inv(u64 x[8], u64* sbuf, int tid, const DevParams& p) {
  using S = NttShape<N>;
  const u64 Q = p.Q, Q2 = p.Q2;
  inv_last<N, S::PLAST>(x, tid, p.itw, p.itwp, Q, Q2);
#pragma unroll
  for (int k = 0; k < 8; k++) sbuf[swz(8 * tid + k)] = x[k];
  __syncwarp();
#pragma unroll
  for (int q = S::NMID - 1; q >= 1; q--) {
    const int T1 = N >> (3 * q + 3);
    const int base = (tid / T1) * 8 * T1 + (tid % T1);
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = sbuf[swz(base + T1 * k)];
    if (q == 1) inv_pass8<N, (N >> 6)>(x, base, p.itw, p.itwp, Q, Q2);
    else if (q == 2) inv_pass8<N, (N >> 9)>(x, base, p.itw, p.itwp, Q, Q2);
#pragma unroll
    for (int k = 0; k < 8; k++) sbuf[swz(base + T1 * k)] = x[k];
    if (q > 1) __syncwarp();
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = sbuf[swz(tid + S::T * k)];
  inv_pass8<N, S::T>(x, 0 + tid, p.itw, p.itwp, Q, Q2);
}
