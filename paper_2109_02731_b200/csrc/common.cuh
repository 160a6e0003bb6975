// common.cuh -- device arithmetic, counter-based PRNG and the per-context parameter
// block shared by all FDFB kernels (sm_100a).  Integer-only: residues mod a prime
// Q < 2^62 held in uint64 with lazy [0, 2Q) / [0, 4Q) ranges (Harvey's NTT trick),
// LWE values mod 2^w with native wrap.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef uint32_t u32;

#define FDFB_DEV __device__ __forceinline__

// ---------------------------------------------------------------- parameters
// Everything a kernel needs, passed by value (fits in the 4 KB param space).
struct DevParams {
  u64 Q, Q2, Q4;          // Q, 2Q, 4Q
  u64 half;               // 2^{-1} mod Q = (Q+1)/2
  u64 q_mask;             // q_lwe - 1
  int N, logN, n, u;      // ring degree, log2 N, LWE dim, |u|
  int log_q_lwe;
  int logL_rgsw, ell_rgsw, logL_boot, ell_boot, logL_pk, ell_pk, logL_ks, ell_ks, logL_pack, ell_pack;
  int lwe_ternary, rlwe_ternary, noiseless, cdt_T;
  u64 t;
  const u64* tw;   const u64* twp;    // forward twiddles psi^{bitrev(k)} and Shoup companions
  const u64* itw;  const u64* itwp;   // inverse twiddles psi^{-bitrev(k)}
  u64 ninv, ninvp;                    // N^{-1} mod Q and its Shoup companion
  const u64* cdt;                     // 2*cdt_T CDT thresholds
  u64 qbar, qbias;                    // floor(2^64 / Q); a multiple of Q >= 2^31 (horner_mod)
};

// ---------------------------------------------------------------- modular arithmetic
// Shoup multiplication by a constant w with precomputed wp = floor(w 2^64 / Q):
// for any a < 2^64 returns a*w mod Q in [0, 2Q)   (Q < 2^63).
FDFB_DEV u64 mul_shoup_lazy(u64 a, u64 w, u64 wp, u64 Q) {
  u64 q = __umul64hi(a, wp);
  return a * w - q * Q;
}
FDFB_DEV u64 csub(u64 x, u64 m) { return x >= m ? x - m : x; }
FDFB_DEV u64 add_mod(u64 a, u64 b, u64 Q) { return csub(a + b, Q); }
FDFB_DEV u64 sub_mod(u64 a, u64 b, u64 Q) { return a >= b ? a - b : a + Q - b; }
FDFB_DEV u64 neg_mod(u64 a, u64 Q) { return a ? Q - a : 0; }
// general a*b mod Q for a, b < 2^64 (slow path; keygen / setup only)
FDFB_DEV u64 mul_mod_slow(u64 a, u64 b, u64 Q) {
  unsigned __int128 p = (unsigned __int128)a * b;
  return (u64)(p % Q);
}
// One Horner step of an exact digit recombination mod Q (GEMM epilogues):
// acc <- (acc 2^s + d) mod Q for acc in [0, Q), s <= 8, |d| < 2^31, Q < 2^55.
// x = acc 2^s + d + qbias < 2^64 is reduced by Barrett with qbar = floor(2^64 / Q):
// the estimate is at most 2 below floor(x / Q), so x - q Q lies in [0, 3Q).
FDFB_DEV u64 horner_mod(u64 acc, int s, long long d, const DevParams& p) {
  const u64 x = (acc << s) + (u64)(d + (long long)p.qbias);
  const u64 q = __umul64hi(x, p.qbar);
  const u64 r = x - q * p.Q;
  return csub(csub(r, p.Q << 1), p.Q);
}
FDFB_DEV u64 from_signed(long long v, u64 Q) {
  long long r = v % (long long)Q;
  if (r < 0) r += (long long)Q;
  return (u64)r;
}

// ---------------------------------------------------------------- Philox4x64-10
// Counter-based generator (Salmon et al., SC'11).  Sampling spec: DESIGN.md
// "Seeded determinism" -- key = (seed, domain), counter = (i0, i1, i2, w / 4).
FDFB_DEV void philox4x64(u64 c0, u64 c1, u64 c2, u64 c3, u64 k0, u64 k1, u64 out[4]) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    if (r > 0) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
    u64 lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    u64 lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    u64 n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}
FDFB_DEV u64 rnd_word(u64 seed, u64 dom, u64 i0, u64 i1, u64 i2, u64 w) {
  u64 o[4];
  philox4x64(i0, i1, i2, w >> 2, seed, dom, o);
  return o[w & 3];
}
// floor(x Q / 2^128) for x = hi:lo  (uniform mod Q)
FDFB_DEV u64 uniform_mod_q(u64 hi, u64 lo, u64 Q) {
  u64 a_lo = hi * Q, a_hi = __umul64hi(hi, Q);
  u64 b_hi = __umul64hi(lo, Q);
  u64 mid = a_lo + b_hi;
  return a_hi + (mid < a_lo ? 1 : 0);
}
FDFB_DEV int key_coeff(u64 x, int ternary) {
  return ternary ? (int)__umul64hi(x, 3ULL) - 1 : (int)(x >> 63);
}
FDFB_DEV long long gauss_cdt(u64 x, const DevParams& p) {
  if (p.noiseless || p.cdt_T == 0) return 0;
  long long e = -p.cdt_T;
  for (int i = 0; i < 2 * p.cdt_T; i++) e += (x >= p.cdt[i]) ? 1 : 0;
  return e;
}

// canonical "X^k * poly" coefficient fetch: coefficient c of X^k a(X), k in [0, 2N)
FDFB_DEV u64 rot_coeff(const u64* a, int c, int k, int N, u64 Q) {
  int e = c - k;
  e &= (2 * N - 1);                       // (c - k) mod 2N
  return e < N ? a[e] : neg_mod(a[e - N], Q);
}
