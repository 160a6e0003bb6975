// kernels_ksgemm.cuh -- key switching as one exact int8 tensor-core GEMM.
//
// KeySwitch(c, K) = [b, 0] - sum_{i,j} Decomp_L(a_i)[j] * K[i,j] is a (digits) x (key) matrix
// product.  Digits d < L = 2^logL are split into NL = ceil(logL / 7) unsigned 7-bit limbs
// (int8), key coefficients into 7 balanced base-256 digits (int8), so
//   D[g*NL + t][l*Wpad + w] = sum_{i,j} limb_t(d_{g,i,j}) * digit_l(K[i,j][w])     (int32, exact:
//   |sum| <= N ell 127 * 128 < 2^31 for every configuration here)
// and out[g][w] = [b_g]_{w=0} - sum_{t,l} 128^t 256^l D[...]  (exact in 128 bits, then mod q).
// Used for the bootstrap's LWE_N -> RLWE switch with pK (W = 2N, mod Q) and the final
// LWE_N -> LWE_n switch with ksK (W = n+1, mod 2^w).  The GEMM itself is a plain cuBLASLt
// int8 GEMM; the operand builders and the recombination are ours.
#pragma once
#include "kernels_core.cuh"

struct KsGemm {
  int NL;       // 7-bit limbs per digit
  int Kd;       // N * ell   (GEMM K, multiple of 16 for N >= 256)
  int W;        // output words (2N or n+1)
  int Wpad;     // W rounded up to 16
  int Nout;     // 7 * Wpad
};
static inline KsGemm ks_gemm_shape(int N, int ell, int logL, int W) {
  KsGemm g;
  g.NL = (logL + 6) / 7;
  g.Kd = N * ell;
  g.W = W;
  g.Wpad = (W + 15) & ~15;
  g.Nout = 7 * g.Wpad;
  return g;
}

// Key digits: GK[l * Wpad + w][i*ell + j] = balanced base-256 digit l of key[(i*ell + j) * W + w]
// (zero for the padding w >= W).  Tile: 32 key rows x 8 words.
__global__ void k_ks_gemm_key(const u64* __restrict__ key, KsGemm g, int8_t* __restrict__ GK) {
  const int r = blockIdx.x * 32 + threadIdx.x;         // key row (i, j)
  const int w = blockIdx.y * 8 + threadIdx.y;
  if (r >= g.Kd || w >= g.Wpad) return;
  u64 v = w < g.W ? key[(size_t)r * g.W + w] : 0;
#pragma unroll
  for (int l = 0; l < 7; l++) {
    int t = (int)(v & 255);
    if (t >= 128) t -= 256;
    v = (u64)((long long)v - t) >> 8;
    GK[((size_t)l * g.Wpad + w) * g.Kd + r] = (int8_t)t;
  }
}
// Digit limbs of `rows` LWE samples [rows][N+1]: A[g*NL + t][i*ell + j] = limb_t(digit_j(a_{g,i})).
__global__ void k_ks_gemm_bits(const u64* __restrict__ lwe, int rows, int N, int ell, int logL, KsGemm g,
                               int8_t* __restrict__ A) {
  const int gi = blockIdx.y;
  const u64 dmask = (1ULL << logL) - 1;
  const u64* a = lwe + (size_t)gi * (N + 1) + 1;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < g.Kd; c += gridDim.x * blockDim.x) {
    const int i = c / ell, j = c % ell;
    const u64 d = (__ldg(a + i) >> (j * logL)) & dmask;
#pragma unroll 1
    for (int t = 0; t < g.NL; t++) A[((size_t)gi * g.NL + t) * g.Kd + c] = (int8_t)((d >> (7 * t)) & 127);
  }
}
// out[g][w] = [b_g]_{w=0} - value(D rows of g) mod q   (q = Q prime if qmask == 0, else 2^w via qmask)
__global__ void k_ks_gemm_finish(DevParams dp, const int* __restrict__ D, const u64* __restrict__ lwe, int rows, int N, KsGemm g,
                                 u64 Q, u64 qmask, u64* __restrict__ out) {
  const size_t total = (size_t)rows * g.W;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    const int gi = (int)(x / g.W), w = (int)(x % g.W);
    const u64 b = w == 0 ? __ldg(lwe + (size_t)gi * (N + 1)) : 0;
    if (!qmask) {                                    // mod Q: Horner over 7-bit groups of 8-bit limbs
      u64 vm = 0;
#pragma unroll 1
      for (int t = g.NL - 1; t >= 0; t--) {
        const int* dr = D + ((size_t)gi * g.NL + t) * g.Nout + w;
        u64 s = 0;
#pragma unroll
        for (int l = 6; l >= 0; l--) s = horner_mod(s, 8, dr[(size_t)l * g.Wpad], dp);
        vm = add_mod(horner_mod(vm, 7, 0, dp), s, Q);
      }
      out[x] = b >= vm ? b - vm : b + Q - vm;
      continue;
    }
    __int128 v = 0;
#pragma unroll 1
    for (int t = g.NL - 1; t >= 0; t--) {
      const int* dr = D + ((size_t)gi * g.NL + t) * g.Nout + w;
      __int128 s = 0;
#pragma unroll
      for (int l = 6; l >= 0; l--) s = s * 256 + dr[(size_t)l * g.Wpad];
      v = v * 128 + s;
    }
    out[x] = (b - (u64)v) & qmask;                   // two's complement wrap: exact mod 2^w
  }
}
