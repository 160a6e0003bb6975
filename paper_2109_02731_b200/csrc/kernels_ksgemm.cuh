// kernels_ksgemm.cuh -- key switching as one exact int8 tensor-core GEMM
// on the hand-written tcgen05 kernel of kernels_imma.cuh.
//
// KeySwitch(c, K) = [b, 0] - sum_{i,j} Decomp_L(a_i)[j] * K[i,j] is a (digits) x (key) matrix
// product.  Digits d < L = 2^logL are split into NL = ceil(logL / 7) unsigned 7-bit limbs
// (int8), padded to NLP = 1, 2 or 4 limb rows per sample (zero rows beyond NL), and key
// coefficients, centred into (-q/2, q/2], into 7 balanced base-256 digits (int8), so
//   D[g NLP + t][(l, w)] = sum_{i,j} limb_t(d_{g,i,j}) * digit_l(K[i,j][w])     (int32, exact:
//   |sum| <= N ell 127 * 128 < 2^31 for every accepted parameter set)
// and out[g][w] = [b_g]_{w=0} - sum_{t,l} 128^t 256^l D[...]  (mod Q, or mod 2^64 then mod 2^w),
// recombined in the GEMM's epilogue.  Used for the bootstrap's LWE_N -> RLWE switch with pK
// (W = 2N, mod Q) and the final LWE_N -> LWE_n switch with ksK (W = n+1, mod 2^w).
#pragma once
#include "kernels_core.cuh"
#include "kernels_imma.cuh"

struct KsGemm {
  int NL;       // 7-bit limbs per digit
  int NLP;      // limb rows per sample (power of two >= NL)
  int Kd;       // N * ell   (GEMM K, multiple of 16 for N >= 256)
  int W;        // output words (2N or n+1)
  int Wpad;     // W rounded up to the epilogue's words per tile (imma::WT)
  int Nout;     // 7 * Wpad key-digit rows
};
static inline KsGemm ks_gemm_shape(int N, int ell, int logL, int W) {
  KsGemm g;
  g.NL = (logL + 6) / 7;
  g.NLP = g.NL <= 1 ? 1 : (g.NL <= 2 ? 2 : 4);
  g.Kd = N * ell;
  g.W = W;
  g.Wpad = (W + imma::WT - 1) / imma::WT * imma::WT;
  g.Nout = 7 * g.Wpad;
  return g;
}
// row of the key-digit matrix holding digit l of output word w (the epilogue's tile layout)
FDFB_DEV size_t imma_key_row(int l, int w) {
  return (size_t)(w / imma::WT) * imma::BN + (size_t)l * imma::WT + (w % imma::WT);
}
// 7 balanced base-256 digits of a signed value |v| < 2^55 (exact)
FDFB_DEV void balanced_digits7(long long v, int8_t (&dg)[7]) {
#pragma unroll
  for (int l = 0; l < 7; l++) {
    int t = (int)(v & 255);
    if (t >= 128) t -= 256;
    v = (v - t) >> 8;
    dg[l] = (int8_t)t;
  }
}
// centred representative of a residue: mod Q (qbits == 0) into (-Q/2, Q/2], mod 2^qbits into
// [-2^(qbits-1), 2^(qbits-1))
FDFB_DEV long long centred(u64 v, u64 Q, int qbits) {
  if (qbits == 0) return v > Q / 2 ? (long long)v - (long long)Q : (long long)v;
  const u64 m = (qbits >= 64) ? ~0ULL : ((1ULL << qbits) - 1);
  v &= m;
  return (v >> (qbits - 1)) & 1 ? (long long)(v | ~m) : (long long)v;
}

// Key digits: GK[imma_key_row(l, w)][i*ell + j] = digit l of key[(i*ell + j) * W + w]
// (zero for the padding w >= W).  Tile: 32 key rows x 8 words.
__global__ void k_ks_gemm_key(const u64* __restrict__ key, KsGemm g, u64 Q, int qbits, int8_t* __restrict__ GK) {
  const int r = blockIdx.x * 32 + threadIdx.x;         // key row (i, j)
  const int w = blockIdx.y * 8 + threadIdx.y;
  if (r >= g.Kd || w >= g.Wpad) return;
  const long long v = w < g.W ? centred(key[(size_t)r * g.W + w], Q, qbits) : 0;
  int8_t dg[7];
  balanced_digits7(v, dg);
#pragma unroll
  for (int l = 0; l < 7; l++) GK[imma_key_row(l, w) * g.Kd + r] = dg[l];
}
// Digit limbs of `rows` LWE samples [rows][N+1]: A[g*NLP + t][i*ell + j] = limb_t(digit_j(a_{g,i}))
// (zero for t >= NL).
__global__ void k_ks_gemm_bits(const u64* __restrict__ lwe, int rows, int N, int ell, int logL, KsGemm g,
                               int8_t* __restrict__ A) {
  const int gi = blockIdx.y;
  const u64 dmask = (1ULL << logL) - 1;
  const u64* a = lwe + (size_t)gi * (N + 1) + 1;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < g.Kd; c += gridDim.x * blockDim.x) {
    const int i = c / ell, j = c % ell;
    const u64 d = (__ldg(a + i) >> (j * logL)) & dmask;
#pragma unroll 1
    for (int t = 0; t < g.NLP; t++)
      A[((size_t)gi * g.NLP + t) * g.Kd + c] = t < g.NL ? (int8_t)((d >> (7 * t)) & 127) : (int8_t)0;
  }
}
