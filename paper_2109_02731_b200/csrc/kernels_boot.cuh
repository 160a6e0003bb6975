// kernels_boot.cuh -- the FDFB bootstrap hot path (Fig. Bootstrap).
#pragma once
#include "kernels_br.cuh"
#include "kernels_ksgemm.cuh"

// ---------------------------------------------------------------------------
// a1: ModSwitch(ct, q_lwe, 2N) -- round half up.
// q_lwe = 2^w, 2N = 2^{logN+1}: round(2N x / q) = ((x >> (w - logN - 2)) + 1) >> 1.
// logm: log2 of the target modulus (logN + 1 for 2N; logN for the shift-based BR's Z_N)
__global__ void k_modswitch_in(DevParams p, const u64* __restrict__ ct, int B, u32* __restrict__ abar,
                               u32* __restrict__ bbar, int logm) {
  const int sh = p.log_q_lwe - logm - 1;
  const u32 m2N = (1u << logm) - 1;
  size_t total = (size_t)B * (p.n + 1);
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    size_t c = x / (p.n + 1); int i = (int)(x % (p.n + 1));
    u64 v = ct[x] & p.q_mask;
    u32 r = (u32)(((v >> sh) + 1) >> 1) & m2N;
    if (i == 0) bbar[c] = r; else abar[c * p.n + (i - 1)] = r;
  }
}

// a2: ladder accumulators acc_{c,i} = [L_boot^{i} 2^{-1} sgnP X^{bbar_c}, 0]  (reading R1),
// sgnP = 1 - sum_{i>=1} X^i.
__global__ void k_ladder_init(DevParams p, const u32* __restrict__ bbar, int B, u64* __restrict__ accs) {
  const int N = p.N, ell = p.ell_boot;
  size_t total = (size_t)B * ell * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    size_t g = x / N; int j = (int)(x % N);
    int c = (int)(g / ell), i = (int)(g % ell);
    u64 cst = mul_mod_slow(pow2_mod(p.logL_boot * i, p.Q), p.half, p.Q);
    // coefficient j of sgnP * X^{bbar}: e = (j - bbar) mod 2N; sgnP[e] for e<N, -sgnP[e-N] else
    int e = (j - (int)bbar[c]) & (2 * N - 1);
    int sgn = (e == 0) ? 1 : (e < N ? -1 : (e == N ? -1 : 1));
    u64* acc = accs + g * 2 * N;
    acc[j] = sgn > 0 ? cst : neg_mod(cst, p.Q);
    acc[N + j] = 0;
  }
}

// a3: batched blind rotation -> kernels_br.cuh

// ---------------------------------------------------------------------------
// a4: ladder SampleExt(acc, 1) + [L_boot^{i} 2^{-1}, 0]
// -> LWE_N mod Q:  b' = b_0,  a'_0 = a_0,  a'_I = -a_{N-I} (I >= 1; NSgn(0) = -1).
__global__ void k_ladder_extract(DevParams p, const u64* __restrict__ accs, int count, u64* __restrict__ lwe) {
  const int N = p.N;
  size_t total = (size_t)count * (N + 1);
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    size_t g = x / (N + 1); int I = (int)(x % (N + 1));
    const u64* acc = accs + g * 2 * N;
    u64 v;
    if (I == 0) {
      int i = (int)(g % p.ell_boot);
      u64 cst = mul_mod_slow(pow2_mod(p.logL_boot * i, p.Q), p.half, p.Q);
      v = add_mod(acc[0], cst, p.Q);
    } else {
      int a = I - 1;
      v = (a == 0) ? acc[N] : neg_mod(acc[N + N - a], p.Q);
    }
    lwe[x] = v;
  }
}

// a6 (first half): c_Q = SampleExt(acc_F, 1), then ModSwitch(Q -> q_lwe) per coefficient:
// floor((2 q x + Q) / (2Q)) mod q  (reading c.3 order, round half up).
__global__ void k_extract_modswitch(DevParams p, const u64* __restrict__ accs, int count, u64* __restrict__ lwe) {
  const int N = p.N;
  size_t total = (size_t)count * (N + 1);
  const unsigned __int128 twoQ = (unsigned __int128)2 * p.Q;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    size_t g = x / (N + 1); int I = (int)(x % (N + 1));
    const u64* acc = accs + g * 2 * N;
    u64 v;
    if (I == 0) v = acc[0];
    else { int a = I - 1; v = (a == 0) ? acc[N] : neg_mod(acc[N + N - a], p.Q); }
    unsigned __int128 num = ((unsigned __int128)v << (p.log_q_lwe + 1)) + p.Q;
    lwe[x] = (u64)(num / twoQ) & p.q_mask;
  }
}

// ---------------------------------------------------------------------------
// a6 CUDA-core LWE KeySwitch N -> n mod q_lwe, the tiled reference
// evaluation behind fdfb_lwe_keyswitch with a NULL workspace (the bootstrap uses the tcgen05
// GEMM of kernels_ksgemm.cuh).  CTA tile: KS_ROWS ciphertexts x KS_COLS output words;
// arithmetic mod 2^w is native u64 wrap.
#define KS_ROWS 16
#define KS_COLS 128
__global__ void __launch_bounds__(KS_COLS)
k_keyswitch_lwe(DevParams p, const u64* __restrict__ ksk, const u64* __restrict__ lwe, int count,
                u64* __restrict__ out) {
  const int N = p.N, n = p.n, ell = p.ell_ks, logL = p.logL_ks;
  const u64 dmask = (1ULL << logL) - 1;
  const int col = blockIdx.x * KS_COLS + threadIdx.x;   // in [0, n+1)
  const int row0 = blockIdx.y * KS_ROWS;
  const bool act = col <= n;
  __shared__ u64 sa[KS_ROWS][33];
  u64 acc[KS_ROWS];
#pragma unroll
  for (int r = 0; r < KS_ROWS; r++) acc[r] = 0;
  for (int i0 = 0; i0 < N; i0 += 32) {
    __syncthreads();
    for (int x = threadIdx.x; x < KS_ROWS * 32; x += KS_COLS) {
      int r = x / 32, ii = x % 32;
      int g = row0 + r;
      sa[r][ii] = (g < count && i0 + ii < N) ? lwe[(size_t)g * (N + 1) + 1 + i0 + ii] : 0;
    }
    __syncthreads();
    if (act) {
      for (int ii = 0; ii < 32 && i0 + ii < N; ii++) {
        const u64* krow = ksk + ((size_t)(i0 + ii) * ell) * (n + 1) + col;
        for (int j = 0; j < ell; j++) {
          u64 kv = __ldg(krow + (size_t)j * (n + 1));
#pragma unroll
          for (int r = 0; r < KS_ROWS; r++) {
            u64 dg = (sa[r][ii] >> (j * logL)) & dmask;
            acc[r] += dg * kv;
          }
        }
      }
    }
  }
  if (!act) return;
#pragma unroll
  for (int r = 0; r < KS_ROWS; r++) {
    int g = row0 + r;
    if (g >= count) continue;
    u64 v = (col == 0 ? lwe[(size_t)g * (N + 1)] : 0) - acc[r];
    out[(size_t)g * (n + 1) + col] = v & p.q_mask;
  }
}

// ---------------------------------------------------------------------------
// a5 (PubMux, readings R1 + F4): per ciphertext c,
//   r_x = rotP_x X^{bbar_c};  p0 := r_1, p1 := r_0 (swap);  P = Decomp_{L_boot}(p1 - p0)
//   acc_F = [p0, 0] + sum_i P[i] * acc_{R,c,i}   (ring products via NTT, Montgomery MAC).
// Step 1: digit polynomials (coef domain) into dig[c][i][N]; accR NTT'd in place by k_ntt_batch.
__global__ void k_pubmux_digits(DevParams p, const u64* __restrict__ rotp, const u32* __restrict__ bbar, int B,
                                u64* __restrict__ dig) {
  const int N = p.N, ell = p.ell_boot, logL = p.logL_boot;
  const u64 dmask = (1ULL << logL) - 1, Q = p.Q;
  size_t total = (size_t)B * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    int c = (int)(x / N), j = (int)(x % N);
    int e = (int)bbar[c];
    u64 r0 = rot_coeff(rotp, j, e, N, Q), r1 = rot_coeff(rotp + N, j, e, N, Q);
    u64 pd = sub_mod(r0, r1, Q);                        // p1 - p0 = r0 - r1
    for (int i = 0; i < ell; i++) dig[((size_t)c * ell + i) * N + j] = (pd >> (i * logL)) & dmask;
  }
}
// Step 2 (NTT domain): F[c][col] = sum_i Dhat[c][i] * Ahat[c][i][col]
__global__ void k_pubmux_mac(DevParams p, const u64* __restrict__ dig_hat, const u64* __restrict__ accR_hat, int B,
                             u64* __restrict__ F, u64 qinv_neg, u64 r2) {
  const int N = p.N, ell = p.ell_boot;
  const u64 Q = p.Q;
  size_t total = (size_t)B * 2 * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    int c = (int)(x / (2 * N)); int cs = (int)(x % (2 * N)); int col = cs / N, s = cs % N;
    u64 acc = 0;
    for (int i = 0; i < ell; i++) {
      u64 dv = dig_hat[((size_t)c * ell + i) * N + s];
      u64 av = accR_hat[(((size_t)c * ell + i) * 2 + col) * N + s];
      acc = add_mod(acc, csub(mont_mul(dv, av, Q, qinv_neg), Q), Q);
    }
    F[x] = csub(mont_mul(acc, r2, Q, qinv_neg), Q);
  }
}
// Step 3 (after inverse NTT of F): acc_F = [p0, 0] + F, p0 = rotP_1 X^{bbar}
__global__ void k_pubmux_finish(DevParams p, const u64* __restrict__ rotp, const u32* __restrict__ bbar, int B,
                                u64* __restrict__ F) {
  const int N = p.N;
  size_t total = (size_t)B * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    int c = (int)(x / N), j = (int)(x % N);
    u64 r1 = rot_coeff(rotp + N, j, (int)bbar[c], N, p.Q);
    u64* f = F + (size_t)c * 2 * N;
    f[j] = add_mod(f[j], r1, p.Q);
  }
}

// Standalone SampleExt with per-item 1-based k.
__global__ void k_sample_extract(DevParams p, const u64* __restrict__ rlwe, const u32* __restrict__ kk, int B,
                                 u64* __restrict__ lwe, int* __restrict__ status) {
  const int N = p.N;
  size_t total = (size_t)B * (N + 1);
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    size_t g = x / (N + 1); int I = (int)(x % (N + 1));
    const u64* ct = rlwe + g * 2 * N;
    int k = (int)kk[g];                      // 1-based
    if (k < 1 || k > N) {                    // out of range: flag, zero output
      if (I == 0) atomicOr(status, 1);
      lwe[x] = 0;
      continue;
    }
    u64 v;
    if (I == 0) v = ct[k - 1];
    else {
      int i = I;                             // 1-based i
      int idx = ((k - i) % N + N) % N;
      u64 a = ct[N + idx];
      v = (k - i + 1 > 0) ? a : neg_mod(a, p.Q);
    }
    lwe[x] = v;
  }
}

// ------------------------------------------------------------------ shift-based bootstrap (NEXT #4)
// Steps 1-2 of PAPER.md:322-323 (readings S2, S3): F[c] = [Shift(rotP, bbar_c), 0], the plaintext
// cyclic rotation rotP_b[x] = rotP[(x - bbar_c) mod N], bbar in Z_N.
__global__ void k_shiftboot_init(DevParams p, const u64* __restrict__ rotp, const u32* __restrict__ bbar, int B,
                                 u64* __restrict__ F) {
  const int N = p.N;
  const size_t total = (size_t)B * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    const int cc = (int)(x / N), j = (int)(x % N);
    F[(size_t)cc * 2 * N + j] = __ldg(rotp + ((j - (int)bbar[cc]) & (N - 1)));
    F[(size_t)cc * 2 * N + N + j] = 0;
  }
}
// Shift amount of step s = i u + j for every ciphertext: -abar_i u_j mod N, with 0 (the
// identity, skipped by the CMux kernel, reading S1) replaced by a valid dummy 1.
__global__ void k_shiftbr_amount(DevParams p, const u32* __restrict__ abar, int B, int s, u32* __restrict__ d) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  const int i = (p.u == 2) ? (s >> 1) : s, j = s - i * p.u;
  const u32 a = abar[(size_t)c * p.n + i];
  const u32 v = (p.u == 2 && j == 0) ? a : ((u32)p.N - a) & (u32)(p.N - 1);
  d[c] = v ? v : 1u;
}

// ------------------------------------------------------------------ decryption helpers
// phase = b - <a, s> mod q_lwe (one warp per ciphertext); msg = round(t phase / q) mod t.
__global__ void k_lwe_decrypt(DevParams p, const int8_t* __restrict__ s, const u64* __restrict__ ct, int count,
                              u32 t, u64* __restrict__ phase, u64* __restrict__ msg) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= count) return;
  const u64* c = ct + (size_t)warp * (p.n + 1);
  u64 acc = 0;                                      // exact mod 2^64, then mod q_lwe
  for (int i = lane; i < p.n; i += 32) acc += c[1 + i] * (u64)(long long)s[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    const u64 ph = (c[0] - acc) & p.q_mask;
    if (phase) phase[warp] = ph;
    if (msg && t) {
      const unsigned __int128 num = (unsigned __int128)ph * t * 2 + ((unsigned __int128)1 << p.log_q_lwe);
      msg[warp] = (u64)((num >> (p.log_q_lwe + 1)) % t);
    }
  }
}
// out = b - prod (prod = a * s in coefficient form, from fdfb_poly_mul's NTT path)
__global__ void k_rlwe_phase_finish(DevParams p, const u64* __restrict__ ct, const u64* __restrict__ prod, int count,
                                    u64* __restrict__ out) {
  const int N = p.N;
  const size_t total = (size_t)count * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    const size_t c = x / N, j = x % N;
    out[x] = sub_mod(ct[c * 2 * N + j], prod[x], p.Q);
  }
}
__global__ void k_rlwe_phase_prep(DevParams p, const u64* __restrict__ ct, const int8_t* __restrict__ s, int count,
                                  u64* __restrict__ a, u64* __restrict__ sp) {
  const int N = p.N;
  const size_t total = (size_t)count * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    const size_t c = x / N, j = x % N;
    a[x] = ct[c * 2 * N + N + j];
    const int v = s[j];
    sp[x] = v >= 0 ? (u64)v : p.Q - (u64)(-v);
  }
}
