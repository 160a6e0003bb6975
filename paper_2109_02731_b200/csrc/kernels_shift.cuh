// kernels_shift.cuh -- Pack / VectorPack / Shift kernels.
//
// Device packing-key format (opaque; built by k_pack_suffix + k_pack_fixup from the
// canonical PackSetup table pK[i][j][v], i in [N], j in [ell], v in [L]):
//   A   canonical pK                     [N][ell][L][2][N]      (direct VectorPack / Pack)
//   T1  T^{(v)}_{1,j}                    [ell][L][2][N]
//   D   Delta^{(v)}_{i,j}, i = 2..N, v>=1 [ell][N-1][L-1][2][N]
//   U   sum_j sum_{i>=2} T^{(0)}_{i,j}   [2][N]
//   Uj  per-j partials of U              [ell][2][N]
//   S0  sum_j T^{(0)}_{1,j}              [2][N]        (L == 2: Shift-as-GEMM key below)
//   GK  int8 [7 * 2N][Kpad] balanced base-256 digits of the Shift GEMM key matrix
//   GP  int8 [7 * 2N][N ell] digits of Delta0_{k,l} = pK[k,l,1] - pK[k,l,0] (Permute GEMM)
// with the key-only suffix sums  T^{(v)}_{i,j} = sum_{i'>=i} X^{i'-i} pK[i',j,v]  and
// Delta^{(v)}_{i,j} = T^{(v)}_{i,j} - T^{(0)}_{i,j}.
//
// Shift: the m LWE samples Shift packs are
// SampleExt(ct, K) at consecutive K = K1 .. K1+m-1, and SampleExt(ct, K).a[i+1] =
// SampleExt(ct, K-1).a[i].  With A_k[i,j] = digit_j(a'_k[i]) this gives the exact identity
//   sum_{k,i} X^{k-1} pK[i,j,A_k[i,j]] = sum_k X^{k-1} T^{(A_k[1,j])}_{1,j}
//        + sum_{i'=1}^{N-1} ( T^{(gamma)}_{i'+1,j} - X^m T^{(beta)}_{i'+1,j} ),
//   gamma = A_1[i'+1,j],  beta = A_m[i',j],
// so VectorPack needs (m + 2(N-1)) * ell key-polynomial additions per ciphertext instead of
// the definition's m * N * ell; the result is the same residue vector mod Q.
#pragma once
#include "kernels_core.cuh"
#include "kernels_ksgemm.cuh"

struct PackLayout {
  size_t P;                 // words per RLWE (2N)
  size_t A, T1, D, U, Uj;   // word offsets
  size_t S0, GK, GP;        // L == 2 only: S0 = sum_j T^(0)_{1,j} [2][N]; Shift / Permute GEMM key digits (int8)
  size_t words;
};
static inline size_t shift_gemm_key_bytes(int N, int ell, int L) {
  if (L != 2) return 0;
  const size_t K = (size_t)ell * (N - 1) + N + (size_t)ell * N, Kpad = (K + 15) & ~(size_t)15;
  return 7 * 2 * (size_t)N * Kpad;
}
static inline PackLayout pack_layout(int N, int ell, int L) {
  PackLayout l;
  l.P = 2 * (size_t)N;
  l.A = 0;
  l.T1 = l.A + (size_t)N * ell * L * l.P;
  l.D = l.T1 + (size_t)ell * L * l.P;
  l.U = l.D + (size_t)ell * (N - 1) * (L - 1) * l.P;
  l.Uj = l.U + l.P;
  l.S0 = l.Uj + (size_t)ell * l.P;
  l.GK = l.S0 + l.P;
  l.GP = l.GK + (shift_gemm_key_bytes(N, ell, L) + 7) / 8;
  l.words = l.GP + ((L == 2 ? (size_t)14 * N * (size_t)N * ell : 0) + 7) / 8;
  return l;
}

// ---------------------------------------------------------------------------
// Suffix recurrence T_i = P_i + X T_{i+1} (T_{N+1} = 0), one CTA per (j, v, column):
//   v == 0: P_i = pK[i,j,0];          writes T1[j][0], accumulates Uj[j] = sum_{i>=2} T_i
//   v >= 1: P_i = pK[i,j,v]-pK[i,j,0]; writes D[j][i][v] (i >= 2) and T1[j][v] (= Delta_1)
// (X T)[c] = T[c-1] for c >= 1, -T[N-1] for c = 0.
__global__ void k_pack_suffix(DevParams p, u64* __restrict__ pk, int ell, int L, PackLayout lay) {
  extern __shared__ u64 sm[];
  const int N = p.N;
  const u64 Q = p.Q;
  const int jv = blockIdx.x, col = blockIdx.y;
  const int j = jv / L, v = jv % L;
  u64* cur = sm;
  u64* nxt = sm + N;
  u64 uacc[8];                      // N <= 2048, blockDim 256 -> <= 8 coefficients per thread
#pragma unroll
  for (int r = 0; r < 8; r++) uacc[r] = 0;
  for (int c = threadIdx.x; c < N; c += blockDim.x) cur[c] = 0;
  __syncthreads();
  for (int i = N; i >= 1; i--) {     // 1-based i
    const u64* base = pk + lay.A + (((size_t)(i - 1) * ell + j) * L) * lay.P + (size_t)col * N;
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int c = threadIdx.x + r * blockDim.x;
      if (c >= N) break;
      u64 pi = base[(size_t)v * lay.P + c];
      if (v) pi = sub_mod(pi, base[c], Q);
      const u64 xt = c ? cur[c - 1] : neg_mod(cur[N - 1], Q);
      const u64 t = add_mod(pi, xt, Q);
      nxt[c] = t;
      if (i >= 2) {
        if (v) pk[lay.D + (((size_t)j * (N - 1) + (i - 2)) * (L - 1) + (v - 1)) * lay.P + (size_t)col * N + c] = t;
        else uacc[r] = add_mod(uacc[r], t, Q);
      } else {
        pk[lay.T1 + ((size_t)j * L + v) * lay.P + (size_t)col * N + c] = t;
      }
    }
    __syncthreads();
    u64* tmp = cur; cur = nxt; nxt = tmp;
  }
  if (v == 0) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int c = threadIdx.x + r * blockDim.x;
      if (c < N) pk[lay.Uj + (size_t)j * lay.P + (size_t)col * N + c] = uacc[r];
    }
  }
}
// T1[j][v] += T1[j][0] for v >= 1 (Delta_1 -> T_1), and U = sum_j Uj[j].
__global__ void k_pack_fixup(DevParams p, u64* __restrict__ pk, int ell, int L, PackLayout lay) {
  const u64 Q = p.Q;
  const size_t P = lay.P;
  const size_t n1 = (size_t)ell * (L - 1) * P;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < n1 + P; x += (size_t)gridDim.x * blockDim.x) {
    if (x < n1) {
      const size_t w = x % P, jv = x / P;
      const size_t j = jv / (L - 1), v = jv % (L - 1) + 1;
      u64* t = pk + lay.T1 + (j * L + v) * P + w;
      *t = add_mod(*t, pk[lay.T1 + (j * L) * P + w], Q);
    } else {
      const size_t w = x - n1;
      u64 s = 0;
      for (int j = 0; j < ell; j++) s = add_mod(s, pk[lay.Uj + (size_t)j * P + w], Q);
      pk[lay.U + w] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// SampleExt mask coefficient a'_K[i] (1-based K, i, NSgn(x) = +1 iff x > 0)
FDFB_DEV u64 sx_mask(const u64* a, int K, int i, int N, u64 Q) {
  const int idx = (K - i) & (N - 1);                  // (K - i) mod N, N a power of two
  const u64 v = a[idx];
  return (K - i + 1 > 0) ? v : neg_mod(v, Q);
}

// Shift (readings F2/F3): one CTA per (tile of C ciphertexts, column h),
// 256 threads, thread owns coefficients x_r = tid + 256 r (CPT = N / 256 of them).
// BIN: L_pack == 2 (one Delta row per (i', j), shared by the whole tile).
template <int CPT, int C, bool BIN>
__global__ void __launch_bounds__(256)
k_shift(DevParams p, const u64* __restrict__ pk, PackLayout lay, const u64* __restrict__ ct,
        const u32* __restrict__ dd, int B, u64* __restrict__ out, int* __restrict__ status) {
  constexpr int TPB = 256;
  const int N = p.N, h = blockIdx.y, tid = threadIdx.x;
  const int ell = p.ell_pack, logL = p.logL_pack, L = 1 << logL;
  const u64 Q = p.Q, dmask = (u64)L - 1;
  extern __shared__ u64 sm[];
  u64* gam = sm;                       // [C][N-1]: a'_{K1}[i'+1]
  u64* bet = sm + (size_t)C * N;       // [C][N-1]: a'_{Km}[i']
  u64* W = sm + (size_t)2 * C * N;     // [N] finalisation buffers
  u64* Pb = W + N;
  int m[C], K1[C], dv[C];
  bool ok[C];
#pragma unroll
  for (int c = 0; c < C; c++) {
    const int g = blockIdx.x * C + c;
    ok[c] = g < B;
    int d = ok[c] ? (int)dd[g] : 1;
    if (d < 1 || d > N - 1) {          // out of range: flag, produce zeros for this item
      if (ok[c] && tid == 0 && h == 0) atomicOr(status, 1);
      ok[c] = false; d = 1;
    }
    dv[c] = d;
    const bool br1 = 2 * d <= N;       // F3: d = N/2 takes branch 1
    m[c] = br1 ? d : N - d;
    K1[c] = br1 ? N - d + 1 : 1;
    const u64* a = ct + (size_t)(ok[c] ? g : 0) * 2 * N + N;
    const int Km = K1[c] + m[c] - 1;
    for (int t = tid; t < N - 1; t += TPB) {
      gam[(size_t)c * N + t] = ok[c] ? sx_mask(a, K1[c], t + 2, N, Q) : 0;
      bet[(size_t)c * N + t] = ok[c] ? sx_mask(a, Km, t + 1, N, Q) : 0;
    }
  }
  __syncthreads();
  u64 G[C][CPT], Bs[C][CPT];
#pragma unroll
  for (int c = 0; c < C; c++)
#pragma unroll
    for (int r = 0; r < CPT; r++) { G[c][r] = 0; Bs[c][r] = 0; }

  // sum_{i'} T^{(gamma)}_{i'+1,j} and sum_{i'} T^{(beta)}_{i'+1,j}, as Delta rows (T^{(0)} part is U)
  for (int j = 0; j < ell; j++) {
    const int sh = j * logL;
    const u64* Dj = pk + lay.D + (size_t)j * (N - 1) * (L - 1) * lay.P + (size_t)h * N + tid;
#pragma unroll 1
    for (int t = 0; t < N - 1; t++) {
      const u64* row = Dj + (size_t)t * (L - 1) * lay.P;
      if (BIN) {
        u64 rv[CPT];
#pragma unroll
        for (int r = 0; r < CPT; r++) rv[r] = __ldg(row + r * TPB);
#pragma unroll
        for (int c = 0; c < C; c++) {
          const u64 mg = 0 - ((gam[(size_t)c * N + t] >> sh) & 1);
          const u64 mb = 0 - ((bet[(size_t)c * N + t] >> sh) & 1);
#pragma unroll
          for (int r = 0; r < CPT; r++) {
            G[c][r] = csub(G[c][r] + (rv[r] & mg), Q);
            Bs[c][r] = csub(Bs[c][r] + (rv[r] & mb), Q);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < C; c++) {
          const u64 vg = (gam[(size_t)c * N + t] >> sh) & dmask;
          const u64 vb = (bet[(size_t)c * N + t] >> sh) & dmask;
          if (vg) {
            const u64* rr = row + (vg - 1) * lay.P;
#pragma unroll
            for (int r = 0; r < CPT; r++) G[c][r] = csub(G[c][r] + __ldg(rr + r * TPB), Q);
          }
          if (vb) {
            const u64* rr = row + (vb - 1) * lay.P;
#pragma unroll
            for (int r = 0; r < CPT; r++) Bs[c][r] = csub(Bs[c][r] + __ldg(rr + r * TPB), Q);
          }
        }
      }
    }
  }
  // sum_k X^{k-1} T^{(A_k[1,j])}_{1,j},  A_k[1,j] = digit_j(a[K_k - 1]),  K_k = K1 + k - 1
  int mmax = 0;
#pragma unroll
  for (int c = 0; c < C; c++) mmax = (ok[c] && m[c] > mmax) ? m[c] : mmax;
  for (int j = 0; j < ell; j++) {
    const u64* T1j = pk + lay.T1 + (size_t)j * L * lay.P + (size_t)h * N;
#pragma unroll 1
    for (int k = 1; k <= mmax; k++) {
#pragma unroll
      for (int c = 0; c < C; c++) {
        if (!ok[c] || k > m[c]) continue;
        const int g = blockIdx.x * C + c;
        const u64 av = __ldg(ct + (size_t)g * 2 * N + N + (K1[c] + k - 2));
        const u64* T = T1j + ((av >> (j * logL)) & dmask) * lay.P;
#pragma unroll
        for (int r = 0; r < CPT; r++) {
          const int e = tid + r * TPB - (k - 1);
          const u64 tv = e >= 0 ? __ldg(T + e) : neg_mod(__ldg(T + e + N), Q);
          G[c][r] = add_mod(G[c][r], tv, Q);
        }
      }
    }
  }
  // finalisation per ciphertext:
  //   S = G + U - X^m (U + Bs);  P = [sum_k b_k X^{k-1}, 0] - S  (column h)
  //   branch 1: out = ct X^d + 2P;  branch 2: out = (2P - ct) X^d
  const u64* U = pk + lay.U + (size_t)h * N;
#pragma unroll
  for (int c = 0; c < C; c++) {
    const int g = blockIdx.x * C + c;
    if (!ok[c]) {                                       // uniform across the CTA
      if (g < B)                                        // out-of-range d: zero row (flag raised)
        for (int x = tid; x < N; x += TPB) out[(size_t)g * 2 * N + (size_t)h * N + x] = 0;
      continue;
    }
    const u64* cth = ct + (size_t)g * 2 * N + (size_t)h * N;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < CPT; r++) {
      const int x = tid + r * TPB;
      W[x] = add_mod(__ldg(U + x), Bs[c][r], Q);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < CPT; r++) {
      const int x = tid + r * TPB;
      const int e = x - m[c];
      const u64 rw = e >= 0 ? W[e] : neg_mod(W[e + N], Q);
      const u64 S = sub_mod(add_mod(G[c][r], __ldg(U + x), Q), rw, Q);
      u64 bs = 0;
      if (h == 0 && x < m[c]) bs = __ldg(ct + (size_t)g * 2 * N + (K1[c] + x - 1));
      Pb[x] = sub_mod(bs, S, Q);
    }
    __syncthreads();
    const int d = dv[c];
    const bool br1 = 2 * d <= N;
    u64* o = out + (size_t)g * 2 * N + (size_t)h * N;
#pragma unroll
    for (int r = 0; r < CPT; r++) {
      const int x = tid + r * TPB;
      const u64 cr = rot_coeff(cth, x, d, N, Q);
      if (br1) {
        o[x] = add_mod(cr, add_mod(Pb[x], Pb[x], Q), Q);
      } else {
        const u64 pr = rot_coeff(Pb, x, d, N, Q);
        o[x] = sub_mod(add_mod(pr, pr, Q), cr, Q);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// VectorPack by definition (Pack 1299-1306):
//   out = sum_{k=1}^m X^{k-1+off} ([b_k, 0] - sum_{i,j} pK[i, j, A_k[i,j]]),  A_k = Decomp(a_k)
// one CTA per (item, column); per k the key rows are summed unrotated (coalesced) into
// smem, then rotated once.  off = 0 (VectorPack) or d-1 per item (Pack(c, pK, d)).
template <int CPT>
__global__ void __launch_bounds__(256)
k_vector_pack(DevParams p, const u64* __restrict__ pk, PackLayout lay, const u64* __restrict__ lwe, int m,
              const u32* __restrict__ off, u64* __restrict__ out) {
  constexpr int TPB = 256;
  const int N = p.N, h = blockIdx.y, b = blockIdx.x, tid = threadIdx.x;
  const int ell = p.ell_pack, logL = p.logL_pack, L = 1 << logL;
  const u64 Q = p.Q, dmask = (u64)L - 1;
  extern __shared__ u64 sm[];
  u64* S = sm;                 // [N]
  u64 acc[CPT];
#pragma unroll
  for (int r = 0; r < CPT; r++) acc[r] = 0;
  const int o0 = off ? (int)off[b] - 1 : 0;   // Pack(c, pK, d): message at X^{d-1}
  for (int k = 1; k <= m; k++) {
    const u64* lw = lwe + ((size_t)b * m + (k - 1)) * (N + 1);
    u64 s[CPT];
#pragma unroll
    for (int r = 0; r < CPT; r++) s[r] = 0;
#pragma unroll 1
    for (int i = 0; i < N; i++) {
      const u64 ai = __ldg(lw + 1 + i);
      for (int j = 0; j < ell; j++) {
        const u64 v = (ai >> (j * logL)) & dmask;
        const u64* row = pk + lay.A + (((size_t)i * ell + j) * L + v) * lay.P + (size_t)h * N + tid;
#pragma unroll
        for (int r = 0; r < CPT; r++) s[r] = add_mod(s[r], __ldg(row + r * TPB), Q);
      }
    }
    // t = [b_k, 0] - s  (column h), then acc += X^{k-1+o0} t
    __syncthreads();
#pragma unroll
    for (int r = 0; r < CPT; r++) {
      const int x = tid + r * TPB;
      u64 t = neg_mod(s[r], Q);
      if (h == 0 && x == 0) t = add_mod(t, __ldg(lw), Q);
      S[x] = t;
    }
    __syncthreads();
    const int e = (k - 1 + o0) % (2 * N);
#pragma unroll
    for (int r = 0; r < CPT; r++) acc[r] = add_mod(acc[r], rot_coeff(S, tid + r * TPB, e, N, Q), Q);
  }
#pragma unroll
  for (int r = 0; r < CPT; r++) out[(size_t)b * 2 * N + (size_t)h * N + tid + r * TPB] = acc[r];
}

// ===========================================================================
// Shift as one exact int8 GEMM (L_pack == 2).
// With A_k[i,j] = bit_j(a'_k[i]) the packed sum of Shift's VectorPack is, per ciphertext,
//   G  = sum_{j,i'} gamma_{i',j} Delta_{i'+1,j} + sum_{k<m} X^k S0 + sum_{j,k<m} A_{k+1}[1,j] X^k Delta_{1,j}
//   Bs = sum_{j,i'} beta_{i',j}  Delta_{i'+1,j}
// (S0 = sum_j T^(0)_{1,j}), i.e. a 0/1 matrix (rows: G and Bs of every ciphertext; columns:
// the GK = ell(N-1) + N + ell N "terms") times the key matrix whose row for each term is
// the term polynomial pair.  Key coefficients (< 2^54) are split into 7 balanced base-256
// digits, so the product is 7 int8 GEMMs done as one (N_out = 7 * 2N), exact in int32
// (|sum| <= GK * 128 < 2^31), on the tcgen05 kernel (kernels_imma.cuh) whose epilogue
// recombines the digits mod Q; k_shift_gemm_finish assembles the output.
struct ShiftGemm {
  int K;        // number of terms ell(N-1) + N + ell N
  int Kpad;     // K rounded up to a multiple of 16
  int Nout;     // 7 * 2N
};
static inline ShiftGemm shift_gemm_shape(int N, int ell) {
  ShiftGemm s;
  s.K = ell * (N - 1) + N + ell * N;
  s.Kpad = (s.K + 15) & ~15;
  s.Nout = 7 * 2 * N;
  return s;
}
// term kk, coefficient w (of the 2N-word pair) of the key matrix
FDFB_DEV u64 shift_term(const DevParams& p, const u64* __restrict__ pk, const PackLayout& lay, const u64* __restrict__ S0,
                        int kk, int w) {
  const int N = p.N, ell = p.ell_pack;
  const int h = w / N, x = w % N;
  const int s1 = ell * (N - 1);
  if (kk < s1) {                                  // Delta_{i'+1, j}, j = kk / (N-1), i'+1 = kk % (N-1) + 2
    const int j = kk / (N - 1), t = kk % (N - 1);
    return pk[lay.D + ((size_t)j * (N - 1) + t) * lay.P + w];
  }
  kk -= s1;
  const u64* src;
  int k;
  if (kk < N) { src = S0 + (size_t)h * N; k = kk; }                         // X^k S0
  else {                                                                    // X^k Delta_{1,j}
    kk -= N;
    const int j = kk / N;
    k = kk % N;
    src = pk + lay.T1 + ((size_t)j * 2 + 1) * lay.P + (size_t)h * N;       // T^(1)_{1,j} ...
    const u64* t0 = pk + lay.T1 + ((size_t)j * 2) * lay.P + (size_t)h * N;  // ... minus T^(0)_{1,j}
    const int e = x - k;
    const int ix = e >= 0 ? e : e + N;
    const u64 v = sub_mod(src[ix], t0[ix], p.Q);
    return e >= 0 ? v : neg_mod(v, p.Q);
  }
  const int e = x - k;
  return e >= 0 ? src[e] : neg_mod(src[e + N], p.Q);
}
// S0[h][x] = sum_j T^(0)_{1,j}
__global__ void k_shift_s0(DevParams p, const u64* __restrict__ pk, PackLayout lay, u64* __restrict__ S0) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= 2 * p.N) return;
  u64 s = 0;
  for (int j = 0; j < p.ell_pack; j++) s = add_mod(s, pk[lay.T1 + ((size_t)j * 2) * lay.P + w], p.Q);
  S0[w] = s;
}
// GK[imma_key_row(l, w)][kk] = balanced digit l of term kk (centred mod Q) at coefficient w.
// Tile: 32 terms x 8 coefficients.
__global__ void k_shift_gemm_key(DevParams p, const u64* __restrict__ pk, PackLayout lay, const u64* __restrict__ S0,
                                 ShiftGemm g, int8_t* __restrict__ GK) {
  const int kk = blockIdx.x * 32 + threadIdx.x;
  const int w = blockIdx.y * 8 + threadIdx.y;
  if (w >= 2 * p.N) return;
  u64 v = 0;
  if (kk < g.K) v = shift_term(p, pk, lay, S0, kk, w);
  if (kk >= g.Kpad) return;
  int8_t dg[7];
  balanced_digits7(centred(v, p.Q, 0), dg);
#pragma unroll
  for (int l = 0; l < 7; l++) GK[imma_key_row(l, w) * g.Kpad + kk] = dg[l];
}
// Per-batch 0/1 matrix: rows 2c (G) and 2c+1 (Bs) of ciphertext c.  Grid (ceil(N / blockDim), B):
// thread t computes the SampleExt coefficients it needs once and writes their ell bits with
// stride N-1 / N (coalesced across the warp for every bit j), no per-element division.
__global__ void k_shift_bits(DevParams p, const u64* __restrict__ ct, const u32* __restrict__ dd, int B, ShiftGemm g,
                             int8_t* __restrict__ A, int* __restrict__ status) {
  const int c = blockIdx.y;
  const int N = p.N, ell = p.ell_pack;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;       // 0 .. N-1
  if (t >= N) return;
  int d = (int)dd[c];
  const bool ok = d >= 1 && d <= N - 1;
  if (!ok) { if (t == 0) atomicOr(status, 1); d = 1; }
  const bool br1 = 2 * d <= N;
  const int m = br1 ? d : N - d, K1 = br1 ? N - d + 1 : 1, Km = K1 + m - 1;
  const u64* a = ct + (size_t)c * 2 * N + N;
  int8_t* rg = A + (size_t)(2 * c) * g.Kpad;
  int8_t* rb = rg + g.Kpad;
  const int s1 = ell * (N - 1);
  if (t < N - 1) {                                            // Delta rows (i' = t + 1, bit j)
    const u64 vgw = ok ? sx_mask(a, K1, t + 2, N, p.Q) : 0;
    const u64 vbw = ok ? sx_mask(a, Km, t + 1, N, p.Q) : 0;
    for (int j = 0; j < ell; j++) {
      rg[j * (N - 1) + t] = (int8_t)((vgw >> j) & 1);
      rb[j * (N - 1) + t] = (int8_t)((vbw >> j) & 1);
    }
  }
  rg[s1 + t] = (int8_t)(ok && t < m);                         // E_m S0 rows
  rb[s1 + t] = 0;
  const u64 bw = (ok && t < m) ? a[K1 + t - 1] : 0;          // Toeplitz rows (bit j, k = t)
  for (int j = 0; j < ell; j++) {
    rg[s1 + N + j * N + t] = (int8_t)((bw >> j) & 1);
    rb[s1 + N + j * N + t] = 0;
  }
  for (int kk = g.K + t; kk < g.Kpad; kk += N) { rg[kk] = 0; rb[kk] = 0; }
}
// Assemble Shift's output from the GEMM's recombined rows (V[row][w] mod Q, rows 2c = G and
// 2c+1 = Bs), one CTA of 256 threads per (ciphertext, column):  S = G + U - X^m (U + Bs);  P = [bsum, 0] - S;
// branch 1: out = ct X^d + 2P;  branch 2: out = (2P - ct) X^d.
template <int CPT>
__global__ void __launch_bounds__(256)
k_shift_gemm_finish(DevParams p, const u64* __restrict__ pk, PackLayout lay, const u64* __restrict__ ct,
                    const u32* __restrict__ dd, const u64* __restrict__ V, u64* __restrict__ out) {
  constexpr int TPB = 256;
  const int N = p.N, c = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
  const u64 Q = p.Q;
  __shared__ u64 W[2048];
  __shared__ u64 Pb[2048];
  u64* o = out + (size_t)c * 2 * N + (size_t)h * N;
  int d = (int)dd[c];
  if (d < 1 || d > N - 1) {                     // flagged by k_shift_bits
    for (int x = tid; x < N; x += TPB) o[x] = 0;
    return;
  }
  const bool br1 = 2 * d <= N;
  const int m = br1 ? d : N - d, K1 = br1 ? N - d + 1 : 1;
  const u64* vgr = V + (size_t)(2 * c) * 2 * N + (size_t)h * N;
  const u64* vbr = vgr + 2 * N;
  const u64* U = pk + lay.U + (size_t)h * N;
  u64 G[CPT];
#pragma unroll
  for (int r = 0; r < CPT; r++) {
    const int x = tid + r * TPB;
    G[r] = __ldg(vgr + x);
    W[x] = add_mod(__ldg(U + x), __ldg(vbr + x), Q);
  }
  __syncthreads();
  const u64* cth = ct + (size_t)c * 2 * N + (size_t)h * N;
#pragma unroll
  for (int r = 0; r < CPT; r++) {
    const int x = tid + r * TPB;
    const int e = x - m;
    const u64 rw = e >= 0 ? W[e] : neg_mod(W[e + N], Q);
    const u64 S = sub_mod(add_mod(G[r], __ldg(U + x), Q), rw, Q);
    u64 bs = 0;
    if (h == 0 && x < m) bs = __ldg(ct + (size_t)c * 2 * N + (K1 + x - 1));
    Pb[x] = sub_mod(bs, S, Q);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < CPT; r++) {
    const int x = tid + r * TPB;
    const u64 cr = rot_coeff(cth, x, d, N, Q);
    if (br1) {
      o[x] = add_mod(cr, add_mod(Pb[x], Pb[x], Q), Q);
    } else {
      const u64 pr = rot_coeff(Pb, x, d, N, Q);
      o[x] = sub_mod(add_mod(pr, pr, Q), cr, Q);
    }
  }
}

// ===========================================================================
// Permute(ct, pK, pi) (reading P1: v[j] = Pack(SampleExt(ct, j), pK, 1)):
//   ct_out = ct + sum_{i : pi(i) = j != i} X^{i-1} (v[j] - v[i]),
//   v[j] - v[i] = [b_j - b_i, 0] - sum_{k,l} (pK[k,l,A_j[k,l]] - pK[k,l,A_i[k,l]])
// (A_j = Decomp(SampleExt(ct, j).a); the constant pK[.,.,0] parts cancel for L = 2).
// L == 2: every moved slot i is one GEMM row with coefficients A_j - A_i in {-1, 0, 1} against
// the key matrix of Delta0_{k,l} = pK[k,l,1] - pK[k,l,0] (7 balanced base-256 digits, int8),
// exact in int32 (|sum| <= N ell 128 < 2^31); the GEMM epilogue recombines the digits mod Q,
// k_permute_partial / k_permute_reduce rotate and add.
struct PermGemm { int K; int Nout; };          // K = N ell (multiple of 16), Nout = 7 * 2N
static inline PermGemm perm_gemm_shape(int N, int ell) { PermGemm g; g.K = N * ell; g.Nout = 14 * N; return g; }
static inline size_t perm_gemm_key_bytes(int N, int ell, int L) {
  return L == 2 ? (size_t)14 * N * (size_t)N * ell : 0;
}
// GP[imma_key_row(l, w)][k*ell + j] = digit l of Delta0_{k,j}[w] (centred mod Q)
__global__ void k_perm_gemm_key(DevParams p, const u64* __restrict__ pk, PackLayout lay, PermGemm g,
                                int8_t* __restrict__ GP) {
  const int kk = blockIdx.x * 32 + threadIdx.x;   // (k, j) row of the canonical table
  const int w = blockIdx.y * 8 + threadIdx.y;
  if (kk >= g.K || w >= 2 * p.N) return;
  const u64* e = pk + lay.A + (size_t)kk * 2 * lay.P;                    // pK[k,j,0], then pK[k,j,1]
  int8_t dg[7];
  balanced_digits7(centred(sub_mod(e[lay.P + w], e[w], p.Q), p.Q, 0), dg);
#pragma unroll
  for (int l = 0; l < 7; l++) GP[imma_key_row(l, w) * g.K + kk] = dg[l];
}
// rows r = c_local * N + (i-1) of a chunk of ciphertexts: A[r][k*ell + l] = bit_l(a'_j[k]) - bit_l(a'_i[k]),
// j = pi(i); zero rows for fixed points (and flag an invalid permutation entry).  One CTA of
// (64, 4) threads per row: threadIdx.x = bit l, threadIdx.y strides over k (coalesced per k).
__global__ void __launch_bounds__(256)
k_perm_bits(DevParams p, const u64* __restrict__ ct, const u32* __restrict__ perm, int c0, int nct,
            PermGemm g, int8_t* __restrict__ A, int* __restrict__ status) {
  const int N = p.N, ell = p.ell_pack;
  const int r = blockIdx.x;                         // local row
  const int c = c0 + r / N, i = r % N + 1;          // 1-based slot
  int j = (int)perm[(size_t)c * N + (i - 1)];
  if (j < 1 || j > N) { if (threadIdx.x == 0 && threadIdx.y == 0) atomicOr(status, 1); j = i; }
  const u64* a = ct + (size_t)c * 2 * N + N;
  int8_t* row = A + (size_t)r * g.K;
  const int l = threadIdx.x;
  if (l >= ell) return;
  for (int k = 1 + threadIdx.y; k <= N; k += blockDim.y) {   // SampleExt index k (1-based)
    int8_t v = 0;
    if (j != i) {
      const int bj = (int)((sx_mask(a, j, k, N, p.Q) >> l) & 1), bi = (int)((sx_mask(a, i, k, N, p.Q) >> l) & 1);
      v = (int8_t)(bj - bi);
    }
    row[(k - 1) * ell + l] = v;
  }
}
// out[c] = ct[c] + sum_{i moved} X^{i-1} ([b_j - b_i, 0] - W_i).  One CTA per (ciphertext,
// column, slice of PERM_SLICES consecutive slots i): partial sums into part[c][h][slice][N]
// (slice 0 also carries ct), summed by k_permute_reduce.
#define PERM_SLICES 32
template <int CPT>
__global__ void __launch_bounds__(256)
k_permute_partial(DevParams p, const u64* __restrict__ ct, const u32* __restrict__ perm, int c0, PermGemm g,
                  const u64* __restrict__ V, u64* __restrict__ part) {
  constexpr int TPB = 256;
  const int N = p.N, cl = blockIdx.x, h = blockIdx.y, sl = blockIdx.z, tid = threadIdx.x;
  const int c = c0 + cl;
  const u64 Q = p.Q;
  __shared__ u64 W[2048];
  const u64* cth = ct + (size_t)c * 2 * N;
  u64 acc[CPT];
#pragma unroll
  for (int r = 0; r < CPT; r++) acc[r] = sl == 0 ? cth[(size_t)h * N + tid + r * TPB] : 0;
  const int per = N / PERM_SLICES;
  for (int i = 1 + sl * per; i <= (sl + 1) * per; i++) {
    int j = (int)perm[(size_t)c * N + (i - 1)];
    if (j < 1 || j > N || j == i) continue;                      // uniform across the CTA
    const u64* vrow = V + ((size_t)cl * N + (i - 1)) * 2 * N + (size_t)h * N;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < CPT; r++) {
      const int x = tid + r * TPB;
      u64 t = neg_mod(__ldg(vrow + x), Q);                        // -W_i
      if (h == 0 && x == 0) t = add_mod(t, sub_mod(cth[j - 1], cth[i - 1], Q), Q);   // + [b_j - b_i, 0]
      W[x] = t;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < CPT; r++) acc[r] = add_mod(acc[r], rot_coeff(W, tid + r * TPB, i - 1, N, Q), Q);
  }
  u64* o = part + (((size_t)cl * 2 + h) * PERM_SLICES + sl) * N;
#pragma unroll
  for (int r = 0; r < CPT; r++) o[tid + r * TPB] = acc[r];
}
__global__ void k_permute_reduce(DevParams p, const u64* __restrict__ part, int c0, int nct, u64* __restrict__ out) {
  const int N = p.N;
  const size_t total = (size_t)nct * 2 * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    const size_t ch = x / N, w = x % N;                           // (local ciphertext, column), coefficient
    const u64* src = part + ch * PERM_SLICES * N + w;
    u64 s = 0;
#pragma unroll 8
    for (int k = 0; k < PERM_SLICES; k++) s = add_mod(s, __ldg(src + (size_t)k * N), p.Q);
    out[(size_t)c0 * 2 * N + x] = s;
  }
}
// Definition path for any L (small N): per (ciphertext, column) CTA, every moved slot's
// v[j] - v[i] gathered from the canonical table, rotated by X^{i-1} and added.
template <int CPT>
__global__ void __launch_bounds__(256)
k_permute_direct(DevParams p, const u64* __restrict__ pk, PackLayout lay, const u64* __restrict__ ct,
                 const u32* __restrict__ perm, u64* __restrict__ out, int* __restrict__ status) {
  constexpr int TPB = 256;
  const int N = p.N, c = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
  const int ell = p.ell_pack, logL = p.logL_pack, L = 1 << logL;
  const u64 Q = p.Q, dmask = (u64)L - 1;
  __shared__ u64 W[2048];
  const u64* cth = ct + (size_t)c * 2 * N;
  const u64* a = cth + N;
  u64 acc[CPT];
#pragma unroll
  for (int r = 0; r < CPT; r++) acc[r] = cth[(size_t)h * N + tid + r * TPB];
  for (int i = 1; i <= N; i++) {
    int j = (int)perm[(size_t)c * N + (i - 1)];
    if (j < 1 || j > N) { if (tid == 0 && h == 0) atomicOr(status, 1); continue; }
    if (j == i) continue;
    u64 s[CPT];
#pragma unroll
    for (int r = 0; r < CPT; r++) s[r] = 0;
    for (int k = 1; k <= N; k++) {
      const u64 aj = sx_mask(a, j, k, N, Q), ai = sx_mask(a, i, k, N, Q);
      for (int l = 0; l < ell; l++) {
        const u64 vj = (aj >> (l * logL)) & dmask, vi = (ai >> (l * logL)) & dmask;
        if (vj == vi) continue;
        const u64* rj = pk + lay.A + (((size_t)(k - 1) * ell + l) * L + vj) * lay.P + (size_t)h * N + tid;
        const u64* ri = pk + lay.A + (((size_t)(k - 1) * ell + l) * L + vi) * lay.P + (size_t)h * N + tid;
#pragma unroll
        for (int r = 0; r < CPT; r++) s[r] = add_mod(s[r], sub_mod(__ldg(ri + r * TPB), __ldg(rj + r * TPB), Q), Q);
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < CPT; r++) {
      const int x = tid + r * TPB;
      u64 t = s[r];                                                  // -(sum pK[.,A_j] - sum pK[.,A_i])
      if (h == 0 && x == 0) t = add_mod(t, sub_mod(cth[j - 1], cth[i - 1], Q), Q);
      W[x] = t;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < CPT; r++) acc[r] = add_mod(acc[r], rot_coeff(W, tid + r * TPB, i - 1, N, Q), Q);
  }
#pragma unroll
  for (int r = 0; r < CPT; r++) out[(size_t)c * 2 * N + (size_t)h * N + tid + r * TPB] = acc[r];
}
