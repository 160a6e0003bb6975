// kernels_core.cuh -- batched NTT utilities, keygen/encryption and key-format kernels.
#pragma once
#include "ntt.cuh"

// Montgomery multiplication (R = 2^64) for products of two variable residues
// (PubMux ring products, keygen).  a, b < 2^64 with a*b < Q*2^64; out in [0, 2Q).
FDFB_DEV u64 mont_mul(u64 a, u64 b, u64 Q, u64 qinv_neg) {
  u64 lo = a * b, hi = __umul64hi(a, b);
  u64 m = lo * qinv_neg;
  u64 mq_hi = __umul64hi(m, Q);
  return hi + mq_hi + (lo != 0 ? 1 : 0);
}

// ---------------------------------------------------------------------------
// Generic batched transform: one polynomial per N/8-thread group, G groups per CTA.
// mode 0: forward NTT of canonical input, output reduced to [0, Q) in bit-reversed slots
// mode 1: inverse NTT of [0, Q) slots, times N^{-1}, natural order output in [0, Q)
template <int N>
__global__ void k_ntt_batch(DevParams p, u64* __restrict__ data, int count, int mode) {
  constexpr int T = N / 8;
  extern __shared__ u64 smem[];
  const int grp = threadIdx.y, tid = threadIdx.x;
  const int poly = blockIdx.x * blockDim.y + grp;
  u64* sb = smem + (size_t)grp * N;
  const bool active = poly < count;
  u64* a = data + (size_t)(active ? poly : 0) * N;
  u64 x[8];
  if (mode == 0) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = active ? a[tid + T * k] : 0;
    ntt_fwd<N>(x, sb, tid, p);
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = csub(csub(x[k], p.Q2), p.Q);
    if (active) {
#pragma unroll
      for (int k = 0; k < 8; k++) a[8 * tid + k] = x[k];
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = active ? a[8 * tid + k] : 0;
    ntt_inv<N>(x, sb, tid, p);
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = csub(mul_shoup_lazy(x[k], p.ninv, p.ninvp, p.Q), p.Q);
    if (active) {
#pragma unroll
      for (int k = 0; k < 8; k++) a[tid + T * k] = x[k];
    }
  }
}

// c[i] = a[i] * b[i] mod Q (pointwise, Montgomery with R^2 correction), both [0, Q)
__global__ void k_pointwise_mul(const u64* __restrict__ a, const u64* __restrict__ b, u64* __restrict__ c,
                                size_t total, size_t b_period, u64 Q, u64 qinv_neg, u64 r2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    u64 t = csub(mont_mul(a[i], b[i % b_period], Q, qinv_neg), Q);
    c[i] = csub(mont_mul(t, r2, Q, qinv_neg), Q);
  }
}

// ---------------------------------------------------------------------------
// Secrets: s: domain 1, s_rlwe: domain 2, word i.
__global__ void k_keygen_secrets(DevParams p, u64 seed, int8_t* s_lwe, int8_t* s_rlwe) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p.n) s_lwe[i] = (int8_t)key_coeff(rnd_word(seed, 1, 0, 0, 0, i), p.lwe_ternary);
  if (i < p.N) s_rlwe[i] = (int8_t)key_coeff(rnd_word(seed, 2, 0, 0, 0, i), p.rlwe_ternary);
}

// Canonical RLWE entry descriptor: which message the encryption carries.
// kind BRK: RGSW row (gadget on b for row<ell, on a otherwise) of Y[i,j];
// BPK: constant s_F[i] L_pk^j; PACK: constant s_F[i] L_pack^j k.
struct EntryDesc {
  int dom;                // Philox domain
  u64 i0, i1, i2;         // object indices
  int gadget_col;         // -1: message in b's constant term only; 0/1: add m*g at coefficient 0 of col
  u64 m0;                 // constant message (mod Q) placed at coefficient 0 of column gadget_col (or b)
};

FDFB_DEV int y_of(int si, int j, int ternary) {
  if (!ternary) return si;
  return (j == 0) ? (si == -1) : (si == 1);
}
FDFB_DEV u64 pow2_mod(int e, u64 Q) {   // 2^e mod Q
  u64 r = 1 % Q, b = 2;
  while (e) { if (e & 1) r = mul_mod_slow(r, b, Q); b = mul_mod_slow(b, b, Q); e >>= 1; }
  return r;
}

// Stage 1 of RLWE encryption for a list of entries: write the uniform mask a (coef domain)
// into out[e][1] and compute its NTT later; errors and messages are added in stage 3.
// entry e's flat canonical index comes from idx[e]; kind selects the decoding.
FDFB_DEV EntryDesc decode_entry(const DevParams& p, int kind, u64 flat, const int8_t* s_lwe, const int8_t* s_rlwe) {
  EntryDesc d;
  const u64 Q = p.Q;
  if (kind == 1) {            // BRK: flat = (i*u + j)*2ell + row
    int ell = p.ell_rgsw;
    int row = (int)(flat % (2 * ell));
    int j = (int)((flat / (2 * ell)) % p.u);
    int i = (int)(flat / (2 * ell * p.u));
    d.dom = 3; d.i0 = i; d.i1 = j; d.i2 = row;
    int y = y_of(s_lwe[i], j, p.lwe_ternary);
    d.m0 = y ? pow2_mod(p.logL_rgsw * (row % ell), Q) : 0;
    d.gadget_col = row < ell ? 0 : 1;
  } else if (kind == 2) {     // BPK: flat = i*ell_pk + j
    int j = (int)(flat % p.ell_pk), i = (int)(flat / p.ell_pk);
    d.dom = 4; d.i0 = i; d.i1 = j; d.i2 = 0;
    d.m0 = mul_mod_slow(from_signed(s_rlwe[i], Q), pow2_mod(p.logL_pk * j, Q), Q);
    d.gadget_col = 0;
  } else {                    // PACK: flat = (i*ell + j)*L + k
    int L = 1 << p.logL_pack;
    int k = (int)(flat % L), j = (int)((flat / L) % p.ell_pack), i = (int)(flat / ((u64)L * p.ell_pack));
    d.dom = 6; d.i0 = i; d.i1 = j; d.i2 = k;
    d.m0 = mul_mod_slow(mul_mod_slow(from_signed(s_rlwe[i], Q), pow2_mod(p.logL_pack * j, Q), Q), (u64)k, Q);
    d.gadget_col = 0;
  }
  return d;
}

// mask a for entry e -> work[e*N ..] (coef domain)
__global__ void k_rlwe_mask(DevParams p, int kind, const u64* __restrict__ idx, u64 idx_base, int count,
                            u64 seed, const int8_t* s_lwe, const int8_t* s_rlwe, u64* __restrict__ outmask) {
  int e = blockIdx.y;
  if (e >= count) return;
  u64 flat = idx ? idx[e] : idx_base + e;
  EntryDesc d = decode_entry(p, kind, flat, s_lwe, s_rlwe);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.N; c += gridDim.x * blockDim.x) {
    u64 hi = rnd_word(seed, d.dom, d.i0, d.i1, d.i2, 2 * (u64)c);
    u64 lo = rnd_word(seed, d.dom, d.i0, d.i1, d.i2, 2 * (u64)c + 1);
    outmask[(size_t)e * p.N + c] = uniform_mod_q(hi, lo, p.Q);
  }
}
// b = INTT(NTT(a) * NTT(s)) + m + e  ->  out[e] = [b, a]; prod holds a*s (coef domain, [0,Q))
__global__ void k_rlwe_finish(DevParams p, int kind, const u64* __restrict__ idx, u64 idx_base, int count,
                              u64 seed, const int8_t* s_lwe, const int8_t* s_rlwe, const u64* __restrict__ mask,
                              const u64* __restrict__ prod, u64* __restrict__ out) {
  int e = blockIdx.y;
  if (e >= count) return;
  u64 flat = idx ? idx[e] : idx_base + e;
  EntryDesc d = decode_entry(p, kind, flat, s_lwe, s_rlwe);
  const u64 Q = p.Q;
  u64* o = out + (size_t)e * 2 * p.N;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.N; c += gridDim.x * blockDim.x) {
    long long err = gauss_cdt(rnd_word(seed, d.dom, d.i0, d.i1, d.i2, 2 * (u64)p.N + c), p);
    u64 b = add_mod(prod[(size_t)e * p.N + c], from_signed(err, Q), Q);
    u64 a = mask[(size_t)e * p.N + c];
    if (c == 0) {
      if (d.gadget_col == 0) b = add_mod(b, d.m0, Q);
      else a = add_mod(a, d.m0, Q);
    }
    o[c] = b;
    o[p.N + c] = a;
  }
}
// generic RLWE encryption of arbitrary message polynomials (domain 8, object c)
__global__ void k_rlwe_enc_mask(DevParams p, u64 seed, int count, u64 obj0, u64* __restrict__ outmask) {
  int e = blockIdx.y;
  const u64 obj = obj0 + e;                          // global object index (sharded batches)
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.N; c += gridDim.x * blockDim.x) {
    u64 hi = rnd_word(seed, 8, obj, 0, 0, 2 * (u64)c), lo = rnd_word(seed, 8, obj, 0, 0, 2 * (u64)c + 1);
    outmask[(size_t)e * p.N + c] = uniform_mod_q(hi, lo, p.Q);
  }
}
__global__ void k_rlwe_enc_finish(DevParams p, u64 seed, int count, u64 obj0, const u64* __restrict__ msg,
                                  const u64* __restrict__ mask, const u64* __restrict__ prod, u64* __restrict__ out) {
  int e = blockIdx.y;
  const u64 Q = p.Q;
  const u64 obj = obj0 + e;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < p.N; c += gridDim.x * blockDim.x) {
    long long err = gauss_cdt(rnd_word(seed, 8, obj, 0, 0, 2 * (u64)p.N + c), p);
    size_t o = (size_t)e * p.N + c;
    out[(size_t)e * 2 * p.N + c] = add_mod(add_mod(prod[o], msg[o] % Q, Q), from_signed(err, Q), Q);
    out[(size_t)e * 2 * p.N + p.N + c] = mask[o];
  }
}

// LWE encryption mod 2^w of mu under s (dim n): one warp per sample.
FDFB_DEV void lwe_encrypt_warp(const DevParams& p, u64 seed, int dom, u64 i0, u64 i1, const int8_t* s, u64 mu,
                               u64* out, int lane) {
  const int sh = 64 - p.log_q_lwe;
  u64 acc = 0;
  for (int i = lane; i < p.n; i += 32) {
    u64 ai = rnd_word(seed, dom, i0, i1, 0, i) >> sh;
    out[1 + i] = ai;
    acc += ai * (u64)(long long)s[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    long long e = gauss_cdt(rnd_word(seed, dom, i0, i1, 0, p.n), p);
    out[0] = (acc + mu + (u64)e) & p.q_mask;
  }
}
// ksK[i,j] = LWE_s(s_F[i] L_ks^j) mod q_lwe  (domain 5)
__global__ void k_ksk_gen(DevParams p, u64 seed, const int8_t* s_lwe, const int8_t* s_rlwe,
                          const u64* __restrict__ idx, u64 idx_base, int count, u64* __restrict__ out) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= count) return;
  u64 flat = idx ? idx[w] : idx_base + w;
  int j = (int)(flat % p.ell_ks), i = (int)(flat / p.ell_ks);
  u64 mu = ((u64)(long long)s_rlwe[i] << (p.logL_ks * j)) & p.q_mask;
  lwe_encrypt_warp(p, seed, 5, i, j, s_lwe, mu, out + (size_t)w * (p.n + 1), lane);
}
// input ciphertexts of m in Z_t (domain 7).  flags bit0: mod-switch-exact variant.
__global__ void k_lwe_encrypt(DevParams p, u64 seed, const int8_t* s_lwe, const u64* __restrict__ msg, int count,
                              u32 flags, u64 obj0, u64* __restrict__ out) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= count) return;
  const u64 obj = obj0 + w;                          // global object index (sharded batches)
  const u64 delta = (1ULL << p.log_q_lwe) / p.t;
  u64* o = out + (size_t)w * (p.n + 1);
  if (flags & 1) {
    const int log2N = p.logN + 1;
    const u64 step = 1ULL << (p.log_q_lwe - log2N);
    u64 acc = 0;
    for (int i = lane; i < p.n; i += 32) {
      u64 ai = (rnd_word(seed, 7, obj, 0, 0, i) >> (64 - log2N)) * step;
      o[1 + i] = ai;
      acc += ai * (u64)(long long)s_lwe[i];
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) o[0] = (acc + delta * msg[w]) & p.q_mask;
  } else {
    lwe_encrypt_warp(p, seed, 7, obj, 0, s_lwe, delta * msg[w], o, lane);
  }
}

