// kernels_br.cuh -- the batched blind rotation, the hot kernel.
//
// One CTA of T = N/8 threads per accumulator; the accumulator (canonical, mod Q) stays in
// shared memory for all n*u CMux steps; 512/T CTAs per SM (<= 128 registers per thread).
// One CMux step (CMux(C, g, h) = extProd(C, g - h) + h; extProd 2906):
//   d = acc X^e - acc,  D_r = Decomp_{L,Q}(d)[r] (unsigned digits < L)
//   acc_c += ( sum_{r < 2 ell} D_r * brK[i,j][r][c] ) mod Q          for c in {b, a}
//
// Exact RNS evaluation of the external product.  The products D_r * K (negacyclic, over
// the integers, K in [0, Q)) have |coefficients| < 2 ell N (L-1) Q (< 2^82 at the Large
// configuration), so they are computed exactly modulo NP word-size NTT primes
// (P = prod p_i > 8/3 bound; 2^27 < p_i < 2^28) with 32-bit Harvey/Shoup arithmetic, and the signed
// integer result is recovered by CRT and reduced mod Q.  The result is the same residue
// vector as the schoolbook definition (bit-exact with any correct evaluation); it costs
// ~4 IMAD slots per 30-bit butterfly instead of ~16-22 for a 54-bit Shoup butterfly.
//
// Per CMux: d once (both halves); then per prime p: 2 ell forward NTT_p of the digit
// polynomials (pairs of digits per transform; registers, radix-8 passes, smem exchanges in
// two alternating buffers), lazy 64-bit MAC against the NTT_p-domain key (u32, N^{-1} y_p 2^32
// folded in), Montgomery reduction, one paired inverse NTT_p of both columns, and the prime's
// CRT term added to acc (the rounding k = round(sum t_i / p_i) and acc -= k P mod Q after the
// last prime).  For Q < 2^28 the single prime p = Q computes the products directly mod Q.
//
// Kernels: k_blind_rotate (batched: one CTA per accumulator, persistent over the batch, also
// the shift-based BR's CMux in GIN mode) and k_blind_rotate_cl (small passes: a thread-block
// cluster of NP or 2 NP CTAs per accumulator, one prime [and one d half] per CTA, partial
// residues combined through distributed shared memory).
//
// Twiddles: pass-grouped tables of (w, w') u32 pairs per prime (fdfb_api.cu
// make_rns_tables), 8 pairs per group (7 used) -> one base per pass, 16-byte loads.
// brK device format: [n*u steps][NP primes][2 ell rows][2 cols][N slots] u32.
#pragma once
#include <cooperative_groups.h>
#include "kernels_core.cuh"
#include "kernels_imma.cuh"   // mbarrier / TMEM helpers

#define RNS_MAXP 3

template <int N>
struct BrShape {
  static constexpr int LOGN = (N == 256) ? 8 : (N == 512) ? 9 : (N == 1024) ? 10 : 11;
  static constexpr int T = N / 8;
  static constexpr int NMID = (LOGN - 1) / 3;      // radix-8 passes on T1-strided positions
  static constexpr int PLAST = LOGN - 3 * NMID;    // stages of the final pass (1..3)
  static constexpr int NLAST = 8 - (8 >> PLAST);   // twiddle pairs per thread in the final pass
  static constexpr int MINB = 512 / T;             // CTAs per SM
  static constexpr int grp(int q) {                // groups before pass q (8 pairs per group)
    int o = 0, g = 1;
    for (int i = 0; i < q; i++) { o += g; g *= 8; }
    return o;
  }
  static constexpr int G_LAST = grp(NMID);
  static constexpr int GROUPS = G_LAST + T;        // one group per thread in the final pass
  static constexpr int PAIRS = 8 * GROUPS;         // per prime and direction
};

// Per-context RNS constants (passed by value).
struct RnsParams {
  int np;
  u32 p[RNS_MAXP], p2[RNS_MAXP];          // primes, 2p
  u32 pinv[RNS_MAXP];                     // -p^{-1} mod 2^32 (Montgomery reduction of the MAC)
  u32 ninv[RNS_MAXP], ninvs[RNS_MAXP];    // N^{-1} y_i 2^32 mod p (key import; y_i: CRT below)
  // CRT: t_i = r_i y_i mod p_i with y_i = (P/p_i)^{-1} mod p_i;  V = sum t_i M_i - k P
  u32 y[RNS_MAXP], ys[RNS_MAXP];          // y_i and its Shoup companion
  u64 M[RNS_MAXP];                        // (P/p_i) mod Q
  u32 Ms32[RNS_MAXP];                     // floor(M_i 2^32 / Q): Shoup quotient for 28-bit t_i
  u64 pq;                                 // P mod Q
  u32 f16[RNS_MAXP];                      // floor(2^36 / p_i): 16 t_i / p_i = umulhi(t_i, f16) (+ < 1)
  u32 zero;                               // 0, opaque to the compiler (see bfw32)
  const uint4* ftab;                      // [np][GROUPS][8 pairs] forward (w, w') u32
  const uint4* itab;                      // inverse
};

FDFB_DEV u32 shoup32(u32 a, u32 w, u32 ws, u32 p) {     // a*w mod p in [0, 2p), any a < 2^32
  const u32 q = __umulhi(a, ws);
  return a * w - q * p;
}
FDFB_DEV u32 csub32(u32 x, u32 m) { return min(x, x - m); }

// Harvey butterflies.  ptxas issues two-input integer adds as IMAD.IADD on the (binding)
// multiply pipe; every add here therefore carries a third, opaque zero operand z (a kernel
// parameter the compiler cannot fold), which keeps it a 3-input IADD3 on the ALU pipe.
// Conditional subtractions are unsigned min (VIADDMNMX).  Needs 6p < 2^32 (p < 2^29).
// Forward butterflies are lazy (no reduction): a stage adds at most 2p to the bound.  With
// p < 2^28 values may grow to 16p < 2^32, so the transform tracks its bound at compile time
// and subtracts 8p conditionally (red8p_all) only before a pass that would overflow: twice per
// 2048-point transform instead of a conditional subtraction per butterfly.
FDFB_DEV void bfw32(u32& X, u32& Y, u32 w, u32 ws, u32 p, u32 p2, u32 z) {   // CT, +2p per stage
  const u32 t = shoup32(Y, w, ws, p);                                   // [0, 2p)
  const u32 x = X;
  X = x + t + z;
  Y = x - t + p2;
}
FDFB_DEV u32 red16(u32 x, u32 p2) {                                                   // [0, 16p) -> [0, 2p)
  return csub32(csub32(csub32(x, p2 << 2), p2 << 1), p2);
}
FDFB_DEV void bin32(u32& X, u32& Y, u32 w, u32 ws, u32 p, u32 p2, u32 z) {   // GS, [0, 2p)
  const u32 x = X, y = Y;
  X = csub32(x + y + z, p2);                                            // [0, 2p)
  Y = shoup32(x - y + p2, w, ws, p);                                    // [0, 2p)
}

// 8 pairs of a group: tw[0] stage-0, tw[1..2] stage-1, tw[3..6] stage-2 (tw[7] padding)
struct Tw8 { u32 w[8], s[8]; };
FDFB_DEV void load_tw8(Tw8& t, const uint4* g) {
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const uint4 v = __ldg(g + i);
    t.w[2 * i] = v.x; t.s[2 * i] = v.y; t.w[2 * i + 1] = v.z; t.s[2 * i + 1] = v.w;
  }
}
// V polynomials (V = 1 or 2) share every twiddle: twice the ILP and half the twiddle
// loads per polynomial when two digit (or two column) transforms run together.
template <int V>
FDFB_DEV void fwd8_32(u32 (&x)[V][8], const uint4* g, u32 p, u32 p2, u32 z) {
  Tw8 t; load_tw8(t, g);
#pragma unroll
  for (int v = 0; v < V; v++) {
#pragma unroll
    for (int k = 0; k < 4; k++) bfw32(x[v][k], x[v][k + 4], t.w[0], t.s[0], p, p2, z);
  }
#pragma unroll
  for (int v = 0; v < V; v++) {
    bfw32(x[v][0], x[v][2], t.w[1], t.s[1], p, p2, z); bfw32(x[v][1], x[v][3], t.w[1], t.s[1], p, p2, z);
    bfw32(x[v][4], x[v][6], t.w[2], t.s[2], p, p2, z); bfw32(x[v][5], x[v][7], t.w[2], t.s[2], p, p2, z);
  }
#pragma unroll
  for (int v = 0; v < V; v++) {
#pragma unroll
    for (int k = 0; k < 4; k++) bfw32(x[v][2 * k], x[v][2 * k + 1], t.w[3 + k], t.s[3 + k], p, p2, z);
  }
}
// bound bookkeeping (in units of p): a radix-8 pass adds 6, the final pass 2 PLAST.  Before a
// pass that would leave [0, 16p), one conditional subtraction of 8p maps [0, B p) to
// [0, max(8, B - 8) p) (B <= 16): one VIADDMNMX per value instead of a full reduction.
template <int V>
FDFB_DEV void red8p_all(u32 (&x)[V][8], u32 p2) {
  const u32 p8 = p2 << 2;
#pragma unroll
  for (int v = 0; v < V; v++)
#pragma unroll
    for (int k = 0; k < 8; k++) x[v][k] = csub32(x[v][k], p8);
}
constexpr int after_red8p(int b) { return b - 8 > 8 ? b - 8 : 8; }
template <int V>
FDFB_DEV void inv8_32(u32 (&x)[V][8], const uint4* g, u32 p, u32 p2, u32 z) {
  Tw8 t; load_tw8(t, g);
#pragma unroll
  for (int v = 0; v < V; v++) {
#pragma unroll
    for (int k = 0; k < 4; k++) bin32(x[v][2 * k], x[v][2 * k + 1], t.w[3 + k], t.s[3 + k], p, p2, z);
  }
#pragma unroll
  for (int v = 0; v < V; v++) {
    bin32(x[v][0], x[v][2], t.w[1], t.s[1], p, p2, z); bin32(x[v][1], x[v][3], t.w[1], t.s[1], p, p2, z);
    bin32(x[v][4], x[v][6], t.w[2], t.s[2], p, p2, z); bin32(x[v][5], x[v][7], t.w[2], t.s[2], p, p2, z);
  }
#pragma unroll
  for (int v = 0; v < V; v++) {
#pragma unroll
    for (int k = 0; k < 4; k++) bin32(x[v][k], x[v][k + 4], t.w[0], t.s[0], p, p2, z);
  }
}
// final pass on positions 8 tid + k: P stages with pair distance t = 2^{P-1-s}; stage s
// uses 8 >> (P - s) consecutive pairs of the thread's group
template <int P, int V>
FDFB_DEV void fwd_last32_t(u32 (&x)[V][8], const Tw8& t, u32 p, u32 p2, u32 z) {
  int o = 0;
#pragma unroll
  for (int s = 0; s < P; s++) {
    const int d = 1 << (P - 1 - s);
#pragma unroll
    for (int v = 0; v < V; v++) {
#pragma unroll
      for (int k = 0; k < 8; k++)
        if ((k & d) == 0) bfw32(x[v][k], x[v][k + d], t.w[o + (k >> (P - s))], t.s[o + (k >> (P - s))], p, p2, z);
    }
    o += 8 >> (P - s);
  }
}
template <int P, int V>
FDFB_DEV void fwd_last32(u32 (&x)[V][8], const uint4* g, u32 p, u32 p2, u32 z) {
  Tw8 t; load_tw8(t, g);
  fwd_last32_t<P, V>(x, t, p, p2, z);
}
// the thread's final-pass group held in TMEM (16 words: (w, w') pairs), see k_blind_rotate_p
FDFB_DEV void load_tw8_tmem(Tw8& t, uint32_t taddr) {
  u32 v[16];
  tmem_ld16(taddr, v);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 8; i++) { t.w[i] = v[2 * i]; t.s[i] = v[2 * i + 1]; }
}
template <int P, int V>
FDFB_DEV void inv_last32_t(u32 (&x)[V][8], const Tw8& t, u32 p, u32 p2, u32 z) {
  int o = 8 - (8 >> P);
#pragma unroll
  for (int s = P - 1; s >= 0; s--) {
    const int d = 1 << (P - 1 - s);
    o -= 8 >> (P - s);
#pragma unroll
    for (int v = 0; v < V; v++) {
#pragma unroll
      for (int k = 0; k < 8; k++)
        if ((k & d) == 0) bin32(x[v][k], x[v][k + d], t.w[o + (k >> (P - s))], t.s[o + (k >> (P - s))], p, p2, z);
    }
  }
}
template <int P, int V>
FDFB_DEV void inv_last32(u32 (&x)[V][8], const uint4* g, u32 p, u32 p2, u32 z) {
  Tw8 t; load_tw8(t, g);
  inv_last32_t<P, V>(x, t, p, p2, z);
}

// Exchange-buffer layouts.  Exchange x (between radix-8 pass x and x+1) stores logical
// position e at L_x(e) = e + m_x (e >> s_x); every (s_x, m_x) below maps each warp's 256
// positions into its own 288-word slab (so warp-local passes never touch another warp's
// slab) and is bank-conflict free for both the writing and the reading pass (checked
// exhaustively).  For a pass pattern e = B(tid) + S k the address is L_x(B) + S k +
// m_x ((S k) >> s_x): a per-thread base plus compile-time offsets.  V polynomials use V
// planes of WORDS words.
template <int N>
struct Lay {
  static constexpr int S(int x) { return (x == BrShape<N>::NMID - 1) ? 3 : (N == 1024 && x == 1) ? 4 : 5; }
  static constexpr int M(int x) { return (x == BrShape<N>::NMID - 1) ? 1 : (N == 1024 && x == 1) ? 2 : 4; }
  static constexpr int WORDS = N + N / 8;
};
template <int N, int X>
FDFB_DEV int lay_base(int e) { return e + Lay<N>::M(X) * (e >> Lay<N>::S(X)); }
template <int N, int X>
FDFB_DEV constexpr int lay_off(int S, int k) { return S * k + Lay<N>::M(X) * ((S * k) >> Lay<N>::S(X)); }

// pass-q position pattern: B = (tid / T1) 8 T1 + tid % T1, stride T1
template <int N, int q>
FDFB_DEV int qbase(int tid) { constexpr int T1 = N >> (3 * q + 3); return (tid / T1) * 8 * T1 + (tid % T1); }

template <int N, int X, int V>
FDFB_DEV void xload(u32 (&x)[V][8], const u32* sb, int base, int S) {
  if constexpr (V == 2) {          // two polynomials per 64-bit word (layouts are conflict-free for 8-byte words too)
    const uint2* s2 = reinterpret_cast<const uint2*>(sb);
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const uint2 v = s2[base + lay_off<N, X>(S, k)];
      x[0][k] = v.x; x[1][k] = v.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; v++)
#pragma unroll
      for (int k = 0; k < 8; k++) x[v][k] = sb[v * Lay<N>::WORDS + base + lay_off<N, X>(S, k)];
  }
}
template <int N, int X, int V>
FDFB_DEV void xstore(const u32 (&x)[V][8], u32* sb, int base, int S) {
  if constexpr (V == 2) {
    uint2* s2 = reinterpret_cast<uint2*>(sb);
#pragma unroll
    for (int k = 0; k < 8; k++) s2[base + lay_off<N, X>(S, k)] = make_uint2(x[0][k], x[1][k]);
  } else {
#pragma unroll
    for (int v = 0; v < V; v++)
#pragma unroll
      for (int k = 0; k < 8; k++) sb[v * Lay<N>::WORDS + base + lay_off<N, X>(S, k)] = x[v][k];
  }
}

template <int N, int q, int V, int BOUND>
FDFB_DEV void fwd_mid(u32 (&x)[V][8], u32* sb, int tid, const uint4* tab, u32 p, u32 p2, u32 z) {
  if constexpr (q < BrShape<N>::NMID) {
    constexpr int T1 = N >> (3 * q + 3);
    constexpr bool RED = BOUND + 6 > 16;              // this pass would leave [0, 16p): reduce first
    constexpr int OUT = (RED ? after_red8p(BOUND) : BOUND) + 6;
    const int B = qbase<N, q>(tid);
    xload<N, q - 1, V>(x, sb, lay_base<N, q - 1>(B), T1);
    if constexpr (RED) red8p_all<V>(x, p2);
    fwd8_32<V>(x, tab + 4 * (BrShape<N>::grp(q) + tid / T1), p, p2, z);
    __syncwarp();
    xstore<N, q, V>(x, sb, lay_base<N, q>(B), T1);
    __syncwarp();
    fwd_mid<N, q + 1, V, OUT>(x, sb, tid, tab, p, p2, z);
  }
}
// bound (in p) of the values entering the final pass
template <int N, int q, int BOUND>
constexpr int fwd_bound_before_last() {
  if constexpr (q < BrShape<N>::NMID) {
    constexpr int OUT = ((BOUND + 6 > 16) ? after_red8p(BOUND) : BOUND) + 6;
    return fwd_bound_before_last<N, q + 1, OUT>();
  } else {
    return BOUND;
  }
}
template <int N, int q, int V, int QMIN = 1>     // inverse passes q .. QMIN, stores layout QMIN - 1 last
FDFB_DEV void inv_mid(u32 (&x)[V][8], u32* sb, int tid, const uint4* tab, u32 p, u32 p2, u32 z) {
  if constexpr (q >= QMIN && q >= 1) {
    constexpr int T1 = N >> (3 * q + 3);
    const int B = qbase<N, q>(tid);
    xload<N, q, V>(x, sb, lay_base<N, q>(B), T1);
    inv8_32<V>(x, tab + 4 * (BrShape<N>::grp(q) + tid / T1), p, p2, z);
    __syncwarp();
    xstore<N, q - 1, V>(x, sb, lay_base<N, q - 1>(B), T1);
    __syncwarp();
    inv_mid<N, q - 1, V, QMIN>(x, sb, tid, tab, p, p2, z);
  }
}

// Forward NTT mod p of V polynomials. In: x[v][k] = coefficient tid + T k, [0, 2p).
// Out: slot 8 tid + k, [0, fwd_out_bound p) <= [0, 16p).  The caller guarantees that no
// thread still reads sb.
template <int N, int V>
FDFB_DEV void ntt_fwd32(u32 (&x)[V][8], u32* sb, int tid, const uint4* tab, u32 p, u32 p2, u32 z) {
  using S = BrShape<N>;
  constexpr int T = S::T, NM = S::NMID;
  fwd8_32<V>(x, tab, p, p2, z);                       // inputs < 2p (digits < L <= p): bound 2 + 6
  xstore<N, 0, V>(x, sb, lay_base<N, 0>(tid), T);
#ifdef FDFB_EXP_NOBAR
  __syncwarp();
#else
  __syncthreads();
#endif
  fwd_mid<N, 1, V, 8>(x, sb, tid, tab, p, p2, z);
  xload<N, NM - 1, V>(x, sb, lay_base<N, NM - 1>(8 * tid), 1);
  constexpr int BL = fwd_bound_before_last<N, 1, 8>();
  if constexpr (BL + 2 * S::PLAST > 16) red8p_all<V>(x, p2);
#ifdef FDFB_EXP_TW   // timing experiment only (wrong results): every thread reads one final-pass group
  fwd_last32<S::PLAST, V>(x, tab + 4 * (S::G_LAST + (tid & FDFB_EXP_TW)), p, p2, z);
#else
  fwd_last32<S::PLAST, V>(x, tab + 4 * (S::G_LAST + tid), p, p2, z);
#endif
}
// bound (in p) of the forward transform's outputs
template <int N>
constexpr int fwd_out_bound() {
  constexpr int BL = fwd_bound_before_last<N, 1, 8>();
  return ((BL + 2 * BrShape<N>::PLAST > 16) ? after_red8p(BL) : BL) + 2 * BrShape<N>::PLAST;
}

// Inverse NTT mod p (unscaled) of V polynomials. In: slot 8 tid + k, [0, 2p).  Out:
// coefficient tid + T k, [0, 2p).  Starts warp-locally; ends after a CTA barrier.
template <int N, int V>
FDFB_DEV void ntt_inv32(u32 (&x)[V][8], u32* sb, int tid, const uint4* tab, u32 p, u32 p2, u32 z) {
  using S = BrShape<N>;
  constexpr int T = S::T, NM = S::NMID;
#ifdef FDFB_EXP_TW
  inv_last32<S::PLAST, V>(x, tab + 4 * (S::G_LAST + (tid & FDFB_EXP_TW)), p, p2, z);
#else
  inv_last32<S::PLAST, V>(x, tab + 4 * (S::G_LAST + tid), p, p2, z);
#endif
  xstore<N, NM - 1, V>(x, sb, lay_base<N, NM - 1>(8 * tid), 1);
  __syncwarp();
  inv_mid<N, NM - 1, V>(x, sb, tid, tab, p, p2, z);
#ifdef FDFB_EXP_NOBAR
  __syncwarp();
#else
  __syncthreads();
#endif
  xload<N, 0, V>(x, sb, lay_base<N, 0>(tid), T);
  inv8_32<V>(x, tab, p, p2, z);
}

// Montgomery reduction of the MAC sum: s < 2^63 -> s 2^{-32} mod p in [0, 2p)  (the 2^32 is
// folded into the RNS brK).  m = s_lo (-p^{-1}) mod 2^32 makes s + m p divisible by 2^32;
// (s + m p) / 2^32 < 2^31 + p < 9p, brought to [0, 2p) by three conditional subtractions.
FDFB_DEV u32 redc64(u64 s, const RnsParams& R, int i) {
  const u32 m = (u32)s * R.pinv[i];
  const u32 t = (u32)((s + (u64)m * R.p[i]) >> 32);
  const u32 p2 = R.p2[i];
  return csub32(csub32(csub32(t, p2 << 2), p2 << 1), p2);
}
// c * m mod Q in [0, 2Q) for c < 2^28 with a 32-bit quotient companion ms32 = floor(m 2^32 / Q):
// q = floor(c ms32 / 2^32) is floor(c m / Q) or one less (the truncation costs < c / 2^32 < 1/16)
FDFB_DEV u64 shoup64_28(u32 c, u64 m, u32 ms32, u64 Q) {
  const u32 q = __umulhi(c, ms32);
  return (u64)c * m - (u64)q * Q;
}

// GIN = false: every step of the loop "for i in [n], j in [u]": CMux(brK[i,j], acc X^{-abar_i u_j}, acc).
// GIN = true (shift-based BR): the rotated accumulator is given in gin
// (Shift(acc, -abar_i u_j mod N), computed by the Shift GEMM); one step per launch; a zero
// amount (abar_i = 0) is the identity step (reading S1) and is skipped.
template <int N, int NP, bool GIN>
__global__ void __launch_bounds__(N / 8, BrShape<N>::MINB)
k_blind_rotate(DevParams p, RnsParams R, const u32* __restrict__ bsk, u64* __restrict__ accs, int n_acc,
               int acc_per_ct, int abar_rows, const u32* __restrict__ abar, const u64* __restrict__ gin,
               int s_begin) {
  using S = BrShape<N>;
  constexpr int T = S::T;
  static_assert(fwd_out_bound<N>() <= 16, "forward outputs must stay below 16p < 2^32 (MAC bound)");
  extern __shared__ u64 smem[];
  u64* sacc = smem;                          // [b | a], natural order, canonical mod Q
  u64* sd = smem + 2 * N;                    // d = acc X^e - acc, both halves (thread-private slots)
  u32* sbuf = (u32*)(smem + 4 * N);          // NTT exchange buffers: 2 x (2 planes of 9N/8 words),
                                             // alternating per transform (no barrier between transforms)
  const int tid = threadIdx.x;
  const u64 Q = p.Q;
  const int ell = p.ell_rgsw, logL = p.logL_rgsw, u = p.u;
  const u32 dmask = (1u << logL) - 1;
  const size_t prime_words = (size_t)2 * ell * 2 * N;
  const size_t step_words = (size_t)NP * prime_words;

  for (int g = blockIdx.x; g < n_acc; g += gridDim.x) {
    u64* acc = accs + (size_t)g * 2 * N;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) sacc[tid + T * k] = acc[tid + T * k];
    const u32* ab = abar + (size_t)((g / acc_per_ct) % abar_rows) * p.n;   // accumulator g uses abar row
    // GIN: the single step s_begin = i0 u + j0; otherwise every (i, j)
    const int i0 = GIN ? s_begin / u : 0, i1 = GIN ? i0 + 1 : p.n;
    const int j0 = GIN ? s_begin - i0 * u : 0, j1 = GIN ? j0 + 1 : u;
#pragma unroll 1
    for (int i = i0; i < i1; i++) {
      const u32 ai = __ldg(ab + i);
      if constexpr (GIN) {
        if (ai == 0) continue;                     // Shift(acc, 0) = acc: CMux(brK, acc, acc) = acc
      }
#pragma unroll 1
      for (int j = j0; j < j1; j++) {
        // exponent -abar_i u_j mod 2N; u = [1] (binary) or [-1, 1] (ternary)
        const int e = (u == 2 && j == 0) ? (int)ai : (int)((2 * N - ai) & (2 * N - 1));
#ifdef FDFB_EXP_KEY  // timing experiment only (wrong results): every step reads step 0's key
        const u32* Kstep = bsk + 8 * tid;
#else
        const u32* Kstep = bsk + ((size_t)i * u + j) * step_words + 8 * tid;
#endif
        int xb = 0;                                // exchange buffer of the next transform
        __syncthreads();                           // acc of the previous step complete
        // d = acc X^e - acc for both halves, once per CMux (thread-private slots of sd; the
        // epilogues below may then update acc prime by prime)
        if constexpr (GIN) {
          const u64* gsrc = gin + (size_t)g * 2 * N;
#pragma unroll
          for (int k = 0; k < 16; k++) {
            const int pos = tid + T * k;
            sd[pos] = sub_mod(__ldg(gsrc + pos), sacc[pos], Q);
          }
        } else {
#pragma unroll
          for (int half = 0; half < 2; half++) {
            const u64* src = sacc + half * N;
#pragma unroll
            for (int k = 0; k < 8; k++) {
              const int pos = tid + T * k;
#ifdef FDFB_EXP_NOD
              sd[half * N + pos] = src[pos] + e;
#else
              const int idx = (pos - e) & (2 * N - 1);     // coefficient pos of X^e a = +-a[idx mod N]
              const u64 v = src[idx & (N - 1)];
              const u64 rv = (idx >= N && v) ? Q - v : v;
              sd[half * N + pos] = sub_mod(rv, src[pos], Q);
#endif
            }
          }
        }
#pragma unroll 1
        for (int pi = 0; pi < NP; pi++) {
          const u32 pr = R.p[pi], pr2 = R.p2[pi];
          const uint4* ft = R.ftab + (size_t)pi * S::GROUPS * 4;
          const uint4* it = R.itab + (size_t)pi * S::GROUPS * 4;
          const u32* K = Kstep + (size_t)pi * prime_words;
          u64 mb[8], ma[8];
#pragma unroll
          for (int k = 0; k < 8; k++) { mb[k] = 0; ma[k] = 0; }
#pragma unroll 1
          for (int half = 0; half < 2; half++) {
            const u64* sdh = sd + half * N;
            // digit pairs (r, r+1) transformed together; an odd ell pairs the last digit with zero
#pragma unroll 1
            for (int r = 0; r < ell; r += 2) {
              const bool two = r + 1 < ell;
              const u32* Kb0 = K + (size_t)((half * ell + r) * 2) * N;
              const u32* Kb1 = Kb0 + 2 * N;
              asm volatile("prefetch.global.L1 [%0];" ::"l"(Kb0));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(Kb0 + N));
              if (two) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(Kb1));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(Kb1 + N));
              }
              u32 x[2][8];
              const int sh = r * logL;
#pragma unroll
              for (int k = 0; k < 8; k++) {
                const u64 dv = sdh[tid + T * k];
                x[0][k] = (u32)(dv >> sh) & dmask;
                x[1][k] = two ? (u32)(dv >> (sh + logL)) & dmask : 0u;
              }
              // transform k writes buffer k % 2 only after its own CTA barrier has seen every warp
              // finish transform k - 1, whose buffer laggards may still read: no barrier here
              ntt_fwd32<N, 2>(x, sbuf + xb * 2 * Lay<N>::WORDS, tid, ft, pr, pr2, R.zero);
              xb ^= 1;
#pragma unroll
              for (int v = 0; v < 2; v++) {
                if (v == 1 && !two) break;
                const u32* Kb = v ? Kb1 : Kb0;
                const u32* Ka = Kb + N;
                const uint4 kb0 = __ldg((const uint4*)Kb), kb1 = __ldg((const uint4*)Kb + 1);
                const uint4 ka0 = __ldg((const uint4*)Ka), ka1 = __ldg((const uint4*)Ka + 1);
                const u32 kb[8] = {kb0.x, kb0.y, kb0.z, kb0.w, kb1.x, kb1.y, kb1.z, kb1.w};
                const u32 ka[8] = {ka0.x, ka0.y, ka0.z, ka0.w, ka1.x, ka1.y, ka1.z, ka1.w};
#pragma unroll
                for (int k = 0; k < 8; k++) {
                  mb[k] += (u64)x[v][k] * kb[k];      // x < fwd_out_bound p, K < p: setup_rns checks that
                  ma[k] += (u64)x[v][k] * ka[k];      // 2 ell terms + the Montgomery term fit redc64
                }
              }
            }
          }
          // both output columns through one paired inverse transform (warp-local start)
          u32 x[2][8];
#pragma unroll
          for (int k = 0; k < 8; k++) { x[0][k] = redc64(mb[k], R, pi); x[1][k] = redc64(ma[k], R, pi); }
          ntt_inv32<N, 2>(x, sbuf + xb * 2 * Lay<N>::WORDS, tid, it, pr, pr2, R.zero);
          xb ^= 1;
          // CRT, accumulated prime by prime (thread-private coefficients tid + T k):
          //   t_i = r_i (P/p_i)^{-1} mod p_i,  V = sum_i t_i P/p_i - round(sum_i t_i / p_i) P,
          // exact because setup_rns picks P with 256 |V| + 17 NP P <= 128 P (crt_rounding_exact).  acc += V mod Q
          // as acc += t_i (P/p_i mod Q) per prime (unreduced: < 7Q < 2^57), while the sum of
          // floor(16 t_i / p_i) (<= 45, error < 3/16) rides in bits 58..63 of the same word.
#pragma unroll
          for (int c = 0; c < 2; c++) {
            u64* sa = sacc + c * N;
#pragma unroll
            for (int k = 0; k < 8; k++) {
              const int pos = tid + T * k;
              const u32 t = csub32(x[c][k], pr);          // t_i = r_i y_i in [0, p) (y_i folded into brK)
              const u32 f = __umulhi(t, R.f16[pi]);                                 // floor(16 t_i / p_i) - {0, 1}
              u64 a = sa[pos] + shoup64_28(t, R.M[pi], R.Ms32[pi], Q);            // + t_i P/p_i (mod Q)
              if (pi < NP - 1) {
                a += (u64)f << 58;
              } else {
                const u32 kk = ((u32)(a >> 58) + f + 8) >> 4;                       // round(sum t_i / p_i)
                a &= (1ull << 58) - 1;
                a += (u64)(NP + 1) * Q - (u64)kk * R.pq;                            // kk <= NP, pq < Q
#ifndef FDFB_EXP_NOCSUB
                a = csub(a, Q << 3);
                a = csub(a, Q << 2);
                a = csub(a, Q << 1);
                a = csub(a, Q);
#endif
              }
              sa[pos] = a;
            }
          }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) acc[tid + T * k] = sacc[tid + T * k];
  }
}

// ---------------------------------------------------------------------------
// k_blind_rotate_p: the batched kernel with the per-transform CTA barrier removed (the
// default; k_blind_rotate above is kept for A/B, FDFB_BR_KERNEL=1).  Same arithmetic, same
// output bytes.  Every transform has exactly one cross-warp exchange (after the forward
// transform's first radix-8 pass, before the inverse transform's last one); here it goes
// through one of two buffers X0/X1 guarded by mbarriers instead of __syncthreads:
//   produce(c): ... -> wait empty[b] -> store the cross-warp layout into X[b] -> arrive full[b]
//   consume(c): wait full[b] -> load from X[b] -> arrive empty[b] -> warp-local passes (own slab)
// (b = c mod 2) and the schedule produces transform c + 1 before consuming transform c, so a
// warp waits on the others only if they lag by more than a whole transform.  The warp-local
// exchanges use a separate buffer (each warp touches only its own slab), so X[b] is released
// as soon as it is loaded.  d = acc X^e - acc is thread-private and lives in TMEM (64 columns
// per CTA: warps w and w + 4 share TMEM lanes and use column groups 0 / 32), which frees the
// shared memory for the second buffer: 16N (acc) + 18N (X0, X1) + 9N (slabs) = 43N bytes
// (86 KB at N = 2048; 2 CTAs per SM as before).  Per CMux:
//   P(F0) P(F1) C(F0) P(F2) C(F1) P(F3) C(F2) C(F3) P(I) P(F0') C(I) P(F1') C(F0') ...
// (F: forward digit-pair transforms of a prime, I: its inverse; ' = next prime).
// brK loads of the pipelined kernel: __ldg after an L1 prefetch at the start of the consume
// (measured per 296-accumulator wave: 91.9 ms; L1::no_allocate loads 103.1 ms without a
// prefetch, 95.3 ms with an L2 prefetch -- the L1 prefetch hides the latency)
FDFB_DEV uint4 ld_key(const uint4* p) { return __ldg(p); }
FDFB_DEV void prefetch_key(const u32* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
// one arrival per warp: __syncwarp orders the lanes' shared-memory accesses before lane 0's
// (release) arrive, so the barriers count warps, not threads
FDFB_DEV void warp_arrive(uint32_t baddr) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(baddr) : "memory");
}
template <int N, int V, bool TWT>
FDFB_DEV void fwd_consume(u32 (&x)[V][8], const u32* X, u32* sl, int tid, const uint4* tab, u32 p, u32 p2, u32 z,
                          uint32_t empty_b, uint32_t tw_taddr) {
  using S = BrShape<N>;
  constexpr int T1 = N >> 6;                       // pass-1 stride
  const int B = qbase<N, 1>(tid);
  xload<N, 0, V>(x, X, lay_base<N, 0>(B), T1);
  warp_arrive(empty_b);                            // this warp is done with X[b]
  fwd8_32<V>(x, tab + 4 * (S::grp(1) + tid / T1), p, p2, z);   // inputs < 8p: no reduction
  __syncwarp();                                    // laggard lanes done reading the slab
  xstore<N, 1, V>(x, sl, lay_base<N, 1>(B), T1);
  __syncwarp();
  fwd_mid<N, 2, V, 14>(x, sl, tid, tab, p, p2, z);
  xload<N, S::NMID - 1, V>(x, sl, lay_base<N, S::NMID - 1>(8 * tid), 1);
  constexpr int BL = fwd_bound_before_last<N, 1, 8>();
  if constexpr (BL + 2 * S::PLAST > 16) red8p_all<V>(x, p2);
  if constexpr (TWT) {
    Tw8 t;
    load_tw8_tmem(t, tw_taddr);
    fwd_last32_t<S::PLAST, V>(x, t, p, p2, z);
  } else {
    fwd_last32<S::PLAST, V>(x, tab + 4 * (S::G_LAST + tid), p, p2, z);
  }
}
// inverse up to the cross-warp store: last pass in registers, warp-local passes through the
// slab, pass 1 -> layout 0 into X[b]
template <int N, int V, bool TWT>
FDFB_DEV void inv_produce(u32 (&x)[V][8], u32* X, u32* sl, int tid, const uint4* tab, u32 p, u32 p2, u32 z,
                          uint32_t empty_b, uint32_t empty_par, uint32_t full_b, uint32_t tw_taddr) {
  using S = BrShape<N>;
  constexpr int NM = S::NMID;
  if constexpr (TWT) {
    Tw8 t;
    load_tw8_tmem(t, tw_taddr);
    inv_last32_t<S::PLAST, V>(x, t, p, p2, z);
  } else {
    inv_last32<S::PLAST, V>(x, tab + 4 * (S::G_LAST + tid), p, p2, z);
  }
  __syncwarp();
  xstore<N, NM - 1, V>(x, sl, lay_base<N, NM - 1>(8 * tid), 1);
  __syncwarp();
  inv_mid<N, NM - 1, V, 2>(x, sl, tid, tab, p, p2, z);     // passes NM-1 .. 2 (slab), layout 1 stored
  constexpr int T1 = N >> 6;
  const int B = qbase<N, 1>(tid);
  xload<N, 1, V>(x, sl, lay_base<N, 1>(B), T1);
  inv8_32<V>(x, tab + 4 * (S::grp(1) + tid / T1), p, p2, z);
  mbar_wait_sleep(empty_b, empty_par);
  xstore<N, 0, V>(x, X, lay_base<N, 0>(B), T1);
  warp_arrive(full_b);
}

// Key-stream pacing of the persistent batched kernel.  brK is read once per step by every
// resident accumulator; the CTAs of a launch only share those reads through L2 while they are
// at nearby steps.  Free-running CTAs drift apart over the ~35 accumulators each processes (a
// key step is 393 KB at the Large set, so L2 holds ~300 steps), and then every CTA streams brK
// from HBM on its own.  Every BR_PACE_CH steps warp 0 publishes the CTA's position
// pos = round * n u + step (tagged with the launch's tag) to prog[blockIdx.x] and waits while
// any CTA of the launch is between wlo and whi steps behind it.  CTAs further behind (late
// starters of a launch that shares the GPU with another one) are ignored, finished CTAs publish
// tag 0.  A wait lasts at most `cap` polls of ~2 us, so CTAs that are faster for a structural
// reason (an SM shared with fewer CTAs) lose a bounded fraction of their time while the small
// steady-state drift is still corrected; CTAs in their first or last round (staggered starts,
// partners leaving) publish but never wait.  The CTA furthest behind never waits, so the launch
// always progresses; the pacing changes no arithmetic.
#ifndef BR_PACE_CH
#define BR_PACE_CH 8
#endif
FDFB_DEV void pace_publish(u64* prog, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(prog), "l"(v) : "memory");
}
FDFB_DEV u64 pace_load(const u64* prog) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(prog) : "memory");
  return v;
}
FDFB_DEV void pace_wait(u64* prog, u32 tag, u32 pos, u32 wlo, u32 whi, u32 cap) {   // all lanes of one warp
  const int lane = threadIdx.x & 31;
  if (lane == 0) pace_publish(prog + blockIdx.x, ((u64)tag << 32) | pos);
  if (cap == 0) return;                            // publish only
  for (u32 it = 0;; it++) {
    bool behind = false;
    for (int c = lane; c < (int)gridDim.x; c += 32) {
      const u64 v = pace_load(prog + c);
      const u32 q = (u32)v;
      if ((u32)(v >> 32) == tag && q + wlo <= pos && q + whi > pos) behind = true;   // pos - whi < q <= pos - wlo
    }
    if (!__any_sync(0xffffffffu, behind) || it == cap) break;   // at most cap sleeps
    __nanosleep(2000);
  }
}

#ifndef BR_NB
#define BR_NB 3      // cross-warp exchange buffers of k_blind_rotate_p
#endif
#ifndef BR_LA
#define BR_LA 2      // transforms produced ahead of the one consumed (<= BR_NB - 1)
#endif
template <int N, int NP, bool GIN>
__global__ void __launch_bounds__(N / 8, BrShape<N>::MINB)
k_blind_rotate_p(DevParams p, RnsParams R, const u32* __restrict__ bsk, u64* __restrict__ accs, int n_acc,
                 int acc_per_ct, int abar_rows, const u32* __restrict__ abar, const u64* __restrict__ gin,
                 int s_begin, u64* __restrict__ prog, u32 tag, u32 wlo, u32 whi, u32 wcap) {
  using S = BrShape<N>;
  constexpr int T = S::T;
  constexpr int W = Lay<N>::WORDS;
  static_assert(fwd_out_bound<N>() <= 16, "forward outputs must stay below 16p < 2^32 (MAC bound)");
  extern __shared__ u64 smem[];
  u64* sacc = smem;                                // [b | a], natural order, canonical mod Q
  u32* Xb = (u32*)(smem + 2 * N);                  // X0, X1: 2 planes of W words each
  u32* sl = Xb + BR_NB * 2 * W;                    // warp-local exchange slabs (2 planes of W words)
  __shared__ uint64_t bars[2 * BR_NB];             // full[0 .. NB-1], empty[NB .. 2 NB-1]
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  const u64 Q = p.Q;
#ifdef FDFB_EXP_UNROLLF
  constexpr int ell = 4;
#else
  const int ell = p.ell_rgsw;
#endif
  const int logL = p.logL_rgsw, u = p.u;
  const u32 dmask = (1u << logL) - 1;
  const int PPH = (ell + 1) / 2;                   // digit pairs per half
  const int NF = 2 * PPH;                          // forward transforms per prime
  const size_t prime_words = (size_t)2 * ell * 2 * N;
  const size_t step_words = (size_t)NP * prime_words;
  if (tid == 0) {
    for (int b = 0; b < 2 * BR_NB; b++) mbar_init(bars + b, T / 32);   // one arrival per warp
  }
  // TMEM per warp group (warps w and w + 4 share TMEM lanes): 32 columns of d, and for N = 2048
  // (TWT) the thread's final-pass twiddle groups of every prime and direction (16 words each)
  constexpr bool TWT = (N >= 1024);               // 128 columns per warp group: fits MINB CTAs per SM
  constexpr int GCOLS = TWT ? 128 : 32;
  constexpr int TCOLS = T > 128 ? 2 * GCOLS : GCOLS;
  static_assert(!TWT || 32 + 16 * 2 * NP <= GCOLS, "twiddle columns");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // this thread's 32 TMEM words: lanes 32 (warp % 4) .., column group warp / 4
  const uint32_t tm = tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(GCOLS * (warp >> 2));
  if constexpr (TWT) {                             // stage the final-pass twiddles once per CTA
#pragma unroll 1
    for (int q = 0; q < 2 * NP; q++) {
      const uint4* g = (q & 1 ? R.itab : R.ftab) + ((size_t)(q >> 1) * S::GROUPS + S::G_LAST + tid) * 4;
      u32 v[16];
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const uint4 a = __ldg(g + i);
        v[4 * i] = a.x; v[4 * i + 1] = a.y; v[4 * i + 2] = a.z; v[4 * i + 3] = a.w;
      }
      tmem_st16(tm + 32 + 16 * q, v);
    }
    tmem_st_wait();
  }
  const uint32_t bar0 = smem_u32(bars);            // full[b] = bar0 + 8 b, empty[b] = bar0 + 8 NB + 8 b
  constexpr uint32_t EO = 8 * BR_NB;
  int cpb = 0, ccb = 0;                            // buffer of the next produced / consumed transform
  uint32_t cpp = 0, ccp = 0;                       // and its use parity (flips when the buffer index wraps)
  u32 x[2][8];
  u64 mb[8], ma[8];

  for (int g = blockIdx.x; g < n_acc; g += gridDim.x) {
    u64* acc = accs + (size_t)g * 2 * N;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) sacc[tid + T * k] = acc[tid + T * k];
    const u32* ab = abar + (size_t)((g / acc_per_ct) % abar_rows) * p.n;
    const int i0 = GIN ? s_begin / u : 0, i1 = GIN ? i0 + 1 : p.n;
    const int j0 = GIN ? s_begin - i0 * u : 0, j1 = GIN ? j0 + 1 : u;
#pragma unroll 1
    for (int i = i0; i < i1; i++) {
      const u32 ai = __ldg(ab + i);
      if constexpr (GIN) {
        if (ai == 0) continue;                     // Shift(acc, 0) = acc: CMux(brK, acc, acc) = acc
      }
#pragma unroll 1
      for (int j = j0; j < j1; j++) {
        const int e = (u == 2 && j == 0) ? (int)ai : (int)((2 * N - ai) & (2 * N - 1));
#ifdef FDFB_EXP_KEY
        const u32* Kstep = bsk + 8 * tid;
#else
        const u32* Kstep = bsk + ((size_t)i * u + j) * step_words + 8 * tid;
#endif
        if constexpr (!GIN) {                      // pacing: publish always, wait only in middle rounds
          const u32 s = (u32)(i * u + j);
          if (wlo && warp == 0 && (s % BR_PACE_CH) == 0) {   // everything derived here: no loop-carried state
            const u32 rnd = (u32)(g - (int)blockIdx.x) / gridDim.x;
            const bool mid = rnd > 0 && g + (int)gridDim.x < n_acc;
            pace_wait(prog, tag, rnd * (u32)(p.n * u) + s, wlo, whi, mid ? wcap : 0u);
          }
        }
        __syncthreads();                           // acc of the previous step complete
        {                                          // d = acc X^e - acc (both halves) -> TMEM
          u32 dw[16];
#pragma unroll
          for (int half = 0; half < 2; half++) {
            const u64* src = sacc + half * N;
#pragma unroll
            for (int k = 0; k < 8; k++) {
              const int pos = tid + T * k;
              u64 dv;
              if constexpr (GIN) {
                dv = sub_mod(__ldg(gin + (size_t)g * 2 * N + half * N + pos), src[pos], Q);
              } else {
                const int idx = (pos - e) & (2 * N - 1);   // coefficient pos of X^e a = +-a[idx mod N]
                const u64 v = src[idx & (N - 1)];
                const u64 rv = (idx >= N && v) ? Q - v : v;
                dv = sub_mod(rv, src[pos], Q);
              }
              dw[2 * k] = (u32)dv;
              dw[2 * k + 1] = (u32)(dv >> 32);
            }
            tmem_st16(tm + 16 * half, dw);
          }
          tmem_st_wait();
        }
        // ---- the transform pipeline over the NP primes
        auto produce_fwd = [&](int pi, int f) {
          const int half = f >= PPH ? 1 : 0, r = 2 * (f - half * PPH);   // f < 2 PPH: no division
          const bool two = r + 1 < ell;
          u32 dw[16];
          tmem_ld16(tm + 16 * half, dw);
          tmem_ld_wait();
          const int sh = r * logL;
#pragma unroll
          for (int k = 0; k < 8; k++) {
            const u64 dv = ((u64)dw[2 * k + 1] << 32) | dw[2 * k];
            x[0][k] = (u32)(dv >> sh) & dmask;
            x[1][k] = two ? (u32)(dv >> (sh + logL)) & dmask : 0u;
          }
          const uint4* ft = R.ftab + (size_t)pi * S::GROUPS * 4;
          fwd8_32<2>(x, ft, R.p[pi], R.p2[pi], R.zero);          // pass 0 (inputs < 2p)
          const int b = cpb;
          mbar_wait_sleep(bar0 + EO + 8 * b, cpp ^ 1);
          xstore<N, 0, 2>(x, Xb + b * 2 * W, lay_base<N, 0>(tid), T);
          warp_arrive(bar0 + 8 * b);
          if (++cpb == BR_NB) { cpb = 0; cpp ^= 1; }
        };
        auto consume_fwd = [&](int pi, int f) {
          const int half = f >= PPH ? 1 : 0, r = 2 * (f - half * PPH);   // f < 2 PPH: no division
          const bool two = r + 1 < ell;
          const u32* K = Kstep + (size_t)pi * prime_words;
          const u32* Kb0 = K + (size_t)((half * ell + r) * 2) * N;
          const u32* Kb1 = Kb0 + 2 * N;
          prefetch_key(Kb0);
          prefetch_key(Kb0 + N);
          if (two) {
            prefetch_key(Kb1);
            prefetch_key(Kb1 + N);
          }
          const int b = ccb;
          mbar_wait_sleep(bar0 + 8 * b, ccp);
          const uint4* ft = R.ftab + (size_t)pi * S::GROUPS * 4;
          fwd_consume<N, 2, TWT>(x, Xb + b * 2 * W, sl, tid, ft, R.p[pi], R.p2[pi], R.zero, bar0 + EO + 8 * b,
                                 tm + 32 + 32 * pi);
          if (++ccb == BR_NB) { ccb = 0; ccp ^= 1; }
#pragma unroll
          for (int v = 0; v < 2; v++) {
            if (v == 1 && !two) break;
            const u32* Kb = v ? Kb1 : Kb0;
            const u32* Ka = Kb + N;
            const uint4 kb0 = ld_key((const uint4*)Kb), kb1 = ld_key((const uint4*)Kb + 1);
            const uint4 ka0 = ld_key((const uint4*)Ka), ka1 = ld_key((const uint4*)Ka + 1);
            const u32 kb[8] = {kb0.x, kb0.y, kb0.z, kb0.w, kb1.x, kb1.y, kb1.z, kb1.w};
            const u32 ka[8] = {ka0.x, ka0.y, ka0.z, ka0.w, ka1.x, ka1.y, ka1.z, ka1.w};
#pragma unroll
            for (int k = 0; k < 8; k++) {
              mb[k] += (u64)x[v][k] * kb[k];       // x < fwd_out_bound p, K < p: setup_rns checks that
              ma[k] += (u64)x[v][k] * ka[k];       // 2 ell terms + the Montgomery term fit redc64
            }
          }
        };
        auto produce_inv = [&](int pi) {
#pragma unroll
          for (int k = 0; k < 8; k++) { x[0][k] = redc64(mb[k], R, pi); x[1][k] = redc64(ma[k], R, pi); }
          const int b = cpb;
          const uint4* it = R.itab + (size_t)pi * S::GROUPS * 4;
          inv_produce<N, 2, TWT>(x, Xb + b * 2 * W, sl, tid, it, R.p[pi], R.p2[pi], R.zero, bar0 + EO + 8 * b,
                                 cpp ^ 1, bar0 + 8 * b, tm + 32 + 32 * pi + 16);
          if (++cpb == BR_NB) { cpb = 0; cpp ^= 1; }
        };
        auto consume_inv = [&](int pi) {
          const int b = ccb;
          mbar_wait_sleep(bar0 + 8 * b, ccp);
          xload<N, 0, 2>(x, Xb + b * 2 * W, lay_base<N, 0>(tid), T);
          warp_arrive(bar0 + EO + 8 * b);
          if (++ccb == BR_NB) { ccb = 0; ccp ^= 1; }
          const u32 pr = R.p[pi];
          inv8_32<2>(x, R.itab + (size_t)pi * S::GROUPS * 4, pr, R.p2[pi], R.zero);
          // CRT, accumulated prime by prime (see k_blind_rotate)
#pragma unroll
          for (int c = 0; c < 2; c++) {
            u64* sa = sacc + c * N;
#pragma unroll
            for (int k = 0; k < 8; k++) {
              const int pos = tid + T * k;
              const u32 t = csub32(x[c][k], pr);
              const u32 f = __umulhi(t, R.f16[pi]);
              u64 a = sa[pos] + shoup64_28(t, R.M[pi], R.Ms32[pi], Q);
              if (pi < NP - 1) {
                a += (u64)f << 58;
              } else {
                const u32 kk = ((u32)(a >> 58) + f + 8) >> 4;
                a &= (1ull << 58) - 1;
                a += (u64)(NP + 1) * Q - (u64)kk * R.pq;
                a = csub(a, Q << 3);
                a = csub(a, Q << 2);
                a = csub(a, Q << 1);
                a = csub(a, Q);
              }
              sa[pos] = a;
            }
          }
        };
#pragma unroll
        for (int k = 0; k < 8; k++) { mb[k] = 0; ma[k] = 0; }
        // lookahead BR_LA transforms (BR_LA <= BR_NB - 1): forward transforms are independent of
        // each other; the inverse of a prime needs its last forward transform consumed (the MAC)
#pragma unroll
        for (int f = 0; f < BR_LA; f++)
          if (f < NF) produce_fwd(0, f);
#pragma unroll
        for (int pi = 0; pi < NP; pi++) {          // unrolled: per-prime constants from the parameter bank
#ifdef FDFB_EXP_UNROLLF
#pragma unroll
#else
#pragma unroll 1
#endif
          for (int f = 0; f < NF; f++) {
            if (f + BR_LA < NF) produce_fwd(pi, f + BR_LA);
            consume_fwd(pi, f);
          }
          produce_inv(pi);
#pragma unroll
          for (int k = 0; k < 8; k++) { mb[k] = 0; ma[k] = 0; }
          if (pi + 1 < NP) {
#pragma unroll
            for (int f = 0; f < BR_LA; f++)
              if (f < NF) produce_fwd(pi + 1, f);
          }
          consume_inv(pi);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; k++) acc[tid + T * k] = sacc[tid + T * k];
  }
  if (!GIN && wlo && tid == 0) pace_publish(prog + blockIdx.x, 0);   // finished: nobody waits on this CTA
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "n"(TCOLS));
}

// Latency variant for small batches: a cluster of NP x SPLIT CTAs per accumulator.  CTA rank
// (prime pi, part sp) evaluates prime p_pi only, and with SPLIT = 2 only the digit pairs of
// half sp (its own d half): its transforms, MAC and inverse transform give the partial
// residue t^(sp) = r^(sp) y_pi mod p_pi of both output columns, published to a double-buffered
// shared-memory slot.  One cluster barrier per CMux makes all slots visible; every CTA reads
// them through distributed shared memory, sums the parts per prime mod p, and applies the
// batched kernel's CRT (terms t (P/p) mod Q, rounding from floor(16 t / p)), so the copies of
// acc in the cluster stay identical and the result is bit-identical to k_blind_rotate.
template <int N, int NP, int SPLIT>
__global__ void __cluster_dims__(NP * SPLIT, 1, 1) __launch_bounds__(N / 8, 1)
k_blind_rotate_cl(DevParams p, RnsParams R, const u32* __restrict__ bsk, u64* __restrict__ accs, int n_acc,
                  int acc_per_ct, int abar_rows, const u32* __restrict__ abar) {
  namespace cg = cooperative_groups;
  using S = BrShape<N>;
  constexpr int T = S::T;
  constexpr int CL = NP * SPLIT;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int pi = rank / SPLIT, sp = rank % SPLIT;     // prime, part (SPLIT = 2: the d half)
  const int g = blockIdx.x / CL;                      // accumulator (grid = CL * n_acc exactly)
  extern __shared__ u64 smem[];
  u64* sacc = smem;                                   // [b | a], canonical mod Q (a copy per CTA)
  u64* sd = smem + 2 * N;                             // d, both halves
  u32* sbuf = (u32*)(smem + 4 * N);                   // 2 exchange buffers (as k_blind_rotate)
  u32* slot = sbuf + 4 * Lay<N>::WORDS;               // 2 x [2][N] partial residues
  const int tid = threadIdx.x;
  const u64 Q = p.Q;
  const int ell = p.ell_rgsw, logL = p.logL_rgsw, u = p.u;
  const u32 dmask = (1u << logL) - 1;
  const size_t prime_words = (size_t)2 * ell * 2 * N;
  const size_t step_words = (size_t)NP * prime_words;
  const u32 pr = R.p[pi], pr2 = R.p2[pi];
  const uint4* ft = R.ftab + (size_t)pi * S::GROUPS * 4;
  const uint4* it = R.itab + (size_t)pi * S::GROUPS * 4;
  const int h0 = SPLIT == 2 ? sp : 0, h1 = SPLIT == 2 ? sp + 1 : 2;   // halves of this CTA
  u64* acc = accs + (size_t)g * 2 * N;
#pragma unroll
  for (int k = 0; k < 16; k++) sacc[tid + T * k] = acc[tid + T * k];
  const u32* ab = abar + (size_t)((g / acc_per_ct) % abar_rows) * p.n;
  int buf = 0;
#pragma unroll 1
  for (int i = 0; i < p.n; i++) {
    const u32 ai = __ldg(ab + i);
#pragma unroll 1
    for (int j = 0; j < u; j++) {
      const int e = (u == 2 && j == 0) ? (int)ai : (int)((2 * N - ai) & (2 * N - 1));
      const u32* K = bsk + ((size_t)i * u + j) * step_words + (size_t)pi * prime_words + 8 * tid;
      int xb = 0;
      __syncthreads();                                // acc of the previous step complete
#pragma unroll 1
      for (int half = h0; half < h1; half++) {
        const u64* src = sacc + half * N;
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int pos = tid + T * k;
          const int idx = (pos - e) & (2 * N - 1);
          const u64 v = src[idx & (N - 1)];
          const u64 rv = (idx >= N && v) ? Q - v : v;
          sd[half * N + pos] = sub_mod(rv, src[pos], Q);
        }
      }
      u64 mb[8], ma[8];
#pragma unroll
      for (int k = 0; k < 8; k++) { mb[k] = 0; ma[k] = 0; }
#pragma unroll 1
      for (int half = h0; half < h1; half++) {
        const u64* sdh = sd + half * N;
#pragma unroll 1
        for (int r = 0; r < ell; r += 2) {
          const bool two = r + 1 < ell;
          const u32* Kb0 = K + (size_t)((half * ell + r) * 2) * N;
          const u32* Kb1 = Kb0 + 2 * N;
          u32 x[2][8];
          const int sh = r * logL;
#pragma unroll
          for (int k = 0; k < 8; k++) {
            const u64 dv = sdh[tid + T * k];
            x[0][k] = (u32)(dv >> sh) & dmask;
            x[1][k] = two ? (u32)(dv >> (sh + logL)) & dmask : 0u;
          }
          ntt_fwd32<N, 2>(x, sbuf + xb * 2 * Lay<N>::WORDS, tid, ft, pr, pr2, R.zero);
          xb ^= 1;
#pragma unroll
          for (int v = 0; v < 2; v++) {
            if (v == 1 && !two) break;
            const u32* Kb = v ? Kb1 : Kb0;
            const u32* Ka = Kb + N;
            const uint4 kb0 = __ldg((const uint4*)Kb), kb1 = __ldg((const uint4*)Kb + 1);
            const uint4 ka0 = __ldg((const uint4*)Ka), ka1 = __ldg((const uint4*)Ka + 1);
            const u32 kb[8] = {kb0.x, kb0.y, kb0.z, kb0.w, kb1.x, kb1.y, kb1.z, kb1.w};
            const u32 ka[8] = {ka0.x, ka0.y, ka0.z, ka0.w, ka1.x, ka1.y, ka1.z, ka1.w};
#pragma unroll
            for (int k = 0; k < 8; k++) {
              mb[k] += (u64)x[v][k] * kb[k];
              ma[k] += (u64)x[v][k] * ka[k];
            }
          }
        }
      }
      u32 x[2][8];
#pragma unroll
      for (int k = 0; k < 8; k++) { x[0][k] = redc64(mb[k], R, pi); x[1][k] = redc64(ma[k], R, pi); }
      ntt_inv32<N, 2>(x, sbuf + xb * 2 * Lay<N>::WORDS, tid, it, pr, pr2, R.zero);
      u32* mine = slot + (size_t)buf * 2 * N;
#pragma unroll
      for (int c = 0; c < 2; c++)
#pragma unroll
        for (int k = 0; k < 8; k++) mine[c * N + tid + T * k] = csub32(x[c][k], pr);   // t^(sp) in [0, p)
      cl.sync();                                      // all CL partial residues published
      const u32* sl[CL];
#pragma unroll
      for (int r2 = 0; r2 < CL; r2++) sl[r2] = cl.map_shared_rank(slot + (size_t)buf * 2 * N, r2);
#pragma unroll
      for (int c = 0; c < 2; c++)
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int pos = tid + T * k;
          u64 a = sacc[c * N + pos];
          u32 F = 0;
#pragma unroll
          for (int q = 0; q < NP; q++) {
            u32 t = sl[q * SPLIT][c * N + pos];
            if (SPLIT == 2) t = csub32(t + sl[q * SPLIT + 1][c * N + pos], R.p[q]);
            F += __umulhi(t, R.f16[q]);
            a += shoup64_28(t, R.M[q], R.Ms32[q], Q);                  // < 2Q each
          }
          const u32 kk = (F + 8) >> 4;                                  // round(sum t_q / p_q)
          a += (u64)(NP + 1) * Q - (u64)kk * R.pq;                      // < 11Q
          a = csub(a, Q << 3);
          a = csub(a, Q << 2);
          a = csub(a, Q << 1);
          sacc[c * N + pos] = csub(a, Q);
        }
      buf ^= 1;
    }
  }
  __syncthreads();
  if (rank == 0) {
#pragma unroll
    for (int k = 0; k < 16; k++) acc[tid + T * k] = sacc[tid + T * k];
  }
  cl.sync();                                          // no CTA leaves while its slots may be read
}

// brK import: canonical RGSW rows (coefficient domain, [0, Q)) -> for each prime p_i:
// NTT_p(row mod p_i) * N^{-1} y_i 2^32 mod p_i, in [0, p_i)  (y_i = (P/p_i)^{-1} mod p_i, the
// CRT weight, so the inverse transform of the MAC yields t_i = r_i y_i directly; 2^32 cancels
// the Montgomery reduction redc64).
// One CTA (T threads) per (poly, prime);
// poly = row*2 + col of the canonical [rows][2][N] block starting at flat row `row0`.
template <int N>
__global__ void __launch_bounds__(N / 8)
k_brk_rns(DevParams p, RnsParams R, const u64* __restrict__ canon, size_t row0, u32* __restrict__ dev) {
  using S = BrShape<N>;
  constexpr int T = S::T;
  __shared__ u32 sb[Lay<N>::WORDS];
  const int tid = threadIdx.x;
  const int pi = blockIdx.y;
  const size_t poly = blockIdx.x;              // local row*2 + col
  const size_t frow = row0 + poly / 2;         // flat canonical row = step*2ell + r
  const int col = (int)(poly % 2);
  const int rows_per_step = 2 * p.ell_rgsw;
  const size_t step = frow / rows_per_step;
  const int r = (int)(frow % rows_per_step);
  const u32 pr = R.p[pi], pr2 = R.p2[pi];
  const u64* src = canon + poly * N;
  u32 x[1][8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[0][k] = (u32)(src[tid + T * k] % pr);
  ntt_fwd32<N, 1>(x, sb, tid, R.ftab + (size_t)pi * S::GROUPS * 4, pr, pr2, R.zero);
  u32* o = dev + ((step * R.np + pi) * rows_per_step + r) * 2 * (size_t)N + (size_t)col * N + 8 * tid;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const u32 v = csub32(red16(x[0][k], pr2), pr);
    o[k] = csub32(shoup32(v, R.ninv[pi], R.ninvs[pi], pr), pr);
  }
}

// brK export (the inverse of k_brk_rns): per prime, the inverse NTT_p of the stored slots
// gives y_i 2^32 row mod p_i (N^{-1} was folded in), times 2^{-32}: t_i = y_i row mod p_i; the
// CRT  row = sum_i t_i (P / p_i) mod P  is exact because row < Q < P.  One CTA per (poly).
struct BrkExportC {
  u32 inv32[RNS_MAXP], inv32s[RNS_MAXP];   // 2^{-32} mod p_i and its Shoup companion
  u64 Pi[RNS_MAXP];                        // P / p_i
  u64 P_lo, P_hi;                          // P
};
template <int N>
__global__ void __launch_bounds__(N / 8)
k_brk_export(DevParams p, RnsParams R, BrkExportC X, const u32* __restrict__ dev, size_t row0, u64* __restrict__ canon) {
  using S = BrShape<N>;
  constexpr int T = S::T;
  __shared__ u32 sb[Lay<N>::WORDS];
  const int tid = threadIdx.x;
  const size_t poly = blockIdx.x;
  const size_t frow = row0 + poly / 2;
  const int col = (int)(poly % 2);
  const int rows_per_step = 2 * p.ell_rgsw;
  const size_t step = frow / rows_per_step;
  const int r = (int)(frow % rows_per_step);
  unsigned __int128 acc[8];
#pragma unroll
  for (int k = 0; k < 8; k++) acc[k] = 0;
  for (int pi = 0; pi < R.np; pi++) {
    const u32 pr = R.p[pi], pr2 = R.p2[pi];
    const u32* src = dev + ((step * R.np + pi) * rows_per_step + r) * 2 * (size_t)N + (size_t)col * N + 8 * tid;
    u32 x[1][8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[0][k] = src[k];
    __syncthreads();                                  // sb of the previous prime fully read
    ntt_inv32<N, 1>(x, sb, tid, R.itab + (size_t)pi * S::GROUPS * 4, pr, pr2, R.zero);
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const u32 t = csub32(shoup32(csub32(x[0][k], pr), X.inv32[pi], X.inv32s[pi], pr), pr);
      acc[k] += (unsigned __int128)t * X.Pi[pi];
    }
  }
  const unsigned __int128 P = ((unsigned __int128)X.P_hi << 64) | X.P_lo;
  u64* o = canon + (2 * row0 + poly) * (size_t)N;
#pragma unroll
  for (int k = 0; k < 8; k++) o[tid + T * k] = (u64)(acc[k] % P);
}
