/*
 * fdfb_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the FDFB hot path
 * (arXiv 2109.02731, /root/reference/PAPER.md).  It exists to PROVE the CUDA
 * path bit-exact; it is never called by the product library.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It shares no code, header, table or helper with
 * paper_2109_02731_b200/ (the CUDA path); the two meet only through the
 * seeded-input module synth/ and the canonical byte layouts in DESIGN.md.
 *
 * Style rules:
 *   - every function follows one paper passage in the paper's order/notation,
 *     cited as PAPER.md:<line> (section / figure);
 *   - ring products are SCHOOLBOOK negacyclic products (no NTT), mod-Q
 *     arithmetic is exact via unsigned __int128;
 *   - indices in comments are the paper's 1-based ones, arrays are 0-based;
 *   - where the paper is garbled the DESIGN.md reading (R1, F1..F6, G*) is
 *     named at the line that depends on it;
 *   - OpenMP is scheduling only: over independent items of a batch, and -- for a
 *     call that carries one item -- over the rows of a ring product, the 2 ell x 2
 *     independent ring products of an extProd (added in the definition's order)
 *     and the m terms of a VectorPack (an exact, order-free sum in Z_Q).
 *
 * Canonical layouts (shared *format*, not code):
 *   LWE  = [b, a_1..a_n]             ([b, a^T]^T)
 *   RLWE = [b(X) coeffs N][a(X) coeffs N]
 *   brK  = [n][u][2*ell][2][N]       (row r<ell: b-gadget rows)
 *   bpK  = [N][ell_pk][2][N]         (KeySwitchSetup(.,N,1,N,Q,s_F,s,L_pK), 2369)
 *   ksK  = [N][ell_ks][n+1]          (KeySwitchSetup(.,N,n,1,q,s_F,s,L_ks), 2371)
 *   pack = [N][ell_pack][L_pack][2][N] (PackSetup)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef unsigned __int128 u128;

/* ---------------- parameter vector (indices fixed in oracle/oracle.py) -------------- */
enum {
  P_N = 0, P_n, P_Q, P_LOGQLWE, P_LWEKEY, P_RLWEKEY, P_LOGL_RGSW, P_ELL_RGSW,
  P_LOGL_BOOT, P_ELL_BOOT, P_LOGL_PK, P_ELL_PK, P_LOGL_KS, P_ELL_KS,
  P_LOGL_PACK, P_ELL_PACK, P_T, P_NOISELESS, P_COUNT
};

/* ======================= Philox4x64-10 (Salmon et al. 2011) ======================
 * Counter-based generator; the sampling spec (which counter feeds which sample)
 * is DESIGN.md "Seeded determinism".  Pinned against numpy.random.Philox. */
static void mulhilo64(u64 a, u64 b, u64* lo, u64* hi) {
  u128 p = (u128)a * b; *lo = (u64)p; *hi = (u64)(p >> 64);
}
void or_philox(const u64 ctr_in[4], const u64 key_in[2], u64 out[4]) {
  u64 c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  u64 k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    if (r > 0) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
    u64 lo0, hi0, lo1, hi1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, &lo0, &hi0);
    mulhilo64(0xCA5A826395121157ULL, c2, &lo1, &hi1);
    u64 n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* word w of the random stream of object (i0,i1,i2) in domain dom */
static u64 rnd_word(u64 seed, u64 dom, u64 i0, u64 i1, u64 i2, u64 w) {
  u64 ctr[4] = {i0, i1, i2, w >> 2}, key[2] = {seed, dom}, out[4];
  or_philox(ctr, key, out);
  return out[w & 3];
}

/* Discrete Gaussian by CDT (sigma = 3.2, support [-T, T], reading G17).
 * The table is computed by oracle/cdt.py (Python decimal) and installed here. */
static u64 g_cdt[128];
static int g_cdt_T = 0;
void or_set_cdt(const u64* thr, int T) {
  g_cdt_T = T;
  for (int i = 0; i < 2 * T; i++) g_cdt[i] = thr[i];
}
static int64_t sample_gauss(u64 x, int noiseless) {
  if (noiseless || g_cdt_T == 0) return 0;
  int64_t e = -g_cdt_T;
  for (int i = 0; i < 2 * g_cdt_T; i++) if (x >= g_cdt[i]) e++;
  return e;
}
/* uniform mod Q from two words: floor(x * Q / 2^128) with x = hi:lo */
static u64 sample_uniform_q(u64 hi, u64 lo, u64 Q) {
  u128 a = (u128)hi * Q;           /* x*Q = a*2^64 + b  where b = lo*Q */
  u128 b = (u128)lo * Q;
  u128 mid = (u128)(u64)a + (b >> 64);
  return (u64)((a >> 64) + (mid >> 64));
}
static int sample_key_coeff(u64 x, int ternary) {
  if (ternary) return (int)((u64)(((u128)x * 3) >> 64)) - 1;  /* U{-1,0,1} */
  return (int)(x >> 63);                                        /* U{0,1}    */
}

/* ============================ scalar arithmetic ================================== */
static inline u64 addq(u64 a, u64 b, u64 Q) { u64 r = a + b; return r >= Q ? r - Q : r; }
static inline u64 subq(u64 a, u64 b, u64 Q) { return a >= b ? a - b : a + Q - b; }
static inline u64 mulq(u64 a, u64 b, u64 Q) { return (u64)(((u128)a * b) % Q); }
static inline u64 negq(u64 a, u64 Q) { return a ? Q - a : 0; }
/* a signed integer reduced into [0, Q) */
static inline u64 fromsigned(int64_t v, u64 Q) {
  int64_t r = v % (int64_t)Q; if (r < 0) r += (int64_t)Q; return (u64)r;
}
static u64 powq(u64 b, u64 e, u64 Q) {
  u64 r = 1 % Q; b %= Q;
  while (e) { if (e & 1) r = mulq(r, b, Q); b = mulq(b, b, Q); e >>= 1; }
  return r;
}
static inline u64 mask_of(int logq) { return logq >= 64 ? ~0ULL : ((1ULL << logq) - 1); }

/* ============================ ring R_{N,Q} = Z_Q[X]/(X^N+1) ======================
 * PAPER.md:1713 (notation), 1560-1566 (X^N = -1). */

/* c = a * b, schoolbook negacyclic: c_k = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j */
void or_ring_mul(int N, u64 Q, const u64* a, const u64* b, u64* c) {
  u64* tmp = (u64*)malloc(sizeof(u64) * N);
  #pragma omp parallel for if (N >= 1024 && !omp_in_parallel()) schedule(static)
  for (int k = 0; k < N; k++) {
    u128 pos = 0, neg = 0;
    for (int i = 0; i <= k; i++) pos += (u128)a[i] * b[k - i];
    for (int i = k + 1; i < N; i++) neg += (u128)a[i] * b[k + N - i];
    u64 p = (u64)(pos % Q), m = (u64)(neg % Q);
    tmp[k] = subq(p, m, Q);
  }
  memcpy(c, tmp, sizeof(u64) * N);
  free(tmp);
}
/* c = X^e * a, e taken mod 2N (X^N = -1) */
void or_monomial_mul(int N, u64 Q, const u64* a, int64_t e, u64* c) {
  int64_t E = ((e % (2 * N)) + 2 * N) % (2 * N);
  u64* tmp = (u64*)malloc(sizeof(u64) * N);
  for (int i = 0; i < N; i++) {
    int64_t j = i + E;               /* a_i X^i * X^E = a_i X^{i+E} */
    int neg = 0;
    while (j >= N) { j -= N; neg ^= 1; }
    tmp[j] = neg ? negq(a[i], Q) : a[i];
  }
  memcpy(c, tmp, sizeof(u64) * N);
  free(tmp);
}
static void poly_add(int N, u64 Q, const u64* a, const u64* b, u64* c) { for (int i = 0; i < N; i++) c[i] = addq(a[i], b[i], Q); }
static void poly_sub(int N, u64 Q, const u64* a, const u64* b, u64* c) { for (int i = 0; i < N; i++) c[i] = subq(a[i], b[i], Q); }
static void poly_scal(int N, u64 Q, const u64* a, u64 s, u64* c) { for (int i = 0; i < N; i++) c[i] = mulq(a[i], s, Q); }

/* ============================ Decomp_{L,q} =======================================
 * PAPER.md:1833-1842 (Def. Decomposition), 1732: ell = ceil(log_L q).
 * Unsigned digits in [0, L) of the representative x in [0, q) (reading G11):
 * x = sum_{r=1}^{ell} x_r L^{r-1}.  L = 2^logL. */
void or_decomp(u64 x, int logL, int ell, u64* digits) {
  u64 L = 1ULL << logL;
  for (int r = 0; r < ell; r++) { digits[r] = x % L; x /= L; }
}

/* ============================ encryption =========================================
 * RLWE (PAPER.md:1755-1763 with n=1, 1782): b = a*s + m + e, sample [b, a].
 * LWE  (N=1):                b = <a,s> + m + e  mod q. */

/* RLWE encryption of message polynomial m under ternary/binary s (int8 coeffs).
 * Randomness: object (i0,i1,i2) of domain dom; mask coeff c from words 2c,2c+1,
 * error coeff c from word 2N+c. */
void or_rlwe_encrypt(const u64* P, u64 seed, u64 dom, u64 i0, u64 i1, u64 i2,
                     const int8_t* s, const u64* m, u64* out) {
  int N = (int)P[P_N]; u64 Q = P[P_Q]; int nl = (int)P[P_NOISELESS];
  u64* a = out + N; u64* b = out;
  u64* sp = (u64*)malloc(sizeof(u64) * N);
  for (int c = 0; c < N; c++) {
    u64 hi = rnd_word(seed, dom, i0, i1, i2, 2 * (u64)c);
    u64 lo = rnd_word(seed, dom, i0, i1, i2, 2 * (u64)c + 1);
    a[c] = sample_uniform_q(hi, lo, Q);
    sp[c] = fromsigned(s[c], Q);
  }
  or_ring_mul(N, Q, a, sp, b);                         /* a * s */
  for (int c = 0; c < N; c++) {
    int64_t e = sample_gauss(rnd_word(seed, dom, i0, i1, i2, 2 * (u64)N + c), nl);
    b[c] = addq(addq(b[c], m[c], Q), fromsigned(e, Q), Q);  /* + m + e */
  }
  free(sp);
}

/* LWE encryption mod 2^logq under s (dim n) of the already-scaled message mu.
 * mask a_i = top logq bits of word i; error from word n. */
void or_lwe_encrypt_one(u64 seed, u64 dom, u64 i0, u64 i1, u64 i2, int n, int logq,
                        const int8_t* s, u64 mu, int noiseless, u64* out) {
  u64 msk = mask_of(logq);
  u64 acc = 0;
  for (int i = 0; i < n; i++) {
    u64 ai = rnd_word(seed, dom, i0, i1, i2, (u64)i) >> (64 - logq);
    out[1 + i] = ai;
    acc += ai * (u64)(int64_t)s[i];      /* exact mod 2^64, then mod 2^logq */
  }
  int64_t e = sample_gauss(rnd_word(seed, dom, i0, i1, i2, (u64)n), noiseless);
  out[0] = (acc + mu + (u64)e) & msk;
}

/* batch of input ciphertexts of messages m[c] in Z_t: mu = Delta_{q,t} * m,
 * Delta = q/t exactly for q = 2^logq.
 * flags bit0: "mod-switch exact" inputs (a_i multiple of q/2N, e = 0), the
 * correctness-gate variant of SURVEY §8(c.5)(i). */
void or_lwe_encrypt_batch(const u64* P, u64 seed, const int8_t* s, const u64* msg, int count,
                          u64 flags, u64* out) {
  int n = (int)P[P_n], logq = (int)P[P_LOGQLWE], N = (int)P[P_N];
  u64 t = P[P_T];
  u64 delta = (1ULL << logq) / t;
  #pragma omp parallel for schedule(static)
  for (int c = 0; c < count; c++) {
    u64* o = out + (size_t)c * (n + 1);
    if (flags & 1) {
      int log2N = 0; while ((1 << log2N) < 2 * N) log2N++;
      u64 step = 1ULL << (logq - log2N), acc = 0;
      for (int i = 0; i < n; i++) {
        u64 ai = (rnd_word(seed, 7, (u64)c, 0, 0, (u64)i) >> (64 - log2N)) * step;
        o[1 + i] = ai; acc += ai * (u64)(int64_t)s[i];
      }
      o[0] = (acc + delta * msg[c]) & mask_of(logq);
    } else {
      or_lwe_encrypt_one(seed, 7, (u64)c, 0, 0, n, logq, s, delta * msg[c], (int)P[P_NOISELESS], o);
    }
  }
}

/* Phase = [1, -s^T] c for LWE mod 2^logq and RLWE mod Q. */
u64 or_lwe_phase(int n, int logq, const int8_t* s, const u64* c) {
  u64 acc = 0;
  for (int i = 0; i < n; i++) acc += c[1 + i] * (u64)(int64_t)s[i];
  return (c[0] - acc) & mask_of(logq);
}
/* LWE phase mod an arbitrary (prime) modulus Q */
u64 or_lwe_phase_q(int n, u64 Q, const int8_t* s, const u64* c) {
  u64 acc = c[0];
  for (int i = 0; i < n; i++) acc = subq(acc, mulq(c[1 + i], fromsigned(s[i], Q), Q), Q);
  return acc;
}
void or_rlwe_phase(int N, u64 Q, const int8_t* s, const u64* c, u64* out) {
  u64* sp = (u64*)malloc(sizeof(u64) * N);
  u64* as = (u64*)malloc(sizeof(u64) * N);
  for (int i = 0; i < N; i++) sp[i] = fromsigned(s[i], Q);
  or_ring_mul(N, Q, c + N, sp, as);
  poly_sub(N, Q, c, as, out);
  free(sp); free(as);
}

/* ============================ key generation ====================================
 * Secrets (reading G16): s ~ U{0,1}^n or U{-1,0,1}^n; s_rlwe ~ U{-1,0,1}^N.
 * s: domain 1 object (0,0,0) word i;  s_rlwe: domain 2 object (0,0,0) word i. */
void or_keygen_secrets(const u64* P, u64 seed, int8_t* s_lwe, int8_t* s_rlwe) {
  int n = (int)P[P_n], N = (int)P[P_N];
  for (int i = 0; i < n; i++) s_lwe[i] = (int8_t)sample_key_coeff(rnd_word(seed, 1, 0, 0, 0, (u64)i), (int)P[P_LWEKEY]);
  for (int i = 0; i < N; i++) s_rlwe[i] = (int8_t)sample_key_coeff(rnd_word(seed, 2, 0, 0, 0, (u64)i), (int)P[P_RLWEKEY]);
}

/* u vector (reading G12): binary u=[1]; ternary u=[-1,+1]. */
static int u_len(const u64* P) { return P[P_LWEKEY] ? 2 : 1; }
static int u_val(const u64* P, int j) { return P[P_LWEKEY] ? (j == 0 ? -1 : 1) : 1; }
/* Y[i,j] with sum_j Y[i,j] u[j] = s[i] (Y=(1,0) for -1, (0,1) for +1, (0,0) for 0) */
static int Y_of(const u64* P, int si, int j) {
  if (!P[P_LWEKEY]) return si;
  return (j == 0) ? (si == -1) : (si == 1);
}

/* RGSW_{s}(m): rows r<ell: RLWE(0) + [m L^r, 0];
 * rows ell+r: RLWE(0) + [0, m L^r]  (G = I_2 (x) g, 1828).  m is an integer
 * constant here (the BRKeyGen use). brK[i,j]: domain 3, object (i, j, row). */
void or_brk_gen(const u64* P, u64 seed, const int8_t* s_lwe, const int8_t* s_rlwe, u64* brk) {
  int N = (int)P[P_N], n = (int)P[P_n], ell = (int)P[P_ELL_RGSW], logL = (int)P[P_LOGL_RGSW];
  int u = u_len(P); u64 Q = P[P_Q];
  size_t rows = (size_t)n * u * 2 * ell;
  #pragma omp parallel for schedule(dynamic, 1)
  for (size_t idx = 0; idx < rows; idx++) {
    int row = (int)(idx % (2 * ell)); int j = (int)((idx / (2 * ell)) % u); int i = (int)(idx / (2 * ell * u));
    u64* out = brk + idx * 2 * N;
    u64* zero = (u64*)calloc(N, sizeof(u64));
    or_rlwe_encrypt(P, seed, 3, (u64)i, (u64)j, (u64)row, s_rlwe, zero, out);   /* RLWE(0) */
    u64 m = (u64)Y_of(P, s_lwe[i], j);
    int r = row % ell;
    u64 g = mulq(m, powq(2, (u64)logL * r, Q), Q);    /* m * L^{r} (0-based r) */
    if (row < ell) out[0] = addq(out[0], g, Q);       /* b-column gadget */
    else           out[N] = addq(out[N], g, Q);       /* a-column gadget */
    free(zero);
  }
}

/* Bootstrap pK = KeySwitchSetup(B, N, 1, N, Q, s_F, s_rlwe, L_pK):
 * pK[i,j] = RLWE_{s}(s_F[i] * L^{j-1}) with a constant message polynomial. Domain 4. */
void or_bpk_gen(const u64* P, u64 seed, const int8_t* s_rlwe, u64* bpk) {
  int N = (int)P[P_N], ell = (int)P[P_ELL_PK], logL = (int)P[P_LOGL_PK]; u64 Q = P[P_Q];
  #pragma omp parallel for schedule(dynamic, 1)
  for (size_t idx = 0; idx < (size_t)N * ell; idx++) {
    int j = (int)(idx % ell), i = (int)(idx / ell);
    u64* m = (u64*)calloc(N, sizeof(u64));
    m[0] = mulq(fromsigned(s_rlwe[i], Q), powq(2, (u64)logL * j, Q), Q);  /* s_F[i] = Coefs(s)[i] (1988) */
    or_rlwe_encrypt(P, seed, 4, (u64)i, (u64)j, 0, s_rlwe, m, bpk + idx * 2 * N);
    free(m);
  }
}

/* ksK = KeySwitchSetup(B, N, n, 1, q_lwe, s_F, s, L_ks),
 * modulus q_lwe per reading c.3: ksK[i,j] = LWE_{s}(s_F[i] L^{j-1}) mod 2^logq. Domain 5. */
void or_ksk_gen(const u64* P, u64 seed, const int8_t* s_lwe, const int8_t* s_rlwe, u64* ksk) {
  int N = (int)P[P_N], n = (int)P[P_n], ell = (int)P[P_ELL_KS], logL = (int)P[P_LOGL_KS];
  int logq = (int)P[P_LOGQLWE];
  #pragma omp parallel for schedule(static)
  for (size_t idx = 0; idx < (size_t)N * ell; idx++) {
    int j = (int)(idx % ell), i = (int)(idx / ell);
    u64 mu = ((u64)(int64_t)s_rlwe[i] << (logL * j)) & mask_of(logq);
    or_lwe_encrypt_one(seed, 5, (u64)i, (u64)j, 0, n, logq, s_lwe, mu, (int)P[P_NOISELESS],
                       ksk + idx * (n + 1));
  }
}

/* PackSetup(B, N, N, Q, s_F, s, L_pack):
 * pK[i,j,k] = RLWE_s(s_F[i] * L^{j-1} * (k-1)), k in [L]. Domain 6, object (i,j,k-1). */
void or_pack_gen_entry(const u64* P, u64 seed, const int8_t* s_rlwe, int i, int j, int k0, u64* out) {
  int N = (int)P[P_N], logL = (int)P[P_LOGL_PACK]; u64 Q = P[P_Q];
  u64* m = (u64*)calloc(N, sizeof(u64));
  m[0] = mulq(mulq(fromsigned(s_rlwe[i], Q), powq(2, (u64)logL * j, Q), Q), (u64)k0, Q);
  or_rlwe_encrypt(P, seed, 6, (u64)i, (u64)j, (u64)k0, s_rlwe, m, out);
  free(m);
}
void or_pack_gen(const u64* P, u64 seed, const int8_t* s_rlwe, u64* pack) {
  int N = (int)P[P_N], ell = (int)P[P_ELL_PACK], L = 1 << (int)P[P_LOGL_PACK];
  #pragma omp parallel for schedule(dynamic, 1)
  for (size_t idx = 0; idx < (size_t)N * ell * L; idx++) {
    int k0 = (int)(idx % L), j = (int)((idx / L) % ell), i = (int)(idx / ((size_t)L * ell));
    or_pack_gen_entry(P, seed, s_rlwe, i, j, k0, pack + idx * 2 * N);
  }
}

/* ============================ extProd / CMux =====================================
 * extProd(C, d) = Decomp_{L,Q}(d^T) * C:
 *   out = sum_r b_r * C[r] + sum_r a_r * C[ell + r]   (rows ordered as RGSW, 1847).
 * CMux(C, g, h) = extProd(C, g - h) + h. */
void or_ext_prod(int N, u64 Q, int logL, int ell, const u64* C, const u64* d, u64* out) {
  u64* dig = (u64*)malloc(sizeof(u64) * ell);
  u64* D = (u64*)malloc(sizeof(u64) * (size_t)2 * ell * N);   /* digit polynomials */
  for (int half = 0; half < 2; half++)
    for (int c = 0; c < N; c++) {
      or_decomp(d[half * N + c], logL, ell, dig);
      for (int r = 0; r < ell; r++) D[((size_t)half * ell + r) * N + c] = dig[r];
    }
  /* Schedule only: the 2 ell x 2 ring products are independent, so a call that is not already
   * inside a parallel region computes them on the host threads (each by the same or_ring_mul,
   * which then runs its rows serially); they are added in the row order of the definition. */
  u64* prod = (u64*)malloc(sizeof(u64) * (size_t)2 * ell * 2 * N);
  memset(out, 0, sizeof(u64) * 2 * N);
  #pragma omp parallel for collapse(2) schedule(static) if (N >= 1024 && !omp_in_parallel())
  for (int row = 0; row < 2 * ell; row++)
    for (int col = 0; col < 2; col++)
      or_ring_mul(N, Q, D + (size_t)row * N, C + ((size_t)row * 2 + col) * N, prod + ((size_t)row * 2 + col) * N);
  for (int row = 0; row < 2 * ell; row++)
    for (int col = 0; col < 2; col++)
      poly_add(N, Q, out + col * N, prod + ((size_t)row * 2 + col) * N, out + col * N);
  free(prod); free(D); free(dig);
}
void or_cmux(int N, u64 Q, int logL, int ell, const u64* C, const u64* g, const u64* h, u64* out) {
  u64* d = (u64*)malloc(sizeof(u64) * 2 * N);
  poly_sub(N, Q, g, h, d); poly_sub(N, Q, g + N, h + N, d + N);       /* d = g - h */
  or_ext_prod(N, Q, logL, ell, C, d, out);
  poly_add(N, Q, out, h, out); poly_add(N, Q, out + N, h + N, out + N); /* + h */
  free(d);
}

/* BlindRotate(brK, acc, ct, u): for i in [n], j in [u]:
 *   acc <- CMux(brK[i,j], acc * X^{-a[i] u[j]}, acc).
 * abar holds the mask of ct in Z_{2N}; only the first n_steps coefficients are
 * used (n_steps = n for the algorithm; smaller for timing samples).  b is not
 * used here: the caller has already placed X^{b} in acc. */
void or_blind_rotate(const u64* P, const u64* brk, u64* acc, const uint32_t* abar, int n_steps) {
  int N = (int)P[P_N], ell = (int)P[P_ELL_RGSW], logL = (int)P[P_LOGL_RGSW], u = u_len(P);
  u64 Q = P[P_Q];
  u64* g = (u64*)malloc(sizeof(u64) * 2 * N);
  u64* out = (u64*)malloc(sizeof(u64) * 2 * N);
  for (int i = 0; i < n_steps; i++)
    for (int j = 0; j < u; j++) {
      int64_t e = -(int64_t)abar[i] * u_val(P, j);
      or_monomial_mul(N, Q, acc, e, g);
      or_monomial_mul(N, Q, acc + N, e, g + N);
      const u64* C = brk + ((size_t)i * u + j) * (size_t)2 * ell * 2 * N;
      or_cmux(N, Q, logL, ell, C, g, acc, out);
      memcpy(acc, out, sizeof(u64) * 2 * N);
    }
  free(g); free(out);
}

/* ============================ ModSwitch / SampleExt / KeySwitch ==================
 * ModSwitch(c, Q, q): x -> round(q x / Q), ties up
 * (reading G10): floor((2 q x + Q) / (2 Q)) mod q, exact in 128 bits. */
u64 or_mod_switch(u64 x, u64 Qfrom, u64 qto) {
  u128 num = (u128)2 * qto * x + Qfrom;
  return (u64)((num / ((u128)2 * Qfrom)) % qto);
}

/* SampleExt(ct, k):  b' = Coefs(b)[k];
 * a'[i] = NSgn(k - i + 1) a[(k - i mod N) + 1],  NSgn(x) = +1 iff x > 0
 * (reading F1: the prose at 2963 -- "image of 0 is -1" -- not the cases display).
 * k is 1-based; the output LWE is [b', a'_1..a'_N] mod Q under s_F = Coefs(s). */
void or_sample_extract(int N, u64 Q, const u64* ct, int k, u64* out) {
  const u64* b = ct; const u64* a = ct + N;
  out[0] = b[k - 1];
  for (int i = 1; i <= N; i++) {
    int x = k - i + 1;
    int idx = (((k - i) % N) + N) % N;            /* (k - i mod N), 0-based index into a */
    u64 v = a[idx];
    out[i] = (x > 0) ? v : negq(v, Q);
  }
}

/* KeySwitch LWE -> LWE mod 2^logq:
 *   out = [b, 0] - sum_{i,j} A[i,j] ksK[i,j], A = Decomp_{L,q}(a). */
void or_keyswitch_lwe(const u64* P, const u64* ksk, const u64* in, u64* out) {
  int N = (int)P[P_N], n = (int)P[P_n], ell = (int)P[P_ELL_KS], logL = (int)P[P_LOGL_KS];
  u64 msk = mask_of((int)P[P_LOGQLWE]);
  u64 dig[64];
  memset(out, 0, sizeof(u64) * (n + 1));
  out[0] = in[0];
  for (int i = 0; i < N; i++) {
    or_decomp(in[1 + i], logL, ell, dig);
    for (int j = 0; j < ell; j++) {
      const u64* row = ksk + ((size_t)i * ell + j) * (n + 1);
      for (int c = 0; c <= n; c++) out[c] -= dig[j] * row[c];
    }
  }
  for (int c = 0; c <= n; c++) out[c] &= msk;
}

/* KeySwitch LWE_N (mod Q) -> RLWE with the bootstrap pK:
 *   out = [b, 0] - sum_{i,j} A[i,j] pK[i,j]  (A = Decomp_{L_pK,Q}(a)). */
void or_keyswitch_rlwe(const u64* P, const u64* bpk, const u64* in, u64* out) {
  int N = (int)P[P_N], ell = (int)P[P_ELL_PK], logL = (int)P[P_LOGL_PK]; u64 Q = P[P_Q];
  u64 dig[64];
  u128* acc = (u128*)calloc((size_t)2 * N, sizeof(u128));
  for (int i = 0; i < N; i++) {
    or_decomp(in[1 + i], logL, ell, dig);
    for (int j = 0; j < ell; j++) {
      if (!dig[j]) continue;
      const u64* row = bpk + ((size_t)i * ell + j) * 2 * N;
      for (int c = 0; c < 2 * N; c++) acc[c] += (u128)dig[j] * row[c];
    }
  }
  for (int c = 0; c < 2 * N; c++) out[c] = negq((u64)(acc[c] % Q), Q);
  out[0] = addq(out[0], in[0], Q);
  free(acc);
}

/* ============================ PubMux / BuildAcc ==================================
 * PubMux([c_i], p0, p1) with reading R1 (Delta := 1):
 *   p = p1 - p0;  P = Decomp_{L,Q}(p) (coefficient-wise digit polynomials);
 *   out = [p0, 0] + sum_i P[i] * c_i      (ring products). */
void or_pubmux(const u64* P, const u64* accR /* ell_boot RLWE */, const u64* p0, const u64* p1, u64* out) {
  int N = (int)P[P_N], ell = (int)P[P_ELL_BOOT], logL = (int)P[P_LOGL_BOOT]; u64 Q = P[P_Q];
  u64* p = (u64*)malloc(sizeof(u64) * N);
  u64* D = (u64*)malloc(sizeof(u64) * (size_t)ell * N);
  u64* prod = (u64*)malloc(sizeof(u64) * N);
  u64 dig[64];
  poly_sub(N, Q, p1, p0, p);
  for (int c = 0; c < N; c++) {
    or_decomp(p[c], logL, ell, dig);
    for (int r = 0; r < ell; r++) D[(size_t)r * N + c] = dig[r];
  }
  memcpy(out, p0, sizeof(u64) * N); memset(out + N, 0, sizeof(u64) * N);
  for (int r = 0; r < ell; r++)
    for (int col = 0; col < 2; col++) {
      or_ring_mul(N, Q, D + (size_t)r * N, accR + ((size_t)r * 2 + col) * N, prod);
      poly_add(N, Q, out + col * N, prod, out + col * N);
    }
  free(p); free(D); free(prod);
}

/* ============================ SetupPolynomial ====================================
 * Fig. SetupPolynomial with reading F6/G9: the windows are
 * half-open, e in [-ceil(N/t), ceil(N/t)), so every y in [0,2N) is written once.
 * bootsmap[m] = BootsMap[m+1] in the paper's 1-based indexing (values mod Q). */
void or_setup_polynomial(const u64* P, const u64* bootsmap, u64* p0, u64* p1) {
  int N = (int)P[P_N]; u64 Q = P[P_Q]; int64_t t = (int64_t)P[P_T];
  memset(p0, 0, sizeof(u64) * N); memset(p1, 0, sizeof(u64) * N);
  int64_t w = (N + t - 1) / t;                             /* ceil(N/t) */
  int64_t step = (2 * N + t / 2) / t;                      /* round(2N/t) (ties up) */
  for (int64_t m = 0; m < t; m++)
    for (int64_t e = -w; e < w; e++) {
      int64_t y = ((step * m + e) % (2 * N) + 2 * N) % (2 * N);
      u64 v = bootsmap[m];
      if (y == 0) p0[0] = v;                                /* p0[1] = BootsMap[m+1]      */
      else if (y <= N - 1) p0[N - y] = negq(v, Q);          /* p0[N-y+1] = -BootsMap      */
      else if (y == N) p1[0] = negq(v, Q);                  /* p1[1] = -BootsMap          */
      else p1[N - (y - N)] = v;                             /* p1[N-y'+1] = BootsMap      */
    }
}

/* ============================ FDFB Bootstrap =====================================
 * Fig. Bootstrap with readings R1 (G7), F4 (G8) and the
 * c.3 output order (ModSwitch Q->q_lwe, then KeySwitch mod q_lwe). */
static void bootstrap_one(const u64* P, const u64* brk, const u64* bpk, const u64* ksk,
                          const u64* rotp0, const u64* rotp1, const u64* ct, u64* out) {
  int N = (int)P[P_N], n = (int)P[P_n], ellb = (int)P[P_ELL_BOOT], logLb = (int)P[P_LOGL_BOOT];
  int logq = (int)P[P_LOGQLWE]; u64 Q = P[P_Q];
  u64 qlwe = 1ULL << logq;
  /* line 2: ct_N = ModSwitch(ct, q, 2N) */
  uint32_t* abar = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t bbar = (uint32_t)or_mod_switch(ct[0], qlwe, 2 * (u64)N);
  for (int i = 0; i < n; i++) abar[i] = (uint32_t)or_mod_switch(ct[1 + i], qlwe, 2 * (u64)N);
  /* line 1, 3: sgnP = 1 - sum_{i=2}^{N} X^{i-1};  sgnP_b = sgnP * X^{b_N} */
  u64* sgnP = (u64*)malloc(sizeof(u64) * N);
  sgnP[0] = 1; for (int i = 1; i < N; i++) sgnP[i] = Q - 1;
  or_monomial_mul(N, Q, sgnP, bbar, sgnP);
  /* lines 5-8: ladder (reading R1: acc_i = [L^{i-1} * 2^{-1} * sgnP_b, 0]) */
  u64 h = (Q + 1) / 2;                                      /* 2^{-1} mod Q (Q odd) */
  u64* accs = (u64*)malloc(sizeof(u64) * (size_t)2 * N);
  u64* lwe = (u64*)malloc(sizeof(u64) * (N + 1));
  u64* accR = (u64*)malloc(sizeof(u64) * (size_t)ellb * 2 * N);
  for (int i = 0; i < ellb; i++) {
    u64 c = mulq(powq(2, (u64)logLb * i, Q), h, Q);        /* L_boot^{i-1} * 2^{-1} */
    poly_scal(N, Q, sgnP, c, accs); memset(accs + N, 0, sizeof(u64) * N);
    or_blind_rotate(P, brk, accs, abar, n);                 /* line 7 */
    or_sample_extract(N, Q, accs, 1, lwe);                  /* line 8: SampleExt(., 1) */
    lwe[0] = addq(lwe[0], c, Q);                            /*   + [L^{i-1} 2^{-1}, 0] */
    /* BuildAcc line 1: acc_{R,i} = KeySwitch(acc_{c,i}, pK) */
    or_keyswitch_rlwe(P, bpk, lwe, accR + (size_t)i * 2 * N);
  }
  /* lines 9-10: rotP'_x = rotP_x * X^{b_N} */
  u64* r0 = (u64*)malloc(sizeof(u64) * N);
  u64* r1 = (u64*)malloc(sizeof(u64) * N);
  or_monomial_mul(N, Q, rotp0, bbar, r0);
  or_monomial_mul(N, Q, rotp1, bbar, r1);
  /* line 11: BuildAcc -> PubMux with the F4 swap: p0 := rotP'_1, p1 := rotP'_0 */
  u64* accF = (u64*)malloc(sizeof(u64) * 2 * N);
  or_pubmux(P, accR, r1, r0, accF);
  /* line 12: BlindRotate; line 13: SampleExt(., 1) */
  or_blind_rotate(P, brk, accF, abar, n);
  or_sample_extract(N, Q, accF, 1, lwe);
  /* c.3: ModSwitch(Q -> q_lwe) then KeySwitch mod q_lwe (lines 14-15 reordered) */
  for (int i = 0; i <= N; i++) lwe[i] = or_mod_switch(lwe[i], Q, qlwe);
  or_keyswitch_lwe(P, ksk, lwe, out);
  free(abar); free(sgnP); free(accs); free(lwe); free(accR); free(r0); free(r1); free(accF);
}
void or_bootstrap(const u64* P, const u64* brk, const u64* bpk, const u64* ksk,
                  const u64* rotp0, const u64* rotp1, const u64* ct_in, int count, u64* ct_out) {
  int n = (int)P[P_n];
  #pragma omp parallel for schedule(dynamic, 1) if (count > 1)
  for (int c = 0; c < count; c++)
    bootstrap_one(P, brk, bpk, ksk, rotp0, rotp1, ct_in + (size_t)c * (n + 1), ct_out + (size_t)c * (n + 1));
}

/* ============================ TFHE (half-domain) bootstrap ======================
 * Fig. TFHE Bootstrapping (Def./Thm 2095-2139) with the output order
 * of reading c.3 (ModSwitch Q -> q_lwe, then KeySwitch mod q_lwe), as for FDFB:
 *   ct_N = ModSwitch(ct, q, 2N); rotP' = rotP X^{b_N}; acc = [rotP', 0];
 *   acc = BlindRotate(brK, acc, ct_N, u); c_Q = SampleExt(acc, 1); out = KS(ModSwitch(c_Q)). */
static void bootstrap_tfhe_one(const u64* P, const u64* brk, const u64* ksk, const u64* rotp, const u64* ct, u64* out) {
  int N = (int)P[P_N], n = (int)P[P_n], logq = (int)P[P_LOGQLWE]; u64 Q = P[P_Q];
  u64 qlwe = 1ULL << logq;
  uint32_t* abar = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t bbar = (uint32_t)or_mod_switch(ct[0], qlwe, 2 * (u64)N);          /* line 1 */
  for (int i = 0; i < n; i++) abar[i] = (uint32_t)or_mod_switch(ct[1 + i], qlwe, 2 * (u64)N);
  u64* acc = (u64*)calloc((size_t)2 * N, sizeof(u64));
  or_monomial_mul(N, Q, rotp, bbar, acc);                                      /* lines 2-3 */
  or_blind_rotate(P, brk, acc, abar, n);                                       /* line 4 */
  u64* lwe = (u64*)malloc(sizeof(u64) * (N + 1));
  or_sample_extract(N, Q, acc, 1, lwe);                                        /* line 5 */
  for (int i = 0; i <= N; i++) lwe[i] = or_mod_switch(lwe[i], Q, qlwe);        /* lines 6-7, c.3 */
  or_keyswitch_lwe(P, ksk, lwe, out);
  free(abar); free(acc); free(lwe);
}
void or_bootstrap_tfhe(const u64* P, const u64* brk, const u64* ksk, const u64* rotp, const u64* ct_in, int count,
                       u64* ct_out) {
  int n = (int)P[P_n];
  #pragma omp parallel for schedule(dynamic, 1) if (count > 1)
  for (int c = 0; c < count; c++)
    bootstrap_tfhe_one(P, brk, ksk, rotp, ct_in + (size_t)c * (n + 1), ct_out + (size_t)c * (n + 1));
}

/* ============================ Pack / VectorPack / Shift ==========================
 * Pack(c, pK, d), precomputed variant (reading G6):
 *   out = [b X^{d-1}, 0] - X^{d-1} sum_{i,j} pK[i, j, A[i,j] + 1],  A = Decomp_{L,Q}(a).
 * The message lands at X^{d-1} (reading G5; the lemma's m X^k is a typo). */
void or_pack(const u64* P, const u64* pack, const u64* c, int d, u64* out) {
  int N = (int)P[P_N], ell = (int)P[P_ELL_PACK], logL = (int)P[P_LOGL_PACK]; u64 Q = P[P_Q];
  int L = 1 << logL;
  u64 dig[64];
  u64* s = (u64*)calloc((size_t)2 * N, sizeof(u64));
  for (int i = 0; i < N; i++) {
    or_decomp(c[1 + i], logL, ell, dig);
    for (int j = 0; j < ell; j++) {
      const u64* e = pack + (((size_t)i * ell + j) * L + dig[j]) * 2 * N;   /* pK[i,j,A+1] */
      poly_add(N, Q, s, e, s); poly_add(N, Q, s + N, e + N, s + N);
    }
  }
  memset(out, 0, sizeof(u64) * 2 * N);
  out[0] = c[0];                                   /* [b, 0] then * X^{d-1} below */
  poly_sub(N, Q, out, s, out); poly_sub(N, Q, out + N, s + N, out + N);
  or_monomial_mul(N, Q, out, d - 1, out); or_monomial_mul(N, Q, out + N, d - 1, out + N);
  free(s);
}
/* VectorPack(v, pK) = sum_{k=1}^{m} Pack(v[k], pK, k). */
/* Schedule only: when the caller is not already running items in parallel, the m terms
 * Pack(v[k], pK, k) are computed by the host threads (each exactly as in the serial loop) and
 * added into `out` one at a time; addition in Z_Q is exact, so the order of the terms does not
 * change the sum. */
void or_vector_pack(const u64* P, const u64* pack, const u64* v, int m, u64* out) {
  int N = (int)P[P_N]; u64 Q = P[P_Q];
  memset(out, 0, sizeof(u64) * 2 * N);
  #pragma omp parallel if (m >= 16 && !omp_in_parallel())
  {
    u64* t = (u64*)malloc(sizeof(u64) * 2 * N);
    #pragma omp for schedule(dynamic, 1)
    for (int k = 1; k <= m; k++) {
      or_pack(P, pack, v + (size_t)(k - 1) * (N + 1), k, t);
      #pragma omp critical(or_vector_pack_sum)
      { poly_add(N, Q, out, t, out); poly_add(N, Q, out + N, t + N, out + N); }
    }
    free(t);
  }
}
/* Shift(ct, pK, d), d in [N-1] with readings F2 (extract N-d+i),
 * F3 (d = N/2 takes branch 1; branch2 selectable for the tie test) and G4. */
void or_shift(const u64* P, const u64* pack, const u64* ct, int d, int force_branch2, u64* out) {
  int N = (int)P[P_N]; u64 Q = P[P_Q];
  int br1 = (2 * d <= N) && !force_branch2;
  int m = br1 ? d : N - d;
  u64* v = (u64*)malloc(sizeof(u64) * (size_t)m * (N + 1));
  for (int i = 1; i <= m; i++)
    or_sample_extract(N, Q, ct, br1 ? (N - d + i) : i, v + (size_t)(i - 1) * (N + 1));
  u64* c = (u64*)malloc(sizeof(u64) * 2 * N);
  or_vector_pack(P, pack, v, m, c);
  u64* tmp = (u64*)malloc(sizeof(u64) * 2 * N);
  for (int h = 0; h < 2; h++) {
    if (br1) {               /* ct * X^d + 2 c */
      or_monomial_mul(N, Q, ct + h * N, d, tmp + h * N);
      for (int x = 0; x < N; x++) out[h * N + x] = addq(tmp[h * N + x], addq(c[h * N + x], c[h * N + x], Q), Q);
    } else {                 /* (2 c - ct) * X^d */
      for (int x = 0; x < N; x++) tmp[h * N + x] = subq(addq(c[h * N + x], c[h * N + x], Q), ct[h * N + x], Q);
      or_monomial_mul(N, Q, tmp + h * N, d, out + h * N);
    }
  }
  free(v); free(c); free(tmp);
}
void or_shift_batch(const u64* P, const u64* pack, const u64* ct, const uint32_t* d, int count, u64* out) {
  int N = (int)P[P_N];
  #pragma omp parallel for schedule(dynamic, 1) if (count > 1)
  for (int c = 0; c < count; c++)
    or_shift(P, pack, ct + (size_t)c * 2 * N, (int)d[c], 0, out + (size_t)c * 2 * N);
}

/* Permute(ct, pK, pi), reading P1: step 1.a packs the extracted sample
 * into slot 1, v[j] = Pack(SampleExt(ct, j), pK, 1) (message at X^0) -- with the printed
 * "Pack(., pK, j)" step 3.a would move m_j to X^{i+j-2} and the lemma fails.
 *   1. for i in [N] with pi(i) = j != i: v[j] = Pack(SampleExt(ct, j), pK, 1)
 *   2. ct_out = ct
 *   3. for i in [N] with pi(i) = j != i: ct_out += (v[j] - v[i]) X^{i-1}
 * perm[i-1] = pi(i) (1-based values).  literal != 0 uses the printed Pack(., pK, j) instead
 * (for the test that shows the reading is needed). */
void or_permute(const u64* P, const u64* pack, const u64* ct, const uint32_t* perm, int literal, u64* out) {
  int N = (int)P[P_N]; u64 Q = P[P_Q];
  u64* v = (u64*)calloc((size_t)N * 2 * N, sizeof(u64));
  u64* lwe = (u64*)malloc(sizeof(u64) * (N + 1));
  for (int i = 1; i <= N; i++) {
    int j = (int)perm[i - 1];
    if (j == i) continue;
    or_sample_extract(N, Q, ct, j, lwe);
    or_pack(P, pack, lwe, literal ? j : 1, v + (size_t)(j - 1) * 2 * N);
  }
  memcpy(out, ct, sizeof(u64) * 2 * N);
  u64* t = (u64*)malloc(sizeof(u64) * 2 * N);
  for (int i = 1; i <= N; i++) {
    int j = (int)perm[i - 1];
    if (j == i) continue;
    const u64* vj = v + (size_t)(j - 1) * 2 * N;
    const u64* vi = v + (size_t)(i - 1) * 2 * N;
    for (int h = 0; h < 2; h++) {
      poly_sub(N, Q, vj + h * N, vi + h * N, t + h * N);
      or_monomial_mul(N, Q, t + h * N, i - 1, t + h * N);
      poly_add(N, Q, out + h * N, t + h * N, out + h * N);
    }
  }
  free(v); free(lwe); free(t);
}
void or_permute_batch(const u64* P, const u64* pack, const u64* ct, const uint32_t* perm, int count, u64* out) {
  int N = (int)P[P_N];
  #pragma omp parallel for schedule(dynamic, 1) if (count > 1)
  for (int c = 0; c < count; c++)
    or_permute(P, pack, ct + (size_t)c * 2 * N, perm + (size_t)c * N, 0, out + (size_t)c * 2 * N);
}

/* ============================ Shift-based blind rotation / bootstrap (NEXT #4) ====
 * BlindRotate_Shift(brK, acc, ct, u, pK) (Def. Shifting Based Blind
 * Rotation): c = ModSwitch(ct, q, N) (done by the caller: abar in [0, N)); for i in [n],
 * j in [u]:  acc <- CMux(brK[i,j], Shift(acc, -a[i] u[j] mod N), acc).
 * Reading S1: Shift is defined for d in [N-1]; an amount of 0 is the
 * identity, so that step is CMux(brK, acc, acc) = acc (exactly: Decomp(0) = 0).
 * n_steps < n runs only the first n_steps LWE coefficients (timing samples). */
void or_blind_rotate_shift(const u64* P, const u64* brk, const u64* pack, u64* acc, const uint32_t* abar,
                           int n_steps) {
  int N = (int)P[P_N], ell = (int)P[P_ELL_RGSW], logL = (int)P[P_LOGL_RGSW], u = u_len(P);
  u64 Q = P[P_Q];
  u64* g = (u64*)malloc(sizeof(u64) * 2 * N);
  u64* out = (u64*)malloc(sizeof(u64) * 2 * N);
  for (int i = 0; i < n_steps; i++)
    for (int j = 0; j < u; j++) {
      int64_t d = (-(int64_t)abar[i] * u_val(P, j)) % N;
      if (d < 0) d += N;
      if (d == 0) memcpy(g, acc, sizeof(u64) * 2 * N);             /* reading S1 */
      else or_shift(P, pack, acc, (int)d, 0, g);
      const u64* C = brk + ((size_t)i * u + j) * (size_t)2 * ell * 2 * N;
      or_cmux(N, Q, logL, ell, C, g, acc, out);
      memcpy(acc, out, sizeof(u64) * 2 * N);
    }
  free(g); free(out);
}
/* Shift-Based Bootstrapping:
 *   1. rotP_b = Shift(rotP, b)        -- a plaintext cyclic shift: rotP_b[x] = rotP[(x - b) mod N]
 *      (the message map of Shift), with b the mod-switched b~ = ModSwitch(b, q, N)
 *      (reading S2: BlindRotate_Shift switches ct to Z_N in its step 1);
 *   2. acc = [rotP_b, 0]               (reading S3: the "RLWE(s, 0)" is the trivial encryption,
 *      as in the FDFB accumulator setup -- bootstrapping holds no secret key);
 *   3. acc_BR = BlindRotate_Shift(brK, acc, ct, u, pK);
 *   4-6. c_Q = SampleExt(acc_BR, 1); ModSwitch(Q -> q_lwe); KeySwitch mod q_lwe (order of c.3). */
static void bootstrap_shift_one(const u64* P, const u64* brk, const u64* pack, const u64* ksk, const u64* rotp,
                                const u64* ct, int n_steps, u64* out) {
  int N = (int)P[P_N], n = (int)P[P_n], logq = (int)P[P_LOGQLWE]; u64 Q = P[P_Q];
  u64 qlwe = 1ULL << logq;
  uint32_t* abar = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t bbar = (uint32_t)or_mod_switch(ct[0], qlwe, (u64)N);
  for (int i = 0; i < n; i++) abar[i] = (uint32_t)or_mod_switch(ct[1 + i], qlwe, (u64)N);
  u64* acc = (u64*)calloc((size_t)2 * N, sizeof(u64));
  for (int x = 0; x < N; x++) acc[x] = rotp[((x - (int)bbar) % N + N) % N];      /* steps 1-2 */
  or_blind_rotate_shift(P, brk, pack, acc, abar, n_steps);                        /* step 3 */
  u64* lwe = (u64*)malloc(sizeof(u64) * (N + 1));
  or_sample_extract(N, Q, acc, 1, lwe);                                            /* step 4 */
  for (int i = 0; i <= N; i++) lwe[i] = or_mod_switch(lwe[i], Q, qlwe);            /* step 5 */
  or_keyswitch_lwe(P, ksk, lwe, out);                                              /* step 6 */
  free(abar); free(acc); free(lwe);
}
void or_bootstrap_shift(const u64* P, const u64* brk, const u64* pack, const u64* ksk, const u64* rotp,
                        const u64* ct_in, int count, int n_steps, u64* ct_out) {
  int n = (int)P[P_n];
  #pragma omp parallel for schedule(dynamic, 1) if (count > 1)
  for (int c = 0; c < count; c++)
    bootstrap_shift_one(P, brk, pack, ksk, rotp, ct_in + (size_t)c * (n + 1), n_steps, ct_out + (size_t)c * (n + 1));
}

/* RLWE encryption of a batch of message polynomials (Shift inputs), domain 8. */
void or_rlwe_encrypt_batch(const u64* P, u64 seed, const int8_t* s, const u64* msgs, int count, u64* out) {
  int N = (int)P[P_N];
  #pragma omp parallel for schedule(dynamic, 1)
  for (int c = 0; c < count; c++)
    or_rlwe_encrypt(P, seed, 8, (u64)c, 0, 0, s, msgs + (size_t)c * N, out + (size_t)c * 2 * N);
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
