/*
 * fdfb.h -- C-ABI of the B200 (sm_100a) FDFB hot-path library libfdfb.so.
 *
 * Paper: "FDFB: Full Domain Functional Bootstrapping Towards Practical Fully
 * Homomorphic Encryption" (arXiv 2109.02731); line numbers are PAPER.md lines.
 *
 * Conventions (all entry points):
 *   - Every compute call is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*, NULL = legacy default stream) and never synchronises the host,
 *     except fdfb_ctx_create / fdfb_keygen* / fdfb_*_host which say so.
 *   - Buffers marked [dev] are caller-owned device memory, [host] host memory.
 *     The library keeps no pointer to caller memory after a call returns.
 *   - Return value: FDFB_OK (0) or a negative FDFB_E_* status; arguments are
 *     validated before any launch, so an error return means nothing ran,
 *     except FDFB_E_CUDA (a launch or runtime call failed; see
 *     fdfb_last_cuda_error).  Nothing throws across the ABI.
 *   - A batch count of 0 (B, count) returns FDFB_OK before any other check except
 *     the context: its data pointers may then be NULL (empty tensors).  The FDFB / TFHE
 *     bootstrap entry points accept B <= 2^24 per call, Shift, RLWE encryption and the
 *     shift-based bootstrap B <= 65535 (FDFB_E_DIMENSION above).
 *   - Calls run on the CUDA device that is current in the calling thread; it must be the
 *     context's device (one process or thread per GPU, as bench.py and dist.py do).
 *   - Ciphertext layouts (canonical, coefficient domain, residues canonical):
 *       LWE  [b, a_1..a_n] as uint64, mod q_lwe = 2^log_q_lwe (inputs/outputs
 *            of bootstrap/keyswitch) or mod Q (SampleExt outputs, VectorPack
 *            inputs)
 *       RLWE [b_0..b_{N-1}, a_0..a_{N-1}] uint64 mod Q
 *   - Key layouts on the device are OPAQUE (NTT domain, Shoup companions,
 *     suffix sums); fdfb_key_import/fdfb_keygen_canonical translate from/to the
 *     canonical layouts documented in DESIGN.md ("Canonical layouts").
 *   - Indices k (SampleExt) and d (Shift) are 1-based, as in the paper.
 */
#ifndef FDFB_H
#define FDFB_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum {
  FDFB_OK = 0,
  FDFB_E_NULL = -1,                 /* a required pointer is NULL                        */
  FDFB_E_NON_NTT_MODULUS = -2,      /* Q not prime or Q != 1 mod 2N          */
  FDFB_E_DIMENSION = -3,            /* N not in {256,512,1024,2048}, n out of range       */
  FDFB_E_DECOMP = -4,               /* ell != ceil(bits/logL) for some gadget             */
  FDFB_E_INDEX = -5,                /* SampleExt k or Shift d out of range                */
  FDFB_E_PLAINTEXT = -6,            /* t does not divide 2N, t_out == 0                   */
  FDFB_E_UNSUPPORTED = -7,          /* combination not implemented                        */
  FDFB_E_CUDA = -8,                 /* CUDA runtime / launch failure                      */
  FDFB_E_WORKSPACE = -9,            /* workspace too small                                */
  FDFB_E_KIND = -10                 /* unknown key kind                                   */
};

/* ------------------------------------------------------------------ params */
typedef struct fdfb_params {
  uint32_t N;          /* ring degree, power of two in [256, 2048]                         */
  uint32_t n;          /* LWE dimension, 1..4096                                           */
  uint64_t Q;          /* RLWE prime, Q = 1 mod 2N, Q < 2^55 (Q prime "to compute NTTs",
                          PAPER.md:2759; the paper's FDFB sets use 62/63-bit Q, PAPER.md:2618;
                          BASELINE's Large set: 54 bits)                                    */
  uint32_t log_q_lwe;  /* LWE modulus q_lwe = 2^log_q_lwe, max(8, log2(2N)+1)..55
                          (reading c.3)                                           */
  uint32_t lwe_key;    /* 0: binary s, u = [1];  1: ternary s, u = [-1, 1] */
  uint32_t rlwe_key;   /* 0: binary, 1: ternary ring secret                                */
  uint32_t logL_rgsw, ell_rgsw;   /* brK gadget   (L = 2^logL, ell = ceil(log_L Q))       */
  uint32_t logL_boot, ell_boot;   /* sign ladder / PubMux base L_boot     */
  uint32_t logL_pk, ell_pk;       /* bootstrap LWE->RLWE key pK            */
  uint32_t logL_ks, ell_ks;       /* LWE->LWE key ksK mod q_lwe            */
  uint32_t logL_pack, ell_pack;   /* Shift packing key               */
  uint32_t t;          /* plaintext modulus of bootstrap inputs, t | 2N                    */
  uint32_t sigma_milli;/* Gaussian sigma * 1000: 3200 (CDT shipped as data,
                          reading G17) or 0 = noiseless keys (tests); others UNSUPPORTED    */
} fdfb_params;

typedef struct fdfb_ctx fdfb_ctx;

/* Key kinds for fdfb_key_import / fdfb_keygen_canonical. Canonical layouts:
 *   BRK  [n][u][2*ell_rgsw][2][N]   RGSW rows, row r<ell: b-gadget
 *   BPK  [N][ell_pk][2][N]          RLWE_s(s_F[i] L^j)
 *        (device formats of BPK/KSK: the canonical table, then its int8 GEMM digits)
 *   KSK  [N][ell_ks][n+1]           LWE_s(s_F[i] L^j) mod q_lwe
 *   PACK [N][ell_pack][L_pack][2][N] RLWE_s(s_F[i] L^j k)
 *   SK_LWE int8[n], SK_RLWE int8[N]                                             */
enum { FDFB_KEY_BRK = 1, FDFB_KEY_BPK = 2, FDFB_KEY_KSK = 3, FDFB_KEY_PACK = 4,
       FDFB_KEY_SK_LWE = 5, FDFB_KEY_SK_RLWE = 6 };

typedef struct fdfb_sizes_t {
  size_t sk_lwe, sk_rlwe;       /* bytes of the int8 secrets                        */
  size_t brk, bpk, ksk, pack;   /* bytes of the OPAQUE device key formats (pack: canonical
                                   table + suffix sums T1, Delta, U)      */
  size_t canon_brk, canon_bpk, canon_ksk, canon_pack;  /* canonical layouts (bytes) */
} fdfb_sizes_t;

/* Create a context on `device`: validates params (FDFB_E_*), derives 2N-th roots,
 * twiddle tables and the CDT table, uploads them.  Synchronises the device. */
int fdfb_ctx_create(const fdfb_params* p, int device, fdfb_ctx** out);
void fdfb_ctx_destroy(fdfb_ctx* ctx);
int fdfb_sizes(const fdfb_ctx* ctx, fdfb_sizes_t* out);
/* Workspace bytes needed by fdfb_bootstrap_batch / fdfb_shift / fdfb_vector_pack for B items. */
size_t fdfb_workspace_bootstrap(const fdfb_ctx* ctx, uint32_t B);
size_t fdfb_workspace_shift(const fdfb_ctx* ctx, uint32_t B);
size_t fdfb_workspace_vector_pack(const fdfb_ctx* ctx, uint32_t m, uint32_t B);

/* ------------------------------------------------------------------ keys
 * Keygen from a 64-bit seed with the counter-based Philox4x64-10 sampling spec of
 * DESIGN.md ("Seeded determinism"): BRKeyGen, KeySwitchSetup
 * for pK and ksK (2369-2371, 2992-3001), PackSetup (1284-1296).  which: bitmask
 * 1=secrets 2=brk 4=bpk 8=ksk 16=pack; pointers of unselected keys may be NULL,
 * but brk/bpk/ksk/pack need the secrets in sk_lwe/sk_rlwe [dev] (generated in the
 * same call if bit 1 is set).  workspace [dev] of fdfb_workspace_keygen(ctx) bytes (may be
 * NULL when only secrets are generated; FDFB_E_WORKSPACE otherwise).  Syncs.  Like every
 * entry point, it allocates no device memory (all scratch comes from the caller). */
size_t fdfb_workspace_keygen(const fdfb_ctx* ctx);
int fdfb_keygen(const fdfb_ctx* ctx, uint64_t seed, uint32_t which, int8_t* sk_lwe, int8_t* sk_rlwe,
                void* brk, void* bpk, void* ksk, void* pack, void* workspace, void* stream);
/* Canonical key entries for parity checks: `count` entries with flat canonical entry
 * indices idx[] [host] (BRK: (i*u+j)*2ell+row; BPK/KSK: i*ell+j; PACK: (i*ell+j)*L+k),
 * written back to back into out [dev] (2N words per RLWE entry, n+1 per LWE entry).
 * workspace [dev] of fdfb_workspace_keygen_canonical(ctx, count) bytes.  Syncs. */
size_t fdfb_workspace_keygen_canonical(const fdfb_ctx* ctx, uint32_t count);
int fdfb_keygen_canonical(const fdfb_ctx* ctx, uint64_t seed, int kind, const int8_t* sk_lwe,
                          const int8_t* sk_rlwe, const uint64_t* idx, uint32_t count, uint64_t* out,
                          void* workspace, void* stream);
/* Convert a canonical key [dev] to the opaque device format [dev].  Syncs. */
int fdfb_key_import(const fdfb_ctx* ctx, int kind, const uint64_t* canonical, void* dev_key, void* stream);

/* Canonical layout of a device key [dev] -> canonical [dev] (all kinds; BRK, held only as
 * RNS residues in the NTT domain, is brought back by inverse NTTs and the CRT -- exact, since
 * every canonical coefficient is below Q < P).  Stream-ordered. */
int fdfb_key_export(const fdfb_ctx* ctx, int kind, const void* dev_key, uint64_t* canonical, void* stream);

/* ------------------------------------------------------------------ inputs
 * LWE encryptions of m[c] in Z_t (Delta = q_lwe/t) under sk_lwe, c = 0 ..
 * count-1 -> out[c], drawn as object first_index + c of domain 7 (a shard of a global batch
 * passes its global offset and encrypts exactly what one device would).  flags bit0:
 * mod-switch-exact inputs. */
int fdfb_lwe_encrypt(const fdfb_ctx* ctx, uint64_t seed, const int8_t* sk_lwe, const uint64_t* msg,
                     uint32_t count, uint32_t flags, uint64_t first_index, uint64_t* out, void* stream);
/* RLWE encryptions of message polynomials msg [dev, count x N] (domain 8, objects
 * first_index + c).  workspace [dev] of fdfb_workspace_rlwe_encrypt(ctx, count) bytes. */
size_t fdfb_workspace_rlwe_encrypt(const fdfb_ctx* ctx, uint32_t count);
int fdfb_rlwe_encrypt(const fdfb_ctx* ctx, uint64_t seed, const int8_t* sk_rlwe, const uint64_t* msg,
                      uint32_t count, uint64_t first_index, uint64_t* out, void* workspace, void* stream);

/* ------------------------------------------------------------------ decryption (secret-key side)
 * Phase of LWE ciphertexts ct [dev, count x (n+1)] mod q_lwe under sk_lwe [dev, n int8]:
 * phase[c] = b - <a, s> mod q_lwe.  With t > 0 also decoded: msg[c] =
 * round(t phase / q_lwe) mod t (PAPER.md:1725 rounding, ties up); msg may be NULL.
 * phase [dev, count] may be NULL when only msg is wanted. */
int fdfb_lwe_decrypt(const fdfb_ctx* ctx, const int8_t* sk_lwe, const uint64_t* ct, uint32_t count, uint32_t t,
                     uint64_t* phase, uint64_t* msg, void* stream);
/* Phase of RLWE ciphertexts ct [dev, count x 2 x N] under sk_rlwe [dev, N int8]:
 * out = b - a * s mod Q (negacyclic product) [dev, count x N].
 * workspace [dev] of fdfb_workspace_rlwe_phase(ctx, count) bytes. */
size_t fdfb_workspace_rlwe_phase(const fdfb_ctx* ctx, uint32_t count);
int fdfb_rlwe_phase(const fdfb_ctx* ctx, const int8_t* sk_rlwe, const uint64_t* ct, uint32_t count, uint64_t* out,
                    void* workspace, void* stream);

/* ------------------------------------------------------------------ LUT
 * BootsMap[x] = round(Q/t_out) * lut[x] then SetupPolynomial
 * (Fig. SetupPolynomial, half-open windows, reading F6).
 * lut [host, t values in Z_t_out]; rotp [dev, 2 x N] = (rotP_0, rotP_1). */
int fdfb_setup_lut(const fdfb_ctx* ctx, const uint64_t* lut, uint32_t t_out, uint64_t* rotp, void* stream);

/* ------------------------------------------------------------------ hot path
 * FDFB Bootstrap (Fig. Bootstrap; readings R1, F4, c.3):
 * ct_in [dev, B x (n+1)] mod q_lwe -> ct_out [dev, B x (n+1)] mod q_lwe encrypting
 * f(m).  workspace [dev] of fdfb_workspace_bootstrap(ctx, B) bytes. */
int fdfb_bootstrap_batch(const fdfb_ctx* ctx, const void* brk, const void* bpk, const void* ksk,
                         const uint64_t* rotp, const uint64_t* ct_in, uint64_t* ct_out, uint32_t B,
                         void* workspace, void* stream);
/* FDFB Bootstrap of B ciphertexts under k LUTs at once (rotp: [dev, k x 2 x N], one
 * fdfb_setup_lut output per function): the ell_boot ladder rotations, their SampleExt and the
 * LWE->RLWE key switch are computed once and reused by all k functions (PAPER.md:2568-2570:
 * ell_boot + k blind rotations instead of k (ell_boot + 1)).  ct_out [dev, k x B x (n+1)];
 * output kk equals fdfb_bootstrap_batch under LUT kk byte for byte.  workspace [dev] of
 * fdfb_workspace_bootstrap_multi(ctx, B, k) bytes. */
size_t fdfb_workspace_bootstrap_multi(const fdfb_ctx* ctx, uint32_t B, uint32_t k);
int fdfb_bootstrap_multi_batch(const fdfb_ctx* ctx, const void* brk, const void* bpk, const void* ksk,
                               const uint64_t* rotp, uint32_t k, const uint64_t* ct_in, uint64_t* ct_out,
                               uint32_t B, void* workspace, void* stream);
/* TFHE (half-domain) bootstrap (Fig. TFHE Bootstrapping PAPER.md:3070-3090, Thm 2109-2139;
 * output order of reading c.3): one blind rotation of [rotP_0 X^{b~}, 0] (rotp [dev, 2 x N]
 * from fdfb_setup_lut; only rotP_0 is used), SampleExt, ModSwitch Q -> q_lwe, KeySwitch.
 * Correct for m < t/2; upper-half inputs return -F(m - t/2) (negacyclicity).  workspace of
 * fdfb_workspace_bootstrap(ctx, B) bytes. */
int fdfb_bootstrap_tfhe_batch(const fdfb_ctx* ctx, const void* brk, const void* ksk, const uint64_t* rotp,
                              const uint64_t* ct_in, uint64_t* ct_out, uint32_t B, void* workspace, void* stream);
/* Shift-based bootstrap (Def. PAPER.md:318-337 over BlindRotate_Shift PAPER.md:207-221,
 * readings S1-S3, output order of c.3): ct_in [dev, B x (n+1)] mod q_lwe is switched to Z_N;
 * acc = [Shift(rotP, b~), 0] with rotp [dev, N] ONE plaintext polynomial in [0, Q) (the
 * cyclic rotation rotP[(x - b~) mod N]); for every (i, j): acc <- CMux(brK[i,j],
 * Shift(acc, -a~_i u_j mod N), acc), the Shift evaluated homomorphically with the packing
 * key `pack` (fdfb_keygen / fdfb_key_import FDFB_KEY_PACK; one int8 GEMM per step for
 * L_pack = 2, else the streaming kernel); then SampleExt(., 1), ModSwitch Q -> q_lwe,
 * KeySwitch -> ct_out [dev, B x (n+1)].  Evaluates ANY map Z_N -> Z_Q placed in rotP
 * (full domain, no sign ladder); n u Shift evaluations per batch.  workspace [dev] of
 * fdfb_workspace_bootstrap_shift(ctx, B) bytes. */
size_t fdfb_workspace_bootstrap_shift(const fdfb_ctx* ctx, uint32_t B);
int fdfb_bootstrap_shift_batch(const fdfb_ctx* ctx, const void* brk, const void* pack, const void* ksk,
                               const uint64_t* rotp, const uint64_t* ct_in, uint64_t* ct_out, uint32_t B,
                               void* workspace, void* stream);
/* Same, with ct_in/ct_out in (pinned) HOST memory: H2D copy, bootstrap, D2H copy,
 * all on `stream`; synchronises the stream before returning. */
int fdfb_bootstrap_batch_host(const fdfb_ctx* ctx, const void* brk, const void* bpk, const void* ksk,
                              const uint64_t* rotp, const uint64_t* ct_in_host, uint64_t* ct_out_host,
                              uint32_t B, void* workspace, void* stream);
/* BlindRotate: acc [dev, count x 2 x N] in/out, abar [dev,
 * count x n] in Z_2N; accumulator g uses abar row g / acc_per_ct. */
int fdfb_blind_rotate(const fdfb_ctx* ctx, const void* brk, uint64_t* acc, const uint32_t* abar,
                      uint32_t count, uint32_t acc_per_ct, void* stream);
/* SampleExt (NSgn(0) = -1): rlwe [dev, B x 2N], k [dev, B, 1..N],
 * lwe [dev, B x (N+1)] mod Q.  A k outside 1..N (device data, not checkable before
 * launch) yields a zero row and raises the flag read by fdfb_device_status. */
int fdfb_sample_extract(const fdfb_ctx* ctx, const uint64_t* rlwe, const uint32_t* k, uint64_t* lwe,
                        uint32_t B, void* stream);
/* LWE KeySwitch N -> n mod q_lwe: in [dev, B x (N+1)] mod q_lwe,
 * out [dev, B x (n+1)].  With workspace [dev] of fdfb_workspace_keyswitch(ctx, B) bytes the
 * switch runs as one exact int8 tensor-core GEMM (digit limbs x balanced base-256 key
 * digits on the tcgen05 kernel, recombined in its epilogue); with workspace NULL
 * through the tiled CUDA-core kernel.  Same bytes. */
size_t fdfb_workspace_keyswitch(const fdfb_ctx* ctx, uint32_t B);
int fdfb_lwe_keyswitch(const fdfb_ctx* ctx, const void* ksk, const uint64_t* lwe_N, uint64_t* lwe_n,
                       uint32_t B, void* workspace, void* stream);
/* VectorPack: lwe [dev, B x m x (N+1)] mod Q under s_F,
 * 1 <= m <= N; out [dev, B x 2N] = sum_k Pack(lwe_k, pK, k), computed by the definition
 * (m N ell key-row additions per item).  workspace may be NULL (size 0). */
int fdfb_vector_pack(const fdfb_ctx* ctx, const void* pack, const uint64_t* lwe, uint32_t m, uint64_t* out,
                     uint32_t B, void* workspace, void* stream);
/* Pack (reading G5): out[b] = [b X^{d-1}, 0] - X^{d-1} sum_{i,j}
 * pK[i, j, A[i,j]+1] for lwe [dev, B x (N+1)] mod Q and d [dev, B, 1-based]. */
int fdfb_pack(const fdfb_ctx* ctx, const void* pack, const uint64_t* lwe, const uint32_t* d, uint64_t* out,
              uint32_t B, void* stream);
/* Shift (readings F2/F3/G4): rlwe_in [dev, B x 2N] mod Q encrypting m,
 * d [dev, B, 1..N-1] -> rlwe_out [dev, B x 2N] encrypting the cyclic rotation of m by d.
 * VectorPack is evaluated through the exact suffix-sum identity of DESIGN.md; for
 * L_pack = 2 as one int8 tensor-core GEMM (bit matrix x balanced base-256 key digits,
 * exact in int32) plus a finishing kernel -- workspace [dev] of fdfb_workspace_shift(ctx, B)
 * bytes is then required (FDFB_E_WORKSPACE if NULL); for L_pack > 2 by the streaming kernel
 * (workspace may be NULL).  A d outside 1..N-1 yields a zero row and raises the
 * fdfb_device_status flag. */
int fdfb_shift(const fdfb_ctx* ctx, const void* pack, const uint64_t* rlwe_in, const uint32_t* d,
               uint64_t* rlwe_out, uint32_t B, void* workspace, void* stream);
/* Permute (reading P1: v[j] = Pack(SampleExt(ct, j), pK, 1)):
 * rlwe_in [dev, B x 2N] encrypting m, perm [dev, B x N] with perm[i-1] = pi(i) (1-based, a
 * permutation of 1..N) -> rlwe_out [dev, B x 2N] encrypting sum_i m_{pi(i)} X^{i-1}.  For
 * L_pack = 2 every moved slot is one row of an exact int8 tensor-core GEMM against the digits
 * of pK[.,.,1] - pK[.,.,0] (workspace [dev] of fdfb_workspace_permute(ctx, B) bytes
 * required); otherwise the definition is evaluated directly (workspace may be NULL).  An
 * entry outside 1..N is treated as a fixed point and raises the fdfb_device_status flag. */
size_t fdfb_workspace_permute(const fdfb_ctx* ctx, uint32_t B);
int fdfb_permute(const fdfb_ctx* ctx, const void* pack, const uint64_t* rlwe_in, const uint32_t* perm,
                 uint64_t* rlwe_out, uint32_t B, void* workspace, void* stream);
/* The same Shift through the streaming (CUDA-core) kernel for any L_pack; no workspace. */
int fdfb_shift_streaming(const fdfb_ctx* ctx, const void* pack, const uint64_t* rlwe_in, const uint32_t* d,
                         uint64_t* rlwe_out, uint32_t B, void* stream);

/* ------------------------------------------------------------------ kernel unit tests
 * Negacyclic ring product through the NTT kernels: c = a * b mod (X^N+1, Q),
 * a, b, c [dev, count x N]; workspace [dev] of fdfb_workspace_poly_mul(ctx, count) bytes. */
size_t fdfb_workspace_poly_mul(const fdfb_ctx* ctx, uint32_t count);
int fdfb_poly_mul(const fdfb_ctx* ctx, const uint64_t* a, const uint64_t* b, uint64_t* c, uint32_t count,
                  void* workspace, void* stream);
/* The int8 tensor-core contraction under both key switches, Shift and Permute
 * (kernels_imma.cuh: TMA loads, tcgen05.mma kind::i8, int32 accumulators in TMEM), with its
 * raw epilogue: D [dev, M x Ncols] int32 = A [dev, M x K] int8 (K-major) x B [dev, Ncols x K]
 * int8 (K-major)^T, exact.  K must be a positive multiple of 16 and the operands 16-byte
 * aligned (FDFB_E_DIMENSION / FDFB_E_CUDA otherwise).  Unit test of the GEMM itself. */
int fdfb_gemm_i8(const fdfb_ctx* ctx, const int8_t* A, const int8_t* B, uint32_t M, uint32_t Ncols, uint32_t K,
                 int32_t* D, void* stream);
/* The library's own CDT thresholds (2T values) into thr [host]; *T = tail cut. */
int fdfb_cdt_table(const fdfb_ctx* ctx, uint64_t* thr, int* T);
/* Per-kernel-class timing for the roofline report: when enabled, every launch of the
 * classes below is bracketed by CUDA events recorded on the launching stream.
 * fdfb_timing_read waits for the recorded events of class `kclass`, returns their
 * summed device time (ms) and launch count, and forgets them. */
enum { FDFB_KCLASS_BLIND_ROTATE = 0, FDFB_KCLASS_KEYSWITCH_RLWE = 1, FDFB_KCLASS_KEYSWITCH_LWE = 2,
       FDFB_KCLASS_SHIFT = 3, FDFB_KCLASS_SHIFT_GEMM = 4 };
int fdfb_timing_enable(const fdfb_ctx* ctx, int on);
int fdfb_timing_read(const fdfb_ctx* ctx, int kclass, double* total_ms, uint64_t* launches);
/* As fdfb_timing_read, but *union_ms is the span covered by the launches (the union of their
 * [start, end] intervals): launches of one call on two streams may overlap. */
int fdfb_timing_read_union(const fdfb_ctx* ctx, int kclass, double* union_ms, uint64_t* launches);
/* Device-side argument errors of earlier stream-ordered calls: synchronises, returns
 * FDFB_E_INDEX if any kernel saw an out-of-range k/d since the last clear, else FDFB_OK. */
int fdfb_device_status(const fdfb_ctx* ctx, int clear);
/* Number of kernel launches issued by this context so far (bench evidence). */
uint64_t fdfb_launch_count(const fdfb_ctx* ctx);
const char* fdfb_status_string(int status);
const char* fdfb_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FDFB_H */
