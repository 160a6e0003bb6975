// fdfb_api.cu -- the C-ABI of libfdfb.so (include/fdfb.h): parameter validation,
// context setup (roots of unity, twiddles, CDT), key generation/import and the
// stream-ordered orchestration of the hot-path kernels.  Unity build: the kernel
// headers are included here.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/fdfb.h"
#include "kernels_boot.cuh"
#include "kernels_shift.cuh"

typedef unsigned __int128 u128;

struct fdfb_ctx {
  fdfb_params prm;
  DevParams dp;
  int device;
  int num_sms;
  u64 qinv_neg, r2;          // Montgomery constants
  u64* d_tables;             // tw | twp | itw | itwp | cdt | omega tables
  int* d_status;             // device-side argument errors (bit 0: index out of range)
  RnsParams rns;             // word-size primes for the exact RNS external product (kernels_br.cuh)
  u32* d_rtab;               // [2 dirs][np][GROUPS][8 pairs] twiddle tables
  u64 omega_off;             // offset of NTT(X) slots (omega) in d_tables
  std::vector<u64> cdt;
  mutable std::atomic<unsigned long long> launches{0};
  // optional per-kernel-class CUDA-event timing (fdfb_timing_enable / fdfb_timing_read)
  mutable std::mutex tmu;
  mutable bool timing = false;
  mutable std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> tev;
  int br_cluster = 1;        // FDFB_BR_CLUSTER: 0 batched only, 1 auto (default), 2 / 3 force clusters of NP / 2 NP
  int imma_cg = 2;           // FDFB_IMMA_CG: int8 GEMM tiles per CTA pair (2, default) or per CTA (1)
  int br_kernel = 2;         // FDFB_BR_KERNEL: 2 pipelined k_blind_rotate_p (default), 1 k_blind_rotate
  int boot_split = 1;        // FDFB_BOOT_SPLIT: 1 run the bootstrap as two stream-overlapped halves, 0 one part
  cudaStream_t helper = nullptr;          // second stream of the two-part bootstrap (created at ctx_create)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  mutable std::mutex boot_mu;             // serialises the fork/join enqueue of concurrent callers
  int imma_wide_k = 65536;   // FDFB_IMMA_WIDE_K: K from which pair tiles are 448 columns wide
  // key-stream pacing of k_blind_rotate_p (kernels_br.cuh pace_wait): FDFB_BR_PACE = "wlo,whi" in
  // steps, "0" off; one position slot per CTA in one of BR_PACE_SLOTS per-launch regions
  u32 br_wlo = 32, br_whi = 160, br_wcap = 8;     // cap: at most 8 sleeps of ~2 us per check
  bool br_pace_split = true;              // FDFB_BR_PACE_SPLIT=0: do not pace the two-part bootstrap's halves
  u64* d_prog = nullptr;                  // [BR_PACE_SLOTS][BR_PACE_MAXGRID], allocated at ctx_create
  mutable std::atomic<u32> br_tag{0};
};
#define BR_PACE_SLOTS 16
#define BR_PACE_MAXGRID 4096

// Bracket one launch of kernel class `cls` with events on its stream when timing is on.
struct TimedLaunch {
  const fdfb_ctx* c; int cls; cudaStream_t st; cudaEvent_t e1 = nullptr;
  TimedLaunch(const fdfb_ctx* c_, int cls_, cudaStream_t st_) : c(c_), cls(cls_), st(st_) {
    if (!c->timing) return;
    cudaEvent_t e0;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    std::lock_guard<std::mutex> g(c->tmu);
    c->tev.push_back({cls, {e0, e1}});
  }
  ~TimedLaunch() { if (e1) cudaEventRecord(e1, st); }
};

static thread_local std::string g_last_cuda;
struct PackLayout;
static size_t shift_pack_bytes(const fdfb_params& p);
static int pack_keygen(const fdfb_ctx* c, u64 seed, const int8_t* s_rlwe, void* pack, u64* shat, u64* tmask,
                       u64* tprod, int CH, cudaStream_t st);
static int pack_import(const fdfb_ctx* c, const u64* canon, void* dev, cudaStream_t st);

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t _e = (x);                                                  \
    if (_e != cudaSuccess) {                                               \
      g_last_cuda = std::string(#x) + ": " + cudaGetErrorString(_e);       \
      return FDFB_E_CUDA;                                                  \
    }                                                                      \
  } while (0)
#define CKL(ctx)                                                           \
  do {                                                                     \
    (ctx)->launches++;                                                     \
    cudaError_t _e = cudaGetLastError();                                   \
    if (_e != cudaSuccess) {                                               \
      g_last_cuda = std::string("launch: ") + cudaGetErrorString(_e);      \
      return FDFB_E_CUDA;                                                  \
    }                                                                      \
  } while (0)

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

// ------------------------------------------------------------------ host number theory
static u64 h_mulmod(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
static u64 h_powmod(u64 b, u64 e, u64 m) {
  u64 r = 1 % m; b %= m;
  while (e) { if (e & 1) r = h_mulmod(r, b, m); b = h_mulmod(b, b, m); e >>= 1; }
  return r;
}
static bool h_is_prime(u64 n) {   // deterministic Miller-Rabin for 64-bit
  if (n < 2) return false;
  for (u64 p : {2ULL, 3ULL, 5ULL, 7ULL, 11ULL, 13ULL, 17ULL, 19ULL, 23ULL, 29ULL, 31ULL, 37ULL}) {
    if (n % p == 0) return n == p;
  }
  u64 d = n - 1; int s = 0;
  while ((d & 1) == 0) { d >>= 1; s++; }
  for (u64 a : {2ULL, 3ULL, 5ULL, 7ULL, 11ULL, 13ULL, 17ULL, 19ULL, 23ULL, 29ULL, 31ULL, 37ULL}) {
    u64 x = h_powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; r++) { x = h_mulmod(x, x, n); if (x == n - 1) { comp = false; break; } }
    if (comp) return false;
  }
  return true;
}
static int bits_of(u64 x) { int b = 0; while (b < 64 && (x >> b)) b++; return b; }   // ceil(log2(x+1))
static int ceil_log2(u64 x) { int b = 0; while ((1ULL << b) < x) b++; return b; }
static u64 shoup_of(u64 w, u64 Q) { return (u64)(((u128)w << 64) / Q); }
static int bitrev(int x, int logn) { int r = 0; for (int i = 0; i < logn; i++) r |= ((x >> i) & 1) << (logn - 1 - i); return r; }

// Library-side CDT (reading G17): the thresholds floor(2^64 CDF(-T + k)) for sigma = 3.2 are
// data, generated once with exact fixed-point arithmetic by tools/gen_cdt_table.py (its own
// derivation, shared with no test code); sigma_milli = 0 means noiseless keys, other sigmas are rejected.
#include "cdt_table.inc"
static bool make_cdt(uint32_t sigma_milli, std::vector<u64>* thr, int* Tout) {
  thr->clear();
  *Tout = 0;
  if (sigma_milli == 0) return true;
  if (sigma_milli != kCdtSigmaMilli) return false;
  thr->assign(kCdtThr, kCdtThr + 2 * kCdtT);
  *Tout = kCdtT;
  return true;
}

// ------------------------------------------------------------------ launch helpers
static int grid_for(size_t total, int threads, int num_sms) {
  size_t g = (total + threads - 1) / threads;
  size_t cap = (size_t)num_sms * 32;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <int N>
static int launch_ntt_batch_t(const fdfb_ctx* c, u64* data, int count, int mode, cudaStream_t st) {
  constexpr int T = N / 8;
  int G = T >= 256 ? 1 : 256 / T;
  dim3 blk(T, G);
  dim3 grd((count + G - 1) / G);
  size_t sm = (size_t)G * N * sizeof(u64);
  k_ntt_batch<N><<<grd, blk, sm, st>>>(c->dp, data, count, mode);
  CKL(c);
  return FDFB_OK;
}
static int launch_ntt_batch(const fdfb_ctx* c, u64* data, size_t count, int mode, cudaStream_t st) {
  // chunk to keep grid.x within limits
  const size_t CH = 1 << 20;
  for (size_t o = 0; o < count; o += CH) {
    int cnt = (int)((count - o) < CH ? (count - o) : CH);
    u64* d = data + o * c->prm.N;
    int rc;
    switch (c->prm.N) {
      case 256: rc = launch_ntt_batch_t<256>(c, d, cnt, mode, st); break;
      case 512: rc = launch_ntt_batch_t<512>(c, d, cnt, mode, st); break;
      case 1024: rc = launch_ntt_batch_t<1024>(c, d, cnt, mode, st); break;
      case 2048: rc = launch_ntt_batch_t<2048>(c, d, cnt, mode, st); break;
      default: return FDFB_E_DIMENSION;
    }
    if (rc) return rc;
  }
  return FDFB_OK;
}

// co-resident clusters of k_blind_rotate_cl (a cluster must fit a GPC, so fewer than
// num_sms / (NP SPLIT) in general)
template <int N, int NP, int SPLIT>
static int br_cluster_slots(const fdfb_ctx* c) {
  const size_t sm = 66 * (size_t)N;
  cudaFuncSetAttribute(k_blind_rotate_cl<N, NP, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(NP * SPLIT * c->num_sms);
  cfg.blockDim = dim3(N / 8);
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = NP * SPLIT; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int num = 0;
  if (cudaOccupancyMaxActiveClusters(&num, k_blind_rotate_cl<N, NP, SPLIT>, &cfg) != cudaSuccess || num < 1) {
    cudaGetLastError();
    num = c->num_sms / (NP * SPLIT);
  }
  return num;
}

template <int N, int NP, int SPLIT>
static int launch_br_cl_t(const fdfb_ctx* c, const u32* bsk, u64* accs, int n_acc, int acc_per_ct, int abar_rows,
                          const u32* abar, cudaStream_t st) {
  constexpr int T = N / 8;
  const size_t sm = 66 * (size_t)N;            // sacc 16N + sd 16N + 2 exchange buffers 18N + 2 residue slots 16N
  cudaFuncSetAttribute(k_blind_rotate_cl<N, NP, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  TimedLaunch tl(c, FDFB_KCLASS_BLIND_ROTATE, st);
  k_blind_rotate_cl<N, NP, SPLIT><<<NP * SPLIT * n_acc, T, sm, st>>>(c->dp, c->rns, bsk, accs, n_acc, acc_per_ct,
                                                                       abar_rows, abar);
  CKL(c);
  return FDFB_OK;
}

// small-batch path selection: 0 = batched kernel, 1 = clusters of NP, 2 = clusters of 2 NP
template <int N, int NP>
static int br_cluster_choice(const fdfb_ctx* c, int n_acc) {
  if (c->br_cluster == 0) return 0;
  if (c->br_cluster == 2) return 1;
  if (c->br_cluster == 3) return 2;
  if (n_acc > c->num_sms) return 0;
  if (n_acc <= br_cluster_slots<N, NP, 2>(c)) return 2;                  // one wave of split clusters
  const int slots = br_cluster_slots<N, NP, 1>(c);
  return n_acc <= (NP == 3 ? 2 : 1) * slots ? 1 : 0;
}

template <int N, int NP>
static int launch_br_small(const fdfb_ctx* c, const u32* bsk, u64* accs, int n_acc, int acc_per_ct, int abar_rows,
                           const u32* abar, cudaStream_t st, bool* done) {
  *done = true;
  switch (br_cluster_choice<N, NP>(c, n_acc)) {
    case 2: return launch_br_cl_t<N, NP, 2>(c, bsk, accs, n_acc, acc_per_ct, abar_rows, abar, st);
    case 1: return launch_br_cl_t<N, NP, 1>(c, bsk, accs, n_acc, acc_per_ct, abar_rows, abar, st);
  }
  *done = false;
  return FDFB_OK;
}

template <int N, int NP, bool GIN>
static int launch_br_t(const fdfb_ctx* c, const u32* bsk, u64* accs, int n_acc, int acc_per_ct, int abar_rows,
                       const u32* abar, const u64* gin, int s_begin, cudaStream_t st, bool pace) {
  constexpr int T = N / 8;
  if (c->br_kernel != 1) {                     // pipelined kernel (mbarrier-decoupled exchanges, d in TMEM)
    const size_t sm = (25 + 9 * BR_NB) * (size_t)N;   // acc 16N + NB cross-warp buffers 9N each + slabs 9N
    cudaFuncSetAttribute(k_blind_rotate_p<N, NP, GIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_blind_rotate_p<N, NP, GIN>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blind_rotate_p<N, NP, GIN>, T, sm);
    // the occupancy query under-reports this kernel (1 per SM at N = 2048 where registers and shared
    // memory both allow 2, as ncu's launch__occupancy_limit_* confirm): also bound it directly
    {
      int smem_sm = 0, regs_sm = 0;
      cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->device);
      cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, c->device);
      int by_smem = smem_sm / (int)(sm + 1024 + 64), by_regs = regs_sm / (T * 128);
      int est = by_smem < by_regs ? by_smem : by_regs;
      if (est > BrShape<N>::MINB) est = BrShape<N>::MINB;
      if (est > per_sm) per_sm = est;
    }
    cudaGetLastError();
    if (getenv("FDFB_DEBUG")) fprintf(stderr, "k_blind_rotate_p<%d,%d,%d>: %d CTAs per SM\n", N, NP, (int)GIN, per_sm);
    if (per_sm < 1) per_sm = 1;
    const int tmem_cap = 512 / ((N >= 1024 ? 128 : 32) * (T > 128 ? 2 : 1));   // TMEM columns per CTA
    if (per_sm > tmem_cap) per_sm = tmem_cap;
    int grid = c->num_sms * per_sm;
    if (grid > n_acc) grid = n_acc;
    // pacing (kernels_br.cuh pace_wait): only where a CTA processes more than one accumulator
    u32 tag = 0, wlo = 0, whi = 0, wcap = 0;
    u64* prog = nullptr;
    if (!GIN && pace && c->br_wlo && grid <= BR_PACE_MAXGRID && n_acc > grid) {
      do tag = ++c->br_tag; while (tag == 0);
      prog = c->d_prog + (size_t)(tag % BR_PACE_SLOTS) * BR_PACE_MAXGRID;
      wlo = c->br_wlo; whi = c->br_whi; wcap = c->br_wcap;
    }
    TimedLaunch tl(c, FDFB_KCLASS_BLIND_ROTATE, st);
    k_blind_rotate_p<N, NP, GIN><<<grid, T, sm, st>>>(c->dp, c->rns, bsk, accs, n_acc, acc_per_ct, abar_rows, abar,
                                                       gin, s_begin, prog, tag, wlo, whi, wcap);
    CKL(c);
    return FDFB_OK;
  }
  const size_t sm = 50 * (size_t)N;            // sacc 16N + sd 16N + 2 exchange buffers x 2 planes 9N bytes
  // function attributes are per device: set on every launch (host-side, ~µs), not once per process
  cudaFuncSetAttribute(k_blind_rotate<N, NP, GIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blind_rotate<N, NP, GIN>, T, sm);
  if (per_sm < 1) per_sm = 1;
  int grid = c->num_sms * per_sm;
  if (grid > n_acc) grid = n_acc;
  TimedLaunch tl(c, FDFB_KCLASS_BLIND_ROTATE, st);
  k_blind_rotate<N, NP, GIN><<<grid, T, sm, st>>>(c->dp, c->rns, bsk, accs, n_acc, acc_per_ct, abar_rows, abar,
                                                   gin, s_begin);
  CKL(c);
  return FDFB_OK;
}
// blind-rotate n_acc accumulators; accumulator g uses mask row (g / acc_per_ct) % abar_rows
// gin != nullptr: one shift-based step s_begin (k_blind_rotate GIN mode), else steps [0, n u)
static int launch_br(const fdfb_ctx* c, const u64* bsk, u64* accs, int n_acc, int acc_per_ct, const u32* abar,
                     cudaStream_t st, int abar_rows = 0, const u64* gin = nullptr, int s_begin = 0, bool pace = true) {
  if (n_acc <= 0) return FDFB_OK;
  if (abar_rows <= 0) abar_rows = (n_acc + acc_per_ct - 1) / acc_per_ct;
  const u32* k = (const u32*)bsk;
  const int np = c->rns.np;
  // small passes: clusters of np (or 2 np) CTAs per accumulator, one RNS prime (and one d half)
  // per CTA, same arithmetic (k_blind_rotate_cl).  Measured at N = 2048, np = 3
  // (profiles/r01/latency): chosen when the batched kernel would run one CTA per SM and the
  // clusters need at most two waves (np = 2: one); FDFB_BR_CLUSTER = 0 / 2 / 3 forces batched /
  // clusters of np / clusters of 2 np.
  if (!gin && np > 1) {
    bool done = false;
    int rc = FDFB_OK;
    switch (c->prm.N) {
      case 256: rc = np == 3 ? launch_br_small<256, 3>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, st, &done)
                             : launch_br_small<256, 2>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, st, &done); break;
      case 512: rc = np == 3 ? launch_br_small<512, 3>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, st, &done)
                             : launch_br_small<512, 2>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, st, &done); break;
      case 1024: rc = np == 3 ? launch_br_small<1024, 3>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, st, &done)
                              : launch_br_small<1024, 2>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, st, &done); break;
      case 2048: rc = np == 3 ? launch_br_small<2048, 3>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, st, &done)
                              : launch_br_small<2048, 2>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, st, &done); break;
    }
    if (done) return rc;
  }
  const int s0 = gin ? s_begin : 0;
#define BR_CASE(NN)                                                                                          \
  case NN:                                                                                                   \
    if (gin)                                                                                                 \
      return np == 3 ? launch_br_t<NN, 3, true>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, gin, s0, st, pace) \
           : np == 2 ? launch_br_t<NN, 2, true>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, gin, s0, st, pace) \
                     : launch_br_t<NN, 1, true>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, gin, s0, st, pace); \
    return np == 3 ? launch_br_t<NN, 3, false>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, gin, s0, st, pace)  \
         : np == 2 ? launch_br_t<NN, 2, false>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, gin, s0, st, pace)  \
                   : launch_br_t<NN, 1, false>(c, k, accs, n_acc, acc_per_ct, abar_rows, abar, gin, s0, st, pace);
  switch (c->prm.N) {
    BR_CASE(256)
    BR_CASE(512)
    BR_CASE(1024)
    BR_CASE(2048)
  }
#undef BR_CASE
  return FDFB_E_DIMENSION;
}

// ------------------------------------------------------------------ exact int8 GEMMs (kernels_imma.cuh)
// TMA descriptors come from the driver's cuTensorMapEncodeTiled, resolved through the runtime
// (no libcuda link); one 2D map per K-major int8 operand [rows][K] with row pitch ld bytes.
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
    cudaGetLastError();
  });
  return fn;
}
static int make_tmap_i8(CUtensorMap* m, const void* base, size_t rows, size_t K, size_t ld, int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) { g_last_cuda = "cuTensorMapEncodeTiled unavailable"; return FDFB_E_CUDA; }
  if (((uintptr_t)base & 15) || (ld & 15) || K > ld) { g_last_cuda = "GEMM operand not 16-byte aligned"; return FDFB_E_CUDA; }
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)imma::BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { g_last_cuda = "cuTensorMapEncodeTiled failed: " + std::to_string((int)r); return FDFB_E_CUDA; }
  return FDFB_OK;
}
// D = A [M][K] (pitch lda) x B [Ncols][K]^T (pitch ldb), both int8 K-major, through the
// epilogue e (kernels_imma.cuh); Ncols is a multiple of imma::BN except in raw mode.  CTA pairs
// (cta_group::2, 256-row tiles) unless FDFB_IMMA_CG=1.
template <int CG, int NSUB>
static int imma_launch(const fdfb_ctx* c, const CUtensorMap& ta, const CUtensorMap& tb, size_t M, size_t Ncols,
                       size_t K, const ImmaEpi& e, int kclass, cudaStream_t st) {
  const int tiles_m = (int)((M + imma::BM * CG - 1) / (imma::BM * CG));
  const int tiles_n = (int)((Ncols + imma::BN * NSUB - 1) / (imma::BN * NSUB));
  const long long nt = (long long)tiles_m * tiles_n;
  const int units = (int)(nt < c->num_sms / CG ? nt : c->num_sms / CG);
  const size_t smem = imma::Cfg<CG, NSUB>::SMEM;
  CK(cudaFuncSetAttribute(k_imma<CG, NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * CG);
  cfg.blockDim = dim3(imma::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = CG; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  TimedLaunch tl(c, kclass, st);
  CK(cudaLaunchKernelEx(&cfg, k_imma<CG, NSUB>, ta, tb, (int)K, tiles_m, tiles_n, c->dp, e));
  CKL(c);
  return FDFB_OK;
}
static int imma_gemm(const fdfb_ctx* c, const int8_t* A, size_t M, size_t lda, const int8_t* B, size_t Ncols,
                     size_t ldb, size_t K, const ImmaEpi& e, int kclass, cudaStream_t st) {
  if (M == 0) return FDFB_OK;
  const int cg = c->imma_cg;
  CUtensorMap ta, tb;
  int rc = make_tmap_i8(&ta, A, M, K, lda, imma::BM);
  if (!rc) rc = make_tmap_i8(&tb, B, Ncols, K, ldb, imma::BN / cg);
  if (rc) return rc;
  // long K (the epilogue is negligible next to a tile's MMAs): 448-column tiles, one accumulator
  const bool wide = cg == 2 && K >= (size_t)c->imma_wide_k && Ncols % (2 * imma::BN) == 0;
  if (cg == 1) return imma_launch<1, 1>(c, ta, tb, M, Ncols, K, e, kclass, st);
  return wide ? imma_launch<2, 2>(c, ta, tb, M, Ncols, K, e, kclass, st)
              : imma_launch<2, 1>(c, ta, tb, M, Ncols, K, e, kclass, st);
}

// ------------------------------------------------------------------ key switching
static KsGemm ks_shape_rlwe(const fdfb_params& p) { return ks_gemm_shape(p.N, p.ell_pk, p.logL_pk, 2 * p.N); }
static KsGemm ks_shape_lwe(const fdfb_params& p) { return ks_gemm_shape(p.N, p.ell_ks, p.logL_ks, p.n + 1); }
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
static const size_t kKsABytes = 1ull << 30;     // int8 limb-matrix chunk cap
static int ks_chunk_rows(const KsGemm& g) {     // LWE samples per GEMM chunk (<= 32768: k_ks_gemm_bits grid.y)
  size_t r = kKsABytes / ((size_t)g.NLP * g.Kd);
  return (int)(r < 1 ? 1 : (r > (1 << 15) ? (1 << 15) : r));
}
static size_t ks_ws_bytes(const KsGemm& g, int count) {
  const int rows = count < ks_chunk_rows(g) ? count : ks_chunk_rows(g);
  return align256((size_t)rows * g.NLP * g.Kd);
}
// device formats: canonical key, then (256-aligned) its int8 digit matrix
static size_t ks_key_bytes(size_t canon, const KsGemm& g) { return align256(canon) + (size_t)g.Nout * g.Kd; }
// qbits = 0: key mod Q; else key mod 2^qbits (digits of the centred representative)
static int ks_build_key(const fdfb_ctx* c, const u64* canon_dev, size_t canon_bytes, const KsGemm& g, int qbits,
                        void* dev, cudaStream_t st) {
  if ((void*)canon_dev != dev) CK(cudaMemcpyAsync(dev, canon_dev, canon_bytes, cudaMemcpyDeviceToDevice, st));
  int8_t* GK = (int8_t*)dev + align256(canon_bytes);
  dim3 grd((g.Kd + 31) / 32, (g.Wpad + 7) / 8), blk(32, 8);
  k_ks_gemm_key<<<grd, blk, 0, st>>>((const u64*)dev, g, c->prm.Q, qbits, GK);
  CKL(c);
  return FDFB_OK;
}
// out = KeySwitch(lwe) for `count` samples: limb matrix, then one tcgen05 GEMM per chunk with
// the recombination and b - v in its epilogue; qmask = 0 -> mod Q, else mod 2^w.
static int ks_gemm(const fdfb_ctx* c, const void* key_dev, size_t canon_bytes, const KsGemm& g, int logL, int ell,
                   const u64* lwe, int count, u64* out, u64 qmask, void* ws, int kclass, cudaStream_t st) {
  const int N = c->prm.N;
  const int8_t* GK = (const int8_t*)key_dev + align256(canon_bytes);
  const int CH = ks_chunk_rows(g);
  int8_t* A = (int8_t*)ws;
  for (int o = 0; o < count; o += CH) {
    const int rows = (count - o) < CH ? (count - o) : CH;
    const u64* in = lwe + (size_t)o * (N + 1);
    dim3 gb((g.Kd + 255) / 256 < 64 ? (g.Kd + 255) / 256 : 64, rows);
    k_ks_gemm_bits<<<gb, 256, 0, st>>>(in, rows, N, ell, logL, g, A);
    CKL(c);
    ImmaEpi e;
    e.mode = qmask ? 1 : 0;
    e.nlp = g.NLP;
    e.rows = rows * g.NLP;
    e.W = g.W;
    e.ldo = g.W;
    e.neg_sub = 1;
    e.qmask = qmask;
    e.out = out + (size_t)o * g.W;
    e.lwe = in;
    e.lwe_ld = N + 1;
    int rc = imma_gemm(c, A, (size_t)rows * g.NLP, g.Kd, GK, g.Nout, g.Kd, g.Kd, e, kclass, st);
    if (rc) return rc;
  }
  return FDFB_OK;
}

static size_t canon_bpk_bytes(const fdfb_params& p) { return (size_t)p.N * p.ell_pk * 2 * p.N * 8; }
static size_t canon_ksk_bytes(const fdfb_params& p) { return (size_t)p.N * p.ell_ks * (p.n + 1) * 8; }

// ------------------------------------------------------------------ context
static int validate(const fdfb_params* p) {
  if (!p) return FDFB_E_NULL;
  // Q < 2^55: the blind rotation's CRT accumulates up to 7Q below the rounding bits 58..63
  if (!(p->N == 256 || p->N == 512 || p->N == 1024 || p->N == 2048)) return FDFB_E_DIMENSION;
  if (p->n < 1 || p->n > 4096) return FDFB_E_DIMENSION;
  if (p->Q < 3 || p->Q >= (1ULL << 55) || !h_is_prime(p->Q) || (p->Q - 1) % (2 * (u64)p->N)) return FDFB_E_NON_NTT_MODULUS;
  // q_lwe <= 2^55: the key switches' int8 GEMM splits the centred key (|v| <= 2^54) into 7
  // balanced base-256 digits
  if (p->log_q_lwe < 8 || p->log_q_lwe > 55 || p->log_q_lwe < (uint32_t)ceil_log2(2 * p->N) + 1) return FDFB_E_DIMENSION;
  if (p->lwe_key > 1 || p->rlwe_key > 1) return FDFB_E_UNSUPPORTED;
  const int qb = bits_of(p->Q - 1) > 0 ? ceil_log2(p->Q) : 1;
  auto ok = [](uint32_t logL, uint32_t ell, int bits) {
    return logL >= 1 && logL <= 32 && ell >= 1 && (int)ell == (bits + (int)logL - 1) / (int)logL;
  };
  if (!ok(p->logL_rgsw, p->ell_rgsw, qb) || p->ell_rgsw > 8 || p->logL_rgsw > 27) return FDFB_E_DECOMP;  // digits < RNS primes
  if (!ok(p->logL_boot, p->ell_boot, qb) || p->ell_boot > 64) return FDFB_E_DECOMP;
  if (!ok(p->logL_pk, p->ell_pk, qb)) return FDFB_E_DECOMP;
  if (!ok(p->logL_ks, p->ell_ks, (int)p->log_q_lwe)) return FDFB_E_DECOMP;
  if (!ok(p->logL_pack, p->ell_pack, qb) || p->logL_pack > 12) return FDFB_E_DECOMP;
  if ((u128)p->N * p->ell_pk * (1ULL << p->logL_pk) >= ((u128)1 << 32)) return FDFB_E_DECOMP;
  // key-switch GEMM sums stay exact in int32: K = N ell terms of |limb x digit| <= 127 * 128
  if ((u64)p->N * p->ell_pk * 127 * 128 >= (1ULL << 31) || (u64)p->N * p->ell_ks * 127 * 128 >= (1ULL << 31))
    return FDFB_E_DECOMP;
  if (p->t < 2 || (2 * p->N) % p->t) return FDFB_E_PLAINTEXT;
  return FDFB_OK;
}

// Pass-grouped RNS twiddle tables for kernels_br.cuh (one prime, one direction): group g of
// radix-8 pass q holds (tw[2^{3q}+g], tw[2^{3q+1}+2g+{0,1}], tw[2^{3q+2}+4g+{0..3}], pad);
// the final pass of P stages has one group per thread with, for stage s, the pairs
// tw[2^{3 NMID+s} + tid c_s + {0..c_s-1}], c_s = 8 >> (P-s).  tw(idx) = psi^{+-bitrev(idx)}
// mod p with its 32-bit Shoup companion.  Appends GROUPS*16 words to out.
template <int N>
static void make_rns_tables(u64 psi, u64 pr, std::vector<u32>& out) {
  using S = BrShape<N>;
  const int logN = S::LOGN;
  std::vector<u32> w(N), ws(N);
  for (int k = 0; k < N; k++) {
    w[k] = (u32)h_powmod(psi, bitrev(k, logN), pr);
    ws[k] = (u32)(((u64)w[k] << 32) / pr);
  }
  const size_t base = out.size();
  out.resize(base + (size_t)S::GROUPS * 16, 0);
  auto put = [&](int grp, int e, int idx) {
    out[base + (size_t)grp * 16 + 2 * e] = w[idx];
    out[base + (size_t)grp * 16 + 2 * e + 1] = ws[idx];
  };
  for (int q = 0; q < S::NMID; q++) {
    const int groups = 1 << (3 * q);
    for (int g = 0; g < groups; g++) {
      const int G = S::grp(q) + g;
      put(G, 0, (1 << (3 * q)) + g);
      for (int e = 0; e < 2; e++) put(G, 1 + e, (1 << (3 * q + 1)) + 2 * g + e);
      for (int e = 0; e < 4; e++) put(G, 3 + e, (1 << (3 * q + 2)) + 4 * g + e);
    }
  }
  for (int tid = 0; tid < S::T; tid++) {
    int o = 0;
    for (int s = 0; s < S::PLAST; s++) {
      const int cnt = 8 >> (S::PLAST - s);
      for (int e = 0; e < cnt; e++) put(S::G_LAST + tid, o + e, (1 << (3 * S::NMID + s)) + tid * cnt + e);
      o += cnt;
    }
  }
}
static u64 h_inv(u64 a, u64 m) { return h_powmod(a % m, m - 2, m); }   // m prime
static u64 h_primroot_2n(u64 pr, int N) {
  for (u64 g = 2; g < 10000; g++) {
    u64 c = h_powmod(g, (pr - 1) / (2 * (u64)N), pr);
    if (h_powmod(c, N, pr) == pr - 1) return c;
  }
  return 0;
}
// The kernel rounds k = floor((sum_i f_i + 8) / 16) with f_i = floor(16 t_i / p_i) - {0, 1}
// (and f16's truncation, < 1/16 each): sum f_i lies in [16 X - 17 NP / 16, 16 X] for
// X = sum t_i / p_i = k + V / P, |V| <= bound.  k is exact iff 16 bound / P + 17 NP / 16 <= 8
// (lower side) and 16 bound / P < 8 (upper side), i.e. 256 bound + 17 NP P <= 128 P.
static bool crt_rounding_exact(u128 bound, u128 P, int np) {
  return (u128)256 * bound + (u128)17 * np * P <= (u128)128 * P;
}
// Choose the RNS primes (largest p < 2^28 so that 16p < 2^32, p = 1 mod 2N) until the CRT
// rounding is exact for bound = 2 ell N (L-1) (Q-1) >= |coefficients| of sum_r D_r * K_r; build
// constants/tables.
static int setup_rns(fdfb_ctx* c) {
  const fdfb_params& p = c->prm;
  const int N = p.N;
  RnsParams& R = c->rns;
  memset(&R, 0, sizeof(R));
  const u128 bound = (u128)(2 * p.ell_rgsw) * N * ((1ULL << p.logL_rgsw) - 1) * (p.Q - 1);
  std::vector<u64> primes;
  u128 P = 1;
  if (p.Q < (1ULL << 28)) {
    // Q itself fits the 32-bit lazy butterflies (16Q < 2^32) and is NTT-friendly: one "RNS"
    // prime p = Q computes the ring products directly mod Q (the CRT below degenerates to
    // t_0 = r_0, P mod Q = 0), half the transforms of a 2-prime exact evaluation.
    primes.push_back(p.Q);
    P = p.Q;
  } else {
    for (u64 cand = ((1ULL << 28) - 1) / (2 * N) * (2 * N) + 1; cand > (1ULL << 27) && primes.size() < RNS_MAXP;
         cand -= 2 * (u64)N) {
      if (cand >= (1ULL << 28) || cand == p.Q || !h_is_prime(cand)) continue;
      primes.push_back(cand);
      P *= cand;
      if (primes.size() >= 2 && crt_rounding_exact(bound, P, (int)primes.size())) break;
    }
    if (primes.size() < 2 || !crt_rounding_exact(bound, P, (int)primes.size())) return FDFB_E_UNSUPPORTED;
  }
  // MAC range of k_blind_rotate: 2 ell products of forward outputs (< B p, B = fwd_out_bound)
  // and key residues (< p) plus the Montgomery term stay below 2^64, and the reduced value
  // below 16p (three conditional subtractions then reach [0, 2p))
  {
    int B = 16;
    switch (N) {
      case 256: B = fwd_out_bound<256>(); break;
      case 512: B = fwd_out_bound<512>(); break;
      case 1024: B = fwd_out_bound<1024>(); break;
      default: B = fwd_out_bound<2048>(); break;
    }
    for (u64 pr : primes) {
      const u128 smax = (u128)(2 * p.ell_rgsw) * B * pr * pr + (u128)0xFFFFFFFFull * pr;
      if (smax >= ((u128)1 << 64) || (u64)(smax >> 32) >= 16 * pr) return FDFB_E_UNSUPPORTED;
    }
  }
  R.np = (int)primes.size();
  const u64 Q = p.Q;
  std::vector<u32> ft, it;
  for (int i = 0; i < R.np; i++) {
    const u64 pr = primes[i];
    R.p[i] = (u32)pr; R.p2[i] = (u32)(2 * pr);
    {                                              // -p^{-1} mod 2^32 by Newton iteration
      u32 inv = (u32)pr;                           // p odd: p p = 1 mod 8
      for (int it2 = 0; it2 < 5; it2++) inv *= 2u - (u32)pr * inv;
      R.pinv[i] = 0u - inv;
    }
    const u64 psi = h_primroot_2n(pr, N);
    if (!psi) return FDFB_E_UNSUPPORTED;
    const u64 psii = h_inv(psi, pr);
    switch (N) {
      case 256: make_rns_tables<256>(psi, pr, ft); make_rns_tables<256>(psii, pr, it); break;
      case 512: make_rns_tables<512>(psi, pr, ft); make_rns_tables<512>(psii, pr, it); break;
      case 1024: make_rns_tables<1024>(psi, pr, ft); make_rns_tables<1024>(psii, pr, it); break;
      default: make_rns_tables<2048>(psi, pr, ft); make_rns_tables<2048>(psii, pr, it); break;
    }
  }
  auto s32 = [](u64 w, u64 m) { return (u32)((w << 32) / m); };
  for (int i = 0; i < R.np; i++) {                 // CRT constants (kernels_br.cuh epilogue)
    u64 Pi_q = 1 % Q, Pi_p = 1;                    // P / p_i mod Q and mod p_i
    for (int j = 0; j < R.np; j++) {
      if (j == i) continue;
      Pi_q = h_mulmod(Pi_q, primes[j] % Q, Q);
      Pi_p = h_mulmod(Pi_p, primes[j] % primes[i], primes[i]);
    }
    R.y[i] = (u32)h_inv(Pi_p, primes[i]); R.ys[i] = s32(R.y[i], primes[i]);
    // the key carries N^{-1} y_i: the inverse NTT then yields t_i = r_i y_i directly
    R.ninv[i] = (u32)h_mulmod(h_mulmod(h_inv(N, primes[i]), R.y[i], primes[i]), (1ULL << 32) % primes[i], primes[i]);
    R.ninvs[i] = s32(R.ninv[i], primes[i]);
    R.M[i] = Pi_q; R.Ms32[i] = (u32)(((u128)Pi_q << 32) / Q);
    R.f16[i] = (u32)((1ULL << 36) / primes[i]);
  }
  R.pq = (u64)(P % Q);
  ft.insert(ft.end(), it.begin(), it.end());
  CK(cudaMalloc(&c->d_rtab, ft.size() * 4));
  CK(cudaMemcpy(c->d_rtab, ft.data(), ft.size() * 4, cudaMemcpyHostToDevice));
  R.ftab = (const uint4*)c->d_rtab;
  R.itab = (const uint4*)(c->d_rtab + it.size());
  return FDFB_OK;
}

extern "C" int fdfb_ctx_create(const fdfb_params* p, int device, fdfb_ctx** out) {
  if (!out) return FDFB_E_NULL;
  *out = nullptr;
  int rc = validate(p);
  if (rc) return rc;
  CK(cudaSetDevice(device));
  fdfb_ctx* c = new fdfb_ctx();
  c->prm = *p;
  c->device = device;
  CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  const u64 Q = p->Q;
  const int N = p->N, logN = ceil_log2(N);
  // primitive 2N-th root of unity: psi = g^{(Q-1)/2N} with psi^N = -1
  u64 psi = 0;
  for (u64 g = 2; g < 1000; g++) {
    u64 c2 = h_powmod(g, (Q - 1) / (2 * (u64)N), Q);
    if (h_powmod(c2, N, Q) == Q - 1) { psi = c2; break; }
  }
  if (!psi) { delete c; return FDFB_E_NON_NTT_MODULUS; }
  u64 psi_inv = h_powmod(psi, Q - 2, Q);
  int T = 0;
  if (!make_cdt(p->sigma_milli, &c->cdt, &T)) { delete c; return FDFB_E_UNSUPPORTED; }
  // tables: tw, twp, itw, itwp (N each), cdt (2T), omega (N)
  size_t ntab = 4 * (size_t)N + c->cdt.size() + N;
  std::vector<u64> h(ntab, 0);
  for (int k = 0; k < N; k++) {
    int br = bitrev(k, logN);
    u64 w = h_powmod(psi, br, Q), wi = h_powmod(psi_inv, br, Q);
    h[k] = w; h[N + k] = shoup_of(w, Q);
    h[2 * N + k] = wi; h[3 * N + k] = shoup_of(wi, Q);
  }
  for (size_t k = 0; k < c->cdt.size(); k++) h[4 * N + k] = c->cdt[k];
  // omega[slot] = value of X at the slot's evaluation point = psi^{2 bitrev(slot) + 1}
  c->omega_off = 4 * (size_t)N + c->cdt.size();
  for (int k = 0; k < N; k++) h[c->omega_off + k] = h_powmod(psi, 2 * (u64)bitrev(k, logN) + 1, Q);
  CK(cudaMalloc(&c->d_tables, ntab * sizeof(u64)));
  CK(cudaMalloc(&c->d_status, sizeof(int)));
  CK(cudaMemset(c->d_status, 0, sizeof(int)));
  CK(cudaMalloc(&c->d_prog, (size_t)BR_PACE_SLOTS * BR_PACE_MAXGRID * sizeof(u64)));
  CK(cudaMemset(c->d_prog, 0, (size_t)BR_PACE_SLOTS * BR_PACE_MAXGRID * sizeof(u64)));
  if (const char* e = getenv("FDFB_BR_PACE_SPLIT")) c->br_pace_split = atoi(e) != 0;
  const bool pace_env = getenv("FDFB_BR_PACE") != nullptr;
  if (const char* e = getenv("FDFB_BR_PACE")) {
    unsigned lo = 0, hi = 0, cap = 0;
    const int nf = sscanf(e, "%u,%u,%u", &lo, &hi, &cap);
    if (nf >= 2 && lo > 0 && hi > lo) { c->br_wlo = lo; c->br_whi = hi; if (nf == 3) c->br_wcap = cap; }
    else c->br_wlo = c->br_whi = 0;
  }
  CK(cudaMemcpy(c->d_tables, h.data(), ntab * sizeof(u64), cudaMemcpyHostToDevice));
  if ((rc = setup_rns(c))) { delete c; return rc; }
  if (!pace_env) {
    // pacing keeps the brK reads of drifting CTAs in L2; a key that stays in L2 as a whole needs none,
    // and the checks then only cost time (FHEW-like, 67 MB of brK: 173 -> 158 ms per 10 rounds unpaced,
    // profiles/r02/fhewexp).  Paced by default only when the device-format brK exceeds 3/4 of L2.
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
    const size_t brk_dev = (size_t)p->n * (p->lwe_key ? 2 : 1) * 2 * p->ell_rgsw * 2 * p->N * c->rns.np * sizeof(u32);
    if (l2 > 0 && brk_dev <= (size_t)l2 / 4 * 3) c->br_wlo = c->br_whi = 0;
  }
  if (const char* e = getenv("FDFB_BR_CLUSTER")) c->br_cluster = atoi(e);
  if (const char* e = getenv("FDFB_IMMA_CG")) c->imma_cg = atoi(e) == 1 ? 1 : 2;
  if (const char* e = getenv("FDFB_BR_KERNEL")) c->br_kernel = atoi(e) == 1 ? 1 : 2;
  if (const char* e = getenv("FDFB_BOOT_SPLIT")) c->boot_split = atoi(e) ? 1 : 0;
  CK(cudaStreamCreateWithFlags(&c->helper, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  if (const char* e = getenv("FDFB_IMMA_WIDE_K")) c->imma_wide_k = atoi(e);
  DevParams& d = c->dp;
  memset(&d, 0, sizeof(d));
  d.Q = Q; d.Q2 = 2 * Q; d.Q4 = 4 * Q; d.half = (Q + 1) / 2;
  d.q_mask = (p->log_q_lwe >= 64) ? ~0ULL : ((1ULL << p->log_q_lwe) - 1);
  d.N = N; d.logN = logN; d.n = p->n; d.u = p->lwe_key ? 2 : 1;
  d.log_q_lwe = p->log_q_lwe;
  d.logL_rgsw = p->logL_rgsw; d.ell_rgsw = p->ell_rgsw;
  d.logL_boot = p->logL_boot; d.ell_boot = p->ell_boot;
  d.logL_pk = p->logL_pk; d.ell_pk = p->ell_pk;
  d.logL_ks = p->logL_ks; d.ell_ks = p->ell_ks;
  d.logL_pack = p->logL_pack; d.ell_pack = p->ell_pack;
  d.lwe_ternary = p->lwe_key; d.rlwe_ternary = p->rlwe_key;
  d.noiseless = p->sigma_milli == 0; d.cdt_T = T;
  d.t = p->t;
  d.tw = c->d_tables; d.twp = c->d_tables + N; d.itw = c->d_tables + 2 * N; d.itwp = c->d_tables + 3 * N;
  d.cdt = c->d_tables + 4 * N;
  d.ninv = h_powmod(N, Q - 2, Q); d.ninvp = shoup_of(d.ninv, Q);
  d.qbar = (u64)((((u128)1) << 64) / Q);
  d.qbias = ((1ULL << 31) / Q + 1) * Q;
  // Montgomery: -Q^{-1} mod 2^64 (Newton), R^2 mod Q
  u64 inv = 1;
  for (int i = 0; i < 7; i++) inv *= 2 - Q * inv;
  c->qinv_neg = 0 - inv;
  u64 r1 = (u64)(((u128)1 << 64) % Q);
  c->r2 = h_mulmod(r1, r1, Q);
  *out = c;
  return FDFB_OK;
}

extern "C" void fdfb_ctx_destroy(fdfb_ctx* c) {
  if (!c) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(c->device);                    // the context's allocations live on its device
  {
    std::lock_guard<std::mutex> g(c->tmu);     // timing events never read back
    for (auto& e : c->tev) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
    c->tev.clear();
  }
  cudaFree(c->d_tables);
  cudaFree(c->d_status);
  cudaFree(c->d_prog);
  cudaFree(c->d_rtab);
  if (c->helper) cudaStreamDestroy(c->helper);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
  cudaSetDevice(cur);
}

static size_t brk_words(const fdfb_params& p) { return (size_t)p.n * (p.lwe_key ? 2 : 1) * 2 * p.ell_rgsw * 2 * p.N; }

extern "C" int fdfb_sizes(const fdfb_ctx* c, fdfb_sizes_t* o) {
  if (!c || !o) return FDFB_E_NULL;
  const fdfb_params& p = c->prm;
  o->sk_lwe = p.n; o->sk_rlwe = p.N;
  o->canon_brk = brk_words(p) * 8;
  o->brk = brk_words(p) * c->rns.np * 4;        // u32 residues per RNS prime
  o->canon_bpk = canon_bpk_bytes(p);
  o->bpk = ks_key_bytes(o->canon_bpk, ks_shape_rlwe(p));      // canonical + int8 GEMM digits
  o->canon_ksk = canon_ksk_bytes(p);
  o->ksk = ks_key_bytes(o->canon_ksk, ks_shape_lwe(p));
  o->canon_pack = (size_t)p.N * p.ell_pack * (1ULL << p.logL_pack) * 2 * p.N * 8;
  o->pack = shift_pack_bytes(p);
  return FDFB_OK;
}

// largest batch per call (keeps every derived count, e.g. B * ell_boot accumulators, in int)
static const uint32_t kMaxBatch = 1u << 24;

// workspace layout of fdfb_bootstrap_batch
struct BootWs {
  u32* abar; u32* bbar; u64* accs; u64* lweN; u64* dig; u64* F; void* ks; size_t ks_part; size_t bytes;
};
static BootWs boot_ws(const fdfb_params& p, uint32_t B, void* base, uint32_t k = 1) {
  BootWs w;
  char* b = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = b + off; off += (bytes + 255) & ~(size_t)255; return r; };
  const size_t ellb = p.ell_boot, N = p.N;
  const size_t nl = ellb + k;                             // LWE_N samples: ladder rows, then output rows
  w.abar = (u32*)take((size_t)B * p.n * 4);
  w.bbar = (u32*)take((size_t)B * 4);
  w.accs = (u64*)take((size_t)B * ellb * 2 * N * 8);
  w.lweN = (u64*)take((size_t)B * nl * (N + 1) * 8);
  w.dig = (u64*)take((size_t)B * ellb * N * 8);
  w.F = (u64*)take((size_t)B * k * 2 * N * 8);
  {                                                       // one key-switch region per part (two parts)
    const int half = (int)((B + 1) / 2);
    const size_t kr = ks_ws_bytes(ks_shape_rlwe(p), (int)(half * ellb ? half * ellb : 1));
    const size_t kl = ks_ws_bytes(ks_shape_lwe(p), (int)(half * k ? half * k : 1));
    w.ks_part = align256(kr > kl ? kr : kl);
    w.ks = take(2 * w.ks_part);
  }
  w.bytes = off;
  return w;
}
extern "C" size_t fdfb_workspace_bootstrap(const fdfb_ctx* c, uint32_t B) {
  if (!c) return 0;
  return boot_ws(c->prm, B, nullptr).bytes + (size_t)B * 2 * (c->prm.n + 1) * 8;  // + host staging
}
extern "C" size_t fdfb_workspace_bootstrap_multi(const fdfb_ctx* c, uint32_t B, uint32_t k) {
  if (!c || k == 0) return 0;
  return boot_ws(c->prm, B, nullptr, k).bytes;
}

// ------------------------------------------------------------------ encryption helpers
// Encrypt `count` canonical RLWE entries of `kind` (BRK/BPK/PACK) into out [count][2][N].
static int rlwe_entries(const fdfb_ctx* c, u64 seed, int kind, const int8_t* s_lwe, const int8_t* s_rlwe,
                        const u64* idx, u64 idx_base, int count, u64* out, u64* shat, u64* tmp_mask,
                        u64* tmp_prod, cudaStream_t st) {
  const int N = c->prm.N;
  dim3 g1((N + 255) / 256, count);
  k_rlwe_mask<<<g1, 256, 0, st>>>(c->dp, kind, idx, idx_base, count, seed, s_lwe, s_rlwe, tmp_mask);
  CKL(c);
  CK(cudaMemcpyAsync(tmp_prod, tmp_mask, (size_t)count * N * 8, cudaMemcpyDeviceToDevice, st));
  int rc = launch_ntt_batch(c, tmp_prod, count, 0, st);
  if (rc) return rc;
  size_t tot = (size_t)count * N;
  k_pointwise_mul<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(tmp_prod, shat, tmp_prod, tot, N, c->dp.Q,
                                                                   c->qinv_neg, c->r2);
  CKL(c);
  rc = launch_ntt_batch(c, tmp_prod, count, 1, st);
  if (rc) return rc;
  k_rlwe_finish<<<g1, 256, 0, st>>>(c->dp, kind, idx, idx_base, count, seed, s_lwe, s_rlwe, tmp_mask, tmp_prod, out);
  CKL(c);
  return FDFB_OK;
}

__global__ void k_secret_to_residues(DevParams p, const int8_t* s, u64* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p.N) out[i] = from_signed(s[i], p.Q);
}
static int make_shat(const fdfb_ctx* c, const int8_t* s_rlwe, u64* shat, cudaStream_t st) {
  k_secret_to_residues<<<(c->prm.N + 255) / 256, 256, 0, st>>>(c->dp, s_rlwe, shat);
  CKL(c);
  return launch_ntt_batch(c, shat, 1, 0, st);
}

// canonical brk rows [rows][2][N] (coef) -> device BRK (RNS NTT domain); rows are consecutive
// canonical rows starting at row0 (flat (i*u+j)*2ell + row).
template <int N>
static int brk_rns_t(const fdfb_ctx* c, const u64* canon, size_t rows, size_t row0, u32* dev, cudaStream_t st) {
  dim3 g((unsigned)(rows * 2), c->rns.np);
  k_brk_rns<N><<<g, N / 8, 0, st>>>(c->dp, c->rns, canon, row0, dev);
  CKL(c);
  return FDFB_OK;
}
static int brk_import_rows(const fdfb_ctx* c, const u64* canon, size_t rows, size_t row0, u64* dev,
                           cudaStream_t st) {
  switch (c->prm.N) {
    case 256: return brk_rns_t<256>(c, canon, rows, row0, (u32*)dev, st);
    case 512: return brk_rns_t<512>(c, canon, rows, row0, (u32*)dev, st);
    case 1024: return brk_rns_t<1024>(c, canon, rows, row0, (u32*)dev, st);
    case 2048: return brk_rns_t<2048>(c, canon, rows, row0, (u32*)dev, st);
  }
  return FDFB_E_DIMENSION;
}

// keygen scratch: the ring secret's NTT, and per chunk of CH RLWE entries the mask, the mask
// product and the encrypted entries
static const int kKeygenChunk = 2048;
struct KeygenWs { u64* shat; u64* tmask; u64* tprod; u64* tout; size_t bytes; };
static KeygenWs keygen_ws(const fdfb_params& p, void* base) {
  KeygenWs w;
  char* b = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = b + off; off += (bytes + 255) & ~(size_t)255; return r; };
  const size_t N = p.N, CH = kKeygenChunk;
  w.shat = (u64*)take(N * 8);
  w.tmask = (u64*)take(CH * N * 8);
  w.tprod = (u64*)take(CH * N * 8);
  w.tout = (u64*)take(CH * 2 * N * 8);
  w.bytes = off;
  return w;
}
extern "C" size_t fdfb_workspace_keygen(const fdfb_ctx* c) { return c ? keygen_ws(c->prm, nullptr).bytes : 0; }

extern "C" int fdfb_keygen(const fdfb_ctx* c, uint64_t seed, uint32_t which, int8_t* sk_lwe, int8_t* sk_rlwe,
                           void* brk, void* bpk, void* ksk, void* pack, void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  cudaStream_t st = S(stream);
  const fdfb_params& p = c->prm;
  const int N = p.N;
  if (!sk_lwe || !sk_rlwe) return FDFB_E_NULL;
  if (((which & 2) && !brk) || ((which & 4) && !bpk) || ((which & 8) && !ksk) || ((which & 16) && !pack))
    return FDFB_E_NULL;
  if ((which & 30) && !workspace) return FDFB_E_WORKSPACE;
  if (which & 1) {
    int m = p.n > p.N ? p.n : p.N;
    k_keygen_secrets<<<(m + 255) / 256, 256, 0, st>>>(c->dp, seed, sk_lwe, sk_rlwe);
    CKL(c);
  }
  if (!(which & 30)) { CK(cudaStreamSynchronize(st)); return FDFB_OK; }
  const int CH = kKeygenChunk;  // RLWE entries per chunk
  KeygenWs w = keygen_ws(p, workspace);
  int rc = make_shat(c, sk_rlwe, w.shat, st);
  if (!rc && (which & 2)) {
    size_t rows = brk_words(p) / (2 * (size_t)N);
    for (size_t o = 0; o < rows && !rc; o += CH) {
      int cnt = (int)((rows - o) < (size_t)CH ? (rows - o) : CH);
      rc = rlwe_entries(c, seed, 1, sk_lwe, sk_rlwe, nullptr, o, cnt, w.tout, w.shat, w.tmask, w.tprod, st);
      if (!rc) rc = brk_import_rows(c, w.tout, cnt, o, (u64*)brk, st);
    }
  }
  if (!rc && (which & 4)) {
    size_t ent = (size_t)N * p.ell_pk;
    for (size_t o = 0; o < ent && !rc; o += CH) {
      int cnt = (int)((ent - o) < (size_t)CH ? (ent - o) : CH);
      rc = rlwe_entries(c, seed, 2, sk_lwe, sk_rlwe, nullptr, o, cnt, (u64*)bpk + o * 2 * N, w.shat, w.tmask,
                        w.tprod, st);
    }
    if (!rc) rc = ks_build_key(c, (const u64*)bpk, canon_bpk_bytes(p), ks_shape_rlwe(p), 0, bpk, st);
  }
  if (!rc && (which & 8)) {
    int ent = N * p.ell_ks;
    k_ksk_gen<<<(ent * 32 + 255) / 256, 256, 0, st>>>(c->dp, seed, sk_lwe, sk_rlwe, nullptr, 0, ent, (u64*)ksk);
    CKL(c);
    rc = ks_build_key(c, (const u64*)ksk, canon_ksk_bytes(p), ks_shape_lwe(p), (int)p.log_q_lwe, ksk, st);
  }
  if (!rc && (which & 16)) rc = pack_keygen(c, seed, sk_rlwe, pack, w.shat, w.tmask, w.tprod, CH, st);
  if (rc) return rc;
  CK(cudaStreamSynchronize(st));
  return FDFB_OK;
}

// keygen_canonical scratch: the entry indices, the ring secret's NTT, mask and mask product
static size_t keycanon_ws_bytes(const fdfb_params& p, uint32_t count) {
  return align256((size_t)count * 8) + align256((size_t)p.N * 8) + 2 * align256((size_t)count * p.N * 8);
}
extern "C" size_t fdfb_workspace_keygen_canonical(const fdfb_ctx* c, uint32_t count) {
  return c ? keycanon_ws_bytes(c->prm, count) : 0;
}
extern "C" int fdfb_keygen_canonical(const fdfb_ctx* c, uint64_t seed, int kind, const int8_t* sk_lwe,
                                     const int8_t* sk_rlwe, const uint64_t* idx, uint32_t count, uint64_t* out,
                                     void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (count == 0) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (!idx || !out || !sk_lwe || !sk_rlwe) return FDFB_E_NULL;
  if (kind != FDFB_KEY_KSK && kind != FDFB_KEY_BRK && kind != FDFB_KEY_BPK && kind != FDFB_KEY_PACK) return FDFB_E_KIND;
  if (!workspace) return FDFB_E_WORKSPACE;
  cudaStream_t st = S(stream);
  const int N = c->prm.N;
  char* b = (char*)workspace;
  u64* didx = (u64*)b;
  u64* shat = (u64*)(b + align256((size_t)count * 8));
  u64* tm = (u64*)((char*)shat + align256((size_t)N * 8));
  u64* tp = (u64*)((char*)tm + align256((size_t)count * N * 8));
  CK(cudaMemcpyAsync(didx, idx, (size_t)count * 8, cudaMemcpyHostToDevice, st));
  int rc = FDFB_OK;
  if (kind == FDFB_KEY_KSK) {
    k_ksk_gen<<<(count * 32 + 255) / 256, 256, 0, st>>>(c->dp, seed, sk_lwe, sk_rlwe, didx, 0, count, out);
    CKL(c);
  } else {
    rc = make_shat(c, sk_rlwe, shat, st);
    int k = kind == FDFB_KEY_BRK ? 1 : (kind == FDFB_KEY_BPK ? 2 : 3);
    if (!rc) rc = rlwe_entries(c, seed, k, sk_lwe, sk_rlwe, didx, 0, count, out, shat, tm, tp, st);
  }
  if (rc) return rc;
  CK(cudaStreamSynchronize(st));
  return FDFB_OK;
}

extern "C" int fdfb_key_import(const fdfb_ctx* c, int kind, const uint64_t* canon, void* dev_key, void* stream) {
  if (!c || !canon || !dev_key) return FDFB_E_NULL;
  cudaStream_t st = S(stream);
  const fdfb_params& p = c->prm;
  fdfb_sizes_t sz;
  fdfb_sizes(c, &sz);
  int rc = FDFB_OK;
  if (kind == FDFB_KEY_BRK) {
    size_t rows = brk_words(p) / (2 * (size_t)p.N);
    const size_t CH = 4096;
    for (size_t o = 0; o < rows && !rc; o += CH) {
      size_t cnt = (rows - o) < CH ? (rows - o) : CH;
      rc = brk_import_rows(c, canon + o * 2 * p.N, cnt, o, (u64*)dev_key, st);
    }
  } else if (kind == FDFB_KEY_BPK) {
    rc = ks_build_key(c, canon, sz.canon_bpk, ks_shape_rlwe(p), 0, dev_key, st);
  } else if (kind == FDFB_KEY_KSK) {
    rc = ks_build_key(c, canon, sz.canon_ksk, ks_shape_lwe(p), (int)p.log_q_lwe, dev_key, st);
  } else if (kind == FDFB_KEY_PACK) {
    rc = pack_import(c, canon, dev_key, st);
  } else {
    return FDFB_E_KIND;
  }
  if (rc) return rc;
  CK(cudaStreamSynchronize(st));
  return FDFB_OK;
}

template <int N>
static int brk_export_t(const fdfb_ctx* c, const u32* dev, u64* canon, size_t rows, cudaStream_t st) {
  const RnsParams& R = c->rns;
  BrkExportC X;
  memset(&X, 0, sizeof(X));
  u128 P = 1;
  for (int i = 0; i < R.np; i++) P *= R.p[i];
  for (int i = 0; i < R.np; i++) {
    const u64 pr = R.p[i];
    X.inv32[i] = (u32)h_inv((1ULL << 32) % pr, pr);
    X.inv32s[i] = (u32)(((u64)X.inv32[i] << 32) / pr);
    X.Pi[i] = (u64)(P / pr);
  }
  X.P_lo = (u64)P; X.P_hi = (u64)(P >> 64);
  const size_t CH = 1 << 20;                        // polynomials per launch
  for (size_t o = 0; o < 2 * rows; o += CH) {
    const size_t cnt = (2 * rows - o) < CH ? (2 * rows - o) : CH;
    k_brk_export<N><<<(unsigned)cnt, N / 8, 0, st>>>(c->dp, R, X, dev, o / 2, canon);
    CKL(c);
  }
  return FDFB_OK;
}
extern "C" int fdfb_key_export(const fdfb_ctx* c, int kind, const void* dev_key, uint64_t* canon, void* stream) {
  if (!c || !dev_key || !canon) return FDFB_E_NULL;
  fdfb_sizes_t sz;
  fdfb_sizes(c, &sz);
  if (kind == FDFB_KEY_BRK) {                        // inverse RNS NTT + CRT (k_brk_export)
    const size_t rows = brk_words(c->prm) / (2 * (size_t)c->prm.N);
    const u32* d = (const u32*)dev_key;
    switch (c->prm.N) {
      case 256: return brk_export_t<256>(c, d, canon, rows, S(stream));
      case 512: return brk_export_t<512>(c, d, canon, rows, S(stream));
      case 1024: return brk_export_t<1024>(c, d, canon, rows, S(stream));
      case 2048: return brk_export_t<2048>(c, d, canon, rows, S(stream));
    }
    return FDFB_E_DIMENSION;
  }
  size_t bytes = kind == FDFB_KEY_BPK ? sz.canon_bpk : kind == FDFB_KEY_KSK ? sz.canon_ksk
               : kind == FDFB_KEY_PACK ? sz.canon_pack : 0;
  if (!bytes) return FDFB_E_KIND;
  CK(cudaMemcpyAsync(canon, dev_key, bytes, cudaMemcpyDeviceToDevice, S(stream)));
  return FDFB_OK;
}

extern "C" int fdfb_lwe_encrypt(const fdfb_ctx* c, uint64_t seed, const int8_t* sk_lwe, const uint64_t* msg,
                                uint32_t count, uint32_t flags, uint64_t first_index, uint64_t* out, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (!count) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (!sk_lwe || !msg || !out) return FDFB_E_NULL;
  k_lwe_encrypt<<<((size_t)count * 32 + 255) / 256, 256, 0, S(stream)>>>(c->dp, seed, sk_lwe, msg, count, flags,
                                                                          first_index, out);
  CKL(c);
  return FDFB_OK;
}

// rlwe_encrypt scratch: the ring secret's NTT, the masks and their products with the secret
static size_t rlwe_enc_ws_bytes(const fdfb_params& p, uint32_t count) {
  return align256((size_t)p.N * 8) + 2 * align256((size_t)count * p.N * 8);
}
extern "C" size_t fdfb_workspace_rlwe_encrypt(const fdfb_ctx* c, uint32_t count) {
  return c ? rlwe_enc_ws_bytes(c->prm, count) : 0;
}
extern "C" int fdfb_rlwe_encrypt(const fdfb_ctx* c, uint64_t seed, const int8_t* sk_rlwe, const uint64_t* msg,
                                 uint32_t count, uint64_t first_index, uint64_t* out, void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (!count) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (count > 65535) return FDFB_E_DIMENSION;   // one grid row per ciphertext
  if (!sk_rlwe || !msg || !out) return FDFB_E_NULL;
  if (!workspace) return FDFB_E_WORKSPACE;
  cudaStream_t st = S(stream);
  const int N = c->prm.N;
  u64* shat = (u64*)workspace;
  u64* tm = (u64*)((char*)shat + align256((size_t)N * 8));
  u64* tp = (u64*)((char*)tm + align256((size_t)count * N * 8));
  int rc = make_shat(c, sk_rlwe, shat, st);
  dim3 g1((N + 255) / 256, count);
  if (!rc) {
    k_rlwe_enc_mask<<<g1, 256, 0, st>>>(c->dp, seed, count, first_index, tm);
    CKL(c);
    CK(cudaMemcpyAsync(tp, tm, (size_t)count * N * 8, cudaMemcpyDeviceToDevice, st));
    rc = launch_ntt_batch(c, tp, count, 0, st);
  }
  if (!rc) {
    size_t tot = (size_t)count * N;
    k_pointwise_mul<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(tp, shat, tp, tot, N, c->dp.Q, c->qinv_neg, c->r2);
    CKL(c);
    rc = launch_ntt_batch(c, tp, count, 1, st);
  }
  if (!rc) {
    k_rlwe_enc_finish<<<g1, 256, 0, st>>>(c->dp, seed, count, first_index, msg, tm, tp, out);
    CKL(c);
  }
  return rc;
}

// ------------------------------------------------------------------ LUT
extern "C" int fdfb_setup_lut(const fdfb_ctx* c, const uint64_t* lut, uint32_t t_out, uint64_t* rotp, void* stream) {
  if (!c || !lut || !rotp) return FDFB_E_NULL;
  if (t_out == 0) return FDFB_E_PLAINTEXT;
  const fdfb_params& p = c->prm;
  const u64 Q = p.Q;
  const long long N = p.N, t = p.t;
  const u64 delta = (u64)(((u128)2 * Q + t_out) / (2 * (u128)t_out));      // round(Q / t')
  std::vector<u64> h(2 * N, 0);
  // closed form of the half-open-window SetupPolynomial (reading F6): every y in [0,2N)
  // is the y of exactly one (m, e); m(y) = floor((t y + N) / 2N) mod t.
  for (long long y = 0; y < 2 * N; y++) {
    long long m = ((t * y + N) / (2 * N)) % t;
    u64 v = h_mulmod(delta, lut[m] % t_out, Q);
    u64 nv = v ? Q - v : 0;
    if (y == 0) h[0] = v;
    else if (y < N) h[N - y] = nv;
    else if (y == N) h[N] = nv;
    else h[N + 2 * N - y] = v;
  }
  CK(cudaMemcpyAsync(rotp, h.data(), 2 * N * 8, cudaMemcpyHostToDevice, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  return FDFB_OK;
}

// ------------------------------------------------------------------ hot path
extern "C" int fdfb_blind_rotate(const fdfb_ctx* c, const void* brk, uint64_t* acc, const uint32_t* abar,
                                 uint32_t count, uint32_t acc_per_ct, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (count == 0) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (!brk || !acc || !abar) return FDFB_E_NULL;
  if (acc_per_ct == 0) return FDFB_E_DIMENSION;
  return launch_br(c, (const u64*)brk, acc, (int)count, (int)acc_per_ct, abar, S(stream));
}

static int keyswitch_rlwe(const fdfb_ctx* c, const u64* bpk, const u64* lwe, int count, u64* out, void* ws,
                          cudaStream_t st) {
  const fdfb_params& p = c->prm;
  return ks_gemm(c, bpk, canon_bpk_bytes(p), ks_shape_rlwe(p), p.logL_pk, p.ell_pk, lwe, count, out, 0, ws,
                 FDFB_KCLASS_KEYSWITCH_RLWE, st);
}
static int keyswitch_lwe(const fdfb_ctx* c, const u64* ksk, const u64* lwe, int count, u64* out, void* ws,
                         cudaStream_t st) {
  if (ws) {
    const fdfb_params& p = c->prm;
    return ks_gemm(c, ksk, canon_ksk_bytes(p), ks_shape_lwe(p), p.logL_ks, p.ell_ks, lwe, count, out, c->dp.q_mask,
                   ws, FDFB_KCLASS_KEYSWITCH_LWE, st);
  }
  dim3 grd((c->prm.n + 1 + KS_COLS - 1) / KS_COLS, (count + KS_ROWS - 1) / KS_ROWS);
  TimedLaunch tl(c, FDFB_KCLASS_KEYSWITCH_LWE, st);
  k_keyswitch_lwe<<<grd, KS_COLS, 0, st>>>(c->dp, ksk, lwe, count, out);
  CKL(c);
  return FDFB_OK;
}

// Steps 3-7 of the bootstrap for ciphertexts [s0, s0 + cnt) of the batch (all workspace arrays
// are indexed by ciphertext, so a part works on sub-ranges): ell_boot blind rotations of the part,
// BuildAcc, the final rotation, extraction and the LWE key switch, on stream st.
static int boot_part(const fdfb_ctx* c, const void* brk, const void* bpk, const void* ksk, const uint64_t* rotp,
                     uint32_t k, uint64_t* ct_out, uint32_t B, const BootWs& w, uint32_t s0, uint32_t cnt,
                     void* ks_ws, cudaStream_t st, bool pace) {
  const fdfb_params& p = c->prm;
  const int N = p.N, ellb = p.ell_boot;
  if (cnt == 0) return FDFB_OK;
  int rc;
  size_t tot;
  u64* accs = w.accs + (size_t)s0 * ellb * 2 * N;
  u64* lad = w.lweN + (size_t)s0 * ellb * (N + 1);                 // ladder samples [B ell][N+1]
  u64* dig = w.dig + (size_t)s0 * ellb * N;
  const u32* abar = w.abar + (size_t)s0 * p.n;
  const u32* bbar = w.bbar + s0;
  // 3. ell_boot blind rotations of every ciphertext, batched
  if ((rc = launch_br(c, (const u64*)brk, accs, (int)(cnt * ellb), ellb, abar, st, 0, nullptr, 0, pace))) return rc;
  // 4. SampleExt(., 1) + L^{i-1}/2
  tot = (size_t)cnt * ellb * (N + 1);
  k_ladder_extract<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, accs, (int)(cnt * ellb), lad);
  CKL(c);
  // 5. BuildAcc: KeySwitch LWE->RLWE (into accs), then PubMux per LUT
  if ((rc = keyswitch_rlwe(c, (const u64*)bpk, lad, (int)(cnt * ellb), accs, ks_ws, st))) return rc;
  if ((rc = launch_ntt_batch(c, accs, (size_t)cnt * ellb * 2, 0, st))) return rc;
  for (uint32_t kk = 0; kk < k; kk++) {
    const uint64_t* rp = rotp + (size_t)kk * 2 * N;
    u64* F = w.F + ((size_t)kk * B + s0) * 2 * N;
    tot = (size_t)cnt * N;
    k_pubmux_digits<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, rp, bbar, (int)cnt, dig);
    CKL(c);
    if ((rc = launch_ntt_batch(c, dig, (size_t)cnt * ellb, 0, st))) return rc;
    tot = (size_t)cnt * 2 * N;
    k_pubmux_mac<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, dig, accs, (int)cnt, F, c->qinv_neg, c->r2);
    CKL(c);
    if ((rc = launch_ntt_batch(c, F, (size_t)cnt * 2, 1, st))) return rc;
    tot = (size_t)cnt * N;
    k_pubmux_finish<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, rp, bbar, (int)cnt, F);
    CKL(c);
  }
  // 6.-7. final blind rotation, SampleExt(., 1), ModSwitch(Q -> q_lwe), KeySwitch mod q_lwe
  //       (reading c.3); output samples after the ladder rows
  for (uint32_t kk = 0; kk < k; kk++) {
    u64* F = w.F + ((size_t)kk * B + s0) * 2 * N;
    u64* o = w.lweN + ((size_t)ellb * B + (size_t)kk * B + s0) * (N + 1);
    if ((rc = launch_br(c, (const u64*)brk, F, (int)cnt, 1, abar, st, (int)cnt, nullptr, 0, pace))) return rc;
    tot = (size_t)cnt * (N + 1);
    k_extract_modswitch<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, F, (int)cnt, o);
    CKL(c);
    if ((rc = keyswitch_lwe(c, (const u64*)ksk, o, (int)cnt, ct_out + ((size_t)kk * B + s0) * (p.n + 1), ks_ws, st)))
      return rc;
  }
  return FDFB_OK;
}

// FDFB Bootstrap (Fig. Bootstrap; readings R1, F4, c.3) of B ciphertexts
// under k LUTs (rotp: k x [2][N]); the ladder rotations, SampleExt and the LWE->RLWE key
// switch are shared by the k functions; out: [k][B][n+1].
// Large single-LUT batches run as two halves, the second on the context's helper stream (forked
// and joined with events, so the call stays stream-ordered and graph-capturable): the blind
// rotations of one half fill the SMs the other half's persistent CTAs leave idle at the end of
// each launch (the wave tail), and one half's BuildAcc / key switches overlap the other's BR.
static int bootstrap_impl(const fdfb_ctx* c, const void* brk, const void* bpk, const void* ksk, const uint64_t* rotp,
                          uint32_t k, const uint64_t* ct_in, uint64_t* ct_out, uint32_t B, void* workspace,
                          cudaStream_t st) {
  const fdfb_params& p = c->prm;
  const int N = p.N, ellb = p.ell_boot;
  BootWs w = boot_ws(p, B, workspace, k);
  size_t tot;
  // 1. ModSwitch(ct, q_lwe, 2N)
  tot = (size_t)B * (p.n + 1);
  k_modswitch_in<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, ct_in, B, w.abar, w.bbar, (int)c->dp.logN + 1);
  CKL(c);
  // 2. ladder accumulators (reading R1)
  tot = (size_t)B * ellb * N;
  k_ladder_init<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, w.bbar, B, w.accs);
  CKL(c);
  void* ks0 = w.ks;
  void* ks1 = (char*)w.ks + w.ks_part;
  const bool split = c->boot_split && k == 1 && B >= 64;
  if (!split) return boot_part(c, brk, bpk, ksk, rotp, k, ct_out, B, w, 0, B, ks0, st, true);
  const uint32_t h = B / 2;
  std::lock_guard<std::mutex> lock(c->boot_mu);
  CK(cudaEventRecord(c->ev_fork, st));
  CK(cudaStreamWaitEvent(c->helper, c->ev_fork, 0));
  int rc = boot_part(c, brk, bpk, ksk, rotp, k, ct_out, B, w, 0, h, ks0, st, c->br_pace_split);
  int rc2 = boot_part(c, brk, bpk, ksk, rotp, k, ct_out, B, w, h, B - h, ks1, c->helper, c->br_pace_split);
  CK(cudaEventRecord(c->ev_join, c->helper));
  CK(cudaStreamWaitEvent(st, c->ev_join, 0));
  return rc ? rc : rc2;
}

extern "C" int fdfb_bootstrap_batch(const fdfb_ctx* c, const void* brk, const void* bpk, const void* ksk,
                                    const uint64_t* rotp, const uint64_t* ct_in, uint64_t* ct_out, uint32_t B,
                                    void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (B == 0) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (B > kMaxBatch) return FDFB_E_DIMENSION;
  if (!brk || !bpk || !ksk || !rotp || !ct_in || !ct_out || !workspace) return FDFB_E_NULL;
  return bootstrap_impl(c, brk, bpk, ksk, rotp, 1, ct_in, ct_out, B, workspace, S(stream));
}

extern "C" int fdfb_bootstrap_multi_batch(const fdfb_ctx* c, const void* brk, const void* bpk, const void* ksk,
                                          const uint64_t* rotp, uint32_t k, const uint64_t* ct_in, uint64_t* ct_out,
                                          uint32_t B, void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (B == 0) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (B > kMaxBatch) return FDFB_E_DIMENSION;
  if (!brk || !bpk || !ksk || !rotp || !ct_in || !ct_out || !workspace) return FDFB_E_NULL;
  if (k == 0) return FDFB_E_DIMENSION;
  return bootstrap_impl(c, brk, bpk, ksk, rotp, k, ct_in, ct_out, B, workspace, S(stream));
}

// TFHE (half-domain) bootstrap (Fig. PAPER.md:3070-3090, output order of reading c.3):
// acc = [rotP_0 X^{b~}, 0], one blind rotation, SampleExt, ModSwitch Q -> q_lwe, KeySwitch.
__global__ void k_tfhe_init(DevParams p, const u64* __restrict__ rotp0, const u32* __restrict__ bbar, int B,
                            u64* __restrict__ F) {
  const int N = p.N;
  const size_t total = (size_t)B * N;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    const int cc = (int)(x / N), j = (int)(x % N);
    F[(size_t)cc * 2 * N + j] = rot_coeff(rotp0, j, (int)bbar[cc], N, p.Q);
    F[(size_t)cc * 2 * N + N + j] = 0;
  }
}
extern "C" int fdfb_bootstrap_tfhe_batch(const fdfb_ctx* c, const void* brk, const void* ksk, const uint64_t* rotp,
                                         const uint64_t* ct_in, uint64_t* ct_out, uint32_t B, void* workspace,
                                         void* stream) {
  if (!c) return FDFB_E_NULL;
  if (B == 0) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (B > kMaxBatch) return FDFB_E_DIMENSION;
  if (!brk || !ksk || !rotp || !ct_in || !ct_out || !workspace) return FDFB_E_NULL;
  cudaStream_t st = S(stream);
  const fdfb_params& p = c->prm;
  const int N = p.N;
  BootWs w = boot_ws(p, B, workspace);
  size_t tot = (size_t)B * (p.n + 1);
  k_modswitch_in<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, ct_in, B, w.abar, w.bbar, (int)c->dp.logN + 1);
  CKL(c);
  tot = (size_t)B * N;
  k_tfhe_init<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, rotp, w.bbar, (int)B, w.F);
  CKL(c);
  int rc = launch_br(c, (const u64*)brk, w.F, (int)B, 1, w.abar, st);
  if (rc) return rc;
  tot = (size_t)B * (N + 1);
  k_extract_modswitch<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, w.F, (int)B, w.lweN);
  CKL(c);
  return keyswitch_lwe(c, (const u64*)ksk, w.lweN, (int)B, ct_out, w.ks, st);
}

extern "C" int fdfb_bootstrap_batch_host(const fdfb_ctx* c, const void* brk, const void* bpk, const void* ksk,
                                         const uint64_t* rotp, const uint64_t* in_h, uint64_t* out_h, uint32_t B,
                                         void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (B == 0) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (B > kMaxBatch) return FDFB_E_DIMENSION;
  if (!in_h || !out_h || !workspace) return FDFB_E_NULL;
  cudaStream_t st = S(stream);
  size_t bytes = (size_t)B * (c->prm.n + 1) * 8;
  BootWs w = boot_ws(c->prm, B, workspace);
  u64* din = (u64*)((char*)workspace + w.bytes);
  u64* dout = din + (size_t)B * (c->prm.n + 1);
  CK(cudaMemcpyAsync(din, in_h, bytes, cudaMemcpyHostToDevice, st));
  int rc = fdfb_bootstrap_batch(c, brk, bpk, ksk, rotp, din, dout, B, workspace, stream);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out_h, dout, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return FDFB_OK;
}

extern "C" int fdfb_sample_extract(const fdfb_ctx* c, const uint64_t* rlwe, const uint32_t* k, uint64_t* lwe,
                                   uint32_t B, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (!B) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (!rlwe || !k || !lwe) return FDFB_E_NULL;
  size_t tot = (size_t)B * (c->prm.N + 1);
  k_sample_extract<<<grid_for(tot, 256, c->num_sms), 256, 0, S(stream)>>>(c->dp, rlwe, k, B, lwe, c->d_status);
  CKL(c);
  return FDFB_OK;
}

extern "C" size_t fdfb_workspace_keyswitch(const fdfb_ctx* c, uint32_t B) {
  return c ? ks_ws_bytes(ks_shape_lwe(c->prm), (int)(B ? B : 1)) : 0;
}
extern "C" int fdfb_lwe_keyswitch(const fdfb_ctx* c, const void* ksk, const uint64_t* lwe_N, uint64_t* lwe_n,
                                  uint32_t B, void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (!B) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (!ksk || !lwe_N || !lwe_n) return FDFB_E_NULL;
  return keyswitch_lwe(c, (const u64*)ksk, lwe_N, (int)B, lwe_n, workspace, S(stream));
}

extern "C" size_t fdfb_workspace_poly_mul(const fdfb_ctx* c, uint32_t count) {
  return c ? align256((size_t)count * c->prm.N * 8) : 0;
}
extern "C" int fdfb_poly_mul(const fdfb_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t count,
                             void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (!count) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (!a || !b || !out) return FDFB_E_NULL;
  if (!workspace) return FDFB_E_WORKSPACE;
  cudaStream_t st = S(stream);
  const int N = c->prm.N;
  u64* tb = (u64*)workspace;
  CK(cudaMemcpyAsync(out, a, (size_t)count * N * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(tb, b, (size_t)count * N * 8, cudaMemcpyDeviceToDevice, st));
  int rc = launch_ntt_batch(c, out, count, 0, st);
  if (!rc) rc = launch_ntt_batch(c, tb, count, 0, st);
  if (!rc) {
    size_t tot = (size_t)count * N;
    k_pointwise_mul<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(out, tb, out, tot, tot, c->dp.Q, c->qinv_neg, c->r2);
    CKL(c);
    rc = launch_ntt_batch(c, out, count, 1, st);
  }
  return rc;
}

extern "C" int fdfb_lwe_decrypt(const fdfb_ctx* c, const int8_t* sk, const uint64_t* ct, uint32_t count, uint32_t t,
                                uint64_t* phase, uint64_t* msg, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (!count) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (!sk || !ct || (!phase && !msg)) return FDFB_E_NULL;
  if (msg && t == 0) return FDFB_E_PLAINTEXT;
  const unsigned blocks = (unsigned)(((size_t)count * 32 + 255) / 256);
  k_lwe_decrypt<<<blocks, 256, 0, S(stream)>>>(c->dp, sk, ct, (int)count, t, phase, msg);
  CKL(c);
  return FDFB_OK;
}

extern "C" size_t fdfb_workspace_rlwe_phase(const fdfb_ctx* c, uint32_t count) {
  return c ? 3 * align256((size_t)count * c->prm.N * 8) + fdfb_workspace_poly_mul(c, count) : 0;
}
extern "C" int fdfb_rlwe_phase(const fdfb_ctx* c, const int8_t* sk, const uint64_t* ct, uint32_t count, uint64_t* out,
                               void* workspace, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (!count) return FDFB_OK;  // empty batch: data pointers may be NULL
  if (!sk || !ct || !out) return FDFB_E_NULL;
  if (!workspace) return FDFB_E_WORKSPACE;
  cudaStream_t st = S(stream);
  const size_t tot = (size_t)count * c->prm.N;
  u64* a = (u64*)workspace;
  u64* sp = (u64*)((char*)a + align256(tot * 8));
  u64* prod = (u64*)((char*)sp + align256(tot * 8));
  void* pm_ws = (char*)prod + align256(tot * 8);
  k_rlwe_phase_prep<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, ct, sk, (int)count, a, sp);
  CKL(c);
  int rc = fdfb_poly_mul(c, a, sp, prod, count, pm_ws, st);
  if (!rc) {
    k_rlwe_phase_finish<<<grid_for(tot, 256, c->num_sms), 256, 0, st>>>(c->dp, ct, prod, (int)count, out);
    CKL(c);
  }
  return rc;
}

extern "C" int fdfb_cdt_table(const fdfb_ctx* c, uint64_t* thr, int* T) {
  if (!c || !T) return FDFB_E_NULL;
  *T = c->dp.cdt_T;
  if (thr) for (size_t i = 0; i < c->cdt.size(); i++) thr[i] = c->cdt[i];
  return FDFB_OK;
}
extern "C" int fdfb_device_status(const fdfb_ctx* c, int clear) {
  if (!c) return FDFB_E_NULL;
  int h = 0;
  CK(cudaMemcpy(&h, c->d_status, sizeof(int), cudaMemcpyDeviceToHost));
  if (clear) CK(cudaMemset(c->d_status, 0, sizeof(int)));
  return (h & 1) ? FDFB_E_INDEX : FDFB_OK;
}
extern "C" int fdfb_timing_enable(const fdfb_ctx* c, int on) {
  if (!c) return FDFB_E_NULL;
  c->timing = on != 0;
  return FDFB_OK;
}
extern "C" int fdfb_timing_read(const fdfb_ctx* c, int kclass, double* total_ms, uint64_t* launches) {
  if (!c || !total_ms || !launches) return FDFB_E_NULL;
  std::lock_guard<std::mutex> g(c->tmu);
  double ms = 0; uint64_t cnt = 0;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> keep;
  for (auto& e : c->tev) {
    if (e.first != kclass) { keep.push_back(e); continue; }
    CK(cudaEventSynchronize(e.second.second));
    float f = 0;
    CK(cudaEventElapsedTime(&f, e.second.first, e.second.second));
    ms += f; cnt++;
    cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second);
  }
  c->tev.swap(keep);
  *total_ms = ms; *launches = cnt;
  return FDFB_OK;
}
// Wall span covered by the launches of one class: the union of their [start, end] intervals
// (launches on the bootstrap's two streams overlap, so their summed durations overcount).
extern "C" int fdfb_timing_read_union(const fdfb_ctx* c, int kclass, double* union_ms, uint64_t* launches) {
  if (!c || !union_ms || !launches) return FDFB_E_NULL;
  std::lock_guard<std::mutex> g(c->tmu);
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> keep, mine;
  for (auto& e : c->tev) (e.first == kclass ? mine : keep).push_back(e);
  std::vector<std::pair<double, double>> iv;
  for (auto& e : mine) CK(cudaEventSynchronize(e.second.second));
  for (auto& e : mine) {
    float a = 0, b = 0;
    CK(cudaEventElapsedTime(&a, mine[0].second.first, e.second.first));   // may be negative
    CK(cudaEventElapsedTime(&b, mine[0].second.first, e.second.second));
    iv.push_back({a, b});
  }
  std::sort(iv.begin(), iv.end());
  double ms = 0, cs = 0, ce = 0;
  bool open = false;
  for (auto& x : iv) {
    if (!open || x.first > ce) { if (open) ms += ce - cs; cs = x.first; ce = x.second; open = true; }
    else if (x.second > ce) ce = x.second;
  }
  if (open) ms += ce - cs;
  for (auto& e : mine) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
  c->tev.swap(keep);
  *union_ms = ms;
  *launches = mine.size();
  return FDFB_OK;
}
extern "C" uint64_t fdfb_launch_count(const fdfb_ctx* c) { return c ? (uint64_t)c->launches.load() : 0; }

// Parity hook of the tcgen05 int8 GEMM itself: D [M][Ncols] int32 = A [M][K] x B [Ncols][K]^T.
extern "C" int fdfb_gemm_i8(const fdfb_ctx* c, const int8_t* A, const int8_t* B, uint32_t M, uint32_t Ncols,
                            uint32_t K, int32_t* D, void* stream) {
  if (!c) return FDFB_E_NULL;
  if (!M || !Ncols) return FDFB_OK;
  if (!A || !B || !D) return FDFB_E_NULL;
  if (K == 0 || K % 16) return FDFB_E_DIMENSION;
  ImmaEpi e;
  e.mode = 2; e.nlp = 1; e.rows = (int)M; e.W = (int)Ncols; e.ldo = (int)Ncols; e.neg_sub = 0;
  e.qmask = 0; e.out = D; e.lwe = nullptr; e.lwe_ld = 0;
  return imma_gemm(c, A, M, K, B, Ncols, K, K, e, FDFB_KCLASS_SHIFT_GEMM, S(stream));
}

extern "C" const char* fdfb_status_string(int s) {
  switch (s) {
    case FDFB_OK: return "ok";
    case FDFB_E_NULL: return "null pointer argument";
    case FDFB_E_NON_NTT_MODULUS: return "Q is not a prime with Q = 1 mod 2N (or Q >= 2^55)";
    case FDFB_E_DIMENSION: return "dimension out of range";
    case FDFB_E_DECOMP: return "gadget decomposition: ell != ceil(bits / logL) or out of range";
    case FDFB_E_INDEX: return "index out of range";
    case FDFB_E_PLAINTEXT: return "plaintext modulus t must divide 2N";
    case FDFB_E_UNSUPPORTED: return "unsupported parameter combination";
    case FDFB_E_CUDA: return "CUDA error";
    case FDFB_E_WORKSPACE: return "workspace too small";
    case FDFB_E_KIND: return "unknown key kind";
  }
  return "unknown status";
}
extern "C" const char* fdfb_last_cuda_error(void) { return g_last_cuda.c_str(); }
#include "shift_host.inc"
