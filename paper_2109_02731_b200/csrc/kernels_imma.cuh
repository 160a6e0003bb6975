// kernels_imma.cuh -- the exact int8 tensor-core contraction behind both key switches
// (PAPER.md:3006-3013), Shift's VectorPack and Permute
// (PAPER.md:124-139): a hand-written sm_100a GEMM on the 5th-generation tensor cores.
//
//   D[r][c] = sum_k A[r][k] * B[c][k]          (int8 x int8 -> int32, exact)
//
// A (rows = digit limbs / 0-1 rows of the ciphertexts) and B (rows = balanced base-256
// digits of the key coefficients) are both K-major in global memory.  CG = 2 (default): a
// CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with tcgen05.mma.cta_group::2,
// each CTA holding its 128 rows of A and BN/2 rows of B per stage, so each SM streams half
// the operand bytes of a 1-CTA 128 x BN tile per MMA (CG = 1 is kept for A/B runs).
// Per CTA (one per SM, persistent over the output tiles, 256 threads, warp-specialised):
//   warp 0      TMA producer: cp.async.bulk.tensor 2D loads of a 128 x 128 B tile of A and
//               a BN/CG x 128 B tile of B per stage (SWIZZLE_128B), STAGES-deep mbarrier ring
//               (CG = 2: both CTAs' loads complete on the leader CTA's barrier);
//   warp 1      MMA issuer (one thread of the leader CTA): tcgen05.mma.kind::i8, M = 128 CG,
//               N = BN, K = 32 per instruction, accumulators (int32) in TMEM, two
//               accumulator buffers so the epilogue of tile t overlaps the MMAs of t + 1;
//               its commits arrive on both CTAs' barriers (multicast);
//   warp 2      TMEM allocator (512 columns);
//   warps 4..7  epilogue: tcgen05.ld of the accumulator rows (one TMEM lane = one row per
//               thread) and the exact recombination of the digit planes, see below.
//
// Column layout of B (built by the key-digit kernels): an output tile of BN = 7 WT
// columns holds the 7 digit planes of WT consecutive output words,
//   column (nb, l, wi) = nb * 7 WT + l * WT + wi,   word w = nb * WT + wi,
// so the epilogue has every digit of a word in one tile and writes the recombined word:
//   v = sum_{l<7} 256^l D_l   (mod Q by Horner/Barrett, or mod 2^64 by wrapping),
//   limb rows: NLP consecutive rows r = g NLP + t of A hold 7-bit limbs t of the same
//   digits, combined across lanes: v_g = sum_t 128^t v_{g,t};
//   out[g][w] = b_g [w = 0] - v_g  (key switch: mod Q or & qmask)  or  out[g][w] = v_g.
// A raw mode writes the int32 accumulators (parity test of the GEMM itself).
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace imma {
constexpr int BM = 128;                      // rows per CTA tile (TMEM lanes)
constexpr int BK = 128;                      // K bytes per stage (one 128-byte swizzle atom)
constexpr int WT = 32;                       // output words per tile
constexpr int BN = 7 * WT;                   // 224 accumulator columns per tile
constexpr int ACC_COLS = 256;                // TMEM columns per accumulator buffer (2 buffers)
constexpr int THREADS = 256;
// NSUB = 2 (long K): a tile is two N = BN MMAs per k-step (448 accumulator columns, one
// accumulator buffer), so each SM streams 27 % fewer operand bytes per MMA; NSUB = 1: one MMA,
// two accumulator buffers (epilogue of tile t overlaps the MMAs of tile t + 1).
template <int CG, int NSUB = 1> struct Cfg {
  static constexpr int NBUF = NSUB == 1 ? 2 : 1;                 // accumulator buffers
  static constexpr int A_BYTES = BM * BK;                        // 16 KB
  static constexpr int BSUB_BYTES = (BN / CG) * BK;              // 28 KB / 14 KB per sub-tile
  static constexpr int STAGE_BYTES = A_BYTES + NSUB * BSUB_BYTES;  // multiple of 1024 (SW128 atoms)
  static constexpr int STAGES = (int)((227 * 1024 - 1024 - 256) / STAGE_BYTES) > 8 ? 8
                              : (int)((227 * 1024 - 1024 - 256) / STAGE_BYTES);
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};
}  // namespace imma

// epilogue parameters
struct ImmaEpi {
  int mode;            // 0: mod Q, 1: mod 2^64 then & qmask, 2: raw int32
  int nlp;             // limb rows per output row (1, 2 or 4); raw: 1
  int rows;            // valid rows of A (M)
  int W;               // valid output words per row (raw: valid columns)
  int ldo;             // output row stride (u64 words; raw: int32 words)
  int neg_sub;         // 1: out = b - v (key switch), 0: out = v
  u64 qmask;
  void* out;
  const u64* lwe;      // b_g = lwe[g * lwe_ld] (neg_sub), may be null
  long long lwe_ld;
};

// ---------------------------------------------------------------- PTX helpers
FDFB_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
FDFB_DEV void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
FDFB_DEV void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
FDFB_DEV void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
FDFB_DEV void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// as mbar_wait, with a suspend-time hint: the waiting warp sleeps until the phase completes (or
// the hint, in ns, expires) instead of re-polling, so waiting warps take no issue slots from
// the ones doing arithmetic
FDFB_DEV void mbar_wait_sleep(uint32_t baddr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(baddr),
      "r"(parity), "r"(1000000u)
      : "memory");
}
FDFB_DEV void tma_load_2d(const CUtensorMap* tm, void* dst, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
FDFB_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
FDFB_DEV uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {   // shared::cluster address in CTA `rank`
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
FDFB_DEV void mbar_arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
FDFB_DEV void cluster_sync_all() {   // every thread of both CTAs (warps reconverged by the caller)
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
// CTA-pair TMA load: lands in this CTA's smem, completes on the barrier at cluster address bar_c
FDFB_DEV void tma_load_2d_pair(const CUtensorMap* tm, void* dst, uint32_t bar_c, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(bar_c), "r"(x), "r"(y)
      : "memory");
}
FDFB_DEV void umma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit of the pair's MMAs: arrive on the barrier at this smem offset in both CTAs
FDFB_DEV void umma_commit_pair(uint64_t* b) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(b))
      : "memory");
}
FDFB_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FDFB_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// K-major, 128-byte-swizzled operand tile: rows of 128 B, 8-row groups 1024 B apart
FDFB_DEV uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                          // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
  return d;
}
// instruction descriptor: kind::i8, D = s32, A = B = signed int8, both K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
FDFB_DEV void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
FDFB_DEV void umma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
// 32 lanes x 32 bits, 8 consecutive columns per thread
FDFB_DEV void tmem_ld8(uint32_t taddr, int (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
FDFB_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 32 lanes x 32 bits, 16 consecutive columns per thread
FDFB_DEV void tmem_ld16(uint32_t taddr, u32 (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
FDFB_DEV void tmem_st16(uint32_t taddr, const u32 (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
FDFB_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- the kernel
template <int CG, int NSUB>
__global__ void __launch_bounds__(imma::THREADS, 1)
k_imma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K, int tiles_m,
       int tiles_n, DevParams dp, ImmaEpi e) {
  using namespace imma;
  using C = Cfg<CG, NSUB>;
  constexpr int STAGES = C::STAGES, A_BYTES = C::A_BYTES, STAGE_BYTES = C::STAGE_BYTES, NBUF = C::NBUF;
  constexpr int BSUB = C::BSUB_BYTES;
  constexpr int TM = BM * CG;                          // rows per (pair) tile
  constexpr int TN = BN * NSUB;                        // accumulator columns per tile
  constexpr int TW = WT * NSUB;                        // output words per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);   // SW128 atoms: 1024-B aligned
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + NBUF;
  uint32_t* tslot = (uint32_t*)(tempty + NBUF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = tiles_m * tiles_n;
  const int nk = (K + BK - 1) / BK;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;     // pair (or CTA) index
  const int nunits = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    for (int s = 0; s < STAGES; s++) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int b = 0; b < NBUF; b++) { mbar_init(tfull + b, 1); mbar_init(tempty + b, 128 * CG); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (warp == 2) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {                                   // ---- TMA producer (each CTA loads its own halves)
      int st = 0;
      uint32_t ph = 0;
      for (int tile = unit; tile < ntiles; tile += nunits) {
        const int tm = tile % tiles_m, tn = tile / tiles_m;
        const int arow = tm * TM + (int)rank * BM, brow = tn * TN + (int)rank * (BN / CG);
        for (int kb = 0; kb < nk; kb++) {
          mbar_wait(empty + st, ph ^ 1);
          uint8_t* sa = smem + st * STAGE_BYTES;
          if constexpr (CG == 2) {
            const uint32_t fb = mapa_rank(smem_u32(full + st), 0);   // the leader's barrier
            if (leader) mbar_expect_tx(full + st, 2 * STAGE_BYTES);
            tma_load_2d_pair(&tmA, sa, fb, kb * BK, arow);
#pragma unroll
            for (int j = 0; j < NSUB; j++) tma_load_2d_pair(&tmB, sa + A_BYTES + j * BSUB, fb, kb * BK, brow + j * BN);
          } else {
            mbar_expect_tx(full + st, STAGE_BYTES);
            tma_load_2d(&tmA, sa, full + st, kb * BK, arow);
#pragma unroll
            for (int j = 0; j < NSUB; j++) tma_load_2d(&tmB, sa + A_BYTES + j * BSUB, full + st, kb * BK, brow + j * BN);
          }
          if (++st == STAGES) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {                         // ---- MMA issuer
      constexpr uint32_t idesc = umma_idesc_i8(TM, BN);   // per MMA: M = 128 CG, N = 224
      int st = 0, ab = 0;
      uint32_t ph = 0, aph = 0;
      for (int tile = unit; tile < ntiles; tile += nunits) {
        mbar_wait(tempty + ab, aph ^ 1);              // epilogues drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(ab * ACC_COLS);
        for (int kb = 0; kb < nk; kb++) {
          mbar_wait(full + st, ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 32; k++) {
#pragma unroll
            for (int j = 0; j < NSUB; j++) {
              const uint64_t ad = umma_desc_sw128(sa + 32 * k), bd = umma_desc_sw128(sb + j * BSUB + 32 * k);
              if constexpr (CG == 2)
                umma_i8_pair(d + j * BN, ad, bd, idesc, (kb | k) != 0);
              else
                umma_i8(d + j * BN, ad, bd, idesc, (kb | k) != 0);
            }
          }
          if constexpr (CG == 2) umma_commit_pair(empty + st); else umma_commit(empty + st);   // slots free
          if (++st == STAGES) { st = 0; ph ^= 1; }
        }
        if constexpr (CG == 2) umma_commit_pair(tfull + ab); else umma_commit(tfull + ab);     // accumulator complete
        if (++ab == NBUF) { ab = 0; aph ^= 1; }
      }
    }
  } else if (warp >= 4) {                              // ---- epilogue (lane quarter = warp % 4)
    const int q = warp & 3;
    const int row_in_tile = (int)rank * BM + q * 32 + lane;
    const uint32_t tempty_c = CG == 2 ? mapa_rank(smem_u32(tempty), 0) : 0;   // the leader's tempty[0]
    int ab = 0;
    uint32_t aph = 0;
    for (int tile = unit; tile < ntiles; tile += nunits) {
      const int tm = tile % tiles_m, tn = tile / tiles_m;
      mbar_wait(tfull + ab, aph);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * ACC_COLS);
      const int row = tm * TM + row_in_tile;
      if (e.mode == 2) {                               // raw int32 accumulators
        int* o = (int*)e.out + (size_t)row * e.ldo;
#pragma unroll 1
        for (int c = 0; c < TN; c += 8) {
          int v[8];
          tmem_ld8(tbase + c, v);
          tmem_ld_wait();
          const int col = tn * TN + c;
          if (row < e.rows) {
#pragma unroll
            for (int i = 0; i < 8; i++)
              if (col + i < e.W) o[col + i] = v[i];
          }
        }
      } else {
        const int nlp = e.nlp;
        const int g = row / nlp, t = row % nlp;       // output row, limb
        const int lbase = lane & ~(nlp - 1);
        u64* o = (u64*)e.out + (size_t)g * e.ldo;
        const bool wrap = e.mode == 1;
#pragma unroll 1
        for (int c8 = 0; c8 < TW; c8 += 8) {
          const int sub = c8 / WT, cw = c8 % WT;         // sub-tile (its own 7 digit planes), word
          int v[7][8];
#pragma unroll
          for (int l = 0; l < 7; l++) tmem_ld8(tbase + sub * BN + l * WT + cw, v[l]);
          tmem_ld_wait();
          u64 val[8];
#pragma unroll
          for (int i = 0; i < 8; i++) {
            u64 s = 0;
            if (wrap) {
#pragma unroll
              for (int l = 6; l >= 0; l--) s = (s << 8) + (u64)(long long)v[l][i];
            } else {
#pragma unroll
              for (int l = 6; l >= 0; l--) s = horner_mod(s, 8, v[l][i], dp);
            }
            // limbs t of output row g sit in lanes lbase .. lbase + nlp - 1: sum_t 128^t s_t
            u64 acc = 0;
            for (int tt = nlp - 1; tt >= 0; tt--) {
              const u64 st = __shfl_sync(0xffffffffu, s, lbase + tt);
              acc = wrap ? (acc << 7) + st : add_mod(horner_mod(acc, 7, 0, dp), st, dp.Q);
            }
            val[i] = acc;
          }
          const int w0 = tn * TW + c8;
          if (row < e.rows) {
#pragma unroll
            for (int i = 0; i < 8; i++) {
              const int w = w0 + i;
              if ((i % nlp) != t || w >= e.W) continue;  // the nlp lanes of a row split the words
              u64 r = val[i];
              if (e.neg_sub) {
                const u64 b = (w == 0 && e.lwe) ? __ldg(e.lwe + (size_t)g * e.lwe_ld) : 0;
                r = wrap ? ((b - r) & e.qmask) : sub_mod(b, r, dp.Q);
              } else if (wrap) {
                r &= e.qmask;
              }
              o[w] = r;
            }
          }
        }
      }
      tc_fence_before();
      if constexpr (CG == 2) mbar_arrive_cluster(tempty_c + 8 * ab); else mbar_arrive(tempty + ab);
      if (++ab == NBUF) { ab = 0; aph ^= 1; }
    }
  }
  __syncwarp();                                        // role loops ran on lane 0 only
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}
