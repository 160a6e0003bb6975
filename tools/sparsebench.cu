// sparsebench.cu -- can the sparse form of the RNS primes move work off the multiply pipe?
// The BR kernel's lazy Harvey butterfly spends 4 multiply-pipe slots (IMAD.HI + 2 IMAD) and
// 2 ALU ops.  For p = 2^28 - 2^16 + 1 the quotient product is q p = (q << 28) - (q << 16) + q,
// so r = y w - q p mod 2^32 can use two LEA (ALU) instead of one IMAD: 3 slots + 5 ALU ops,
// the same 32-bit result.  This measures butterflies per SM per clock (whole chip, 2 CTAs of
// 256 threads per SM as in k_blind_rotate_p) for all-Shoup, all-sparse and mixes.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o sparsebench tools/sparsebench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 16;     // independent butterflies per thread (V = 2 polynomials x 8)
constexpr int IT = 1024;
constexpr uint32_t P0 = 268369921u;   // 2^28 - 2^16 + 1

__device__ __forceinline__ uint32_t lea(uint32_t a, uint32_t b, int s) { return (a << s) + b; }
// q << S as a funnel shift with an opaque zero low word: ptxas cannot turn it into IMAD.SHL
template <int S>
__device__ __forceinline__ uint32_t shl_alu(uint32_t q, uint32_t z) {
  uint32_t r;
  asm("shf.l.clamp.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(z), "r"(q), "n"(S));
  return r;
}

// SPARSE_MASK bit c: chain c uses the shift form
template <uint32_t SPARSE_MASK, bool FORCE>
__global__ void __launch_bounds__(256, 2) k_bf(uint32_t* out, uint32_t p, uint32_t w0, uint32_t ws0, uint32_t z,
                                               long long* cyc) {
  uint32_t x[CH], y[CH];
  for (int c = 0; c < CH; c++) { x[c] = (threadIdx.x * 977 + c * 131) % p; y[c] = (threadIdx.x * 613 + c * 71) % p; }
  const uint32_t p2 = 2 * p;
  const uint32_t w = w0 + (threadIdx.x & 1), ws = ws0 + (threadIdx.x & 1);
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < IT; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      const uint32_t q = __umulhi(y[c], ws);
      const uint32_t xx = x[c];
      if (FORCE && (SPARSE_MASK >> c & 1)) {
        const uint32_t s16 = shl_alu<16>(q, z), s28 = shl_alu<28>(q, z);
        const uint32_t r = y[c] * w + s16 - q;             // IADD3 (u, s16, -q)
        x[c] = xx + r - s28;
        y[c] = xx - r + s28 + p2;
      } else if (SPARSE_MASK >> c & 1) {
        const uint32_t t1 = lea(q, y[c] * w, 16);          // y w + (q << 16)
        const uint32_t t2 = lea(q, q, 28);                 // (q << 28) + q
        x[c] = xx + t1 - t2;                               // x + t
        y[c] = xx - t1 + t2 + p2;                          // x - t + 2p
      } else {
        const uint32_t t = y[c] * w - q * p;
        x[c] = xx + t + z;
        y[c] = xx - t + p2;
      }
    }
    // keep the values bounded-ish (timing only): rotate chains so they stay dependent
    const uint32_t tmp = x[0];
#pragma unroll
    for (int c = 0; c < CH - 1; c++) x[c] = x[c + 1];
    x[CH - 1] = tmp;
  }
  long long t1 = clock64();
  uint32_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c] ^ y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_check(uint32_t p, uint32_t* bad, unsigned long long n) {   // sparse r == Shoup r
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t y = (uint32_t)(k * 2654435761ull);
    const uint32_t w = (uint32_t)((k * 40503ull + 17) % p);
    const uint32_t ws = (uint32_t)(((unsigned long long)w << 32) / p);
    const uint32_t q = __umulhi(y, ws);
    const uint32_t a = y * w - q * p;
    const uint32_t b = lea(q, y * w, 16) - lea(q, q, 28);
    if (a != b || a >= 2 * p || (a % p) != (uint32_t)(((unsigned long long)y * w) % p)) atomicAdd(bad, 1u);
  }
}

template <uint32_t M, bool F = false>
void run(const char* name, int sms, uint32_t* d_out, long long* d_cyc, uint32_t w, uint32_t ws) {
  const int grid = 2 * sms;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_bf<M, F><<<grid, 256>>>(d_out, P0, w, ws, 0u, d_cyc);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) k_bf<M, F><<<grid, 256>>>(d_out, P0, w, ws, 0u, d_cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double bf = 5.0 * grid * 256.0 * IT * CH;
  const double per_sm_clk = bf / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("{\"variant\": \"%s\", \"sparse_chains\": %d, \"ms\": %.3f, \"butterflies_per_sm_per_clk_nominal\": %.2f, \"err\": \"%s\"}\n",
         name, __builtin_popcount(M), ms, per_sm_clk, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t w = 123456789u % P0;
  const uint32_t ws = (uint32_t)(((uint64_t)w << 32) / P0);
  uint32_t *d_out, *d_bad;
  long long* d_cyc;
  cudaMalloc(&d_out, 4 * sms * 256 * sizeof(uint32_t));
  cudaMalloc(&d_cyc, 4 * sms * sizeof(long long));
  cudaMalloc(&d_bad, 4);
  cudaMemset(d_bad, 0, 4);
  k_check<<<4 * sms, 256>>>(P0, d_bad, 1ull << 30);
  uint32_t bad = 0;
  cudaMemcpy(&bad, d_bad, 4, cudaMemcpyDeviceToHost);
  printf("{\"sparse_form_check\": {\"samples\": %llu, \"bad\": %u}}\n", 1ull << 30, bad);
  for (int rep = 0; rep < 2; rep++) {
    run<0x0000>("shoup", sms, d_out, d_cyc, w, ws);
    run<0x1111>("sparse 1/4", sms, d_out, d_cyc, w, ws);
    run<0x5555>("sparse 1/2", sms, d_out, d_cyc, w, ws);
    run<0x7777>("sparse 3/4", sms, d_out, d_cyc, w, ws);
    run<0xFFFF>("sparse all", sms, d_out, d_cyc, w, ws);
    run<0x1111, true>("shf 1/4", sms, d_out, d_cyc, w, ws);
    run<0x5555, true>("shf 1/2", sms, d_out, d_cyc, w, ws);
    run<0xFFFF, true>("shf all", sms, d_out, d_cyc, w, ws);
  }
  return 0;
}
