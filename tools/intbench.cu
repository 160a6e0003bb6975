// intbench.cu -- integer-pipe microbenchmark for the roofline denominator (DESIGN.md
// "Integer-pipe roofline").  Measures, on the whole chip, lane-ops per SM per clock of
//   imad32   : 32-bit IMAD  (d = a*b + c)                      -- the fma-pipe unit op
//   imadwide : IMAD.WIDE.U32 (64-bit = 32x32 + 64)
//   imadhi   : IMAD.HI.U32
//   shoup64  : one lazy 64-bit Shoup modmul  a*w - umulhi(a, w')*Q  (the NTT/MAC op)
// and prints one JSON line.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8;        // independent chains per thread
constexpr int IT = 4096;     // iterations

__global__ void k_imad32(uint32_t* out, uint32_t s, long long* cyc) {
  uint32_t x[CH];
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c * s;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < IT; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = x[c] * s + (uint32_t)c;
  }
  long long t1 = clock64();
  uint32_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_imadwide(uint64_t* out, uint32_t s, long long* cyc) {
  uint64_t x[CH];
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c * s;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < IT; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = (uint64_t)(uint32_t)x[c] * s + x[c];
  }
  long long t1 = clock64();
  uint64_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_imadhi(uint32_t* out, uint32_t s, long long* cyc) {
  uint32_t x[CH];
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 2654435761u + c * s;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < IT; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = __umulhi(x[c], s) + x[c];
  }
  long long t1 = clock64();
  uint32_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_shoup64(uint64_t* out, uint64_t w, uint64_t wp, uint64_t Q, long long* cyc) {
  uint64_t x[CH];
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 0x9E3779B97F4A7C15ULL + c;
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < IT / 4; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      uint64_t q = __umul64hi(x[c], wp);
      x[c] = x[c] * w - q * Q;
    }
  }
  long long t1 = clock64();
  uint64_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int TPB = 512, BPS = 4;  // 64 warps per SM
  const int grid = sms * BPS;
  uint64_t* out; long long* cyc;
  cudaMalloc(&out, (size_t)grid * TPB * 8);
  cudaMalloc(&cyc, grid * 8);
  long long* hc = new long long[grid];
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint64_t Q = 18014398509404161ULL, w = 1234567890123ULL;
  const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / Q);
  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f", sms, clk_khz / 1000.0);
  for (int which = 0; which < 4; which++) {
    double best_ms = 1e30, best_cyc = 0;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(e0);
      if (which == 0) k_imad32<<<grid, TPB>>>((uint32_t*)out, 3u, cyc);
      if (which == 1) k_imadwide<<<grid, TPB>>>(out, 3u, cyc);
      if (which == 2) k_imadhi<<<grid, TPB>>>((uint32_t*)out, 2654435761u, cyc);
      if (which == 3) k_shoup64<<<grid, TPB>>>(out, w, wp, Q, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost);
      double mc = 0; for (int i = 0; i < grid; i++) mc = hc[i] > mc ? hc[i] : mc;
      if (ms < best_ms) { best_ms = ms; best_cyc = mc; }
    }
    const int iters = which == 3 ? IT / 4 : IT;
    double ops = (double)grid * TPB * CH * iters;              // lane-ops
    double per_sm_clk = ops / sms / best_cyc;                   // lane-ops / SM / clock
    double eff_mhz = best_cyc / (best_ms * 1e3);                // cycles per us
    const char* nm[4] = {"imad32", "imadwide", "imadhi", "shoup64"};
    printf(", \"%s\": {\"ops_per_sm_clk\": %.2f, \"ms\": %.3f, \"eff_mhz\": %.0f, \"Gops\": %.1f}", nm[which],
           per_sm_clk, best_ms, eff_mhz, ops / best_ms / 1e6);
  }
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
