// bfbench.cu -- butterfly-throughput microbenchmark for the BR kernel's NTT arithmetic.
// Compares, on the whole chip (butterflies per SM per clock), the lazy 32-bit Harvey/Shoup
// butterfly used by k_blind_rotate with a variant that takes the quotient from an FP64 FMA
// (q = round(y w / p) via the 1.5*2^52 magic constant), moving the IMAD.HI off the
// integer-multiply pipe.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;      // independent butterflies per thread
constexpr int IT = 2048;

__device__ __forceinline__ uint32_t csub(uint32_t a, uint32_t m) { return min(a, a - m); }

__global__ void k_bf_shoup(uint32_t* out, uint32_t p, uint32_t w0, uint32_t ws0, long long* cyc) {
  uint32_t x[CH], y[CH];
  for (int c = 0; c < CH; c++) { x[c] = (threadIdx.x * 977 + c * 131) % p; y[c] = (threadIdx.x * 613 + c * 71) % p; }
  const uint32_t p2 = 2 * p;
  const uint32_t w = w0 + (threadIdx.x & 1), ws = ws0 + (threadIdx.x & 1);
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < IT; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      const uint32_t q = __umulhi(y[c], ws);
      const uint32_t t = y[c] * w - q * p;            // [0, 2p)
      const uint32_t nx = x[c] + t, ny = x[c] - t + p2;
      x[c] = csub(nx, p2);
      y[c] = csub(ny, p2);
    }
  }
  long long t1 = clock64();
  uint32_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c] ^ y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_bf_fp64(uint32_t* out, uint32_t p, uint32_t w0, double wd0, long long* cyc) {
  uint32_t x[CH], y[CH];
  for (int c = 0; c < CH; c++) { x[c] = (threadIdx.x * 977 + c * 131) % p; y[c] = (threadIdx.x * 613 + c * 71) % p; }
  const uint32_t p2 = 2 * p;
  const uint32_t w = w0 + (threadIdx.x & 1);
  const double wd = wd0 * (1.0 + 1e-12 * (threadIdx.x & 1));
  const double M = 4503599627370496.0;            // 2^52
  const double R = 6755399441055744.0;            // 1.5 * 2^52: round-to-nearest integer magic
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < IT; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      const double yd = __hiloint2double(0x43300000, (int)y[c]) - M;   // exact y
      const double qd = fma(yd, wd, R);
      const uint32_t q = (uint32_t)__double2loint(qd);                  // round(y w / p) (+-1)
      const uint32_t t = y[c] * w - q * p + p;                          // (0, 2p)
      const uint32_t nx = x[c] + t, ny = x[c] - t + p2;
      x[c] = csub(nx, p2);
      y[c] = csub(ny, p2);
    }
  }
  long long t1 = clock64();
  uint32_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c] ^ y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_bf_i2f(uint32_t* out, uint32_t p, uint32_t w0, double wd0, long long* cyc) {
  uint32_t x[CH], y[CH];
  for (int c = 0; c < CH; c++) { x[c] = (threadIdx.x * 977 + c * 131) % p; y[c] = (threadIdx.x * 613 + c * 71) % p; }
  const uint32_t p2 = 2 * p;
  const uint32_t w = w0 + (threadIdx.x & 1);
  const double wd = wd0 * (1.0 + 1e-12 * (threadIdx.x & 1));
  const double R = 6755399441055744.0;
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < IT; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      const double qd = fma((double)y[c], wd, R);
      const uint32_t q = (uint32_t)__double2loint(qd);
      const uint32_t t = y[c] * w - q * p + p;
      const uint32_t nx = x[c] + t, ny = x[c] - t + p2;
      x[c] = csub(nx, p2);
      y[c] = csub(ny, p2);
    }
  }
  long long t1 = clock64();
  uint32_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c] ^ y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// mixed: NF of the CH chains take the FP64 quotient (fp64 pipe), the others the Shoup IMAD.HI
// (multiply pipe): the two pipes run in parallel
template <int NF>
__global__ void k_bf_mix(uint32_t* out, uint32_t p, uint32_t w0, uint32_t ws0, double wd0, long long* cyc) {
  uint32_t x[CH], y[CH];
  for (int c = 0; c < CH; c++) { x[c] = (threadIdx.x * 977 + c * 131) % p; y[c] = (threadIdx.x * 613 + c * 71) % p; }
  const uint32_t p2 = 2 * p;
  const uint32_t w = w0 + (threadIdx.x & 1), ws = ws0 + (threadIdx.x & 1);
  const double wd = wd0 * (1.0 + 1e-12 * (threadIdx.x & 1));
  const double M = 4503599627370496.0, R = 6755399441055744.0;
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < IT; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      uint32_t t;
      if (c < NF) {
        const double yd = __hiloint2double(0x43300000, (int)y[c]) - M;
        const uint32_t q = (uint32_t)__double2loint(fma(yd, wd, R));
        t = y[c] * w - q * p + p;
      } else {
        const uint32_t q = __umulhi(y[c], ws);
        t = y[c] * w - q * p;
      }
      const uint32_t nx = x[c] + t, ny = x[c] - t + p2;
      x[c] = csub(nx, p2);
      y[c] = csub(ny, p2);
    }
  }
  long long t1 = clock64();
  uint32_t r = 0;
  for (int c = 0; c < CH; c++) r ^= x[c] ^ y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// correctness of the FP64 quotient over many (y, w): t must land in (0, 2p) and equal y w mod p
__global__ void k_check(uint32_t p, uint32_t* bad, unsigned long long n) {
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t y = (uint32_t)((k * 2654435761ull) % (16ull * p));   // lazy inputs up to 16p
    const uint32_t w = (uint32_t)((k * 40503ull + 17) % p);
    const double wd = (double)w / (double)p;
    const double qd = fma(__hiloint2double(0x43300000, (int)y) - 4503599627370496.0, wd, 6755399441055744.0);
    const uint32_t q = (uint32_t)__double2loint(qd);
    const uint32_t t = y * w - q * p + p;
    const uint32_t ref = (uint32_t)(((unsigned long long)y * w) % p);
    if (!(t > 0 && t < 2 * p && (t % p) == ref)) atomicAdd(bad, 1u);
  }
}

int main() {
  const uint32_t p = 268369921u;   // 2^28 - 2^16 + 1 (prime, = 1 mod 4096)
  const uint32_t w = 123456789u % p;
  const uint32_t ws = (uint32_t)(((uint64_t)w << 32) / p);
  const double wd = (double)w / (double)p;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out; long long* cyc; uint32_t* bad;
  const int TPB = 256;
  cudaMalloc(&out, 64ull * sms * TPB * 4);
  cudaMalloc(&cyc, 64ull * sms * 8);
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  k_check<<<sms * 8, 256>>>(p, bad, 1ull << 30);
  uint32_t hbad = 0;
  cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost);
  printf("{\"fp64_quotient_check\": {\"samples\": %llu, \"bad\": %u}}\n", 1ull << 30, hbad);
  for (int blocks_per_sm = 2; blocks_per_sm <= 8; blocks_per_sm *= 2) {
    for (int v = 0; v < 7; v++) {
      const int grid = sms * blocks_per_sm;
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        if (v == 0) k_bf_shoup<<<grid, TPB>>>(out, p, w, ws, cyc);
        else if (v == 1) k_bf_fp64<<<grid, TPB>>>(out, p, w, wd, cyc);
        else if (v == 2) k_bf_i2f<<<grid, TPB>>>(out, p, w, wd, cyc);
        else if (v == 3) k_bf_mix<1><<<grid, TPB>>>(out, p, w, ws, wd, cyc);
        else if (v == 4) k_bf_mix<2><<<grid, TPB>>>(out, p, w, ws, wd, cyc);
        else if (v == 5) k_bf_mix<3><<<grid, TPB>>>(out, p, w, ws, wd, cyc);
        else k_bf_mix<4><<<grid, TPB>>>(out, p, w, ws, wd, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bfly = (double)grid * TPB * CH * IT;
      const double per_sm_clk = bfly / (ms * 1e-3) / sms / (clk * 1e3);
      printf("{\"variant\": \"%s\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"butterflies_per_sm_per_clk_nominal\": %.2f, "
             "\"err\": \"%s\"}\n", (const char*[]){"shoup", "fp64_magic", "fp64_i2f", "mix1of8", "mix2of8", "mix3of8", "mix4of8"}[v], blocks_per_sm, ms,
             per_sm_clk, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
