// Latencies (SM clocks, one warp, dependent chains) of what one step of the warp-level FMA sweep
// is built from: DFMA, DADD, 64-bit SHFL, LDS.64, the FP64 tanh (table in shared vs global memory),
// __syncthreads with one warp, and one q = 16 matvec step as the sweep issues it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2007_07336_b200/csrc -I include \
//        -o tools/latency_probe.bin tools/latency_probe.cu && tools/latency_probe.bin
#include <cstdio>

#include <cuda_runtime.h>

#include "lmg.h"
#include "lmg_gemm.cuh"

using namespace lmg;

constexpr int R = 256;

__global__ void probe(double* out, long long* cyc, double seed) {
  __shared__ double sm[1024];
  __shared__ double2 tab[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = 1.0 + i * 1e-9;
  for (int i = lane; i < 64; i += 32) tab[i] = kTanhExp2[i];
  __syncthreads();
  double x = seed + lane * 1e-7, acc = 0.0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < R; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = fma(x, acc, 1e-3);
  }
  t1 = clock64();
  cyc[0] = (t1 - t0) / (R * 16);
  // DADD chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < R; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = __dadd_rn(acc, x);
  }
  t1 = clock64();
  cyc[1] = (t1 - t0) / (R * 16);
  // SHFL (64-bit) chain
  double y = acc;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < R; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) y = __shfl_sync(0xffffffffu, y, (lane + 1) & 31);
  }
  t1 = clock64();
  cyc[2] = (t1 - t0) / (R * 16);
  // LDS.64 pointer chase
  int idx = lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < R * 16; ++i) idx = (int)sm[idx] & 1023;
  t1 = clock64();
  cyc[3] = (t1 - t0) / (R * 16);
  // tanh chain, table in shared memory
  double z = 0.3 + lane * 1e-3;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < R; ++i) z = fast_tanh_impl(z + 0.5, [&](int j) { return tab[j]; });
  t1 = clock64();
  cyc[4] = (t1 - t0) / R;
  // tanh chain, global table
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < R; ++i) z = fast_tanh(z + 0.5);
  t1 = clock64();
  cyc[5] = (t1 - t0) / R;
  // __syncthreads, one warp
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < R; ++i) __syncthreads();
  t1 = clock64();
  cyc[6] = (t1 - t0) / R;
  // one q = 16 step: 16 shuffles + LDS + a k-ascending DFMA chain, then tanh (the sweep's step)
  double xa = x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < R; ++i) {
    double a2 = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double xk = __shfl_sync(0xffffffffu, xa, k);
      a2 = fma(sm[(lane & 15) * 17 + k], xk, a2);
    }
    xa = __dadd_rn(xa, __dmul_rn(0.01, fast_tanh_impl(a2, [&](int j) { return tab[j]; })));
  }
  t1 = clock64();
  cyc[7] = (t1 - t0) / R;
  out[lane] = acc + y + idx + z + xa;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  probe<<<1, 32>>>(out, cyc, 0.5);
  probe<<<1, 32>>>(out, cyc, 0.5);
  cudaDeviceSynchronize();
  const char* names[8] = {"DFMA", "DADD", "SHFL.64", "LDS.64 chase", "tanh (smem table)",
                          "tanh (global table)", "__syncthreads (1 warp)", "q16 step (matvec + tanh)"};
  for (int i = 0; i < 8; ++i) printf("%-26s %lld cycles\n", names[i], cyc[i]);
  printf("cuda: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
