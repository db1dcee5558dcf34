// DMMA (mma.sync.m8n8k4.f64) throughput vs independent accumulator chains per warp and warps
// per CTA (one CTA per SM, registers only).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_probe tools/dmma_probe.cu && /tmp/dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void probe(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double acc[C][2];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int C>
void run(int warps) {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096 / C * 8;
  probe<C><<<148, warps * 32>>>(out, iters);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(s);
  probe<C><<<148, warps * 32>>>(out, iters);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  const double dmma = 148.0 * warps * (double)iters * C;
  const double tflops = dmma * 512.0 / (ms * 1e-3) / 1e12;
  const double clk_per_dmma_smsp = (ms * 1e-3) * 1.965e9 / (dmma / 148.0 / 4.0);
  printf("chains/warp %2d warps/SM %2d (chains/SMSP %3d): %6.2f TF/s  %5.1f clk per DMMA per SMSP\n", C,
         warps, C * warps / 4, tflops, clk_per_dmma_smsp);
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    run<1>(w);
    run<2>(w);
    run<4>(w);
    run<8>(w);
    run<16>(w);
  }
  return 0;
}
