// Is one DMMA (mma.sync.m8n8k4.f64) bitwise a k-ascending chain of FMAs?  Compares every output
// of many random m8n8k4 products against three host-side hypotheses:
//   seq   : fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0, c))))
//   exact : the exact a.b + c rounded once (long double is not enough; uses two-sum/two-prod)
// If `seq` matches everywhere, a warp-level FMA path over k ascending is bitwise the DMMA path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_fma tools/dmma_fma_probe.cu && /tmp/dmma_fma
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include <cuda_runtime.h>

__global__ void dmma_kernel(const double* A, const double* B, const double* C, double* D, int n) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (w >= n) return;
  const double* a = A + w * 32;  // 8x4 row-major
  const double* b = B + w * 32;  // 4x8 (k, n) row-major
  const double* c = C + w * 64;  // 8x8
  double* d = D + w * 64;
  const int r = lane >> 2, q4 = lane & 3;
  double af = a[r * 4 + q4];
  double bf = b[q4 * 8 + r];
  double d0 = c[r * 8 + 2 * q4], d1 = c[r * 8 + 2 * q4 + 1];
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(af), "d"(bf));
  d[r * 8 + 2 * q4] = d0;
  d[r * 8 + 2 * q4 + 1] = d1;
}

__global__ void fma_kernel(const double* A, const double* B, const double* C, double* D, int n, int order) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * 64) return;
  const int w = t / 64, e = t % 64, i = e / 8, j = e % 8;
  const double* a = A + w * 32;
  const double* b = B + w * 32;
  double acc = C[w * 64 + e];
  if (order == 0) {
    for (int k = 0; k < 4; ++k) acc = fma(a[i * 4 + k], b[k * 8 + j], acc);
  } else if (order == 1) {
    for (int k = 3; k >= 0; --k) acc = fma(a[i * 4 + k], b[k * 8 + j], acc);
  } else {  // products summed pairwise then added to c
    const double p0 = __dmul_rn(a[i * 4 + 0], b[0 * 8 + j]);
    const double s01 = fma(a[i * 4 + 1], b[1 * 8 + j], p0);
    const double p2 = __dmul_rn(a[i * 4 + 2], b[2 * 8 + j]);
    const double s23 = fma(a[i * 4 + 3], b[3 * 8 + j], p2);
    acc = __dadd_rn(__dadd_rn(s01, s23), acc);
  }
  D[t] = acc;
}

int main() {
  const int n = 1 << 16;
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::uniform_int_distribution<int> ex(-30, 30);
  std::vector<double> A(n * 32), B(n * 32), C(n * 64);
  for (auto& x : A) x = std::ldexp(u(g), ex(g) / 3);
  for (auto& x : B) x = std::ldexp(u(g), ex(g) / 3);
  for (auto& x : C) x = std::ldexp(u(g), ex(g));
  double *dA, *dB, *dC, *dD, *dF;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8);
  cudaMalloc(&dD, C.size() * 8); cudaMalloc(&dF, C.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
  dmma_kernel<<<n / 4, 128>>>(dA, dB, dC, dD, n);
  std::vector<double> D(n * 64), F(n * 64);
  cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost);
  const char* names[3] = {"fma k ascending", "fma k descending", "pairwise"};
  for (int o = 0; o < 3; ++o) {
    fma_kernel<<<n * 64 / 256, 256>>>(dA, dB, dC, dF, n, o);
    cudaMemcpy(F.data(), dF, F.size() * 8, cudaMemcpyDeviceToHost);
    long mism = 0;
    for (size_t i = 0; i < D.size(); ++i) mism += D[i] != F[i];
    printf("%-18s mismatches %ld of %zu\n", names[o], mism, D.size());
  }
  // chains of 128 k4 steps (a q = 512 layer step): DMMA chain vs FMA chain k ascending
  printf("cuda: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
