// Step-GEMM tile-shape probe on the c2 forward layer step (256 tasks x B 256 x q 512, E_PROP
// tanh epilogue): TF/s per tile configuration of lmg::step_gemm and a bitwise check against the
// production 32x32 tile (every configuration runs the same k-ascending DMMA chain per output).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -I<venv>/flashinfer/data/cutlass/include \
//        -o /tmp/tile_probe tools/tile_probe.cu && /tmp/tile_probe [tasks] [M] [N] [K]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2007_07336_b200/csrc/lmg_gemm.cuh"
#include "gemmx_experiment.cuh"
#include "cutlass_experiment.cuh"

using namespace lmg;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

template <class T, bool BKM = true, bool ASC = false>
float run(const StepArgs& a, int reps, const char* name, const double* ref, double* out_host, size_t nout) {
  using C = GemmCfg<T, true, BKM, ASC>;
  auto kern = step_gemm<T, true, BKM, ASC, 2, true>;
  if (C::SMEM > 227 * 1024) {
    printf("%-34s smem %zu too big\n", name, C::SMEM);
    return 0;
  }
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NTHREADS, C::SMEM));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  dim3 grid(a.N / T::BN, a.M / T::BM, a.ntasks);
  StepArgs al = a;
  al.pdl_late = 1;
  kern<<<grid, C::NTHREADS, C::SMEM>>>(al);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(s);
    kern<<<grid, C::NTHREADS, C::SMEM>>>(al);
    cudaEventRecord(e);
    CK(cudaEventSynchronize(e));
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * a.ntasks * (double)a.M * a.N * a.K;
  bool same = true;
  if (ref) {
    CK(cudaMemcpy(out_host, a.out, nout * 8, cudaMemcpyDeviceToHost));
    same = !memcmp(out_host, ref, nout * 8);
  }
  const double waves = (double)grid.x * grid.y * grid.z / (per_sm * 148.0);
  printf("%-34s %6.3f ms %6.2f TF/s  regs %3d  smem %6zu  CTAs/SM %d  waves %5.2f  %s\n", name, best,
         flops / (best * 1e-3) / 1e12, fa.numRegs, C::SMEM, per_sm, waves,
         ref ? (same ? "bitwise" : "DIFFERS") : "(reference)");
  return best;
}

template <bool DB>
float run_x(const StepArgs& a, int reps, const char* name, const double* ref, double* out_host, size_t nout) {
  using X = TileX;
  auto kern = step_gemm_x<DB>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)X::SMEM));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, X::NT, X::SMEM));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  dim3 grid(a.N / X::BN, a.M / X::BM, a.ntasks);
  StepArgs al = a;
  al.pdl_late = 1;
  kern<<<grid, X::NT, X::SMEM>>>(al);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(s);
    kern<<<grid, X::NT, X::SMEM>>>(al);
    cudaEventRecord(e);
    CK(cudaEventSynchronize(e));
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * a.ntasks * (double)a.M * a.N * a.K;
  bool same = true;
  if (ref) {
    CK(cudaMemcpy(out_host, a.out, nout * 8, cudaMemcpyDeviceToHost));
    same = !memcmp(out_host, ref, nout * 8);
  }
  const double waves = (double)grid.x * grid.y * grid.z / (per_sm * 148.0);
  printf("%-34s %6.3f ms %6.2f TF/s  regs %3d  smem %6zu  CTAs/SM %d  waves %5.2f  %s (spill-local %zu)\n", name, best,
         flops / (best * 1e-3) / 1e12, fa.numRegs, X::SMEM, per_sm, waves,
         ref ? (same ? "bitwise" : "DIFFERS") : "(reference)", fa.localSizeBytes);
  return best;
}

float run_c(const StepArgs& a, int reps, const char* name, const double* ref, double* out_host, size_t nout) {
  using CF = CutlassFwd;
  auto kern = step_gemm_cutlass;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CF::NT, CF::SMEM));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  dim3 grid(a.N / CF::BN, a.M / CF::BM, a.ntasks);
  StepArgs al = a;
  al.pdl_late = 1;
  kern<<<grid, CF::NT, CF::SMEM>>>(al);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(s);
    kern<<<grid, CF::NT, CF::SMEM>>>(al);
    cudaEventRecord(e);
    CK(cudaEventSynchronize(e));
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * a.ntasks * (double)a.M * a.N * a.K;
  bool same = true;
  if (ref) {
    CK(cudaMemcpy(out_host, a.out, nout * 8, cudaMemcpyDeviceToHost));
    same = !memcmp(out_host, ref, nout * 8);
  }
  const double waves = (double)grid.x * grid.y * grid.z / (per_sm * 148.0);
  printf("%-34s %6.3f ms %6.2f TF/s  regs %3d  smem %6zu  CTAs/SM %d  waves %5.2f  %s (spill-local %zu)\n", name, best,
         flops / (best * 1e-3) / 1e12, fa.numRegs, CF::SMEM, per_sm, waves,
         ref ? (same ? "bitwise" : "DIFFERS") : "(reference)", fa.localSizeBytes);
  return best;
}

int main(int argc, char** argv) {
  const int tasks = argc > 1 ? atoi(argv[1]) : 256;
  const int M = argc > 2 ? atoi(argv[2]) : 256;
  const int N = argc > 3 ? atoi(argv[3]) : 512;
  const int K = argc > 4 ? atoi(argv[4]) : 512;
  const size_t na = (size_t)tasks * M * K, nw = (size_t)tasks * N * K, nout = (size_t)tasks * M * N;
  std::vector<double> h(std::max(na, nw));
  uint64_t x = 88172645463325252ull;
  auto rnd = [&] {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    return (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  };
  double *A, *W, *bias, *S, *out;
  CK(cudaMalloc(&A, na * 8));
  CK(cudaMalloc(&W, nw * 8));
  CK(cudaMalloc(&bias, (size_t)tasks * N * 8));
  CK(cudaMalloc(&S, nout * 8));
  CK(cudaMalloc(&out, nout * 8));
  for (size_t i = 0; i < na; ++i) h[i] = rnd();
  CK(cudaMemcpy(A, h.data(), na * 8, cudaMemcpyHostToDevice));
  for (size_t i = 0; i < nw; ++i) h[i] = rnd() * 0.09;
  CK(cudaMemcpy(W, h.data(), nw * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(bias, h.data(), (size_t)tasks * N * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(S, 0, nout * 8));

  StepArgs a;
  memset(&a, 0, sizeof(a));
  a.M = M; a.N = N; a.K = K; a.ntasks = tasks;
  a.epi = E_PROP; a.act = LMG_ACT_TANH; a.h = 1.0 / 1024;
  a.A = A; a.A_ts = (int64_t)M * K; a.lda = K;
  a.Bm = W; a.B_ts = (int64_t)N * K; a.ldb = K;
  a.bias = bias; a.bias_ts = N;
  a.x = A; a.x_ts = (int64_t)M * K;  // M x K == M x N when K == N
  a.s = S; a.s_ts = (int64_t)M * N;
  a.out = out; a.out_ts = (int64_t)M * N; a.ldc = N;

  std::vector<double> ref(nout), tmp(nout);
  const int reps = 10;
  const int group = argc > 5 ? atoi(argv[5]) : 0;
  printf("tasks %d  M %d  N %d  K %d  group %d\n", tasks, M, N, K, group);
  if (group == 3) {  // big-warp-tile kernel vs the production forward tile
    run<Tile<32, 32, 16, 2, 2, 2>>(a, reps, "TFwd 32x32x16 2st (production)", nullptr, nullptr, 0);
    CK(cudaMemcpy(ref.data(), out, nout * 8, cudaMemcpyDeviceToHost));
    run_c(a, reps, "CUTLASS mainloop 64x128 + staged epi", ref.data(), tmp.data(), nout);
    run_x<true>(a, reps, "X 64x128 4w 32x64 3st DB", ref.data(), tmp.data(), nout);
    run_x<false>(a, reps, "X 64x128 4w 32x64 3st", ref.data(), tmp.data(), nout);
    a.act = LMG_ACT_IDENTITY;
    run<Tile<32, 32, 16, 2, 2, 2>>(a, reps, "identity TFwd", nullptr, nullptr, 0);
    CK(cudaMemcpy(ref.data(), out, nout * 8, cudaMemcpyDeviceToHost));
    run_c(a, reps, "identity CUTLASS mainloop", ref.data(), tmp.data(), nout);
    run_x<true>(a, reps, "identity X 64x128 DB", ref.data(), tmp.data(), nout);
    run_x<false>(a, reps, "identity X 64x128", ref.data(), tmp.data(), nout);
    a.act = LMG_ACT_TANH;
  }
  if (group == 0 || group == 1) {  // forward layout, E_PROP tanh
    run<Tile<32, 32, 16, 2, 2, 4>>(a, reps, "32x32x16 2x2w 4st (production)", nullptr, nullptr, 0);
    CK(cudaMemcpy(ref.data(), out, nout * 8, cudaMemcpyDeviceToHost));
    run<Tile<32, 32, 16, 2, 2, 3>>(a, reps, "32x32x16 2x2w 3st", ref.data(), tmp.data(), nout);
    run<Tile<32, 32, 16, 2, 2, 2>>(a, reps, "32x32x16 2x2w 2st", ref.data(), tmp.data(), nout);
    run<Tile<32, 32, 8, 2, 2, 4>>(a, reps, "32x32x8 2x2w 4st", ref.data(), tmp.data(), nout);
    run<Tile<32, 32, 8, 2, 2, 6>>(a, reps, "32x32x8 2x2w 6st", ref.data(), tmp.data(), nout);
    run<Tile<32, 32, 8, 2, 2, 2>>(a, reps, "32x32x8 2x2w 2st", ref.data(), tmp.data(), nout);
    run<Tile<32, 32, 8, 2, 2, 3>>(a, reps, "32x32x8 2x2w 3st", ref.data(), tmp.data(), nout);
    run<Tile<32, 64, 16, 2, 4, 2>>(a, reps, "32x64x16 2x4w 2st", ref.data(), tmp.data(), nout);
    run<Tile<32, 32, 32, 2, 2, 2>>(a, reps, "32x32x32 2x2w 2st", ref.data(), tmp.data(), nout);
    run<Tile<64, 128, 16, 2, 4, 3>>(a, reps, "64x128x16 2x4w 3st", ref.data(), tmp.data(), nout);
    run<Tile<64, 64, 16, 2, 2, 3>>(a, reps, "64x64x16 2x2w 3st", ref.data(), tmp.data(), nout);
    a.act = LMG_ACT_RELU;
    run<Tile<32, 32, 16, 2, 2, 4>>(a, reps, "relu 32x32x16 (production)", nullptr, nullptr, 0);
    a.act = LMG_ACT_IDENTITY;
    run<Tile<32, 32, 16, 2, 2, 4>>(a, reps, "identity 32x32x16 (production)", nullptr, nullptr, 0);
    run<Tile<32, 32, 16, 2, 2, 3>>(a, reps, "identity 32x32x16 3st", nullptr, nullptr, 0);
    run<Tile<32, 32, 16, 2, 2, 2>>(a, reps, "identity 32x32x16 2st", nullptr, nullptr, 0);
    run<Tile<64, 128, 16, 2, 4, 3>>(a, reps, "identity 64x128x16 2x4w 3st", nullptr, nullptr, 0);
    a.act = LMG_ACT_TANH;
  }
  if (group == 0 || group == 2) {  // adjoint layout: A = mu * D (K-major, scaled), B = W MN-major
    a.act = LMG_ACT_IDENTITY;
    a.Ds = S; a.Ds_ts = (int64_t)M * K;
    CK(cudaMemcpy(S, h.data(), std::min(nout, nw) * 8, cudaMemcpyHostToDevice));
    a.bias = nullptr; a.s = nullptr;
    run<Tile<32, 64, 16, 2, 4, 4>, false, true>(a, reps, "adj 32x64x16 2x4w 4st (TWide)", nullptr, nullptr, 0);
    CK(cudaMemcpy(ref.data(), out, nout * 8, cudaMemcpyDeviceToHost));
    run<Tile<32, 64, 16, 2, 4, 3>, false, true>(a, reps, "adj 32x64x16 2x4w 3st", ref.data(), tmp.data(), nout);
    run<Tile<32, 64, 16, 2, 4, 2>, false, true>(a, reps, "adj 32x64x16 2x4w 2st", ref.data(), tmp.data(), nout);
    run<Tile<32, 32, 16, 2, 2, 4>, false, true>(a, reps, "adj 32x32x16 2x2w 4st", ref.data(), tmp.data(), nout);
    run<Tile<32, 32, 16, 2, 2, 2>, false, true>(a, reps, "adj 32x32x16 2x2w 2st", ref.data(), tmp.data(), nout);
    run<TileR<32, 128, 16, 2, 4>, false, true>(a, reps, "adj RS 32x128x16 2x4w", ref.data(), tmp.data(), nout);
    // residual-compatible (canonical partials: BN 32, two 16-column warps)
    run<TileR<64, 32, 16, 2, 2>, false, true>(a, reps, "adj RS 64x32x16 2x2w", ref.data(), tmp.data(), nout);
    run<TileR<64, 32, 16, 4, 2>, false, true>(a, reps, "adj RS 64x32x16 4x2w", ref.data(), tmp.data(), nout);
    run<TileR<128, 32, 16, 4, 2>, false, true>(a, reps, "adj RS 128x32x16 4x2w", ref.data(), tmp.data(), nout);
    run<TileR<128, 32, 16, 8, 2>, false, true>(a, reps, "adj RS 128x32x16 8x2w", ref.data(), tmp.data(), nout);
    run<TileR<32, 64, 16, 2, 4>, false, true>(a, reps, "adj RS 32x64x16 2x4w", ref.data(), tmp.data(), nout);
    run<TileR<32, 32, 16, 2, 2>, false, true>(a, reps, "adj RS 32x32x16 2x2w", ref.data(), tmp.data(), nout);
    run<TileR<64, 128, 16, 2, 4>, false, true>(a, reps, "adj RS 64x128x16 2x4w", ref.data(), tmp.data(), nout);
    run<TileR<32, 128, 8, 2, 4>, false, true>(a, reps, "adj RS 32x128x8 2x4w", ref.data(), tmp.data(), nout);
    run<Tile<64, 128, 16, 2, 4, 3>, false, true>(a, reps, "adj 64x128x16 2x4w 3st", ref.data(), tmp.data(), nout);
    run<Tile<64, 128, 16, 2, 4, 2>, false, true>(a, reps, "adj 64x128x16 2x4w 2st", ref.data(), tmp.data(), nout);
    run<Tile<64, 64, 16, 2, 4, 2>, false, true>(a, reps, "adj 64x64x16 2x4w 2st", ref.data(), tmp.data(), nout);
    run<Tile<32, 128, 16, 2, 4, 2>, false, true>(a, reps, "adj 32x128x16 2x4w 2st", ref.data(), tmp.data(), nout);
    // without the act' scaling: what the scaling costs
    run<Tile<32, 64, 16, 2, 4, 4>, false, false>(a, reps, "adj-noscale 32x64x16 (TWide)", nullptr, nullptr, 0);
    run<Tile<32, 64, 16, 2, 4, 2>, false, false>(a, reps, "adj-noscale 32x64x16 2st", nullptr, nullptr, 0);
    run<Tile<64, 128, 16, 2, 4, 3>, false, false>(a, reps, "adj-noscale 64x128x16 2x4w 3st", nullptr, nullptr, 0);
  }
  return 0;
}
