// Experiment harness (not part of the library): cfg4 order segments (N = 30,
// D = 1, unranking mode, R in shared memory) through the shipped group
// kernel and the bordered one-thread-per-unit kernel (eval_hybrid.cu).
//   nvcc ... -I include scripts/exp_hyb.cu paper_2501_03381_b200/csrc/common.cu
#include "../paper_2501_03381_b200/csrc/eval_group.cu"
#include "../paper_2501_03381_b200/csrc/eval_k13_16.cu"
#include "../paper_2501_03381_b200/csrc/eval_hybrid.cu"

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <random>
#include <vector>

using namespace hoib;

static uint64_t binom_h(int n, int k) { return host_binom(n, k); }

int main(int argc, char **argv) {
  const int N = 30, D = 1;
  std::mt19937_64 rng(3);
  std::normal_distribution<double> nd;
  std::vector<double> A0(N * N), S(N * N), R(N * N);
  for (auto &v : A0) v = nd(rng);
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int q = 0; q < N; ++q) s += A0[i * N + q] * A0[j * N + q];
      S[i * N + j] = s;
    }
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) R[i * N + j] = i == j ? 1.0 : S[i * N + j] / std::sqrt(S[i * N + i] * S[j * N + j]);
  double *dR, *o1, *o2;
  int32_t *cnt;
  int64_t *co;
  cudaMalloc(&dR, N * N * 8);
  cudaMemcpy(dR, R.data(), N * N * 8, cudaMemcpyHostToDevice);
  const int64_t Bmax = (int64_t)binom_h(30, 15);
  cudaMalloc(&o1, 4 * Bmax * 8);
  cudaMalloc(&o2, 4 * Bmax * 8);
  cudaMalloc(&cnt, 4);
  cudaMalloc(&co, 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int k0 = argc > 1 ? atoi(argv[1]) : 17, k1 = argc > 2 ? atoi(argv[2]) : 22;
  for (int K = k0; K <= k1; ++K) {
    const int64_t B = (int64_t)binom_h(30, K);
    EvalArgs A{};
    A.src = dR; A.N = N; A.D = D; A.B = B; A.r0 = 0; A.plane = B;
    A.err_count = cnt; A.err_coords = co; A.err_cap = 64;
    auto timeit = [&](const char *name, auto fn) {
      for (int w = 0; w < 2; ++w) fn();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int w = 0; w < 3; ++w) fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 3;
      const double F = 2.0 * (K * K * K - K) / 3.0 + K * (K + 1.0);
      printf("K=%d %-6s %8.3f ms  %6.2f TF/s  %s\n", K, name, ms, B * F / (ms * 1e-3) / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    };
    timeit("base", [&] { A.out = o1; if (K <= 16) launch_eval_k13_16(A, K, 0); else launch_eval_group(A, K, 0); });
    cudaMemset(o2, 0, 4 * B * 8);
#ifdef HYB_VARIANTS
    if (K == 17) {
      timeit("kr10", [&] { A.out = o2; launch_hyb<17, 10, 128>(A, 0); });
      timeit("kr11", [&] { A.out = o2; launch_hyb<17, 11, 128>(A, 0); });
      timeit("kr12", [&] { A.out = o2; launch_hyb<17, 12, 128>(A, 0); });
      timeit("kr12x64", [&] { A.out = o2; launch_hyb<17, 12, 64>(A, 0); });
      timeit("kr11x64", [&] { A.out = o2; launch_hyb<17, 11, 64>(A, 0); });
      timeit("kr13x64", [&] { A.out = o2; launch_hyb<17, 13, 64>(A, 0); });
    } else if (K == 18) {
      timeit("kr12x64", [&] { A.out = o2; launch_hyb<18, 12, 64>(A, 0); });
      timeit("kr11", [&] { A.out = o2; launch_hyb<18, 11, 128>(A, 0); });
      timeit("kr12", [&] { A.out = o2; launch_hyb<18, 12, 128>(A, 0); });
    }
#endif
    timeit("hybrid", [&] { A.out = o2; launch_eval_hybrid(A, K, 0); });
    cudaDeviceSynchronize();
    std::vector<double> h1(4 * B), h2(4 * B);
    cudaMemcpy(h1.data(), o1, 4 * B * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), o2, 4 * B * 8, cudaMemcpyDeviceToHost);
    double worst = 0;
    int64_t nbad = 0;
    for (int64_t q = 0; q < 4 * B; ++q) {
      const double dlt = std::fabs(h1[q] - h2[q]) - 1e-9 * std::fabs(h1[q]);
      if (!(dlt <= 1e-11)) ++nbad;
      if (dlt > worst) worst = dlt;
    }
    printf("K=%d max(|a-b| - 1e-9|a|) = %.3e, rows over tolerance %lld\n", K, worst, (long long)nbad);
  }
  int c = 0;
  cudaMemcpy(&c, cnt, 4, cudaMemcpyDeviceToHost);
  printf("not-PD %d\n", c);
  return 0;
}
