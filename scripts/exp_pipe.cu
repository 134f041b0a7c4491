// Experiment harness (not part of the library): cfg5-shaped batched
// evaluation (N = 400, D = 16, order 10, 4M n-plets) through the shipped
// k_eval_pipe<10> and candidate variants, plus FP64 latency probes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     --expt-relaxed-constexpr -I include scripts/exp_pipe.cu \
//     paper_2501_03381_b200/csrc/common.cu -o exp_pipe && ./exp_pipe
#include "../paper_2501_03381_b200/csrc/eval_pipe.cu"

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace hoib {
namespace {

// V1: two units per thread, factorisations interleaved by the scheduler
template <int K>
__global__ void __launch_bounds__(kPipeThreads, 2) k_pipe2(const EvalArgs A) {
  constexpr int NE = K * (K - 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *st0 = reinterpret_cast<double *>(smem_raw) + threadIdx.x;
  double *st1 = st0 + NE * kPipeThreads;
  __shared__ double2 s_plog[256];
  const int tid = threadIdx.x;
  for (int x = tid; x < 256; x += kPipeThreads) s_plog[x] = c_plog[x];
  __syncthreads();
  const int D = A.D, N = A.N;
  const int64_t t0 = blockIdx.x * (int64_t)kPipeThreads + tid;
  const int64_t step = (int64_t)gridDim.x * kPipeThreads;
  const int d = (int)(t0 % D);
  const int64_t db = step / D;
  const double *Rd = A.src + d;
  const int rowN = N * D;
  auto issue = [&](int64_t b, double *stage) {
    if (b < A.B) {
      const int32_t *ix = A.idx + b * A.idx_stride;
      int col[K], row[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int v = __ldg(ix + i);
        col[i] = v * D;
        row[i] = v * rowN;
      }
#pragma unroll
      for (int i = 1; i < K; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j)
          cp_async8(stage + (TRI(i, j) - i) * kPipeThreads, Rd + (row[i] + col[j]));
    }
  };
  int64_t b = t0 / D;
  issue(b, st0);
  issue(b + db, st1);
  cp_async_commit();
  const int s_dummy[K] = {};
  const double cs_dummy[K] = {};
  for (; b < A.B; b += 2 * db) {
    cp_async_wait_all();
    double a0[K * (K + 1) / 2], a1[K * (K + 1) / 2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) {
        a0[TRI(i, j)] = st0[(TRI(i, j) - i) * kPipeThreads];
        a1[TRI(i, j)] = st1[(TRI(i, j) - i) * kPipeThreads];
      }
      a0[TRI(i, i)] = 1.0;
      a1[TRI(i, i)] = 1.0;
    }
    LogProd pd0, pd1;
    const bool ok0 = ldl_fast<K>(a0, pd0);
    const bool ok1 = ldl_fast<K>(a1, pd1);
    issue(b + 2 * db, st0);
    issue(b + 3 * db, st1);
    cp_async_commit();
    const LogProd pl0 = inv_diag_logprod<K>(a0);
    const LogProd pl1 = inv_diag_logprod<K>(a1);
    if (!ok0)
      eval_retry<K, true, false>(A, A.src, b, d, K);
    else
      finish_unit<K, true, false>(A, b, d, K, s_dummy, true, logprod_value(pd0, s_plog),
                                  logprod_value(pl0, s_plog), cs_dummy);
    if (b + db < A.B) {
      if (!ok1)
        eval_retry<K, true, false>(A, A.src, b + db, d, K);
      else
        finish_unit<K, true, false>(A, b + db, d, K, s_dummy, true, logprod_value(pd1, s_plog),
                                    logprod_value(pl1, s_plog), cs_dummy);
    }
  }
}

// V2: 16-byte gathers -- the 16 dataset threads of one n-plet load two
// datasets of one entry per cp.async (23 instead of 45 per thread)
template <int K>
__global__ void __launch_bounds__(kPipeThreads, 3) k_pipe16(const EvalArgs A) {
  constexpr int NE = K * (K - 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *stage = reinterpret_cast<double *>(smem_raw) + threadIdx.x;
  double *stage_grp = reinterpret_cast<double *>(smem_raw) + (threadIdx.x & ~15);
  __shared__ double2 s_plog[256];
  const int tid = threadIdx.x;
  for (int x = tid; x < 256; x += kPipeThreads) s_plog[x] = c_plog[x];
  __syncthreads();
  const int D = A.D, N = A.N;   // D == 16
  const int64_t t0 = blockIdx.x * (int64_t)kPipeThreads + tid;
  const int64_t step = (int64_t)gridDim.x * kPipeThreads;
  const int d = (int)(t0 % D);
  const int h = d >> 3, p2 = (d & 7) * 2;
  const int64_t db = step / D;
  const double *Rp = A.src + p2;
  const int rowN = N * D;
  auto issue = [&](int64_t b) {
    if (b < A.B) {
      const int32_t *ix = A.idx + b * A.idx_stride;
      int col[K], row[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int v = __ldg(ix + i);
        col[i] = v * D;
        row[i] = v * rowN;
      }
      // entry list in TRI order: e -> (i, j)
#pragma unroll
      for (int u = 0; 2 * u < NE; ++u) {
        int e0 = 2 * u, e1 = 2 * u + 1;
        // decode compile-time (i, j) of e0, e1
        int i0 = 1, j0 = 0, i1 = 1, j1 = 0;
        {
          int e = 0;
#pragma unroll
          for (int i = 1; i < K; ++i)
#pragma unroll
            for (int j = 0; j < i; ++j) {
              if (e == e0) { i0 = i; j0 = j; }
              if (e == e1) { i1 = i; j1 = j; }
              ++e;
            }
        }
        if (e1 >= NE && h) continue;
        const int off0 = row[i0] + col[j0];
        const int off1 = e1 < NE ? row[i1] + col[j1] : off0;
        const int off = h ? off1 : off0;
        const int e = h ? e1 : e0;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(stage_grp + e * kPipeThreads + p2))),
                     "l"(Rp + off)
                     : "memory");
      }
    }
    cp_async_commit();
  };
  int64_t b = t0 / D;
  issue(b);
  const int s_dummy[K] = {};
  const double cs_dummy[K] = {};
  for (; b < A.B; b += db) {
    cp_async_wait_all();
    __syncwarp();
    double a[K * (K + 1) / 2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) a[TRI(i, j)] = stage[(TRI(i, j) - i) * kPipeThreads];
      a[TRI(i, i)] = 1.0;
    }
    __syncwarp();
    LogProd pd;
    const bool ok = ldl_fast<K>(a, pd);
    issue(b + db);
    if (!ok) {
      eval_retry<K, true, false>(A, A.src, b, d, K);
      continue;
    }
    const LogProd pl = inv_diag_logprod<K>(a);
    finish_unit<K, true, false>(A, b, d, K, s_dummy, true, logprod_value(pd, s_plog),
                                logprod_value(pl, s_plog), cs_dummy);
  }
}


// V3: the shipped kernel + an L2 prefetch of the id row two units ahead and
// 8-byte id loads
template <int K, bool PF, bool V2>
__global__ void __launch_bounds__(kPipeThreads, 3) k_pipe_pf(const EvalArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *stage = reinterpret_cast<double *>(smem_raw) + threadIdx.x;
  __shared__ double2 s_plog[256];
  const int tid = threadIdx.x;
  for (int x = tid; x < 256; x += kPipeThreads) s_plog[x] = c_plog[x];
  __syncthreads();
  const int D = A.D, N = A.N;
  const int64_t t0 = blockIdx.x * (int64_t)kPipeThreads + tid;
  const int64_t step = (int64_t)gridDim.x * kPipeThreads;
  const int d = (int)(t0 % D);
  const int64_t db = step / D;
  const double *Rd = A.src + d;
  const int rowN = N * D;
  auto issue = [&](int64_t b) {
    if (b < A.B) {
      const int32_t *ix = A.idx + b * A.idx_stride;
      int col[K], row[K];
      if (V2 && (K % 2 == 0)) {
#pragma unroll
        for (int i = 0; i < K; i += 2) {
          const int2 v = __ldg(reinterpret_cast<const int2 *>(ix + i));
          col[i] = v.x * D; row[i] = v.x * rowN;
          col[i + 1] = v.y * D; row[i + 1] = v.y * rowN;
        }
      } else {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const int v = __ldg(ix + i);
          col[i] = v * D;
          row[i] = v * rowN;
        }
      }
#pragma unroll
      for (int i = 1; i < K; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j)
          cp_async8(stage + (TRI(i, j) - i) * kPipeThreads, Rd + (row[i] + col[j]));
    }
    if (PF && b + db < A.B && d == 0)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(A.idx + (b + db) * A.idx_stride));
    cp_async_commit();
  };
  int64_t b = t0 / D;
  issue(b);
  const int s_dummy[K] = {};
  const double cs_dummy[K] = {};
  for (; b < A.B; b += db) {
    cp_async_wait_all();
    double a[K * (K + 1) / 2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) a[TRI(i, j)] = stage[(TRI(i, j) - i) * kPipeThreads];
      a[TRI(i, i)] = 1.0;
    }
    LogProd pd;
    const bool ok = ldl_fast<K>(a, pd);
    issue(b + db);
    if (!ok) {
      eval_retry<K, true, false>(A, A.src, b, d, K);
      continue;
    }
    const LogProd pl = inv_diag_logprod<K>(a);
    finish_unit<K, true, false>(A, b, d, K, s_dummy, true, logprod_value(pd, s_plog),
                                logprod_value(pl, s_plog), cs_dummy);
  }
}


// V4: the shipped kernel with other CTA sizes / register caps
template <int K, int T, int MB>
__global__ void __launch_bounds__(T, MB) k_pipe_occ(const EvalArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *stage = reinterpret_cast<double *>(smem_raw) + threadIdx.x;
  __shared__ double2 s_plog[256];
  const int tid = threadIdx.x;
  for (int x = tid; x < 256; x += T) s_plog[x] = c_plog[x];
  __syncthreads();
  const int D = A.D, N = A.N;
  const int64_t t0 = blockIdx.x * (int64_t)T + tid;
  const int64_t step = (int64_t)gridDim.x * T;
  const int d = (int)(t0 % D);
  const int64_t db = step / D;
  const double *Rd = A.src + d;
  const int rowN = N * D;
  auto issue = [&](int64_t b) {
    if (b < A.B) {
      const int32_t *ix = A.idx + b * A.idx_stride;
      int col[K], row[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int v = __ldg(ix + i);
        col[i] = v * D;
        row[i] = v * rowN;
      }
#pragma unroll
      for (int i = 1; i < K; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j)
          cp_async8(stage + (TRI(i, j) - i) * T, Rd + (row[i] + col[j]));
    }
    cp_async_commit();
  };
  int64_t b = t0 / D;
  issue(b);
  const int s_dummy[K] = {};
  const double cs_dummy[K] = {};
  for (; b < A.B; b += db) {
    cp_async_wait_all();
    double a[K * (K + 1) / 2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) a[TRI(i, j)] = stage[(TRI(i, j) - i) * T];
      a[TRI(i, i)] = 1.0;
    }
    LogProd pd;
    const bool ok = ldl_fast<K>(a, pd);
    issue(b + db);
    if (!ok) {
      eval_retry<K, true, false>(A, A.src, b, d, K);
      continue;
    }
    const LogProd pl = inv_diag_logprod<K>(a);
    finish_unit<K, true, false>(A, b, d, K, s_dummy, true, logprod_value(pd, s_plog),
                                logprod_value(pl, s_plog), cs_dummy);
  }
}

__global__ void k_lat_dfma(double *out, long long *cyc, int n) {
  double x = out[0], y = 1.0000001, z = 1e-300;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fma(x, y, z);
  }
  long long t1 = clock64();
  out[1] = x;
  cyc[0] = t1 - t0;
}
__global__ void k_lat_rcp(double *out, long long *cyc, int n) {
  double x = out[0] + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
  }
  long long t1 = clock64();
  out[1] = x;
  cyc[0] = t1 - t0;
}

}  // namespace
}  // namespace hoib

using namespace hoib;

int main(int argc, char **argv) {
  const int N = 400, D = 16, K = 10;
  const int64_t B = argc > 1 ? atoll(argv[1]) : 4000000;
  // correlation stack (N, N, D): low-rank + diagonal, unit diagonal
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  std::vector<double> R((size_t)N * N * D);
  const int r = 40;
  std::vector<double> Am((size_t)N * r);
  for (int dd = 0; dd < D; ++dd) {
    for (auto &v : Am) v = nd(rng);
    std::vector<double> S((size_t)N * N);
    for (int i = 0; i < N; ++i)
      for (int j = 0; j <= i; ++j) {
        double s = 0;
        for (int q = 0; q < r; ++q) s += Am[i * r + q] * Am[j * r + q];
        if (i == j) s += 5.0;
        S[i * N + j] = S[j * N + i] = s;
      }
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j)
        R[((size_t)i * N + j) * D + dd] = i == j ? 1.0 : S[i * N + j] / sqrt(S[i * N + i] * S[j * N + j]);
  }
  std::vector<int32_t> idx((size_t)B * K);
  std::uniform_int_distribution<int> ud(0, N - 1);
  for (int64_t b = 0; b < B; ++b) {
    int s[K];
    for (int i = 0; i < K; ++i) {
      for (;;) {
        int v = ud(rng);
        bool dup = false;
        for (int j = 0; j < i; ++j) dup |= s[j] == v;
        if (!dup) { s[i] = v; break; }
      }
    }
    for (int i = 0; i < K; ++i) idx[b * K + i] = s[i];
  }
  double *dR, *dout, *dout2;
  int32_t *didx, *dcnt;
  int64_t *dco;
  cudaMalloc(&dR, R.size() * 8);
  cudaMalloc(&didx, idx.size() * 4);
  cudaMalloc(&dout, (size_t)4 * B * D * 8);
  cudaMalloc(&dout2, (size_t)4 * B * D * 8);
  cudaMalloc(&dcnt, 4);
  cudaMalloc(&dco, 1024);
  cudaMemcpy(dR, R.data(), R.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(didx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dcnt, 0, 4);
  EvalArgs A{};
  A.src = dR; A.N = N; A.D = D; A.idx = didx; A.idx_stride = K; A.B = B;
  A.out = dout; A.plane = B * D; A.err_count = dcnt; A.err_coords = dco; A.err_cap = 64;
  upload_binomials();
  upload_plog();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double flops = 770.0 * B * D;
  auto timeit = [&](const char *name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    const int it = 10;
    for (int w = 0; w < it; ++w) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= it;
    printf("%-10s %8.4f ms  %6.2f TF/s  err=%s\n", name, ms, flops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  };
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  constexpr int NE = 45;
  timeit("base", [&] { A.out = dout; launch_pipe<10>(A, 0); });
  {
    const int smem = 2 * NE * kPipeThreads * 8;
    cudaFuncSetAttribute(k_pipe2<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pipe2<10>, kPipeThreads, smem);
    printf("pipe2: %d CTAs/SM\n", per);
    timeit("pipe2", [&] {
      A.out = dout2;
      k_pipe2<10><<<sms * per, kPipeThreads, smem>>>(A);
    });
    cudaDeviceSynchronize();
    std::vector<double> h1((size_t)4 * B * D), h2((size_t)4 * B * D);
    cudaMemcpy(h1.data(), dout, h1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), dout2, h2.size() * 8, cudaMemcpyDeviceToHost);
    size_t nd2 = 0;
    for (size_t i = 0; i < h1.size(); ++i) nd2 += memcmp(&h1[i], &h2[i], 8) != 0;
    printf("pipe2 differing values: %zu\n", nd2);
  }
  {
    const int smem = NE * kPipeThreads * 8;
    cudaFuncSetAttribute(k_pipe16<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pipe16<10>, kPipeThreads, smem);
    printf("pipe16: %d CTAs/SM\n", per);
    cudaMemset(dout2, 0, (size_t)4 * B * D * 8);
    timeit("pipe16", [&] {
      A.out = dout2;
      k_pipe16<10><<<sms * per, kPipeThreads, smem>>>(A);
    });
    cudaDeviceSynchronize();
    std::vector<double> h1((size_t)4 * B * D), h2((size_t)4 * B * D);
    cudaMemcpy(h1.data(), dout, h1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), dout2, h2.size() * 8, cudaMemcpyDeviceToHost);
    size_t nd2 = 0;
    for (size_t i = 0; i < h1.size(); ++i) nd2 += memcmp(&h1[i], &h2[i], 8) != 0;
    printf("pipe16 differing values: %zu\n", nd2);
  }
  auto variant = [&](const char *name, auto kern, int smem, int T = kPipeThreads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, T, smem);
    cudaMemset(dout2, 0, (size_t)4 * B * D * 8);
    timeit(name, [&] {
      A.out = dout2;
      kern<<<sms * per, T, smem>>>(A);
    });
    cudaDeviceSynchronize();
    std::vector<double> h1((size_t)4 * B * D), h2((size_t)4 * B * D);
    cudaMemcpy(h1.data(), dout, h1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), dout2, h2.size() * 8, cudaMemcpyDeviceToHost);
    size_t nd2 = 0;
    for (size_t i = 0; i < h1.size(); ++i) nd2 += memcmp(&h1[i], &h2[i], 8) != 0;
    printf("   %s: %d CTAs/SM, differing values: %zu\n", name, per, nd2);
  };
  variant("pf", k_pipe_pf<10, true, false>, NE * kPipeThreads * 8);
  variant("v2", k_pipe_pf<10, false, true>, NE * kPipeThreads * 8);
  variant("pf+v2", k_pipe_pf<10, true, true>, NE * kPipeThreads * 8);
  variant("occ128x2", k_pipe_occ<10, 128, 2>, NE * 128 * 8, 128);
  variant("occ64x6", k_pipe_occ<10, 64, 6>, NE * 64 * 8, 64);
  variant("occ64x7", k_pipe_occ<10, 64, 7>, NE * 64 * 8, 64);
  variant("occ64x8", k_pipe_occ<10, 64, 8>, NE * 64 * 8, 64);
  variant("occ32x14", k_pipe_occ<10, 32, 14>, NE * 32 * 8, 32);
  timeit("base", [&] { A.out = dout; launch_pipe<10>(A, 0); });
  {
    long long *dc;
    cudaMalloc(&dc, 8);
    long long c = 0;
    k_lat_dfma<<<1, 1>>>(dout, dc, 1000);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", c / 16000.0);
    k_lat_rcp<<<1, 1>>>(dout, dc, 1000);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("RCP64H dependent latency: %.2f cycles\n", c / 16000.0);
  }
  int cnt = 0;
  cudaMemcpy(&cnt, dcnt, 4, cudaMemcpyDeviceToHost);
  printf("not-PD count %d\n", cnt);
  return 0;
}
