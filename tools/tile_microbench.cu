// tile_microbench.cu -- isolates the pieces of the TMA-tiled SpMV on the config-2
// pattern (27-point 128^3, fp16 values): (a) tile streaming only (gather returns a
// constant), (b) + gathers of an fp16 vector, (c) + gathers of an fp32 vector,
// (d) a plain coalesced read of the same bytes. Tuning tool, not product code.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//        -I paper_2505_20719_b200/csrc tools/tile_microbench.cu -o build/tile_microbench
#include <cstdio>
#include <vector>

#include "spmv.cuh"
#include "levels.cuh"
#include "richardson.cuh"

using namespace f3rg;

template <int C>
struct GatherConst {
  using Raw = __half;
  __device__ __forceinline__ Raw load(uint32_t) const { return __float2half(1.0f); }
  __device__ __forceinline__ T_<C> value(Raw r) const { return cvt<C>(r); }
};

template <int C, int PY>
struct EpiSink {
  void* y;
  __device__ __forceinline__ void prefetch(uint32_t) {}
  __device__ __forceinline__ void row(uint32_t i, T_<C> acc) { st<PY>(y, i, cvt<PY>(acc)); }
};

template <int MODE, int IDX = 0>
__global__ void __launch_bounds__(256, F3RG_TILE_MINB) k_bench(CsrDev A, TilesDev T, const void* x, void* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  if constexpr (MODE == 0) {
    GatherConst<P32> g;
    EpiSink<P32, P32> e{y};
    spmv_tiles<P16, P32, IDX>(A, T, g, e, smem);
  } else if constexpr (MODE == 1) {
    GatherPlain<P16, P32> g{x};
    EpiSink<P32, P32> e{y};
    spmv_tiles<P16, P32, IDX>(A, T, g, e, smem);
  } else {
    GatherPlain<P32, P32> g{x};
    EpiSink<P32, P32> e{y};
    spmv_tiles<P16, P32, IDX>(A, T, g, e, smem);
  }
}

// epilogue variant with a compile-time projection count
template <int C, int PW, int ND>
struct EpiDotsT {
  void* w;
  void* V;
  uint64_t n;
  T_<PW> sk[ND], d[ND], vk[ND];
  __device__ __forceinline__ void prefetch(uint32_t i) {
#pragma unroll
    for (int k = 0; k < ND; ++k) vk[k] = ld<PW>(V, (uint64_t)k * n + i);
  }
  __device__ __forceinline__ void row(uint32_t i, T_<C> acc) {
    const T_<PW> wi = cvt<PW>(acc);
#pragma unroll
    for (int k = 0; k < ND; ++k) d[k] = Ar<PW>::add(d[k], Ar<PW>::mul(wi, Ar<PW>::mul(sk[k], vk[k])));
    st<PW>(w, i, wi);
  }
};

template <int ND>
__global__ void __launch_bounds__(256, 2) k_dotsT(CsrDev A, TilesDev T, const void* z, void* V, uint64_t n,
                                                  double* dots) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[64];
  GatherPlain<P16, P32> g{z};
  EpiDotsT<P32, P32, ND> e;
  e.w = static_cast<float*>(V) + 5 * n;
  e.V = V;
  e.n = n;
#pragma unroll
  for (int k = 0; k < ND; ++k) e.d[k] = 0.f, e.sk[k] = 1.0f;
  spmv_tiles<P16, P32, 0>(A, T, g, e, smem);
  float dd[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) dd[k] = e.d[k];
  block_sum<P32, ND>(dd, scratch);
  if (threadIdx.x == 0)
    for (int k = 0; k < ND; ++k) dots[(size_t)blockIdx.x * 16 + k] = dd[k];
}

__global__ void k_read(const uint4* p, size_t n16, uint4* out) {
  uint4 acc = {0, 0, 0, 0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(p + i);
    acc.x ^= v.x, acc.y ^= v.y, acc.z ^= v.z, acc.w ^= v.w;
  }
  if (acc.x == 0x12345678u) out[0] = acc;
}

int main() {
  const int N = 128, n = N * N * N;
  std::vector<uint32_t> rp(n + 1, 0), ci;
  ci.reserve((size_t)n * 27);
  for (int z = 0; z < N; ++z)
    for (int y = 0; y < N; ++y)
      for (int x = 0; x < N; ++x) {
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              const int xx = x + dx, yy = y + dy, zz = z + dz;
              if (xx < 0 || yy < 0 || zz < 0 || xx >= N || yy >= N || zz >= N) continue;
              ci.push_back((uint32_t)(xx + N * (yy + N * zz)));
            }
        rp[(size_t)(x + N * (y + N * z)) + 1] = (uint32_t)ci.size();
      }
  const size_t nnz = ci.size();
  std::vector<uint16_t> dc(nnz + 16, 0);
  std::vector<uint32_t> fc(n + 16, 0);
  for (int i = 0; i < n; ++i) {
    fc[i] = ci[rp[i]];
    for (uint32_t k = rp[i] + 1; k < rp[i + 1]; ++k) dc[k] = (uint16_t)(ci[k] - ci[k - 1]);
  }
  std::vector<uint32_t> r0, k0;
  for (uint32_t i = 0; i < (uint32_t)n;) {
    r0.push_back(i);
    k0.push_back(rp[i]);
    uint32_t j = i;
    while (j < (uint32_t)n && j - i < 256 && rp[j + 1] - rp[i] <= (uint32_t)TileCfg<P16>::TNNZ) ++j;
    i = j;
  }
  r0.push_back(n);
  k0.push_back(rp[n]);
  uint32_t *d_rp, *d_ci, *d_r0, *d_k0;
  __half* d_val;
  float *d_x, *d_y;
  cudaMalloc(&d_rp, (n + 16) * 4);
  cudaMalloc(&d_ci, (nnz + 16) * 4);
  cudaMalloc(&d_val, (nnz + 16) * 2);
  cudaMalloc(&d_x, (size_t)n * 4 + 64);
  cudaMalloc(&d_y, (size_t)n * 4 + 64);
  cudaMalloc(&d_r0, r0.size() * 4);
  cudaMalloc(&d_k0, k0.size() * 4);
  cudaMemcpy(d_rp, rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemset(d_val, 0x3c, (nnz + 16) * 2);
  cudaMemset(d_x, 0, (size_t)n * 4);
  cudaMemcpy(d_r0, r0.data(), r0.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_k0, k0.data(), k0.size() * 4, cudaMemcpyHostToDevice);
  uint16_t* d_dc;
  uint32_t* d_fc;
  cudaMalloc(&d_dc, dc.size() * 2);
  cudaMalloc(&d_fc, fc.size() * 4);
  cudaMemcpy(d_dc, dc.data(), dc.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(d_fc, fc.data(), fc.size() * 4, cudaMemcpyHostToDevice);
  CsrDev A;
  A.n = n, A.nnz = nnz, A.rp = d_rp, A.ci = d_ci, A.val[0] = d_val;
  CsrDev A16 = A;
  A16.dcol = d_dc, A16.first = d_fc;
  TilesDev T{d_r0, d_k0, (uint32_t)(r0.size() - 1)};
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = TileCfg<P16>::SMEM_BYTES;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = nnz * 6.0 + 4.0 * (n + 1) + (double)n * 4;
  auto run = [&](auto kern, const char* name, double extra_bytes, int occ_req) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    const int grid = occ * sms;
    for (int w = 0; w < 3; ++w) kern<<<grid, 256, smem>>>(A, T, d_x, d_y);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) kern<<<grid, 256, smem>>>(A, T, d_x, d_y);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    printf("%-28s occ=%d grid=%d %8.1f us  %7.1f GB/s\n", name, occ, grid, ms * 1e3, (bytes + extra_bytes) / (ms * 1e-3) / 1e9);
    (void)occ_req;
  };
  run(k_bench<0>, "tiles only (const gather)", 0, 2);
  run(k_bench<1>, "tiles + f16 gather", n * 2.0, 2);
  run(k_bench<2>, "tiles + f32 gather", n * 4.0, 2);
  {
    const double b16 = nnz * 4.0 + 4.0 * (n + 1) + (double)n * 8;
    auto run16 = [&](auto kern, const char* name, double extra) {
      const int sm16 = TileCfg<P16, 1>::SMEM_BYTES;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm16);
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, sm16);
      const int grid = occ * sms;
      for (int w = 0; w < 3; ++w) kern<<<grid, 256, sm16>>>(A16, T, d_x, d_y);
      cudaEventRecord(e0);
      for (int it = 0; it < 20; ++it) kern<<<grid, 256, sm16>>>(A16, T, d_x, d_y);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 20;
      printf("%-28s occ=%d grid=%d %8.1f us  %7.1f GB/s\n", name, occ, grid, ms * 1e3, (b16 + extra) / (ms * 1e-3) / 1e9);
    };
    run16(k_bench<0, 1>, "D16 tiles only", 0);
    run16(k_bench<1, 1>, "D16 tiles + f16 gather", n * 2.0);
    run16(k_bench<2, 1>, "D16 tiles + f32 gather", n * 4.0);
  }
  {
    uint4* d_o;
    cudaMalloc(&d_o, 64);
    const size_t n16 = nnz * 4 / 16;  // the column array only (in bounds)
    for (int w = 0; w < 3; ++w) k_read<<<sms * 8, 256>>>((const uint4*)d_ci, n16, d_o);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) k_read<<<sms * 8, 256>>>((const uint4*)d_ci, n16, d_o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    printf("%-28s %8.1f us  %7.1f GB/s\n", "coalesced read (same bytes)", ms * 1e3, n16 * 16.0 / (ms * 1e-3) / 1e9);
  }
  // ---- product kernels on the same matrix ----
  {
    float* V;  // 5 basis vectors (fp32) + w
    __half* Z;
    cudaMalloc(&V, (size_t)n * 4 * 6 + 64);
    cudaMalloc(&Z, (size_t)n * 2 + 64);
    cudaMemset(V, 0, (size_t)n * 4 * 6);
    cudaMemset(Z, 0, (size_t)n * 2);
    double *H, *sc, *partials;
    int* dead;
    unsigned *counter, *bar;
    unsigned long long* cnt;
    LevelState hs{};
    cudaMalloc(&H, 4096 * 8);
    cudaMemset(H, 0, 4096 * 8);
    cudaMalloc(&partials, sms * 8 * 16 * 8 * 4);
    cudaMalloc(&dead, 64);
    cudaMemset(dead, 0, 64);
    cudaMalloc(&counter, 64);
    cudaMemset(counter, 0, 64);
    cudaMalloc(&bar, 64);
    cudaMemset(bar, 0, 64);
    cudaMalloc(&cnt, 64 * 8);
    hs.m = 8;
    hs.H = H, hs.cs = H + 100, hs.sn = H + 200, hs.g = H + 300, hs.y = H + 400, hs.scale = H + 500;
    LevelState* dL;
    cudaMalloc(&dL, sizeof hs);
    cudaMemcpy(dL, &hs, sizeof hs, cudaMemcpyHostToDevice);
    Gate gate{dead, 2};
    Sync sync{partials, counter};
    auto timeit = [&](const char* name, double b, auto&& launch) {
      for (int w = 0; w < 3; ++w) launch();
      cudaEventRecord(e0);
      for (int it = 0; it < 20; ++it) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 20;
      printf("%-28s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, b / (ms * 1e-3) / 1e9);
    };
    auto kd = k_spmv_dots<P16, P16, P32, 0>;
    cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int j = 0; j < 4; ++j) {
      char nm[64];
      snprintf(nm, sizeof nm, "spmv_dots[f16,f16,f32] j=%d", j);
      const double b = nnz * 6.0 + 4.0 * (n + 1) + n * (2.0 + 4.0 + 4.0 * (j + 1));
      timeit(nm, b, [&] { kd<<<2 * sms, 256, smem>>>(A, T, Z, V, n, j, dL, gate, sync, partials + 4096 * 4, 1); });
    }
    {
      auto t1 = k_dotsT<1>; auto t4 = k_dotsT<4>;
      cudaFuncSetAttribute(t1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(t4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      timeit("dotsT<1>", nnz * 6.0 + 4.0 * (n + 1) + n * 10.0, [&] { t1<<<2 * sms, 256, smem>>>(A, T, Z, V, n, partials + 4096 * 4); });
      timeit("dotsT<4>", nnz * 6.0 + 4.0 * (n + 1) + n * 22.0, [&] { t4<<<2 * sms, 256, smem>>>(A, T, Z, V, n, partials + 4096 * 4); });
    }
    // make the basis non-degenerate so k_cgs / k_richardson are not gated off
    {
      std::vector<float> ones((size_t)n * 5, 1.0f);
      cudaMemcpy(V, ones.data(), ones.size() * 4, cudaMemcpyHostToDevice);
    }
    auto kc = k_cgs<P32>;
    for (int j = 0; j < 4; ++j) {
      char nm[64];
      snprintf(nm, sizeof nm, "cgs[f32] j=%d", j);
      timeit(nm, n * 4.0 * (j + 3), [&] {
        cudaMemsetAsync(dead, 0, 64);
        kc<<<sms * 4, 256>>>(V, n, j, dL, dead, gate, 1, 0, 0, nullptr, sync, partials + 4096 * 4, 2 * sms);
      });
    }
    for (int g8 : {2, 4, 8}) {
      for (int deferred : {0, 1}) {
        char nm[64];
        snprintf(nm, sizeof nm, "cgs j=3 grid=%dxSM dots=%d", g8, deferred);
        timeit(nm, n * 4.0 * 6, [&] {
          cudaMemsetAsync(dead, 0, 64);
          kc<<<sms * g8, 256>>>(V, n, 3, dL, dead, gate, 1, 0, 0, nullptr, sync, deferred ? partials + 4096 * 4 : nullptr, 2 * sms);
        });
      }
    }
    // Richardson (non-update call: call_count 1, c = 64)
    double* om;
    int* wupd;
    unsigned long long* calls;
    cudaMalloc(&om, 64);
    cudaMalloc(&wupd, 64);
    cudaMalloc(&calls, 64);
    const double one[2] = {1.0, 1.0};
    cudaMemcpy(om, one, 16, cudaMemcpyHostToDevice);
    RichState rs{};
    rs.m = 2, rs.cycle = 1000000000ull, rs.omegas = om, rs.wused = om + 4, rs.wupd = wupd, rs.calls = calls;
    rs.R = V + (size_t)n * 5, rs.Za = V + (size_t)n * 5, rs.Zb = V + (size_t)n * 5;
    const unsigned long long c0[4] = {1, 0, 0, 0};
    cudaMemcpy(calls, c0, 32, cudaMemcpyHostToDevice);
    RichState* dR;
    cudaMalloc(&dR, sizeof rs);
    cudaMemcpy(dR, &rs, sizeof rs, cudaMemcpyHostToDevice);
    auto kr = k_richardson<P16, P16, P32, 0>;
    cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(dead, 0, 64);
    timeit("richardson[f16,f16,f32]", nnz * 6.0 + 4.0 * (n + 1) + n * 6.0, [&] {
      kr<<<2 * sms, 256, smem>>>(A, T, V, nullptr, Z, n, dR, gate, 2, cnt, sync, bar, bar + 1, nullptr);
    });
  }
  printf("tiles=%u nnz=%zu bytes/launch=%.0f err=%s\n", T.ntiles, nnz, bytes, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
