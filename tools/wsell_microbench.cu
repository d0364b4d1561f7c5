// wsell_microbench.cu -- the windowed SELL engine (csrc/wsell.cuh) in isolation on a
// binary CSR cache file (csr_cache.py; config 5 by default), for kernel-design
// iterations that do not need the 10-minute library build: only the four kernels
// below are compiled, against the layout libf3rg.so's DeviceMatrix builds.
//   S   fp16 SpMV            (GatherPlain<f16>, store f16)
//   R   plain Richardson     (GatherZ1 from fp32 v, fused m = 2 sweep, f16 out)
//   D   L3 spmv_dots, ND = 2 (fp16 A, fp16 z, fp32 w + 2 projections)
//   D32 L2 spmv_dots, ND = 4 (fp32 A, fp32 z, fp32 w + 4 projections)
// Prints mean microseconds per launch and an FNV hash of each output (variants must
// keep the hashes: every row sum is bit-exact by construction). Tuning tool.
//   nvcc -std=c++17 -O3 -lineinfo -fmad=false -gencode arch=compute_100a,code=sm_100a \
//        --expt-relaxed-constexpr -I paper_2505_20719_b200/csrc tools/wsell_microbench.cu \
//        -o build/wsell_microbench -L paper_2505_20719_b200/lib -lf3rg \
//        -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2505_20719_b200/lib'
//   build/wsell_microbench /tmp/f3rg_cache/config5_20000000.csr [reps]
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "engine.hpp"
#include "levels.cuh"
#include "richardson.cuh"
#include "spmv.cuh"

using namespace f3rg;

constexpr int IDXW = 16;

template <int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) kb_spmv(CsrDev A, TilesDev T, const void* x, void* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  GatherPlain<P16, P16> g{x};
  EpiStore<P16, P16> e{y};
  spmv_tiles<P16, P16, IDX>(A, T, g, e, smem);
}

template <int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) kb_rich(CsrDev A, TilesDev T, const void* v, void* out, float w0f,
                                                          float w1f) {
  extern __shared__ __align__(128) uint8_t smem[];
  RhsView<P32, P16> rhs{v, 1.0f, false, 0};
  const __half w0 = __float2half_rn(w0f), w1 = __float2half_rn(w1f);
  GatherZ1<P32, P16, P16> g{rhs, w0};
  EpiStep<P32, P16, P16, true> e{rhs, w0, w1, nullptr, out, {}, {}};
  spmv_tiles<P16, P16, IDX>(A, T, g, e, smem);
}

template <int PA, int PZ, int ND, int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) kb_dots(CsrDev A, TilesDev T, const void* z, void* V, uint64_t ld,
                                                          double* dots) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX)];
  constexpr int C = pmax(PA, P32);
  GatherPlain<PZ, C> g{z};
  EpiDots<C, P32, ND> e;
  e.w = static_cast<uint8_t*>(V) + (size_t)ND * ld * 4;
  e.V = V;
  e.ld = ld;
#pragma unroll
  for (int k = 0; k < ND; ++k) e.d[k] = 0.0f, e.sk[k] = 0.5f + 0.125f * k;
  spmv_tiles<PA, C, IDX>(A, T, g, e, smem);
  float dd[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) dd[k] = e.d[k];
  block_sum<P32, ND>(dd, scratch);
  if (threadIdx.x == 0)
    for (int k = 0; k < ND; ++k) dots[(size_t)blockIdx.x * 8 + k] = dd[k];
}

__global__ void k_fill16(__half* p, uint64_t n, uint32_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    p[i] = __float2half_rn((float)(h & 0xffff) / 65536.0f - 0.5f);
  }
}
__global__ void k_fill32(float* p, uint64_t n, uint32_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    p[i] = (float)(h & 0xffffff) / 16777216.0f - 0.5f;
  }
}

static uint64_t fnv(const void* d, size_t bytes) {
  const uint8_t* p = static_cast<const uint8_t*>(d);
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < bytes; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

template <class F>
static double time_us(int reps, F&& launch) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) launch();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) launch();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaGetLastError());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms * 1e3 / reps;
}

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/tmp/f3rg_cache/config5_20000000.csr";
  const int reps = argc > 2 ? std::atoi(argv[2]) : 10;
  const char* only = argc > 3 ? argv[3] : "SRDE";
  int fd = open(path, O_RDONLY);
  if (fd < 0) {
    std::perror(path);
    return 1;
  }
  struct stat st;
  fstat(fd, &st);
  const uint8_t* base = static_cast<const uint8_t*>(mmap(nullptr, st.st_size, PROT_READ, MAP_PRIVATE, fd, 0));
  uint64_t n, nnz;
  std::memcpy(&n, base + 8, 8);
  std::memcpy(&nnz, base + 16, 8);
  const uint32_t* rp = reinterpret_cast<const uint32_t*>(base + 24);
  const uint32_t* ci = rp + n + 1;
  const double* val = reinterpret_cast<const double*>(reinterpret_cast<const uint8_t*>(ci) + nnz * 4);
  const bool check = std::getenv("WS_CHECK") != nullptr;  // also run the row-tile engine and compare hashes
  setenv("F3RG_WSELL", "1", 1);
  DeviceMatrix M(n, rp, ci, val);
  std::printf("n %llu nnz %llu ws_entries %llu shape %d stream bytes f16 %.0f f32 %.0f\n", (unsigned long long)n,
              (unsigned long long)nnz, (unsigned long long)M.ws_entries(), M.shape(), M.stream_bytes(0), M.stream_bytes(1));
  DeviceMatrix* M0 = nullptr;
  if (check) {
    setenv("F3RG_WSELL", "0", 1);
    M0 = new DeviceMatrix(n, rp, ci, val);
    std::printf("reference engine: shape %d sorted %d d16 %d\n", M0->shape(), (int)M0->sorted_rows(), (int)M0->d16());
  }
  const CsrDev A = M.csr();
  const int G = (int)M.tiles(0).ws_G;

  __half *x16, *y16;
  float *v32, *V;
  double* dots;
  const uint64_t ld = (n + 7) & ~7ull;
  CK(cudaMalloc(&x16, n * 2 + 64));
  CK(cudaMalloc(&y16, n * 2 + 64));
  CK(cudaMalloc(&v32, n * 4 + 64));
  CK(cudaMalloc(&V, ld * 4 * 6));
  CK(cudaMalloc(&dots, (size_t)4096 * 8 * 8));
  k_fill16<<<1184, 256>>>(x16, n, 1);
  k_fill32<<<1184, 256>>>(v32, n, 2);
  k_fill32<<<1184, 256>>>(V, ld * 6, 3);
  CK(cudaDeviceSynchronize());
  constexpr int IR = 8;  // the row-tile engine's gather-bound shape, u32 columns
  constexpr int SR16 = TileCfg<P16, IR>::SMEM_BYTES, SR32 = TileCfg<P32, IR>::SMEM_BYTES;
  CK(cudaFuncSetAttribute(kb_spmv<IDXW>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmem));
  CK(cudaFuncSetAttribute(kb_rich<IDXW>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmem));
  CK(cudaFuncSetAttribute(kb_dots<P16, P16, 2, IDXW>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmem));
  CK(cudaFuncSetAttribute(kb_dots<P32, P32, 4, IDXW>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmem));
  CK(cudaFuncSetAttribute(kb_spmv<IR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SR16));
  CK(cudaFuncSetAttribute(kb_rich<IR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SR16));
  CK(cudaFuncSetAttribute(kb_dots<P16, P16, 2, IR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SR16));
  CK(cudaFuncSetAttribute(kb_dots<P32, P32, 4, IR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SR32));
  const int GR = 148 * 3;

  std::vector<uint8_t> host(n * 4);
  auto hash_of = [&](const void* dev, size_t bytes) {
    CK(cudaMemcpy(host.data(), dev, bytes, cudaMemcpyDeviceToHost));
    return (unsigned long long)fnv(host.data(), bytes);
  };
  auto report = [&](const char* name, double us, double bytes, unsigned long long h, unsigned long long href) {
    std::printf("%-22s %9.2f us  %7.1f GB/s streamed  hash %016llx %s\n", name, us, bytes / us * 1e-3, h,
                !check ? "" : h == href ? "== row tiles" : "MISMATCH vs row tiles");
  };
  const double nb16 = (double)M.stream_bytes(0), nb32 = (double)M.stream_bytes(1);
  if (std::strchr(only, 'S')) {
    unsigned long long href = 0;
    if (check) {
      const CsrDev A0 = M0->csr();
      const TilesDev T0 = M0->tiles(0);
      kb_spmv<IR><<<GR, 256, SR16>>>(A0, T0, x16, y16);
      href = hash_of(y16, n * 2);
      CK(cudaMemset(y16, 0xff, n * 2));
    }
    const TilesDev T = M.tiles(0);
    const double us = time_us(reps, [&] { kb_spmv<IDXW><<<G, kWsThreads, kWsSmem>>>(A, T, x16, y16); });
    report("S   fp16 spmv", us, nb16 + n * 4.0, hash_of(y16, n * 2), href);
  }
  if (std::strchr(only, 'R')) {
    unsigned long long href = 0;
    if (check) {
      const CsrDev A0 = M0->csr();
      const TilesDev T0 = M0->tiles(0);
      kb_rich<IR><<<GR, 256, SR16>>>(A0, T0, v32, y16, 0.4f, 0.3f);
      href = hash_of(y16, n * 2);
      CK(cudaMemset(y16, 0xff, n * 2));
    }
    const TilesDev T = M.tiles(0);
    const double us = time_us(reps, [&] { kb_rich<IDXW><<<G, kWsThreads, kWsSmem>>>(A, T, v32, y16, 0.4f, 0.3f); });
    report("R   richardson plain", us, nb16 + n * 10.0, hash_of(y16, n * 2), href);
  }
  if (std::strchr(only, 'D')) {
    unsigned long long href = 0;
    if (check) {
      const CsrDev A0 = M0->csr();
      const TilesDev T0 = M0->tiles(0);
      kb_dots<P16, P16, 2, IR><<<GR, 256, SR16>>>(A0, T0, x16, V, ld, dots);
      href = hash_of(V + 2 * ld, n * 4);
      CK(cudaMemset(V + 2 * ld, 0xff, n * 4));
    }
    const TilesDev T = M.tiles(0);
    const double us = time_us(reps, [&] { kb_dots<P16, P16, 2, IDXW><<<G, kWsThreads, kWsSmem>>>(A, T, x16, V, ld, dots); });
    report("D   L3 spmv_dots(2)", us, nb16 + n * 14.0, hash_of(V + 2 * ld, n * 4), href);
  }
  if (std::strchr(only, 'E')) {
    unsigned long long href = 0;
    if (check) {
      const CsrDev A0 = M0->csr();
      const TilesDev T0 = M0->tiles(1);
      kb_dots<P32, P32, 4, IR><<<GR, 256, SR32>>>(A0, T0, v32, V, ld, dots);
      href = hash_of(V + 4 * ld, n * 4);
      CK(cudaMemset(V + 4 * ld, 0xff, n * 4));
    }
    const TilesDev T = M.tiles(1);
    const double us = time_us(reps, [&] { kb_dots<P32, P32, 4, IDXW><<<G, kWsThreads, kWsSmem>>>(A, T, v32, V, ld, dots); });
    report("D32 L2 spmv_dots(4)", us, nb32 + n * 24.0, hash_of(V + 4 * ld, n * 4), href);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
