// Can a collective's CTAs run on the SMs that already host cuBLASLt GEMM
// CTAs, instead of on SMs carved out of the GEMM (the SM partition)?
//
// One GPU. Stream g runs R back-to-back bf16 GEMMs (the bench's shapes, the
// cuBLASLt heuristic's first algorithm); stream c (high priority) runs K
// back-to-back 25 MiB copies with a low-footprint LSU kernel (no shared
// memory, register-capped) or the copy engine. Reports, per copy config:
// copy GB/s alone and under the GEMMs, GEMM ms alone and under the copies,
// and how long each copy's first CTA waited after its launch event (a copy
// whose CTAs cannot co-reside waits for a GEMM to drain).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/coresident_probe \
//        tools/coresident_probe.cu -lcublasLt
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1); } } while (0)
#define LK(x) do { cublasStatus_t st_ = (x); if (st_ != CUBLAS_STATUS_SUCCESS) { printf("%s: %d\n", #x, (int)st_); exit(1); } } while (0)

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// first-CTA start per launch (atomicMin), last-CTA end (atomicMax)
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) lsu_copy(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                      size_t n16, unsigned long long* span) {
  if (threadIdx.x == 0) atomicMin(span, (unsigned long long)gtime());
  constexpr int U = 4;
  const size_t stride = (size_t)gridDim.x * NT;
  size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n16; i += stride) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(span + 1, (unsigned long long)gtime());
}

struct Gemm {
  int m, n, k;
  cublasLtMatmulDesc_t desc;
  cublasLtMatrixLayout_t a, b, d;
  cublasLtMatmulAlgo_t algo;
  void *A, *B, *D;
};

static cublasLtHandle_t lt;
static void* ws;
static size_t ws_bytes = 64 << 20;

Gemm make_gemm(int m, int n, int k) {
  Gemm g{m, n, k};
  LK(cublasLtMatmulDescCreate(&g.desc, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  LK(cublasLtMatmulDescSetAttribute(g.desc, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof ta));
  LK(cublasLtMatmulDescSetAttribute(g.desc, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof tb));
  LK(cublasLtMatrixLayoutCreate(&g.a, CUDA_R_16BF, k, m, k));
  LK(cublasLtMatrixLayoutCreate(&g.b, CUDA_R_16BF, k, n, k));
  LK(cublasLtMatrixLayoutCreate(&g.d, CUDA_R_16BF, m, n, m));
  cublasLtMatmulPreference_t pref;
  LK(cublasLtMatmulPreferenceCreate(&pref));
  LK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes, sizeof ws_bytes));
  cublasLtMatmulHeuristicResult_t res{};
  int found = 0;
  LK(cublasLtMatmulAlgoGetHeuristic(lt, g.desc, g.a, g.b, g.d, g.d, pref, 1, &res, &found));
  g.algo = res.algo;
  CK(cudaMalloc(&g.A, (size_t)m * k * 2));
  CK(cudaMalloc(&g.B, (size_t)n * k * 2));
  CK(cudaMalloc(&g.D, (size_t)m * n * 2));
  CK(cudaMemset(g.A, 0x3c, (size_t)m * k * 2));
  CK(cudaMemset(g.B, 0x3c, (size_t)n * k * 2));
  return g;
}

void run_gemm(Gemm& g, cudaStream_t s) {
  const float alpha = 1.f, beta = 0.f;
  LK(cublasLtMatmul(lt, g.desc, &alpha, g.A, g.a, g.B, g.b, &beta, g.D, g.d, g.D, g.d, &g.algo, ws, ws_bytes, s));
}

using CopyFn = void (*)(const uint4*, uint4*, size_t, unsigned long long*);
struct CopyCfg {
  const char* name;
  const void* fn;
  int nt;
  int grid;  // 0 = copy engine
};

int main(int argc, char** argv) {
  const int R = 30, K = 24;
  const size_t bytes = 25ull << 20;
  CK(cudaSetDevice(0));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  LK(cublasLtCreate(&lt));
  CK(cudaMalloc(&ws, ws_bytes));
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cudaStream_t sg, sc;
  CK(cudaStreamCreateWithPriority(&sg, cudaStreamNonBlocking, lo));
  CK(cudaStreamCreateWithPriority(&sc, cudaStreamNonBlocking, hi));
  std::vector<Gemm> gemms = {make_gemm(8192, 8192, 2048), make_gemm(2048, 8192, 8192),
                             make_gemm(8192, 2048, 8192), make_gemm(8192, 6144, 2048)};
  uint4 *src, *dst;
  CK(cudaMalloc(&src, bytes * K));
  CK(cudaMalloc(&dst, bytes * K));
  CK(cudaMemset(src, 1, bytes * K));
  unsigned long long* spans;
  CK(cudaMalloc(&spans, 2 * K * sizeof(unsigned long long)));
  std::vector<unsigned long long> hs(2 * K);
  cudaEvent_t g0, g1, cb[K], ce[K];
  CK(cudaEventCreate(&g0));
  CK(cudaEventCreate(&g1));
  for (int i = 0; i < K; ++i) {
    CK(cudaEventCreate(&cb[i]));
    CK(cudaEventCreate(&ce[i]));
  }
  // the copy kernels' per-SM footprint
  std::vector<CopyCfg> cfgs;
  auto add = [&](const char* nm, const void* fn, int nt) {
    for (int grid : {8, 16, 37, 74, 148, 296}) cfgs.push_back({nm, fn, nt, grid});
  };
  add("lsu64_r32", (const void*)lsu_copy<64, 32>, 64);
  add("lsu128_r32", (const void*)lsu_copy<128, 16>, 128);
  add("lsu256_r32", (const void*)lsu_copy<256, 8>, 256);
  add("lsu512_r64", (const void*)lsu_copy<512, 2>, 512);
  cfgs.push_back({"copy_engine", nullptr, 0, 0});
  for (auto& c : cfgs)
    if (c.fn) {
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, c.fn));
      if (c.grid == 8) printf("# %s regs=%d smem=%zu\n", c.name, fa.numRegs, fa.sharedSizeBytes);
    }
  auto launch_copy = [&](const CopyCfg& c, int i) {
    const uint4* s = src + (bytes / 16) * i;
    uint4* d = dst + (bytes / 16) * i;
    if (!c.fn) {
      CK(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, sc));
      return;
    }
    size_t n16 = bytes / 16;
    unsigned long long* sp = spans + 2 * i;
    void* args[] = {&s, &d, &n16, &sp};
    CK(cudaLaunchKernel(c.fn, dim3(c.grid), dim3(c.nt), args, 0, sc));
  };
  auto gemm_loop = [&](int reps) {
    for (int r = 0; r < reps; ++r) run_gemm(gemms[r % gemms.size()], sg);
  };
  auto ms = [](cudaEvent_t a, cudaEvent_t b) {
    float t;
    CK(cudaEventElapsedTime(&t, a, b));
    return (double)t;
  };
  // warm-up
  gemm_loop(8);
  CK(cudaDeviceSynchronize());
  // GEMM alone
  double g_alone = 1e30;
  for (int t = 0; t < 3; ++t) {
    CK(cudaEventRecord(g0, sg));
    gemm_loop(R);
    CK(cudaEventRecord(g1, sg));
    CK(cudaStreamSynchronize(sg));
    g_alone = std::min(g_alone, ms(g0, g1));
  }
  double flops = 0;
  for (int r = 0; r < R; ++r) {
    Gemm& g = gemms[r % gemms.size()];
    flops += 2.0 * g.m * g.n * g.k;
  }
  printf("{\"what\": \"gemm_alone\", \"ms\": %.3f, \"tflops\": %.1f, \"sms\": %d}\n", g_alone,
         flops / (g_alone * 1e-3) / 1e12, sms);
  for (const CopyCfg& c : cfgs) {
    // copy alone: median per-copy time
    std::vector<double> alone;
    for (int i = 0; i < K; ++i) {
      CK(cudaEventRecord(cb[i], sc));
      launch_copy(c, i);
      CK(cudaEventRecord(ce[i], sc));
    }
    CK(cudaStreamSynchronize(sc));
    for (int i = 0; i < K; ++i) alone.push_back(ms(cb[i], ce[i]));
    std::sort(alone.begin(), alone.end());
    // overlapped: copies issued while the GEMM loop runs; spans record the
    // kernel's active window so queueing behind GEMM CTAs is visible
    CK(cudaMemset(spans, 0xff, 2 * K * sizeof(unsigned long long)));
    for (int i = 0; i < K; ++i) CK(cudaMemset(spans + 2 * i + 1, 0, sizeof(unsigned long long)));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(g0, sg));
    gemm_loop(R);
    CK(cudaEventRecord(g1, sg));
    CK(cudaStreamWaitEvent(sc, g0, 0));
    for (int i = 0; i < K; ++i) {
      CK(cudaEventRecord(cb[i], sc));
      launch_copy(c, i);
      CK(cudaEventRecord(ce[i], sc));
    }
    CK(cudaDeviceSynchronize());
    std::vector<double> over, active;
    CK(cudaMemcpy(hs.data(), spans, hs.size() * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < K; ++i) {
      over.push_back(ms(cb[i], ce[i]));
      if (c.fn) active.push_back((hs[2 * i + 1] - hs[2 * i]) * 1e-6);
    }
    const double g_over = ms(g0, g1);
    const double copies_end = ms(g0, ce[K - 1]);
    std::sort(over.begin(), over.end());
    std::sort(active.begin(), active.end());
    const double med = over[K / 2];
    printf("{\"what\": \"copy\", \"cfg\": \"%s\", \"grid\": %d, \"nt\": %d, \"alone_us\": %.1f, "
           "\"alone_gbs\": %.0f, \"over_us_med\": %.1f, \"over_us_max\": %.1f, \"over_active_us_med\": %.1f, "
           "\"over_gbs\": %.0f, \"gemm_ms_over\": %.3f, \"gemm_slowdown\": %.4f, \"copies_done_ms\": %.3f}\n",
           c.name, c.grid, c.nt, alone[K / 2] * 1e3, 2.0 * bytes / (alone[K / 2] * 1e-3) / 1e9, med * 1e3,
           over[K - 1] * 1e3, active.empty() ? 0.0 : active[K / 2] * 1e3, 2.0 * bytes / (med * 1e-3) / 1e9, g_over,
           g_over / g_alone, copies_end);
    fflush(stdout);
  }
  return 0;
}
