// PM sampling self-test on one GPU: a bf16 GEMM loop (cuBLASLt) under
// sampling, one sampler per metric set; prints per-set sample counts and the
// summed values. Build: see tools/gpu_session.sh (links liblagom_b200).
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <string>
#include <vector>

#include "lagom/b200.hpp"

int main(int argc, char** argv) {
  cudaSetDevice(0);
  cudaFree(nullptr);
  const int m = 8192, n = 8192, k = 8192;
  void *A, *B, *D, *ws;
  cudaMalloc(&A, (size_t)m * k * 2);
  cudaMalloc(&B, (size_t)n * k * 2);
  cudaMalloc(&D, (size_t)m * n * 2);
  size_t wsb = 64 << 20;
  cudaMalloc(&ws, wsb);
  cudaMemset(A, 0x3c, (size_t)m * k * 2);
  cudaMemset(B, 0x3c, (size_t)n * k * 2);
  cublasLtHandle_t lt;
  cublasLtCreate(&lt);
  cublasLtMatmulDesc_t desc;
  cublasLtMatmulDescCreate(&desc, CUBLAS_COMPUTE_32F, CUDA_R_32F);
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof ta);
  cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof tb);
  cublasLtMatrixLayout_t la, lb, ld;
  cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, k, m, k);
  cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, k, n, k);
  cublasLtMatrixLayoutCreate(&ld, CUDA_R_16BF, m, n, m);
  const float alpha = 1.f, beta = 0.f;
  auto gemms = [&](int r) {
    for (int i = 0; i < r; ++i)
      cublasLtMatmul(lt, desc, &alpha, A, la, B, lb, &beta, D, ld, D, ld, nullptr, ws, wsb, 0);
    cudaDeviceSynchronize();
  };
  gemms(3);
  std::vector<std::vector<std::string>> sets = {
      lagom::b200::default_pm_metrics(),
      {"dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg"},
      {"dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active_realtime.avg"},
      {"dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"},
      {"dram__bytes_read.sum", "dram__bytes_write.sum", "nvltx__bytes.sum", "nvlrx__bytes.sum"},
      {"sm__cycles_active.avg", "sm__cycles_elapsed.avg", "sm__pipe_tensor_cycles_active_realtime.avg"},
      {"dram__bytes_read.sum", "dram__bytes_write.sum", "nvltx__bytes.sum", "nvlrx__bytes.sum",
       "sm__cycles_active.avg", "sm__pipe_tensor_cycles_active_realtime.avg"},
      {"dram__bytes.sum", "nvltx__bytes.sum", "nvlrx__bytes.sum", "sm__cycles_active.avg",
       "sm__pipe_tensor_cycles_active_realtime.avg", "gpc__cycles_elapsed.max"}};
  for (int i = 1; i < argc; ++i) sets.push_back({argv[i]});
  for (auto& s : sets) {
    try {
      lagom::b200::PmSampler ps(0, s, 20000, 20000);
      ps.start();
      gemms(20);
      auto samples = ps.stop();
      std::vector<double> tot(s.size(), 0.0);
      int nonzero = 0;
      for (auto& x : samples) {
        for (size_t j = 0; j < s.size(); ++j) tot[j] += x.values[j];
        if (x.values[0] != 0) ++nonzero;
      }
      printf("[%zu] %-40s samples=%zu nonzero=%d", s.size(), s[0].c_str(), samples.size(), nonzero);
      for (double v : tot) printf(" sum=%.4g", v);
      if (!samples.empty()) printf(" t0=%llu t1=%llu", (unsigned long long)samples.front().start_ns,
                                   (unsigned long long)samples.back().end_ns);
      printf("\n");
    } catch (const std::exception& e) {
      printf("%-50s error: %s\n", s[0].c_str(), e.what());
    }
    fflush(stdout);
  }
}
