// Attention victims of the replay: fused scaled-dot-product attention
// (flash-style, cuDNN's sm_100 SDPA engines through the cuDNN frontend graph
// API) — the training step's attention kernels the collectives contend
// against, next to the cuBLASLt GEMMs (victim workload, not the product).
// Layout: Q, K, V, O, dO, dQ, dK, dV bf16 [b, h, s, d] (d contiguous), the
// softmax statistics fp32 [b, h, s, 1]; fp32 softmax / accumulation.
#include "attention.hpp"

#include <cudnn.h>
#include <cudnn_frontend.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <unordered_map>

#include "lagom/error.hpp"
#include "lagom_coll.h"

namespace lagom::b200 {

namespace fe = cudnn_frontend;

namespace {

void fe_check(fe::error_t e, const char* what) {
  if (e.is_bad()) throw Error(ErrorCode::IoFailure, "cudnn", std::string(what) + ": " + e.get_message());
}
void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(ErrorCode::IoFailure, "cuda", std::string(what) + ": " + cudaGetErrorString(e));
}

enum Uid : int64_t { kQ = 1, kK, kV, kO, kStats, kdO, kdQ, kdK, kdV };

}  // namespace

struct Attention::Impl {
  AttentionShape shape;
  std::unordered_map<int, std::shared_ptr<fe::graph::Graph>> graphs;  // per SM count target (0 = all)
  std::unordered_map<int64_t, void*> ptrs;
  std::vector<void*> owned;
  int64_t workspace = 0;
  void build(cudnnHandle_t handle, int sm_target);
};

// One cuDNN graph and plan per SM count target: the replay's SM partition
// asks the attention victims for the GEMMs' SM budget too (the graph's
// sm_count knob, CUDNN_ATTR_ENGINE_SM_COUNT_TARGET) where an engine supports
// it.
void Attention::Impl::build(cudnnHandle_t handle, int sm_target) {
  const AttentionShape& s = shape;
  const int64_t b = s.batch, h = s.heads, n = s.seq, d = s.head_dim;
  const std::vector<int64_t> dim{b, h, n, d}, stride{h * n * d, n * d, d, 1};
  const std::vector<int64_t> sdim{b, h, n, 1}, sstride{h * n, n, 1, 1};
  auto g = std::make_shared<fe::graph::Graph>();
  g->set_io_data_type(fe::DataType_t::BFLOAT16)
      .set_intermediate_data_type(fe::DataType_t::FLOAT)
      .set_compute_data_type(fe::DataType_t::FLOAT);
  if (sm_target > 0) g->set_sm_count(sm_target);
  auto tensor = [&](const char* name, int64_t uid) {
    return g->tensor(fe::graph::Tensor_attributes().set_name(name).set_dim(dim).set_stride(stride).set_uid(uid));
  };
  auto Q = tensor("Q", kQ), K = tensor("K", kK), V = tensor("V", kV);
  const float scale = 1.0f / std::sqrt(static_cast<float>(d));
  if (!s.backward) {
    auto opt = fe::graph::SDPA_attributes().set_name("sdpa").set_generate_stats(true).set_causal_mask(s.causal)
                   .set_attn_scale(scale);
    auto [O, Stats] = g->sdpa(Q, K, V, opt);
    O->set_output(true).set_dim(dim).set_stride(stride).set_uid(kO);
    Stats->set_output(true).set_data_type(fe::DataType_t::FLOAT).set_dim(sdim).set_stride(sstride).set_uid(kStats);
  } else {
    auto O = tensor("O", kO), dO = tensor("dO", kdO);
    auto Stats = g->tensor(fe::graph::Tensor_attributes().set_name("Stats").set_dim(sdim).set_stride(sstride)
                               .set_data_type(fe::DataType_t::FLOAT).set_uid(kStats));
    auto opt = fe::graph::SDPA_backward_attributes().set_name("sdpa_bwd").set_causal_mask(s.causal)
                   .set_attn_scale(scale);
    auto [dQ, dK, dV] = g->sdpa_backward(Q, K, V, O, dO, Stats, opt);
    dQ->set_output(true).set_dim(dim).set_stride(stride).set_uid(kdQ);
    dK->set_output(true).set_dim(dim).set_stride(stride).set_uid(kdK);
    dV->set_output(true).set_dim(dim).set_stride(stride).set_uid(kdV);
  }
  fe_check(g->validate(), "validate");
  fe_check(g->build_operation_graph(handle), "build_operation_graph");
  fe_check(g->create_execution_plans({fe::HeurMode_t::A}), "create_execution_plans");
  fe_check(g->check_support(handle), "check_support");
  fe_check(g->build_plans(handle), "build_plans");
  int64_t ws = 0;
  fe_check(g->get_workspace_size(ws), "workspace size");
  workspace = std::max(workspace, ws);
  graphs[sm_target] = g;
}

Attention::Attention(const AttentionShape& s, void* cudnn_handle, std::uint64_t seed, void* stream)
    : impl_(std::make_unique<Impl>()) {
  Impl& I = *impl_;
  I.shape = s;
  const int64_t b = s.batch, h = s.heads, n = s.seq, d = s.head_dim;
  I.build(static_cast<cudnnHandle_t>(cudnn_handle), 0);
  // device tensors: bf16 operands filled with N-like synthetic data, fp32 stats
  const int64_t elems = b * h * n * d;
  auto alloc = [&](int64_t uid, int64_t bytes, bool fill, int dtype) {
    void* p = nullptr;
    cuda_ok(cudaMalloc(&p, static_cast<size_t>(bytes)), "attention buffer");
    I.owned.push_back(p);
    I.ptrs[uid] = p;
    if (fill && lagom_fill_random(p, bytes / (dtype == LAGOM_F32 ? 4 : 2), dtype, seed + static_cast<std::uint64_t>(uid),
                                  dtype == LAGOM_F32 ? 1.0f : 0.5f, stream) != LAGOM_OK)
      throw Error(ErrorCode::IoFailure, "attention", "fill failed");
  };
  for (int64_t uid : {kQ, kK, kV}) alloc(uid, elems * 2, true, LAGOM_BF16);
  alloc(kO, elems * 2, s.backward, LAGOM_BF16);
  alloc(kStats, b * h * n * 4, s.backward, LAGOM_F32);
  if (s.backward) {
    alloc(kdO, elems * 2, true, LAGOM_BF16);
    for (int64_t uid : {kdQ, kdK, kdV}) alloc(uid, elems * 2, false, LAGOM_BF16);
  }
}

Attention::~Attention() {
  if (!impl_) return;
  for (void* p : impl_->owned) cudaFree(p);
}

std::int64_t Attention::workspace_bytes() const { return impl_->workspace; }
const AttentionShape& Attention::shape() const { return impl_->shape; }

void Attention::prepare(void* cudnn_handle, int sm_target) {
  if (impl_->graphs.count(sm_target)) return;
  try {
    impl_->build(static_cast<cudnnHandle_t>(cudnn_handle), sm_target);
  } catch (const Error&) {
    // cuDNN 9.22's sm_100 SDPA engines reject SM carveouts ("SM carveout not
    // supported for this engine"): the attention then runs on every SM, and
    // the collectives' stream priority (replay.cpp) gets their CTAs the next
    // SM that frees up.
    impl_->graphs[sm_target] = impl_->graphs.at(0);
  }
}

void Attention::launch(void* cudnn_handle, void* stream, void* workspace, int sm_target) {
  auto* handle = static_cast<cudnnHandle_t>(cudnn_handle);
  if (cudnnSetStream(handle, static_cast<cudaStream_t>(stream)) != CUDNN_STATUS_SUCCESS)
    throw Error(ErrorCode::IoFailure, "cudnn", "cudnnSetStream failed");
  auto it = impl_->graphs.find(sm_target);
  if (it == impl_->graphs.end()) throw Error(ErrorCode::InvalidInput, "attention", "graph not prepared for the SM target");
  fe_check(it->second->execute(handle, impl_->ptrs, workspace), "sdpa execute");
}

void* create_cudnn_handle() {
  cudnnHandle_t h = nullptr;
  if (cudnnCreate(&h) != CUDNN_STATUS_SUCCESS) throw Error(ErrorCode::IoFailure, "cudnn", "cudnnCreate failed");
  return h;
}
void destroy_cudnn_handle(void* h) {
  if (h) cudnnDestroy(static_cast<cudnnHandle_t>(h));
}

}  // namespace lagom::b200
