// Internal: cuDNN SDPA attention victims of the replay engine (attention.cpp).
#pragma once
#include <cstdint>
#include <memory>

#include "lagom/b200.hpp"

namespace lagom::b200 {

class Attention {
 public:
  // Builds the cuDNN graph and plan for one shape and allocates its tensors
  // (synthetic data filled on `stream`).
  Attention(const AttentionShape& shape, void* cudnn_handle, std::uint64_t seed, void* stream);
  ~Attention();
  Attention(const Attention&) = delete;
  Attention& operator=(const Attention&) = delete;
  // workspace the prepared graphs need (max over SM targets)
  std::int64_t workspace_bytes() const;
  const AttentionShape& shape() const;
  // builds the graph for `sm_target` SMs (0 = all) if not built yet
  void prepare(void* cudnn_handle, int sm_target);
  void launch(void* cudnn_handle, void* stream, void* workspace, int sm_target);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

void* create_cudnn_handle();
void destroy_cudnn_handle(void* handle);

}  // namespace lagom::b200
