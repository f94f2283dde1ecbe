#include "nccl_dl.hpp"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <vector>

#include "lagom/error.hpp"

namespace lagom::b200 {

namespace {

template <typename F>
void bind(void* h, F& fn, const char* name) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  if (!fn) throw Error(ErrorCode::IoFailure, "nccl", std::string("missing symbol ") + name);
}

NcclApi load() {
  std::vector<std::string> candidates;
  if (const char* env = std::getenv("LAGOM_NCCL_LIB")) candidates.emplace_back(env);
  candidates.emplace_back("libnccl.so.2");  // already loaded (torch) or on the loader path
  candidates.emplace_back("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2");
  candidates.emplace_back("/usr/lib/x86_64-linux-gnu/libnccl.so.2");
  void* h = nullptr;
  NcclApi api;
  for (const auto& c : candidates) {
    // Prefer a copy that is already resident in the process.
    h = dlopen(c.c_str(), RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen(c.c_str(), RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.path = c;
      break;
    }
  }
  if (!h) throw Error(ErrorCode::IoFailure, "nccl", "libnccl.so.2 not found (set LAGOM_NCCL_LIB)");
  bind(h, api.GetUniqueId, "ncclGetUniqueId");
  bind(h, api.CommInitRank, "ncclCommInitRank");
  bind(h, api.CommDestroy, "ncclCommDestroy");
  bind(h, api.AllReduce, "ncclAllReduce");
  bind(h, api.AllGather, "ncclAllGather");
  bind(h, api.ReduceScatter, "ncclReduceScatter");
  bind(h, api.Send, "ncclSend");
  bind(h, api.Recv, "ncclRecv");
  bind(h, api.GroupStart, "ncclGroupStart");
  bind(h, api.GroupEnd, "ncclGroupEnd");
  bind(h, api.GetErrorString, "ncclGetErrorString");
  bind(h, api.GetVersion, "ncclGetVersion");
  return api;
}

}  // namespace

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  static std::string error;
  std::call_once(once, [] {
    try {
      api = load();
    } catch (const Error& e) {
      error = e.what();
    }
  });
  if (!api.GetUniqueId) throw Error(ErrorCode::IoFailure, "nccl", error);
  return api;
}

}  // namespace lagom::b200
