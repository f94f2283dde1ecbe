// Cost model: the collective-kernel model (x and V, reference commperf.cpp)
// and the victim-side wave model (paper Eq. 4-6, reference contention.cpp).
//
// Bit-parity note: every expression below keeps the reference's operand order
// and association (e.g. ((alpha + zeta*NC) + chunks*c_over) + m/bw), and the
// library is built with -ffp-contract=off so no FMA can change a rounding.
#include <algorithm>
#include <cmath>

#include "lagom/commperf.hpp"
#include "lagom/contention.hpp"
#include "lagom/error.hpp"

namespace lagom {

// ------------------------------------------------------------ subspaces ----

std::string to_string(const SubspaceKey& key) {
  std::string s = to_string(key.algorithm);
  s.push_back('/');
  s += to_string(key.protocol);
  s.push_back('/');
  s += to_string(key.transport);
  return s;
}

SubspaceKey subspace_key_from_string(const std::string& s) {
  const std::size_t a = s.find('/');
  const std::size_t b = a == std::string::npos ? a : s.find('/', a + 1);
  if (b == std::string::npos)
    throw Error(ErrorCode::InvalidInput, "subspace",
                "expected 'ALGO/PROTO/TRANSPORT', got '" + s + "'");
  SubspaceKey key;
  key.algorithm = algorithm_from_string(s.substr(0, a));
  key.protocol = protocol_from_string(s.substr(a + 1, b - a - 1));
  key.transport = transport_from_string(s.substr(b + 1));
  return key;
}

SubspaceKey subspace_key(const CommConfig& cfg) {
  return {cfg.algorithm, cfg.protocol, cfg.transport};
}

void SubspaceParams::set(const SubspaceKey& key, const SubspaceCoeffs& coeffs) {
  table_.insert_or_assign(key, coeffs);
}

bool SubspaceParams::contains(const SubspaceKey& key) const {
  return table_.find(key) != table_.end();
}

const SubspaceCoeffs& SubspaceParams::at(const SubspaceKey& key) const {
  const auto it = table_.find(key);
  if (it != table_.end()) return it->second;
  throw Error(ErrorCode::UnknownSubspace, "subspace",
              "no coefficients for '" + to_string(key) + "'");
}

std::vector<SubspaceKey> SubspaceParams::keys() const {
  std::vector<SubspaceKey> ks;
  ks.reserve(table_.size());
  for (const auto& entry : table_) ks.push_back(entry.first);
  return ks;
}

double SubspaceParams::collective_factor(Collective c) const {
  const auto it = factors_.find(c);
  return it != factors_.end() ? it->second : 1.0;
}

void SubspaceParams::set_collective_factor(Collective c, double factor) {
  factors_.insert_or_assign(c, factor);
}

// The shipped synthetic table (reference commperf.cpp:67-106,
// data/default_params.json): ring vs tree base, scaled per protocol, then
// per transport. The multiply/add order matches the reference exactly.
SubspaceParams SubspaceParams::defaults() {
  struct ProtoAdj { double lat_scale, bw_scale, mem_coeff; bool set_mem; };
  struct TransAdj { double lat_add, bw_scale; bool scale; };
  static constexpr ProtoAdj kProto[] = {
      {1.0, 1.0, 0.5, false}, {0.4, 0.72, 0.35, true}, {0.6, 0.92, 0.45, true}};
  static constexpr TransAdj kTrans[] = {
      {0.0, 1.0, false}, {2.0, 0.8, true}, {10.0, 0.6, true}};

  SubspaceParams out;
  for (int a = 0; a < 2; ++a) {
    for (int p = 0; p < 3; ++p) {
      for (int t = 0; t < 3; ++t) {
        SubspaceCoeffs c;
        c.base_latency = a == 0 ? 15.0 : 10.0;
        c.per_channel_bw = a == 0 ? 25.0 : 22.0;
        if (kProto[p].set_mem) {
          c.base_latency *= kProto[p].lat_scale;
          c.per_channel_bw *= kProto[p].bw_scale;
          c.mem_coeff = kProto[p].mem_coeff;
        }
        if (kTrans[t].scale) {
          c.base_latency += kTrans[t].lat_add;
          c.per_channel_bw *= kTrans[t].bw_scale;
        }
        out.set({static_cast<Algorithm>(a), static_cast<Protocol>(p),
                 static_cast<Transport>(t)},
                c);
      }
    }
  }
  return out;
}

// ---------------------------------------------------------- comm model -----

double thread_efficiency(int num_threads, double nt_floor) {
  const double headroom = 1.0 - nt_floor;
  return nt_floor + headroom * static_cast<double>(num_threads) / 640.0;
}

double comm_time(const CommOp& op, const CommConfig& cfg, const GpuSpec& gpu,
                 const SubspaceParams& params) {
  const SubspaceCoeffs& k = params.at(subspace_key(cfg));
  const double bytes = static_cast<double>(op.message_bytes) *
                       params.collective_factor(op.collective);
  const double channels = static_cast<double>(cfg.num_channels);
  const double pipeline_steps =
      std::ceil(bytes / (channels * static_cast<double>(cfg.chunk_size)));
  const double channel_bw = channels * k.per_channel_bw *
                            thread_efficiency(cfg.num_threads, k.nt_floor);
  const double bw = std::min(channel_bw, gpu.link_bw);
  double x = k.base_latency + k.per_channel_setup * channels;
  x = x + pipeline_steps * k.per_chunk_overhead;
  return x + bytes / bw;
}

double mem_footprint(const CommConfig& cfg, const GpuSpec& gpu,
                     const SubspaceParams& params) {
  const SubspaceCoeffs& k = params.at(subspace_key(cfg));
  const double c = static_cast<double>(cfg.chunk_size);
  const double fill = c / (c + static_cast<double>(k.chunk_knee));
  const double demand =
      k.mem_coeff * static_cast<double>(cfg.num_channels) * fill * k.per_channel_bw;
  return std::min(gpu.comm_bw_cap_fraction * gpu.peak_mem_bw, demand);
}

// ------------------------------------------------------- victim model -----

namespace {

inline int held_sms(const std::optional<ActiveComm>& a) {
  return a.has_value() ? a->num_channels : 0;
}
inline double held_bw(const std::optional<ActiveComm>& a) {
  return a.has_value() ? a->footprint : 0.0;
}

}  // namespace

std::int64_t wave_count(const ComputeOp& op, const std::optional<ActiveComm>& active,
                        const GpuSpec& gpu) {
  const int nc = held_sms(active);
  if (nc >= gpu.num_sms)
    throw Error(ErrorCode::SmExhaustion, op.id,
                "communication occupies all " + std::to_string(gpu.num_sms) + " SMs");
  const std::int64_t per_wave =
      static_cast<std::int64_t>(gpu.num_sms - nc) * op.blocks_per_sm;
  return (op.total_blocks + per_wave - 1) / per_wave;
}

double wave_time(const ComputeOp& op, std::int64_t blocks_in_wave,
                 const std::optional<ActiveComm>& active, const GpuSpec& gpu) {
  const double left = gpu.peak_mem_bw - held_bw(active);
  if (!(left > 0))
    throw Error(ErrorCode::BandwidthExhaustion, op.id,
                "communication footprint consumes the full memory bandwidth");
  const double moved =
      static_cast<double>(blocks_in_wave) * static_cast<double>(op.bytes_per_block);
  return op.base_wave_time + moved / left;
}

double comp_time_static(const ComputeOp& op, const GpuSpec& gpu,
                        std::span<const WaveShare> assignment) {
  if (assignment.empty()) return 0.0;
  double time = 0.0;
  std::int64_t covered = 0;
  std::int64_t final_capacity = 0;
  for (const WaveShare& s : assignment) {
    const int nc = held_sms(s.active);
    if (nc >= gpu.num_sms)
      throw Error(ErrorCode::SmExhaustion, op.id, "no SMs left for computation");
    const std::int64_t cap =
        static_cast<std::int64_t>(gpu.num_sms - nc) * op.blocks_per_sm;
    time += static_cast<double>(s.waves) * wave_time(op, cap, s.active, gpu);
    covered += s.waves * cap;
    if (s.waves > 0) final_capacity = cap;
  }
  const bool short_of_op = covered < op.total_blocks;
  const bool overshoot = covered - final_capacity >= op.total_blocks;
  if (short_of_op || overshoot)
    throw Error(ErrorCode::PartitionMismatch, op.id,
                "wave shares cover " + std::to_string(covered) +
                    " blocks for an op of " + std::to_string(op.total_blocks));
  return time;
}

}  // namespace lagom
