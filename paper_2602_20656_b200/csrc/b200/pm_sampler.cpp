// CUPTI PM sampling: hardware counters (DRAM bytes, NVLink bytes, SM and
// tensor-pipe activity, L2 traffic) sampled on a fixed GPU-time interval
// while the replay's kernels run concurrently. Unlike ncu there is no kernel
// replay and no serialisation, so it measures exactly what the contention
// model needs — how much HBM bandwidth a collective takes (the reference's
// mem_footprint V, commperf.cpp:127-135), how many HBM bytes a compute op
// moves per CTA (ComputeOp.bytes_per_block D, model.hpp:27-35) and how busy
// the SMs and tensor pipes are while a collective overlaps them — on every
// rank of a multi-GPU replay at once.
//
// libcupti is opened at run time (dlopen), so liblagom_b200.so loads on
// machines without it and ncu (which injects its own CUPTI) is unaffected
// unless sampling is switched on.
#include <cupti_pmsampling.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_target.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "lagom/b200.hpp"
#include "lagom/error.hpp"

namespace lagom::b200 {

namespace {

struct Cupti {
  void* so = nullptr;
#define LAGOM_CUPTI_FN(name) decltype(&::name) name = nullptr;
  LAGOM_CUPTI_FN(cuptiGetResultString)
  LAGOM_CUPTI_FN(cuptiProfilerInitialize)
  LAGOM_CUPTI_FN(cuptiDeviceGetChipName)
  LAGOM_CUPTI_FN(cuptiPmSamplingGetCounterAvailability)
  LAGOM_CUPTI_FN(cuptiProfilerHostInitialize)
  LAGOM_CUPTI_FN(cuptiProfilerHostDeinitialize)
  LAGOM_CUPTI_FN(cuptiProfilerHostConfigAddMetrics)
  LAGOM_CUPTI_FN(cuptiProfilerHostGetConfigImageSize)
  LAGOM_CUPTI_FN(cuptiProfilerHostGetConfigImage)
  LAGOM_CUPTI_FN(cuptiProfilerHostEvaluateToGpuValues)
  LAGOM_CUPTI_FN(cuptiPmSamplingEnable)
  LAGOM_CUPTI_FN(cuptiPmSamplingDisable)
  LAGOM_CUPTI_FN(cuptiPmSamplingSetConfig)
  LAGOM_CUPTI_FN(cuptiPmSamplingGetCounterDataSize)
  LAGOM_CUPTI_FN(cuptiPmSamplingCounterDataImageInitialize)
  LAGOM_CUPTI_FN(cuptiPmSamplingStart)
  LAGOM_CUPTI_FN(cuptiPmSamplingStop)
  LAGOM_CUPTI_FN(cuptiPmSamplingDecodeData)
  LAGOM_CUPTI_FN(cuptiPmSamplingGetCounterDataInfo)
  LAGOM_CUPTI_FN(cuptiPmSamplingCounterDataGetSampleInfo)
#undef LAGOM_CUPTI_FN
};

const Cupti& cupti() {
  static Cupti c;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libcupti.so", "libcupti.so.12", "/usr/local/cuda/lib64/libcupti.so"})
      if ((c.so = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
    if (!c.so) return;
#define LAGOM_CUPTI_SYM(name) c.name = reinterpret_cast<decltype(c.name)>(dlsym(c.so, #name));
    LAGOM_CUPTI_SYM(cuptiGetResultString)
    LAGOM_CUPTI_SYM(cuptiProfilerInitialize)
    LAGOM_CUPTI_SYM(cuptiDeviceGetChipName)
    LAGOM_CUPTI_SYM(cuptiPmSamplingGetCounterAvailability)
    LAGOM_CUPTI_SYM(cuptiProfilerHostInitialize)
    LAGOM_CUPTI_SYM(cuptiProfilerHostDeinitialize)
    LAGOM_CUPTI_SYM(cuptiProfilerHostConfigAddMetrics)
    LAGOM_CUPTI_SYM(cuptiProfilerHostGetConfigImageSize)
    LAGOM_CUPTI_SYM(cuptiProfilerHostGetConfigImage)
    LAGOM_CUPTI_SYM(cuptiProfilerHostEvaluateToGpuValues)
    LAGOM_CUPTI_SYM(cuptiPmSamplingEnable)
    LAGOM_CUPTI_SYM(cuptiPmSamplingDisable)
    LAGOM_CUPTI_SYM(cuptiPmSamplingSetConfig)
    LAGOM_CUPTI_SYM(cuptiPmSamplingGetCounterDataSize)
    LAGOM_CUPTI_SYM(cuptiPmSamplingCounterDataImageInitialize)
    LAGOM_CUPTI_SYM(cuptiPmSamplingStart)
    LAGOM_CUPTI_SYM(cuptiPmSamplingStop)
    LAGOM_CUPTI_SYM(cuptiPmSamplingDecodeData)
    LAGOM_CUPTI_SYM(cuptiPmSamplingGetCounterDataInfo)
    LAGOM_CUPTI_SYM(cuptiPmSamplingCounterDataGetSampleInfo)
#undef LAGOM_CUPTI_SYM
  });
  if (!c.so || !c.cuptiPmSamplingEnable || !c.cuptiProfilerHostInitialize)
    throw Error(ErrorCode::IoFailure, "cupti", "libcupti with the PM sampling API is not available");
  return c;
}

void check(CUptiResult r, const char* what) {
  if (r == CUPTI_SUCCESS) return;
  const char* s = nullptr;
  if (cupti().cuptiGetResultString) cupti().cuptiGetResultString(r, &s);
  throw Error(ErrorCode::IoFailure, "cupti", std::string(what) + ": " + (s ? s : std::to_string(r)));
}

}  // namespace

std::vector<std::string> default_pm_metrics() {
  return {"dram__bytes_read.sum",   "dram__bytes_write.sum",          "nvltx__bytes.sum",
          "nvlrx__bytes.sum",       "sm__cycles_active.avg",          "sm__cycles_elapsed.avg",
          "sm__pipe_tensor_cycles_active_realtime.avg", "lts__t_bytes.sum"};
}

struct PmSampler::Impl {
  int device = 0;
  std::vector<std::string> metrics;
  std::vector<const char*> names;
  std::uint64_t interval_ns = 20000;
  std::size_t max_samples = 20000;
  CUpti_Profiler_Host_Object* host = nullptr;
  CUpti_PmSampling_Object* pm = nullptr;
  std::vector<std::uint8_t> config, counter_data;
  bool running = false;

  Impl(int dev, std::vector<std::string> m, std::uint64_t interval, std::size_t max)
      : device(dev), metrics(std::move(m)), interval_ns(interval), max_samples(max) {
    const Cupti& C = cupti();
    for (const std::string& s : metrics) names.push_back(s.c_str());
    CUpti_Profiler_Initialize_Params ip{};
    ip.structSize = CUpti_Profiler_Initialize_Params_STRUCT_SIZE;
    check(C.cuptiProfilerInitialize(&ip), "cuptiProfilerInitialize");
    CUpti_Device_GetChipName_Params cn{};
    cn.structSize = CUpti_Device_GetChipName_Params_STRUCT_SIZE;
    cn.deviceIndex = static_cast<std::size_t>(device);
    check(C.cuptiDeviceGetChipName(&cn), "cuptiDeviceGetChipName");
    CUpti_PmSampling_GetCounterAvailability_Params ca{};
    ca.structSize = CUpti_PmSampling_GetCounterAvailability_Params_STRUCT_SIZE;
    ca.deviceIndex = static_cast<std::size_t>(device);
    check(C.cuptiPmSamplingGetCounterAvailability(&ca), "counter availability size");
    std::vector<std::uint8_t> avail(ca.counterAvailabilityImageSize);
    ca.pCounterAvailabilityImage = avail.data();
    check(C.cuptiPmSamplingGetCounterAvailability(&ca), "counter availability");
    CUpti_Profiler_Host_Initialize_Params hp{};
    hp.structSize = CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE;
    hp.profilerType = CUPTI_PROFILER_TYPE_PM_SAMPLING;
    hp.pChipName = cn.pChipName;
    hp.pCounterAvailabilityImage = avail.data();
    check(C.cuptiProfilerHostInitialize(&hp), "cuptiProfilerHostInitialize");
    host = hp.pHostObject;
    CUpti_Profiler_Host_ConfigAddMetrics_Params am{};
    am.structSize = CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE;
    am.pHostObject = host;
    am.ppMetricNames = names.data();
    am.numMetrics = names.size();
    check(C.cuptiProfilerHostConfigAddMetrics(&am), "add metrics");
    CUpti_Profiler_Host_GetConfigImageSize_Params cs{};
    cs.structSize = CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE;
    cs.pHostObject = host;
    check(C.cuptiProfilerHostGetConfigImageSize(&cs), "config image size");
    config.resize(cs.configImageSize);
    CUpti_Profiler_Host_GetConfigImage_Params ci{};
    ci.structSize = CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE;
    ci.pHostObject = host;
    ci.configImageSize = config.size();
    ci.pConfigImage = config.data();
    check(C.cuptiProfilerHostGetConfigImage(&ci), "config image");
    CUpti_PmSampling_Enable_Params en{};
    en.structSize = CUpti_PmSampling_Enable_Params_STRUCT_SIZE;
    en.deviceIndex = static_cast<std::size_t>(device);
    check(C.cuptiPmSamplingEnable(&en), "cuptiPmSamplingEnable");
    pm = en.pPmSamplingObject;
    CUpti_PmSampling_SetConfig_Params sc{};
    sc.structSize = CUpti_PmSampling_SetConfig_Params_STRUCT_SIZE;
    sc.pPmSamplingObject = pm;
    sc.configSize = config.size();
    sc.pConfig = config.data();
    sc.hardwareBufferSize = 512ull << 20;
    sc.samplingInterval = interval_ns;
    sc.triggerMode = CUPTI_PM_SAMPLING_TRIGGER_MODE_GPU_TIME_INTERVAL;
    sc.hwBufferAppendMode = CUPTI_PM_SAMPLING_HARDWARE_BUFFER_APPEND_MODE_KEEP_OLDEST;
    check(C.cuptiPmSamplingSetConfig(&sc), "cuptiPmSamplingSetConfig");
    CUpti_PmSampling_GetCounterDataSize_Params ds{};
    ds.structSize = CUpti_PmSampling_GetCounterDataSize_Params_STRUCT_SIZE;
    ds.pPmSamplingObject = pm;
    ds.pMetricNames = names.data();
    ds.numMetrics = names.size();
    ds.maxSamples = static_cast<std::uint32_t>(max_samples);
    check(C.cuptiPmSamplingGetCounterDataSize(&ds), "counter data size");
    counter_data.resize(ds.counterDataSize);
  }

  ~Impl() {
    const Cupti& C = cupti();
    if (running) {
      CUpti_PmSampling_Stop_Params sp{};
      sp.structSize = CUpti_PmSampling_Stop_Params_STRUCT_SIZE;
      sp.pPmSamplingObject = pm;
      C.cuptiPmSamplingStop(&sp);
    }
    if (pm) {
      CUpti_PmSampling_Disable_Params dp{};
      dp.structSize = CUpti_PmSampling_Disable_Params_STRUCT_SIZE;
      dp.pPmSamplingObject = pm;
      C.cuptiPmSamplingDisable(&dp);
    }
    if (host) {
      CUpti_Profiler_Host_Deinitialize_Params hd{};
      hd.structSize = CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE;
      hd.pHostObject = host;
      C.cuptiProfilerHostDeinitialize(&hd);
    }
  }

  void start() {
    const Cupti& C = cupti();
    if (running) throw Error(ErrorCode::InvalidInput, "pm_sampler", "already started");
    CUpti_PmSampling_CounterDataImage_Initialize_Params ii{};
    ii.structSize = CUpti_PmSampling_CounterDataImage_Initialize_Params_STRUCT_SIZE;
    ii.pPmSamplingObject = pm;
    ii.counterDataSize = counter_data.size();
    ii.pCounterData = counter_data.data();
    check(C.cuptiPmSamplingCounterDataImageInitialize(&ii), "counter data init");
    CUpti_PmSampling_Start_Params sp{};
    sp.structSize = CUpti_PmSampling_Start_Params_STRUCT_SIZE;
    sp.pPmSamplingObject = pm;
    check(C.cuptiPmSamplingStart(&sp), "cuptiPmSamplingStart");
    running = true;
  }

  std::vector<PmSample> stop() {
    const Cupti& C = cupti();
    if (!running) throw Error(ErrorCode::InvalidInput, "pm_sampler", "not started");
    CUpti_PmSampling_Stop_Params sp{};
    sp.structSize = CUpti_PmSampling_Stop_Params_STRUCT_SIZE;
    sp.pPmSamplingObject = pm;
    check(C.cuptiPmSamplingStop(&sp), "cuptiPmSamplingStop");
    running = false;
    for (int guard = 0; guard < 1024; ++guard) {  // drain the hardware buffer
      CUpti_PmSampling_DecodeData_Params dd{};
      dd.structSize = CUpti_PmSampling_DecodeData_Params_STRUCT_SIZE;
      dd.pPmSamplingObject = pm;
      dd.pCounterDataImage = counter_data.data();
      dd.counterDataImageSize = counter_data.size();
      check(C.cuptiPmSamplingDecodeData(&dd), "cuptiPmSamplingDecodeData");
      if (dd.overflow) throw Error(ErrorCode::IoFailure, "pm_sampler", "hardware buffer overflow");
      if (dd.decodeStopReason != CUPTI_PM_SAMPLING_DECODE_STOP_REASON_OTHER) break;
    }
    CUpti_PmSampling_GetCounterDataInfo_Params gi{};
    gi.structSize = CUpti_PmSampling_GetCounterDataInfo_Params_STRUCT_SIZE;
    gi.pCounterDataImage = counter_data.data();
    gi.counterDataImageSize = counter_data.size();
    check(C.cuptiPmSamplingGetCounterDataInfo(&gi), "counter data info");
    std::vector<PmSample> out;
    out.reserve(gi.numCompletedSamples);
    std::vector<double> vals(names.size());
    for (std::size_t i = 0; i < gi.numCompletedSamples; ++i) {
      CUpti_PmSampling_CounterData_GetSampleInfo_Params si{};
      si.structSize = CUpti_PmSampling_CounterData_GetSampleInfo_Params_STRUCT_SIZE;
      si.pPmSamplingObject = pm;
      si.pCounterDataImage = counter_data.data();
      si.counterDataImageSize = counter_data.size();
      si.sampleIndex = i;
      check(C.cuptiPmSamplingCounterDataGetSampleInfo(&si), "sample info");
      CUpti_Profiler_Host_EvaluateToGpuValues_Params ev{};
      ev.structSize = CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE;
      ev.pHostObject = host;
      ev.pCounterDataImage = counter_data.data();
      ev.counterDataImageSize = counter_data.size();
      ev.rangeIndex = i;
      ev.ppMetricNames = names.data();
      ev.numMetrics = names.size();
      ev.pMetricValues = vals.data();
      check(C.cuptiProfilerHostEvaluateToGpuValues(&ev), "evaluate sample");
      out.push_back(PmSample{si.startTimestamp, si.endTimestamp, vals});
    }
    return out;
  }
};

PmSampler::PmSampler(int device, std::vector<std::string> metrics, std::uint64_t interval_ns,
                     std::size_t max_samples)
    : impl_(std::make_unique<Impl>(device, metrics.empty() ? default_pm_metrics() : std::move(metrics),
                                   interval_ns, max_samples)) {}
PmSampler::~PmSampler() = default;
const std::vector<std::string>& PmSampler::metrics() const { return impl_->metrics; }
void PmSampler::start() { impl_->start(); }
std::vector<PmSample> PmSampler::stop() { return impl_->stop(); }

}  // namespace lagom::b200
