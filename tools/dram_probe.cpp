// dram_probe.cpp — DRAM bytes of the kernels launched between begin() and end(), read from
// the GPU's counters with CUPTI's range profiler (CUDA 12.9), so bench.py can report the
// walk kernel's DRAM traffic measured in the same run (one extra, untimed launch) instead
// of a number from an earlier ncu capture.  Measurement infrastructure, not the product:
// the walk library never links it.
//
//   grape_dram_probe_begin()  -> 0 on success (profiling the current CUDA context)
//   ... launch the kernel(s) ...
//   grape_dram_probe_end(&read, &write, &ns) -> 0 on success: dram__bytes_read.sum and
//       dram__bytes_write.sum of one user range around the launches (single pass; ns: 0)
//   grape_probe_begin_set(1) / grape_probe_end_set(double out[4]) -> the same for the issue
//       counters (warp instructions, thread instructions, issue-active cycles, active cycles)
//   grape_dram_probe_error() -> the last failure as text
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>

namespace {

std::string g_err;
CUpti_RangeProfiler_Object* g_obj = nullptr;
CUpti_Profiler_Host_Object* g_host = nullptr;
std::vector<uint8_t> g_config, g_counter;
CUcontext g_ctx = nullptr;
bool g_inited = false;
// metric sets: 0 = the DRAM bytes; 1 = the issue counters (warp instructions, thread
// instructions, cycles with an instruction issued, active cycles — summed over the SM
// sub-partitions), for the issue-slot utilisation of an instruction-bound kernel
const char* kSet0[] = {"dram__bytes_read.sum", "dram__bytes_write.sum"};
const char* kSet1[] = {"smsp__inst_executed.sum", "smsp__thread_inst_executed.sum", "smsp__issue_active.sum",
                       "smsp__cycles_active.sum"};
const char** kMetrics = kSet0;
size_t kNumMetrics = 2;
constexpr size_t kMaxMetrics = 4;
constexpr size_t kMaxRanges = 64;

bool fail(const char* what, CUptiResult r)
{
    const char* s = nullptr;
    cuptiGetResultString(r, &s);
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, s ? s : "?");
    g_err = buf;
    return false;
}

#define TRY(call, what)                                     \
    do {                                                    \
        CUptiResult r_ = (call);                            \
        if (r_ != CUPTI_SUCCESS) return fail(what, r_) ? 0 : 1; \
    } while (0)

void cleanup()
{
    if (g_obj) {
        CUpti_RangeProfiler_Disable_Params p{CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
        p.pRangeProfilerObject = g_obj;
        cuptiRangeProfilerDisable(&p);
        g_obj = nullptr;
    }
    if (g_host) {
        CUpti_Profiler_Host_Deinitialize_Params p{CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
        p.pHostObject = g_host;
        cuptiProfilerHostDeinitialize(&p);
        g_host = nullptr;
    }
}

}  // namespace

extern "C" {

const char* grape_dram_probe_error(void) { return g_err.c_str(); }

// Initialise CUPTI's profiler early (before the process launches kernels); begin() does it
// otherwise.
int grape_dram_probe_init(void)
{
    if (g_inited) return 0;
    CUpti_Profiler_Initialize_Params p{CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
    CUptiResult r = cuptiProfilerInitialize(&p);
    if (r != CUPTI_SUCCESS) {
        fail("cuptiProfilerInitialize", r);
        return 1;
    }
    g_inited = true;
    return 0;
}

static int begin_impl(void);

int grape_probe_begin_set(int set)
{
    if (g_obj != nullptr) {
        g_err = "a probe is already running";
        return 1;
    }
    if (set == 1) { kMetrics = kSet1; kNumMetrics = 4; }
    else { kMetrics = kSet0; kNumMetrics = 2; }
    const int rc = begin_impl();
    if (rc != 0) cleanup();
    return rc;
}

int grape_dram_probe_begin(void)
{
    kMetrics = kSet0;
    kNumMetrics = 2;
    const int rc = begin_impl();
    if (rc != 0) cleanup();
    return rc;
}

static int begin_impl(void)
{
    g_err.clear();
    if (cuCtxGetCurrent(&g_ctx) != CUDA_SUCCESS || g_ctx == nullptr) {
        g_err = "no current CUDA context";
        return 1;
    }
    if (!g_inited) {
        CUpti_Profiler_Initialize_Params p{CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
        TRY(cuptiProfilerInitialize(&p), "cuptiProfilerInitialize");
        g_inited = true;
    }
    CUdevice dev;
    if (cuCtxGetDevice(&dev) != CUDA_SUCCESS) {
        g_err = "cuCtxGetDevice";
        return 1;
    }
    // host side: the chip, the counters this context can read, the metrics' configuration
    CUpti_Device_GetChipName_Params chip{CUpti_Device_GetChipName_Params_STRUCT_SIZE};
    chip.deviceIndex = (size_t)dev;
    TRY(cuptiDeviceGetChipName(&chip), "cuptiDeviceGetChipName");
    CUpti_Profiler_GetCounterAvailability_Params av{CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
    av.ctx = g_ctx;
    TRY(cuptiProfilerGetCounterAvailability(&av), "cuptiProfilerGetCounterAvailability (size)");
    std::vector<uint8_t> avail(av.counterAvailabilityImageSize);
    av.pCounterAvailabilityImage = avail.data();
    TRY(cuptiProfilerGetCounterAvailability(&av), "cuptiProfilerGetCounterAvailability");
    CUpti_Profiler_Host_Initialize_Params hi{CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
    hi.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
    hi.pChipName = chip.pChipName;
    hi.pCounterAvailabilityImage = avail.data();
    TRY(cuptiProfilerHostInitialize(&hi), "cuptiProfilerHostInitialize");
    g_host = hi.pHostObject;
    CUpti_Profiler_Host_ConfigAddMetrics_Params am{CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
    am.pHostObject = g_host;
    am.ppMetricNames = kMetrics;
    am.numMetrics = kNumMetrics;
    TRY(cuptiProfilerHostConfigAddMetrics(&am), "cuptiProfilerHostConfigAddMetrics");
    CUpti_Profiler_Host_GetConfigImageSize_Params cs{CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
    cs.pHostObject = g_host;
    TRY(cuptiProfilerHostGetConfigImageSize(&cs), "cuptiProfilerHostGetConfigImageSize");
    g_config.assign(cs.configImageSize, 0);
    CUpti_Profiler_Host_GetConfigImage_Params ci{CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
    ci.pHostObject = g_host;
    ci.pConfigImage = g_config.data();
    ci.configImageSize = g_config.size();
    TRY(cuptiProfilerHostGetConfigImage(&ci), "cuptiProfilerHostGetConfigImage");
    // target side: enable on this context, the counter-data image, kernel replay of auto ranges
    CUpti_RangeProfiler_Enable_Params en{CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
    en.ctx = g_ctx;
    TRY(cuptiRangeProfilerEnable(&en), "cuptiRangeProfilerEnable");
    g_obj = en.pRangeProfilerObject;
    CUpti_RangeProfiler_GetCounterDataSize_Params ds{CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
    ds.pRangeProfilerObject = g_obj;
    ds.pMetricNames = kMetrics;
    ds.numMetrics = kNumMetrics;
    ds.maxNumOfRanges = kMaxRanges;
    ds.maxNumRangeTreeNodes = kMaxRanges;
    TRY(cuptiRangeProfilerGetCounterDataSize(&ds), "cuptiRangeProfilerGetCounterDataSize");
    g_counter.assign(ds.counterDataSize, 0);
    CUpti_RangeProfiler_CounterDataImage_Initialize_Params di{
        CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
    di.pRangeProfilerObject = g_obj;
    di.pCounterData = g_counter.data();
    di.counterDataSize = g_counter.size();
    TRY(cuptiRangeProfilerCounterDataImageInitialize(&di), "cuptiRangeProfilerCounterDataImageInitialize");
    CUpti_RangeProfiler_SetConfig_Params sc{CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
    sc.pRangeProfilerObject = g_obj;
    sc.pConfig = g_config.data();
    sc.configSize = g_config.size();
    sc.pCounterDataImage = g_counter.data();
    sc.counterDataImageSize = g_counter.size();
    sc.range = CUPTI_UserRange;        // one range around everything launched until end()
    sc.replayMode = CUPTI_UserReplay;  // (the two DRAM counters need a single pass)
    sc.maxRangesPerPass = kMaxRanges;
    sc.numNestingLevels = 1;
    sc.minNestingLevel = 1;
    sc.passIndex = 0;
    sc.targetNestingLevel = 1;
    TRY(cuptiRangeProfilerSetConfig(&sc), "cuptiRangeProfilerSetConfig");
    CUpti_RangeProfiler_Start_Params st{CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
    st.pRangeProfilerObject = g_obj;
    TRY(cuptiRangeProfilerStart(&st), "cuptiRangeProfilerStart");
    CUpti_RangeProfiler_PushRange_Params pr{CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
    pr.pRangeProfilerObject = g_obj;
    pr.pRangeName = "probe";
    TRY(cuptiRangeProfilerPushRange(&pr), "cuptiRangeProfilerPushRange");
    return 0;
}

static int end_impl(double* out);

int grape_dram_probe_end(double* read_bytes, double* write_bytes, double* ns)
{
    double v[kMaxMetrics] = {0, 0, 0, 0};
    const int rc = end_impl(v);
    *read_bytes = v[0];
    *write_bytes = v[1];
    *ns = 0;   // (durations are CUDA-event measurements in bench.py)
    return rc;
}

// The running set's metric values, in the set's order (out: 4 doubles).
int grape_probe_end_set(double* out) { return end_impl(out); }

static int end_impl(double* out)
{
    if (g_obj == nullptr) {
        g_err = "grape_dram_probe_end without begin";
        return 1;
    }
    int rc = 0;
    auto run = [&]() -> int {
        CUpti_RangeProfiler_PopRange_Params pp{CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
        pp.pRangeProfilerObject = g_obj;
        TRY(cuptiRangeProfilerPopRange(&pp), "cuptiRangeProfilerPopRange");
        CUpti_RangeProfiler_Stop_Params sp{CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
        sp.pRangeProfilerObject = g_obj;
        TRY(cuptiRangeProfilerStop(&sp), "cuptiRangeProfilerStop");
        if (!sp.isAllPassSubmitted) {
            g_err = "the counters needed more than one pass";
            return 1;
        }
        CUpti_RangeProfiler_DecodeData_Params dd{CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
        dd.pRangeProfilerObject = g_obj;
        TRY(cuptiRangeProfilerDecodeData(&dd), "cuptiRangeProfilerDecodeData");
        if (getenv("GRAPE_DRAM_PROBE_DEBUG"))
            fprintf(stderr, "dram probe: all passes submitted %d, ranges dropped %zu\n", (int)sp.isAllPassSubmitted,
                    dd.numOfRangeDropped);
        CUpti_RangeProfiler_GetCounterDataInfo_Params gi{CUpti_RangeProfiler_GetCounterDataInfo_Params_STRUCT_SIZE};
        gi.pCounterDataImage = g_counter.data();
        gi.counterDataImageSize = g_counter.size();
        TRY(cuptiRangeProfilerGetCounterDataInfo(&gi), "cuptiRangeProfilerGetCounterDataInfo");
        double sum[kMaxMetrics] = {0, 0, 0, 0};
        for (size_t r = 0; r < gi.numTotalRanges; ++r) {
            double v[kMaxMetrics] = {0, 0, 0, 0};
            CUpti_Profiler_Host_EvaluateToGpuValues_Params ev{CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
            ev.pHostObject = g_host;
            ev.pCounterDataImage = g_counter.data();
            ev.counterDataImageSize = g_counter.size();
            ev.ppMetricNames = kMetrics;
            ev.numMetrics = kNumMetrics;
            ev.rangeIndex = r;
            ev.pMetricValues = v;
            TRY(cuptiProfilerHostEvaluateToGpuValues(&ev), "cuptiProfilerHostEvaluateToGpuValues");
            for (size_t q = 0; q < kNumMetrics; ++q) sum[q] += v[q];
        }
        for (size_t q = 0; q < kMaxMetrics; ++q) out[q] = sum[q];
        if (gi.numTotalRanges == 0) {
            g_err = "no kernel ranges were recorded";
            return 1;
        }
        return 0;
    };
    rc = run();
    cleanup();
    return rc;
}

}  // extern "C"
