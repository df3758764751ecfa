// dram_meter.cpp -- in-process hardware counters for one stream-ordered region (bench.py's
// roofline: the DRAM bytes a walk launch really moves, measured in the same run).
//
// CUPTI range profiler (cupti_range_profiler.h + cupti_profiler_host.h): one user range
// around the caller's launches, user replay (the caller re-runs the region while
// dm_pass_end() returns 0 -- dram__bytes_{read,write}.sum fit one pass).  Measurement
// infrastructure only; libbingo does not link it.  C ABI:
//   dm_begin(metrics_csv)  -> 0 ok, else a negative step code (profiling unavailable,
//                             e.g. under ncu, which holds the counters itself)
//   dm_pass_begin()        -> start + push the range
//   dm_pass_end()          -> pop + stop; 1 when every pass has been submitted
//   dm_end(values, n)      -> decode, evaluate the metrics of range 0 into values[n]
//   dm_abort()             -> tear down after an error
#include <cuda.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace {

struct Meter {
    bool host = false, enabled = false, initialized = false;
    CUcontext ctx = nullptr;
    CUpti_Profiler_Host_Object *hobj = nullptr;
    CUpti_RangeProfiler_Object *robj = nullptr;
    std::string chip;
    std::vector<std::string> names;
    std::vector<const char *> cnames;
    std::vector<uint8_t> avail, config, data;
};
Meter M;

void teardown() {
    if (M.enabled) {
        CUpti_RangeProfiler_Disable_Params p{CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
        p.pRangeProfilerObject = M.robj;
        cuptiRangeProfilerDisable(&p);
        M.enabled = false;
        M.robj = nullptr;
    }
    if (M.host) {
        CUpti_Profiler_Host_Deinitialize_Params p{CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
        p.pHostObject = M.hobj;
        cuptiProfilerHostDeinitialize(&p);
        M.host = false;
        M.hobj = nullptr;
    }
}

}  // namespace

extern "C" int dm_begin(const char *metrics_csv) {
    teardown();
    M.names.clear();
    M.cnames.clear();
    std::string s(metrics_csv ? metrics_csv : "");
    size_t pos = 0;
    while (pos <= s.size()) {
        size_t c = s.find(',', pos);
        if (c == std::string::npos) c = s.size();
        if (c > pos) M.names.push_back(s.substr(pos, c - pos));
        pos = c + 1;
    }
    if (M.names.empty()) return -1;
    for (auto &n : M.names) M.cnames.push_back(n.c_str());
    if (cuCtxGetCurrent(&M.ctx) != CUDA_SUCCESS || !M.ctx) return -2;
    CUdevice dev;
    if (cuCtxGetDevice(&dev) != CUDA_SUCCESS) return -2;
    if (!M.initialized) {
        CUpti_Profiler_Initialize_Params ip{CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
        if (cuptiProfilerInitialize(&ip) != CUPTI_SUCCESS) return -3;
        M.initialized = true;
    }
    CUpti_Profiler_DeviceSupported_Params sp{CUpti_Profiler_DeviceSupported_Params_STRUCT_SIZE};
    sp.cuDevice = dev;
    sp.api = CUPTI_PROFILER_RANGE_PROFILING;
    if (cuptiProfilerDeviceSupported(&sp) != CUPTI_SUCCESS || sp.isSupported != CUPTI_PROFILER_CONFIGURATION_SUPPORTED)
        return -4;
    CUpti_Device_GetChipName_Params cp{CUpti_Device_GetChipName_Params_STRUCT_SIZE};
    cp.deviceIndex = (size_t)dev;
    if (cuptiDeviceGetChipName(&cp) != CUPTI_SUCCESS) return -5;
    M.chip = cp.pChipName;
    CUpti_Profiler_GetCounterAvailability_Params ap{CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
    ap.ctx = M.ctx;
    if (cuptiProfilerGetCounterAvailability(&ap) != CUPTI_SUCCESS) return -6;
    M.avail.assign(ap.counterAvailabilityImageSize, 0);
    ap.pCounterAvailabilityImage = M.avail.data();
    if (cuptiProfilerGetCounterAvailability(&ap) != CUPTI_SUCCESS) return -6;
    CUpti_Profiler_Host_Initialize_Params hp{CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
    hp.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
    hp.pChipName = M.chip.c_str();
    hp.pCounterAvailabilityImage = M.avail.data();
    if (cuptiProfilerHostInitialize(&hp) != CUPTI_SUCCESS) return -7;
    M.hobj = hp.pHostObject;
    M.host = true;
    CUpti_Profiler_Host_ConfigAddMetrics_Params am{CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
    am.pHostObject = M.hobj;
    am.ppMetricNames = M.cnames.data();
    am.numMetrics = M.cnames.size();
    if (cuptiProfilerHostConfigAddMetrics(&am) != CUPTI_SUCCESS) { teardown(); return -8; }
    CUpti_Profiler_Host_GetConfigImageSize_Params gs{CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
    gs.pHostObject = M.hobj;
    if (cuptiProfilerHostGetConfigImageSize(&gs) != CUPTI_SUCCESS) { teardown(); return -9; }
    M.config.assign(gs.configImageSize, 0);
    CUpti_Profiler_Host_GetConfigImage_Params gi{CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
    gi.pHostObject = M.hobj;
    gi.pConfigImage = M.config.data();
    gi.configImageSize = M.config.size();
    if (cuptiProfilerHostGetConfigImage(&gi) != CUPTI_SUCCESS) { teardown(); return -9; }
    CUpti_RangeProfiler_Enable_Params ep{CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
    ep.ctx = M.ctx;
    if (cuptiRangeProfilerEnable(&ep) != CUPTI_SUCCESS) { teardown(); return -10; }
    M.robj = ep.pRangeProfilerObject;
    M.enabled = true;
    CUpti_RangeProfiler_GetCounterDataSize_Params ds{CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
    ds.pRangeProfilerObject = M.robj;
    ds.pMetricNames = M.cnames.data();
    ds.numMetrics = M.cnames.size();
    ds.maxNumOfRanges = 1;
    ds.maxNumRangeTreeNodes = 1;
    if (cuptiRangeProfilerGetCounterDataSize(&ds) != CUPTI_SUCCESS) { teardown(); return -11; }
    M.data.assign(ds.counterDataSize, 0);
    CUpti_RangeProfiler_CounterDataImage_Initialize_Params di{
        CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
    di.pRangeProfilerObject = M.robj;
    di.pCounterData = M.data.data();
    di.counterDataSize = M.data.size();
    if (cuptiRangeProfilerCounterDataImageInitialize(&di) != CUPTI_SUCCESS) { teardown(); return -12; }
    CUpti_RangeProfiler_SetConfig_Params sc{CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
    sc.pRangeProfilerObject = M.robj;
    sc.pConfig = M.config.data();
    sc.configSize = M.config.size();
    sc.pCounterDataImage = M.data.data();
    sc.counterDataImageSize = M.data.size();
    sc.maxRangesPerPass = 1;
    sc.numNestingLevels = 1;
    sc.minNestingLevel = 1;
    sc.passIndex = 0;
    sc.targetNestingLevel = 1;
    sc.range = CUPTI_UserRange;
    sc.replayMode = CUPTI_UserReplay;
    if (cuptiRangeProfilerSetConfig(&sc) != CUPTI_SUCCESS) { teardown(); return -13; }
    return 0;
}

extern "C" int dm_pass_begin() {
    CUpti_RangeProfiler_Start_Params st{CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
    st.pRangeProfilerObject = M.robj;
    if (cuptiRangeProfilerStart(&st) != CUPTI_SUCCESS) return -1;
    CUpti_RangeProfiler_PushRange_Params pr{CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
    pr.pRangeProfilerObject = M.robj;
    pr.pRangeName = "region";
    if (cuptiRangeProfilerPushRange(&pr) != CUPTI_SUCCESS) return -2;
    return 0;
}

extern "C" int dm_pass_end() {
    CUpti_RangeProfiler_PopRange_Params pp{CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
    pp.pRangeProfilerObject = M.robj;
    if (cuptiRangeProfilerPopRange(&pp) != CUPTI_SUCCESS) return -1;
    CUpti_RangeProfiler_Stop_Params sp{CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
    sp.pRangeProfilerObject = M.robj;
    if (cuptiRangeProfilerStop(&sp) != CUPTI_SUCCESS) return -2;
    return sp.isAllPassSubmitted ? 1 : 0;
}

extern "C" int dm_end(double *values, int n) {
    CUpti_RangeProfiler_DecodeData_Params dd{CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
    dd.pRangeProfilerObject = M.robj;
    if (cuptiRangeProfilerDecodeData(&dd) != CUPTI_SUCCESS) { teardown(); return -1; }
    CUpti_RangeProfiler_GetCounterDataInfo_Params gi{CUpti_RangeProfiler_GetCounterDataInfo_Params_STRUCT_SIZE};
    gi.pCounterDataImage = M.data.data();
    gi.counterDataImageSize = M.data.size();
    if (cuptiRangeProfilerGetCounterDataInfo(&gi) != CUPTI_SUCCESS || gi.numTotalRanges < 1) { teardown(); return -2; }
    std::vector<double> v(M.cnames.size(), 0.0);
    CUpti_Profiler_Host_EvaluateToGpuValues_Params ev{CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
    ev.pHostObject = M.hobj;
    ev.pCounterDataImage = M.data.data();
    ev.counterDataImageSize = M.data.size();
    ev.ppMetricNames = M.cnames.data();
    ev.numMetrics = M.cnames.size();
    ev.rangeIndex = 0;
    ev.pMetricValues = v.data();
    const CUptiResult r = cuptiProfilerHostEvaluateToGpuValues(&ev);
    teardown();
    if (r != CUPTI_SUCCESS) return -3;
    for (int i = 0; i < n && i < (int)v.size(); i++) values[i] = v[i];
    return 0;
}

extern "C" void dm_abort() { teardown(); }
