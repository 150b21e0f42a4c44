// fc_internal.h -- private types shared by the host planner, the runtime and
// the CUDA launcher of libfc.so.  Not part of the ABI (include/fc.h is).
#pragma once
#include <nvtx3/nvToolsExt.h>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "fc.h"

namespace fc {

constexpr int kPatch = 14;
constexpr int kTps = 2;
constexpr int kMerge = 2;
constexpr int kBlock = kPatch * kMerge;  // 28: merge-block side in pixels
constexpr int kCols = FC_TOKEN_COLS;     // 1176
constexpr int kPrecisionBits = 22;       // Pillow 8bpc fixed point (R4)

// One resize axis (R4): per output index o the first
// source index xmin[o], the tap count cnt[o] and Pillow's 22-bit integer
// weights iw[o][0..cnt) (ksize slots per output).  The kernels' tables (MMA
// fragments / weight digits) are derived from these per device.
struct AxisTable {
  int in = 0, out = 0;
  int ksize = 0;   // Pillow ksize
  int max_cnt = 0; // widest window actually used
  std::vector<int32_t> xmin, cnt;
  std::vector<int32_t> iw;       // out x ksize integer weights, 22-bit fixed point
  int prec = kPrecisionBits;     // the backend's rounding precision (iw = round(w*2^prec) << (22-prec))
};

struct RankPlan {
  fc_rank_plan p{};
};

// Device copies of a plan's tables (see fc_kernels.cu: MMA fragment tables).
// Held by shared_ptr: the bounded process-wide cache and every plan that uses
// them keep a reference; the device memory is freed with the last one.
struct DeviceTables {
  DeviceTables() = default;
  DeviceTables(const DeviceTables&) = delete;
  DeviceTables& operator=(const DeviceTables&) = delete;
  ~DeviceTables();  // fc_kernels.cu
  uint64_t serial = 0;         // unique per table set (keys the launch-configuration cache)
  int ksh = 1, ksv = 1;        // MMA k-steps of the H / V windows
  int32_t* hx = nullptr;       // H xmin per output column
  int32_t* hxs = nullptr;      // H window start per 8-column tile
  uint32_t* hfr = nullptr;     // H B fragments
  int32_t* vx = nullptr;       // V ymin per output row
  int32_t* vcnt = nullptr;     // V taps per output row
  int32_t* vys = nullptr;      // V window start per (band, 8-row group)
  uint32_t* vfr = nullptr;     // V B fragments
  uint32_t* lut = nullptr;     // 3 x 256 normalisation table (R5), token-dtype bits
};

}  // namespace fc

struct fc_plan_s {
  fc_video_meta meta{};
  std::vector<int64_t> gop_start;
  fc_model_cfg cfg{};
  std::vector<int64_t> sampled;  // global frame indices, ascending
  int64_t n = 0;
  int32_t h2 = 0, w2 = 0;
  int64_t gt = 0, gh = 0, gw = 0;
  double sampled_fps = 0, second_per_grid = 0;
  int32_t world = 1, ranks_used = 0;
  std::vector<fc::RankPlan> ranks;
  // horizontal (W -> W'), vertical (H -> H'); shared, immutable, cached per (in, out)
  std::shared_ptr<const fc::AxisTable> th, tv;
  std::vector<float> lut;    // 3 x 256 (R5)
  std::vector<uint32_t> lut_dev;  // what the kernel stores: fp32 bits, or bf16 bits (R16)
  std::mutex mu;             // guards dev, tc
  std::unordered_map<int, std::shared_ptr<const fc::DeviceTables>> dev;  // per (device, strip width)
  std::unordered_map<int, std::shared_ptr<const void>> tc;  // per device: the tcgen05 kernel's tables
};

namespace fc {
void set_error(const std::string& msg);
fc_status fail(fc_status s, const std::string& msg);
fc_status build_axis(int in, int out, int backend, AxisTable* t);
fc_status axis_cached(int in, int out, int backend, std::shared_ptr<const AxisTable>* t);

// NVTX range around a C-ABI entry point (nvtx3, header-only: a no-op unless a
// profiler injects itself), so nsys / ncu timelines show the library's calls.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace fc
