// fc_launch.h -- host-side launch helpers shared by the two kernel families
// (fc_kernels.cu: the mma.sync kernel and the entry points; fc_tc.cu: the
// tcgen05 kernel).  Private to libfc.so.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <list>
#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "fc_internal.h"

namespace fc {

// One launch job: a (plan, rank)'s frame list, its surfaces and its token buffer.
struct Job {
  std::vector<int64_t> frames;
  const fc_nv12_surface* surfaces;
  void* tokens;
};

// Bounded LRU cache of device table sets (keys are POD with operator<).
// Plans hold their own shared_ptr references, so an evicted entry's device
// memory is freed when the last plan using it is destroyed (fc.h: a plan must
// not be destroyed with work in flight).  Callers serialise access.
template <typename K, typename V>
class LruCache {
 public:
  explicit LruCache(size_t cap) : cap_(cap) {}
  std::shared_ptr<V> get(const K& k) {
    auto it = m_.find(k);
    if (it == m_.end()) return nullptr;
    l_.splice(l_.begin(), l_, it->second);  // most recently used first
    return it->second->second;
  }
  void put(const K& k, std::shared_ptr<V> v) {
    l_.emplace_front(k, std::move(v));
    m_[k] = l_.begin();
    while (l_.size() > cap_) {
      m_.erase(l_.back().first);
      l_.pop_back();
    }
  }
  size_t size() const { return l_.size(); }

 private:
  size_t cap_;
  std::list<std::pair<K, std::shared_ptr<V>>> l_;
  std::map<K, typename std::list<std::pair<K, std::shared_ptr<V>>>::iterator> m_;
};
constexpr size_t kTableCacheEntries = 32;  // distinct (device, shape, normalisation) table sets kept

fc_status cuda_fail(cudaError_t e, const char* what);
// fc_kernel_launches(): kernels this library has launched
std::atomic<uint64_t>& launch_counter();
// fc_last_kernel(): the calling thread's last fused-kernel launch (fc_kernel_id)
int32_t& last_kernel();
// 2-D u8 tensor map [rows][pitch] with a (bw x bh) box, cached per surface.
fc_status tensor_map(const uint8_t* base, int64_t pitch, int64_t rows, int bw, int bh, CUtensorMap* out);
// Compute capability major, opt-in shared memory per block, SM count (cached per device).
void device_attrs(int dev, int* major, int* max_smem, int* nsm);
// Raise a kernel's dynamic shared-memory limit to at least smem (monotone per device).
fc_status ensure_smem_attr(int dev, const void* fn, size_t smem);
// Library-owned stream-ordered pool for launch descriptors.
cudaMemPool_t descriptor_pool(int dev);
// Colour-matrix constants (R3, R15) as dp2a operand pairs and biases.
void color_words(fc_color m, uint32_t* kR, uint32_t* kG, uint32_t* kGv, uint32_t* kB, int* bR, int* bG, int* bB);
// Integer Pillow weight of output o at source index src (0 outside the window).
int32_t weight_at(const AxisTable& t, int o, int src);

// The tcgen05 kernel (fc_tc.cu).  *handled = false when the request's shape
// or variant is outside what that kernel is built for (the caller then
// launches the mma.sync kernel); otherwise the status of the launch.  dry:
// validate and prepare only, enqueue nothing.
fc_status launch_tc(fc_plan_s* P, const std::vector<Job>& jobs, void* stream, uint8_t* dbg_src, uint8_t* dbg_rs,
                    bool* handled, bool dry = false);

}  // namespace fc
