// fc_sched.cpp -- stall-free GOP_s dispatch (Alg. 2, P:397-443;
// SURVEY 8(f) f3, the host half of the decode front end).
//
// A request's decode work is split into GOP_s segments (runs of GOPs, each
// decoded by one decode unit from its keyframe).  T worker threads
// own segment lists (Alg. 2 l.6); a gate admits at most N segments in flight,
// N = the decode units (l.10: num_nvdec_in_use vs N).  When a worker finishes
// a segment and still has segments, it keeps its unit and starts the next one
// at once -- "the scheduler prioritizes waking the same worker to dispatch its
// remaining GOP_s segments" (l.12-13) -- so a unit is never idle while
// its worker has work, and units are released only when a worker runs dry,
// waking one waiter.  The granularity (segments instead of whole videos) is
// what removes the stall of Fig. 9: a unit that finishes early takes the next
// segment instead of waiting for the slowest unit.
#include <condition_variable>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "fc_internal.h"

namespace fc {
namespace {

struct Gate {
  std::mutex mu;
  std::condition_variable cv;
  int in_use = 0;
  int cap = 1;
  bool failed = false;
  int64_t seq = 0;  // completion counter (trace)
};

}  // namespace
}  // namespace fc

using namespace fc;

extern "C" fc_status fc_dispatch_segments(const int32_t* worker_of, int64_t num_segments, int32_t num_workers,
                                          int32_t max_in_flight, fc_segment_fn fn, void* ctx, int64_t* trace) {
  NvtxRange nvtx("fc_dispatch_segments");
  if (num_segments < 0 || num_workers < 1 || num_workers > 1024 || max_in_flight < 1 || !fn ||
      (num_segments > 0 && !worker_of))
    return fail(FC_ERR_INVALID_ARG, "bad segment dispatch arguments");
  std::vector<std::vector<int64_t>> own;
  try {
    own.resize(num_workers);
    for (int64_t s = 0; s < num_segments; ++s) {
      if (worker_of[s] < 0 || worker_of[s] >= num_workers) return fail(FC_ERR_INVALID_ARG, "segment worker out of range");
      own[worker_of[s]].push_back(s);
    }
  } catch (const std::bad_alloc&) {
    return fail(FC_ERR_OOM, "segment lists");
  }
  Gate g;
  g.cap = max_in_flight;
  int32_t first_err = 0;
  auto worker = [&](int w) {
    const std::vector<int64_t>& mine = own[w];
    if (mine.empty()) return;
    {  // acquire a decode unit (Alg. 2 l.8-17)
      std::unique_lock<std::mutex> lk(g.mu);
      g.cv.wait(lk, [&] { return g.failed || g.in_use < g.cap; });
      if (g.failed) return;
      ++g.in_use;
    }
    for (size_t i = 0; i < mine.size(); ++i) {
      const int32_t rc = fn(ctx, mine[i], w);
      std::lock_guard<std::mutex> lk(g.mu);
      if (trace) {
        trace[3 * g.seq] = mine[i];
        trace[3 * g.seq + 1] = w;
        trace[3 * g.seq + 2] = rc;
      }
      ++g.seq;
      if (rc != 0 && !g.failed) {
        g.failed = true;
        first_err = rc;
      }
      if (g.failed) break;
      // the same worker keeps its unit for its next segment (l.12-13)
    }
    {
      std::lock_guard<std::mutex> lk(g.mu);
      --g.in_use;
    }
    g.cv.notify_all();
  };
  std::vector<std::thread> th;
  try {
    th.reserve(num_workers);
    for (int w = 0; w < num_workers; ++w) th.emplace_back(worker, w);
  } catch (...) {
    {
      std::lock_guard<std::mutex> lk(g.mu);
      g.failed = true;
    }
    g.cv.notify_all();
    for (auto& t : th) t.join();
    return fail(FC_ERR_OOM, "worker threads");
  }
  for (auto& t : th) t.join();
  if (g.failed) return fail(FC_ERR_CUDA, "a segment decode failed (callback status " + std::to_string(first_err) + ")");
  return FC_OK;
}
