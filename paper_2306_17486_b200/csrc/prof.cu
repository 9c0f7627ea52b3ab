#include <mutex>
#include <vector>

#include "../../include/helmsolve_b200.h"
#include "prof.h"

namespace hs {
namespace prof {

std::atomic<long long> launches{0};
std::atomic<int> active_now{0};

namespace {
struct Rec {
  int tag, label;
  cudaEvent_t a, b;
  double work;
};
std::mutex mu;
unsigned mask = 0;
std::vector<Rec> recs;
std::vector<cudaEvent_t> pool;
thread_local int cur_label = 0;

cudaEvent_t get_event() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

bool on(int tag) { return (mask >> tag) & 1u; }

void set_label(int label) { cur_label = label; }

int start(int tag, cudaStream_t st) {
  if (!on(tag)) return -1;
  std::lock_guard<std::mutex> g(mu);
  Rec r{tag, cur_label, get_event(), get_event(), 0.0};
  cudaEventRecord(r.a, st);
  recs.push_back(r);
  return (int)recs.size() - 1;
}

void stop(int slot, cudaStream_t st, double work) {
  if (slot < 0) return;
  std::lock_guard<std::mutex> g(mu);
  cudaEventRecord(recs[slot].b, st);
  recs[slot].work = work;
}

}  // namespace prof
}  // namespace hs

using namespace hs::prof;

HS_API void hs_profile_enable(unsigned tag_mask) {
  std::lock_guard<std::mutex> g(mu);
  mask = tag_mask;
}

HS_API void hs_profile_reset(void) {
  std::lock_guard<std::mutex> g(mu);
  for (auto& r : recs) {
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  recs.clear();
  launches.store(0);
}

HS_API long long hs_launch_count(void) { return launches.load(); }

/* Per-launch records of the timed tags, in launch order: tag, label (convolutions: cin * 100000 +
   cout * 100 + mode, mode 0/1 = stride 1/2, 2 = transposed), milliseconds.  Returns the record count
   (at most max are written). */
HS_API int hs_profile_records(int* tags, int* labels, double* ms, int max) {
  std::lock_guard<std::mutex> g(mu);
  int n = 0;
  for (auto& r : recs) {
    if (n >= max) break;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return -HS_ECUDA;
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    tags[n] = r.tag;
    labels[n] = r.label;
    ms[n] = t;
    ++n;
  }
  return n;
}

HS_API int hs_profile_query(int tag, double* total_ms, double* total_work, long long* count) {
  std::lock_guard<std::mutex> g(mu);
  double ms = 0.0, work = 0.0;
  long long n = 0;
  for (auto& r : recs) {
    if (r.tag != tag) continue;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return HS_ECUDA;
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    ms += t;
    work += r.work;
    ++n;
  }
  *total_ms = ms;
  *total_work = work;
  *count = n;
  return HS_OK;
}

namespace hs {
extern bool conv_tc_enabled;
}
/* 1 = tcgen05 convolutions where supported (default), 0 = SIMT everywhere (tests) */
HS_API void hs_set_conv_path(int tensor_cores) { hs::conv_tc_enabled = tensor_cores != 0; }
