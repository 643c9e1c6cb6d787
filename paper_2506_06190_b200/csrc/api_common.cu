// Error handling and small shared utilities of libnat.
#include <mutex>
#include <vector>

#include "nat_internal.cuh"

namespace nat {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

nat_status fail(nat_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int device_sm_count() {
  int dev = 0, n = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// ------------------------------------------------------------------------------------
// Kernel timer (diagnostics, off by default): CUDA events on the launching stream around
// the main kernel of each category; the skip word (GMRES iterations enqueued after
// convergence) is copied next to the events so skipped launches are not counted.
// ------------------------------------------------------------------------------------
namespace {
struct TimerEntry {
  cudaEvent_t e0, e1, done;  // done: after the skip-word copy (drain waits on it)
  int cat, n_modes;
  double pairs;
  int slot;  // pinned skip-word slot or -1
};
constexpr int kMaxBucket = 64;  // wavenumbers per launch
struct KTimer {
  std::mutex mu;
  bool on = false;
  std::vector<TimerEntry> live;
  std::vector<cudaEvent_t> pool;
  unsigned long long* slots = nullptr;  // pinned host
  int n_slots = 0, used_slots = 0;
  // totals per category and per wavenumbers-in-launch (bucket 0 = all launches)
  double sec[kTimerCats][kMaxBucket + 1] = {}, pairs[kTimerCats][kMaxBucket + 1] = {};
  long long launches[kTimerCats][kMaxBucket + 1] = {};
};
KTimer& timer() {
  static KTimer t;
  return t;
}
thread_local TimerEntry t_open{nullptr, nullptr, nullptr, -1, 0, 0.0, -1};

cudaEvent_t take_event(KTimer& t) {
  if (!t.pool.empty()) {
    cudaEvent_t e = t.pool.back();
    t.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}

// sums the recorded entries (synchronising their events) into the totals
void drain(KTimer& t) {
  for (auto& e : t.live) {
    if (cudaEventSynchronize(e.done) != cudaSuccess) {  // the skip word has landed too
      cudaGetLastError();
      continue;
    }
    const bool skipped = e.slot >= 0 && t.slots[e.slot] == 0ull;
    float ms = 0.f;
    if (!skipped && cudaEventElapsedTime(&ms, e.e0, e.e1) == cudaSuccess) {
      const int b = e.n_modes >= 1 && e.n_modes <= kMaxBucket ? e.n_modes : 0;
      for (int q : {0, b}) {
        t.sec[e.cat][q] += 1e-3 * ms;
        t.pairs[e.cat][q] += e.pairs;
        t.launches[e.cat][q] += 1;
        if (b == 0) break;  // launches without a mode count only enter the total
      }
    }
    cudaGetLastError();
    t.pool.push_back(e.e0);
    t.pool.push_back(e.e1);
    if (e.done != e.e1) t.pool.push_back(e.done);
  }
  t.live.clear();
  t.used_slots = 0;
}
}  // namespace

bool ktimer_on() { return timer().on; }

void ktimer_begin(int cat, cudaStream_t s) {
  KTimer& t = timer();
  std::lock_guard<std::mutex> lk(t.mu);
  if (!t.on) return;
  cudaEvent_t e0 = take_event(t), e1 = take_event(t);
  if (!e0 || !e1) return;
  cudaEventRecord(e0, s);
  t_open = TimerEntry{e0, e1, e1, cat, 0, 0.0, -1};
}

void ktimer_end(int cat, cudaStream_t s, double pairs, const unsigned long long* skip, int n_modes) {
  KTimer& t = timer();
  std::lock_guard<std::mutex> lk(t.mu);
  if (!t.on || t_open.cat != cat || !t_open.e0) return;
  TimerEntry e = t_open;
  t_open = TimerEntry{nullptr, nullptr, nullptr, -1, 0, 0.0, -1};
  cudaEventRecord(e.e1, s);
  e.pairs = pairs;
  e.n_modes = n_modes;
  if (skip) {
    if (t.used_slots >= t.n_slots) drain(t);  // (rare) recycle the slots
    e.slot = t.used_slots++;
    cudaMemcpyAsync(&t.slots[e.slot], skip, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    // drain() waits on an event recorded after the copy, so it never reads a stale word
    cudaEvent_t d = take_event(t);
    if (d) {
      cudaEventRecord(d, s);
      e.done = d;
    } else {
      cudaStreamSynchronize(s);
    }
  }
  t.live.push_back(e);
}

}  // namespace nat

extern "C" void nat_kernel_timer_enable(int on) {
  nat::KTimer& t = nat::timer();
  std::lock_guard<std::mutex> lk(t.mu);
  nat::drain(t);
  for (int c = 0; c < nat::kTimerCats; ++c)
    for (int b = 0; b <= nat::kMaxBucket; ++b) {
      t.sec[c][b] = t.pairs[c][b] = 0.0;
      t.launches[c][b] = 0;
    }
  if (on && !t.slots) {
    t.n_slots = 4096;
    if (cudaHostAlloc(&t.slots, sizeof(unsigned long long) * t.n_slots, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      t.slots = nullptr;
      t.n_slots = 0;
      return;
    }
  }
  t.on = on != 0;
}

extern "C" nat_status nat_kernel_timer_read_modes(int category, int n_modes, double* seconds, double* pairs,
                                                  int64_t* launches) {
  NAT_REQUIRE(category >= 0 && category < nat::kTimerCats, "category %d out of range", category);
  NAT_REQUIRE(n_modes >= 0 && n_modes <= nat::kMaxBucket, "n_modes %d out of range [0, 64]", n_modes);
  NAT_REQUIRE(seconds && pairs && launches, "outputs must be non-null host pointers");
  nat::KTimer& t = nat::timer();
  std::lock_guard<std::mutex> lk(t.mu);
  nat::drain(t);
  *seconds = t.sec[category][n_modes];
  *pairs = t.pairs[category][n_modes];
  *launches = t.launches[category][n_modes];
  return NAT_OK;
}

extern "C" nat_status nat_kernel_timer_read(int category, double* seconds, double* pairs, int64_t* launches) {
  return nat_kernel_timer_read_modes(category, 0, seconds, pairs, launches);
}

extern "C" int nat_abi_version(void) { return NAT_ABI_VERSION; }

extern "C" const char* nat_last_error(void) { return nat::g_last_error.c_str(); }
