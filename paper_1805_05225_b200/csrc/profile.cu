#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "profile.h"

namespace sl {
namespace {

struct Rec {
  std::string name;
  cudaEvent_t start, stop;
  double flops, bytes;
  bool closed;
};

std::atomic<bool> g_enabled{false};
std::atomic<unsigned long long> g_launches{0};
std::mutex g_mu;
std::vector<Rec> g_recs;

struct Acc {
  std::string name;
  int calls = 0;
  double ms = 0, flops = 0, bytes = 0;
};
std::vector<Acc> g_acc;

Acc& acc_for(const std::string& n) {
  for (auto& a : g_acc)
    if (a.name == n) return a;
  g_acc.push_back(Acc{n});
  return g_acc.back();
}

}  // namespace

bool profile_enabled() { return g_enabled.load(std::memory_order_relaxed); }
void count_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

Phase::Phase(cudaStream_t s, const char* name, double flops, double bytes) : stream_(s) {
  if (!profile_enabled()) return;
  Rec r{name, nullptr, nullptr, flops, bytes, false};
  cudaEventCreate(&r.start);
  cudaEventCreate(&r.stop);
  cudaEventRecord(r.start, s);
  std::lock_guard<std::mutex> lk(g_mu);
  slot_ = (int)g_recs.size();
  g_recs.push_back(r);
}

Phase::~Phase() {
  if (slot_ < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(g_recs[slot_].stop, stream_);
  g_recs[slot_].closed = true;
}

}  // namespace sl

extern "C" {

int sl_profile_enable(int enable) {
  sl::g_enabled.store(enable != 0);
  return 0;
}

unsigned long long sl_launch_count(void) { return sl::g_launches.load(); }

// Synchronizes every recorded phase, folds it into per-name totals, and
// copies up to max_entries totals out.  reset != 0 clears the totals after.
int sl_profile_read(sl_profile_entry* out, int max_entries, int reset) {
  using namespace sl;
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& r : g_recs) {
    if (!r.closed) continue;
    cudaEventSynchronize(r.stop);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.start, r.stop);
    Acc& a = acc_for(r.name);
    a.calls += 1;
    a.ms += ms;
    a.flops += r.flops;
    a.bytes += r.bytes;
    cudaEventDestroy(r.start);
    cudaEventDestroy(r.stop);
  }
  g_recs.erase(std::remove_if(g_recs.begin(), g_recs.end(), [](const Rec& r) { return r.closed; }),
               g_recs.end());
  int n = 0;
  for (auto& a : g_acc) {
    if (n >= max_entries || !out) break;
    std::memset(&out[n], 0, sizeof(sl_profile_entry));
    std::strncpy(out[n].name, a.name.c_str(), sizeof(out[n].name) - 1);
    out[n].calls = a.calls;
    out[n].ms = a.ms;
    out[n].flops = a.flops;
    out[n].bytes = a.bytes;
    ++n;
  }
  if (reset) g_acc.clear();
  return n;
}

}  // extern "C"
