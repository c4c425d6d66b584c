// ob_prof.cu -- CUDA-event kernel profiler used by bench.py's roofline.
//
// When enabled, the hot launches are bracketed by events on their own stream;
// the block counters they ran over are snapshotted into pinned memory at the
// end of each request so the algorithmic bytes of every launch can be
// computed after the fact without a host round trip inside the request.
#include <algorithm>
#include <cstdlib>

#include "ob_engine.h"

namespace ob {

Profiler* g_prof = nullptr;

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("OB_NO_PDL");
    return !(v && v[0] && v[0] != '0');
  }();
  return on;
}

cudaEvent_t Profiler::take() {
  if (next == pool.size()) {
    cudaEvent_t ev;
    OB_CUDA(cudaEventCreate(&ev));
    pool.push_back(ev);
  }
  return pool[next++];
}

int Profiler::slot_for(const BlockCounters* d) {
  for (auto& p : pending)
    if (p.first == d) return p.second;
  if (!pinned) {
    nslots = 1 << 14;
    OB_CUDA(cudaMallocHost(&pinned, sizeof(BlockCounters) * nslots));
  }
  OB_CHECK(used_slots < nslots, OB_ESTATE, "profiler snapshot slots exhausted; re-enable to reset");
  int idx = used_slots++;
  pending.push_back({d, idx});
  return idx;
}

void Profiler::request_end(cudaStream_t s) {
  for (auto& p : pending)
    OB_CUDA(cudaMemcpyAsync(pinned + p.second, p.first, sizeof(BlockCounters), cudaMemcpyDeviceToHost, s));
  pending.clear();
}

uint32_t* Profiler::bits(int64_t words, cudaStream_t s) {
  if (words > rowbits_words) {
    if (rowbits) OB_CUDA(cudaFree(rowbits));
    rowbits_words = std::max<int64_t>(words, 2 * rowbits_words);
    OB_CUDA(cudaMalloc(&rowbits, rowbits_words * 4));
  }
  OB_CUDA(cudaMemsetAsync(rowbits, 0, words * 4, s));
  return rowbits;
}

void Profiler::prime(size_t events) {
  while (pool.size() < events) {
    cudaEvent_t ev;
    OB_CUDA(cudaEventCreate(&ev));
    pool.push_back(ev);
  }
  if (!pinned) {
    nslots = 1 << 14;
    OB_CUDA(cudaMallocHost(&pinned, sizeof(BlockCounters) * nslots));
  }
}

void Profiler::reset() {
  next = 0;
  recs.clear();
  used_slots = 0;
  pending.clear();
}

cudaEvent_t prof_begin(cudaStream_t s) {
  if (!g_prof || !g_prof->on) return nullptr;
  cudaEvent_t a = g_prof->take();
  OB_CUDA(cudaEventRecord(a, s));
  return a;
}

void prof_end(cudaStream_t s, cudaEvent_t a, int cls, const BlockCounters* cnt, int width, int pw, int K, int Nc,
              int gemm_rows) {
  if (!a || !g_prof || !g_prof->on) return;
  cudaEvent_t b = g_prof->take();
  OB_CUDA(cudaEventRecord(b, s));
  ProfRec r{};
  r.cls = cls;
  r.a = a;
  r.b = b;
  r.slot = cnt ? g_prof->slot_for(cnt) : -1;
  r.width = width;
  r.pw = pw;
  r.K = K;
  r.Nc = Nc;
  r.gemm_rows = gemm_rows;
  g_prof->recs.push_back(r);
}

}  // namespace ob
