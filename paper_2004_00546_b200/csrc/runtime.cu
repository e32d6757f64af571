// runtime.cu — errors, device allocation, dynamic shared-memory opt-in, timing windows
// (CUDA events + NVTX ranges) and the CUDA-graph segments of the captured gradient.
#include <map>
#include <mutex>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / Nsight timelines

#include "internal.h"

namespace pxi {

thread_local std::string g_last_error;

int fail(Handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  g_last_error = msg;
  return code;
}

int dalloc(Handle* h, void** p, size_t bytes) {
  if (bytes == 0) bytes = 8;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess)
    return fail(h, e == cudaErrorMemoryAllocation ? PX_ERR_NOMEM : PX_ERR_CUDA,
                "cudaMalloc(" + std::to_string(bytes) + " B): " + cudaGetErrorString(e));
  h->allocs.push_back(*p);
  return PX_OK;
}

// Opt a kernel into `bytes` of dynamic shared memory once per (kernel, device): the
// attribute belongs to the device's context, so a process driving several GPUs needs it
// on each. The table is shared by all handles (one per device, possibly on different
// host threads), hence the lock.
int smem_attr(Handle* h, const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  PX_CUDA(h, cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kernel, dev}];
  if (have >= bytes) return PX_OK;
  PX_CUDA(h, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
  return PX_OK;
}

cudaEvent_t take_event(Handle* h) {
  if (!h->event_pool.empty()) {
    cudaEvent_t e = h->event_pool.back();
    h->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void seg_open(Handle* h, int phase) {
  h->cap_phase = phase;
  h->cap_launches0 = h->stats.kernel_launches;
  h->cap_bytes0 = h->stats.algorithmic_bytes;
  if (cudaStreamBeginCapture(h->gstream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) h->cap_error = 1;
}

void seg_close(Handle* h) {
  cudaGraph_t g = nullptr;
  if (cudaStreamEndCapture(h->gstream, &g) != cudaSuccess || !g) {
    h->cap_error = 1;
    return;
  }
  size_t nn = 0;
  cudaGraphGetNodes(g, nullptr, &nn);
  if (nn > 0) {
    cudaGraphExec_t ex = nullptr;
    if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) h->cap_error = 1;
    else
      h->segs.push_back({h->cap_phase, ex, h->stats.kernel_launches - h->cap_launches0,
                         h->stats.algorithmic_bytes - h->cap_bytes0});
  }
  cudaGraphDestroy(g);
}

void drop_segments(Handle* h) {
  for (auto& sg : h->segs) cudaGraphExecDestroy(sg.exec);
  h->segs.clear();
}

const char* phase_name(int phase) {
  static const char* names[] = {"px.rk4_direct", "px.rk4_adjoint", "px.exp_direct", "px.exp_adjoint", "px.other"};
  return (phase >= 0 && phase < PX_PHASE_COUNT) ? names[phase] : "px.phase";
}

// Open a timing window for `phase` (returns -1 when timing is off; while capturing a
// graph the window becomes its own graph segment, timed at replay). Eager windows are
// also NVTX ranges (the reference's recorder hooks, `workers.py:26-36`, become timeline
// ranges).
int tbegin(Handle* h, int phase, cudaStream_t s) {
  if (h->capturing) {
    seg_close(h);
    seg_open(h, phase);
    return -2;
  }
  nvtxRangePushA(phase_name(phase));
  if (!h->timing) return -1;
  Handle::TMark m{phase, take_event(h), take_event(h), h->stats.kernel_launches, h->stats.algorithmic_bytes};
  cudaEventRecord(m.a, s);
  h->marks.push_back(m);
  return (int)h->marks.size() - 1;
}

void tend(Handle* h, int idx, cudaStream_t s) {
  if (idx == -2 && h->capturing) {
    seg_close(h);
    seg_open(h, -1);
    return;
  }
  nvtxRangePop();
  if (idx < 0) return;
  Handle::TMark& m = h->marks[idx];
  cudaEventRecord(m.b, s);
  m.launches = h->stats.kernel_launches - m.launches;
  m.bytes = h->stats.algorithmic_bytes - m.bytes;
}

int kbegin(Handle* h, int cls, cudaStream_t s) {
  if (h->timing < 2 || h->capturing) return -1;
  Handle::KMark m{cls, take_event(h), take_event(h)};
  cudaEventRecord(m.a, s);
  h->kmarks.push_back(m);
  return (int)h->kmarks.size() - 1;
}

void kend(Handle* h, int idx, cudaStream_t s) {
  if (idx < 0) return;
  cudaEventRecord(h->kmarks[idx].b, s);
}

}  // namespace pxi
