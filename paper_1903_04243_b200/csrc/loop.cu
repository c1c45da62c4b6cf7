// Device-resident while loops: a CUDA graph with a conditional WHILE node
// (reference interp.py:133-154 runs `while` on the host, one condition read
// per trip).
//
//   G = head --> WHILE(h) { iter }
//   head: the condition sub-graph on the carried state, then
//         pfb_set_condition(h, flag)
//   iter: the body sub-graph, copies of its results into the carried state,
//         the condition again, pfb_set_condition(h, flag)
// head and iter are graphs captured by the executor (their kernels are the
// ordinary libpfb launches); this file only creates the handle, assembles G
// and launches it.  One graph launch runs the whole loop with no host round
// trip per trip.
#include "common.cuh"

namespace pfb {
struct DeviceLoop {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
};

// also counts its own invocations (head + one per trip) for launch accounting
__global__ void set_condition_kernel(cudaGraphConditionalHandle h, const uint8_t* flag,
                                     unsigned long long* counter) {
  cudaGraphSetConditional(h, flag[0] ? 1u : 0u);
  if (counter) *counter += 1;
}
// the predicated while's test, any(active) (vectorize._convert_while_masked:
// less(0, reduce_sum(cast(active, i64)))), straight into the handle: one
// launch instead of cast + reduction + compare + set
__global__ void __launch_bounds__(1024) set_condition_any_kernel(cudaGraphConditionalHandle h,
                                                                 const uint8_t* mask, int64_t n,
                                                                 unsigned long long* counter) {
  int any = 0;
  const int64_t n4 = ((reinterpret_cast<uintptr_t>(mask) & 3) == 0) ? n / 4 : 0;
  for (int64_t i = threadIdx.x; i < n4; i += blockDim.x)
    any |= reinterpret_cast<const uint32_t*>(mask)[i] != 0u;
  for (int64_t i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) any |= mask[i] != 0;
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    cudaGraphSetConditional(h, any ? 1u : 0u);
    if (counter) *counter += 1;
  }
}
}  // namespace pfb

using namespace pfb;

extern "C" int pfb_loop_create(void** loop, uint64_t* handle) {
  DeviceLoop* L = new DeviceLoop();
  if (cudaGraphCreate(&L->graph, 0) != cudaSuccess) { delete L; return launch_status(); }
  if (cudaGraphConditionalHandleCreate(&L->handle, L->graph, 0, 0) != cudaSuccess) {
    cudaGraphDestroy(L->graph);
    delete L;
    return launch_status();
  }
  *loop = L;
  *handle = (uint64_t)L->handle;
  return 0;
}

// the condition flag (a device bool) -> the loop's conditional handle;
// `counter` (nullable, device u64) counts the invocations
extern "C" int pfb_set_condition(uint64_t handle, const void* flag, void* counter,
                                 void* stream) {
  kernel_launches()++;
  set_condition_kernel<<<1, 1, 0, as_stream(stream)>>>((cudaGraphConditionalHandle)handle,
                                                       (const uint8_t*)flag,
                                                       (unsigned long long*)counter);
  return launch_status();
}

// any(mask[0..n)) -> the loop's conditional handle (mask: dense u8 bools)
extern "C" int pfb_set_condition_any(uint64_t handle, const void* mask, int64_t n, void* counter,
                                     void* stream) {
  if (n < 0) return PFB_E_ARG;
  kernel_launches()++;
  const int threads = n >= 4096 ? 1024 : 256;
  set_condition_any_kernel<<<1, threads, 0, as_stream(stream)>>>(
      (cudaGraphConditionalHandle)handle, (const uint8_t*)mask, n, (unsigned long long*)counter);
  return launch_status();
}

extern "C" int pfb_loop_finalize(void* loop, void* head_graph, void* iter_graph) {
  DeviceLoop* L = static_cast<DeviceLoop*>(loop);
  cudaGraphNode_t head;
  if (cudaGraphAddChildGraphNode(&head, L->graph, nullptr, 0, (cudaGraph_t)head_graph) != cudaSuccess)
    return launch_status();
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = L->handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wnode;
  if (cudaGraphAddNode(&wnode, L->graph, &head, 1, &cp) != cudaSuccess) return launch_status();
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaGraphNode_t it;
  if (cudaGraphAddChildGraphNode(&it, body, nullptr, 0, (cudaGraph_t)iter_graph) != cudaSuccess)
    return launch_status();
  if (cudaGraphInstantiate(&L->exec, L->graph, 0) != cudaSuccess) return launch_status();
  return 0;
}

extern "C" int pfb_loop_launch(void* loop, void* stream) {
  DeviceLoop* L = static_cast<DeviceLoop*>(loop);
  if (!L->exec) return PFB_E_ARG;
  cudaGraphLaunch(L->exec, as_stream(stream));
  return launch_status();
}

extern "C" int pfb_loop_destroy(void* loop) {
  DeviceLoop* L = static_cast<DeviceLoop*>(loop);
  if (!L) return 0;
  if (L->exec) cudaGraphExecDestroy(L->exec);
  if (L->graph) cudaGraphDestroy(L->graph);
  delete L;
  return 0;
}
