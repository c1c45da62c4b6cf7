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
