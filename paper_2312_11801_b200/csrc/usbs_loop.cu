// Device-controlled repetition of a launch sequence: the kernels a caller
// enqueues between usbs_loop_begin and usbs_loop_end become the body of a
// CUDA-graph WHILE node whose condition a one-thread kernel at the end of the
// body sets on the device -- the alternating maximisation of the bundle
// subproblem (subqp.py:552-614: "repeat the pass until ||nu' - nu|| <= tol
// (1 + ||b||) or max_passes") then runs with no host read between passes.
// The stopping test is the reference's, evaluated in the same arithmetic
// (sqrt(max(.,0)) <= thresh), so the pass count equals the host-driven loop's.
#include <cmath>

#include "usbs_common.cuh"

namespace usbs {

struct LoopState {
  cudaGraph_t graph = nullptr;
  cudaGraph_t body = nullptr;
  cudaGraphConditionalHandle handle = 0;
  bool capturing = false;
  // the body is captured on a private non-blocking stream (the context's
  // stream may be the legacy default stream, which cannot capture); the
  // context launches into it between begin and end
  cudaStream_t cap = nullptr;
  cudaStream_t saved = nullptr;
};

static LoopState& loop_state(usbs_ctx* ctx) {
  static std::mutex mu;
  static std::map<usbs_ctx*, LoopState> st;
  std::lock_guard<std::mutex> g(mu);
  return st[ctx];
}

// counter[0] += 1 (passes done inside the loop); continue while the squared
// step red[0] is above thresh^2-equivalent (tested as the host does) and the
// budget lasts
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const double* __restrict__ red, double thresh,
                            int max_iters, int* __restrict__ counter) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int c = counter[0] + 1;
    counter[0] = c;
    const double step = sqrt(fmax(red[0], 0.0));
    const bool done = (step <= thresh) || c >= max_iters;
    cudaGraphSetConditional(h, done ? 0u : 1u);
  }
}

}  // namespace usbs

using namespace usbs;

extern "C" usbs_status usbs_loop_begin(usbs_ctx* ctx) {
  USBS_API_BEGIN
  LoopState& L = loop_state(ctx);
  if (L.capturing) fail(USBS_ERR_CONFIG, "loop: already capturing");
  USBS_CUDA(cudaGraphCreate(&L.graph, 0));
  USBS_CUDA(cudaGraphConditionalHandleCreate(&L.handle, L.graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = L.handle;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  USBS_CUDA(cudaGraphAddNode(&node, L.graph, nullptr, 0, &np));
  L.body = np.conditional.phGraph_out[0];
  if (!L.cap) USBS_CUDA(cudaStreamCreateWithFlags(&L.cap, cudaStreamNonBlocking));
  USBS_CUDA(cudaStreamBeginCaptureToGraph(L.cap, L.body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  L.saved = ctx->stream;
  ctx->stream = L.cap;
  L.capturing = true;
  USBS_API_END
}

extern "C" usbs_status usbs_loop_end(usbs_ctx* ctx, const double* red_dev, double thresh, int max_iters,
                                     int* counter_dev) {
  USBS_API_BEGIN
  LoopState& L = loop_state(ctx);
  if (!L.capturing) fail(USBS_ERR_CONFIG, "loop: usbs_loop_end without usbs_loop_begin");
  L.capturing = false;
  k_loop_cond<<<1, 32, 0, L.cap>>>(L.handle, red_dev, thresh, max_iters, counter_dev);
  cudaError_t e1 = cudaGetLastError();
  cudaGraph_t out = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(L.cap, &out);
  ctx->stream = L.saved;
  cudaGraphExec_t exec = nullptr;
  cudaError_t e3 = (e1 == cudaSuccess && e2 == cudaSuccess) ? cudaGraphInstantiate(&exec, L.graph, 0) : cudaSuccess;
  cudaError_t e4 = cudaSuccess;
  if (e1 == cudaSuccess && e2 == cudaSuccess && e3 == cudaSuccess) {
    e4 = cudaGraphLaunch(exec, ctx->stream);
    note_launch(ctx);
  }
  if (exec) cudaGraphExecDestroy(exec);  // deferred by the runtime until the launch has run
  cudaGraphDestroy(L.graph);
  L.graph = nullptr;
  L.body = nullptr;
  USBS_CUDA(e1);
  USBS_CUDA(e2);
  USBS_CUDA(e3);
  USBS_CUDA(e4);
  USBS_API_END
}

// Abandon a capture after an error inside the body (the stream leaves capture mode).
extern "C" usbs_status usbs_loop_abort(usbs_ctx* ctx) {
  USBS_API_BEGIN
  LoopState& L = loop_state(ctx);
  if (L.capturing) {
    cudaGraph_t out = nullptr;
    cudaStreamEndCapture(L.cap, &out);
    ctx->stream = L.saved;
    cudaGetLastError();
    if (L.graph) cudaGraphDestroy(L.graph);
    L.graph = nullptr;
    L.body = nullptr;
    L.capturing = false;
  }
  USBS_API_END
}
