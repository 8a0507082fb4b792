// dispatch.cu — NEXT-4: on-device verify-graph dispatch.
//
// SGLang pre-captures one verify graph per verification length
// and "dispatch[es] the one matching the selected length" — on the host, which
// needs k* (device) on the host first: a device→host sync per decoding step.
// Here the choice stays on the device: one CUDA graph
//
//     [optional pre graph] → k_dispatch → SWITCH(handle) { body 0 | … | body n−1 }
//
// k_dispatch (one thread) reads the verify row count T the step produced
// (e.g. verify_offsets[B] of evict_build_verify_tree / the fused call), picks the
// smallest captured length ≥ T and sets the switch value with
// cudaGraphSetConditional; the switch node then runs that body (a clone of the
// caller's captured verify graph) — no host round trip between selection and
// verification.  The pre graph (e.g. the captured draft + EVICT step) runs
// first in the same launch.
#include <cuda_runtime.h>
#include <stdint.h>

#include <new>

#include "evict.h"
#include "evict_launch.h"

struct evict_dispatch_s {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
};

namespace evict {
namespace dispatch {

struct Lengths {
    int32_t n;
    int32_t v[EVICT_DISPATCH_MAX];
};

__global__ void k_dispatch(cudaGraphConditionalHandle h, const int32_t *rows, Lengths lens, int32_t *chosen)
{
    const int32_t T = *rows;
    int idx = lens.n;                       // ≥ size: the switch runs no body
    for (int i = lens.n - 1; i >= 0; i--)
        if (lens.v[i] >= T) idx = i;        // lengths ascending: the smallest one ≥ T
    cudaGraphSetConditional(h, (unsigned)idx);
    if (chosen) *chosen = idx < lens.n ? idx : -1;
}

}  // namespace dispatch
}  // namespace evict

using namespace evict::dispatch;

extern "C" evict_status_t evict_dispatch_create(int32_t n_bodies, const int32_t *lengths, void *const *body_graphs,
                                                void *pre_graph, const int32_t *rows, int32_t *chosen,
                                                evict_dispatch_t *out)
{
    if (!out) return EVICT_ERR_INVALID_ARG;
    *out = nullptr;
    if (n_bodies < 1 || n_bodies > EVICT_DISPATCH_MAX || !lengths || !body_graphs || !rows) return EVICT_ERR_INVALID_ARG;
    Lengths lens{};
    lens.n = n_bodies;
    for (int i = 0; i < n_bodies; i++) {
        if (!body_graphs[i] || lengths[i] < 0 || (i && lengths[i] <= lengths[i - 1])) return EVICT_ERR_INVALID_ARG;
        lens.v[i] = lengths[i];
    }
    if (!evict::dev_supported()) return EVICT_ERR_UNSUPPORTED;
    evict_dispatch_s *d = new (std::nothrow) evict_dispatch_s();
    if (!d) return EVICT_ERR_CUDA;
    auto fail = [&](void) {
        if (d->exec) cudaGraphExecDestroy(d->exec);
        if (d->graph) cudaGraphDestroy(d->graph);
        delete d;
        return EVICT_ERR_CUDA;
    };
    if (cudaGraphCreate(&d->graph, 0) != cudaSuccess) return fail();
    cudaGraphConditionalHandle h;
    // default value n_bodies (no body) is re-applied at every launch
    if (cudaGraphConditionalHandleCreate(&h, d->graph, (unsigned)n_bodies, cudaGraphCondAssignDefault) != cudaSuccess)
        return fail();
    cudaGraphNode_t pre = nullptr, kn = nullptr, cn = nullptr;
    if (pre_graph && cudaGraphAddChildGraphNode(&pre, d->graph, nullptr, 0, (cudaGraph_t)pre_graph) != cudaSuccess)
        return fail();
    void *args[] = {&h, (void *)&rows, &lens, (void *)&chosen};
    cudaKernelNodeParams kp = {};
    kp.func = (void *)k_dispatch;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    if (cudaGraphAddKernelNode(&kn, d->graph, pre ? &pre : nullptr, pre ? 1 : 0, &kp) != cudaSuccess) return fail();
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeSwitch;
    cp.conditional.size = (unsigned)n_bodies;
    if (cudaGraphAddNode(&cn, d->graph, &kn, 1, &cp) != cudaSuccess) return fail();
    for (int i = 0; i < n_bodies; i++) {
        cudaGraphNode_t child;
        if (cudaGraphAddChildGraphNode(&child, cp.conditional.phGraph_out[i], nullptr, 0,
                                       (cudaGraph_t)body_graphs[i]) != cudaSuccess)
            return fail();
    }
    if (cudaGraphInstantiate(&d->exec, d->graph, 0) != cudaSuccess) return fail();
    *out = d;
    return EVICT_OK;
}

extern "C" evict_status_t evict_dispatch_launch(evict_dispatch_t d, void *stream)
{
    if (!d || !d->exec) return EVICT_ERR_INVALID_ARG;
    return cudaGraphLaunch(d->exec, (cudaStream_t)stream) == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}

extern "C" void evict_dispatch_destroy(evict_dispatch_t d)
{
    if (!d) return;
    if (d->exec) cudaGraphExecDestroy(d->exec);
    if (d->graph) cudaGraphDestroy(d->graph);
    delete d;
}
