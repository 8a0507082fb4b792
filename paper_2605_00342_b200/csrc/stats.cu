// stats.cu — A9 batch statistics (north_star: the only cross-GPU exchange is an
// all-reduce of these aggregates).  Grid-stride over trees, shared-memory
// partials, one global atomic per non-zero entry per CTA.
#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"
#include "evict_launch.h"

namespace evict {
// ------------------------------------------------------------ stats
// Scalars (k*, n, status, e_hat, utility) and the k* histogram: one thread per
// tree (coalesced), block partials in shared memory.  Per-layer union sums:
// one warp per tree row with lane = layer (coalesced row reads), register
// accumulators, one atomic per layer per warp at the end — never one shared
// atomic per (tree, layer).
__global__ void k_stats(int B, int N, int L, const int32_t *n_nodes, const int32_t *k_star,
                        const float *e_hat, const float *utility, const int32_t *union_count,
                        const uint32_t *status, unsigned long long *stats, double *dstats)
{
    extern __shared__ unsigned long long sh[];  // [6 + N + L]
    const int len = 6 + N + L;
    for (int i = threadIdx.x; i < len; i += blockDim.x) sh[i] = 0ull;
    __shared__ double sd[2];
    if (threadIdx.x < 2) sd[threadIdx.x] = 0.0;
    __syncthreads();
    unsigned long long nt = 0, sk = 0, sn = 0, su = 0, sbad = 0;
    double de = 0.0, du = 0.0;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
        nt++;
        if (status && status[b]) {
            sbad++;
            atomicAdd(&sh[5], 1ull);
            continue;
        }
        const int k = k_star[b];
        sk += k;
        sn += n_nodes ? n_nodes[b] : N;
        atomicAdd(&sh[5 + k], 1ull);
        de += e_hat[b];
        du += utility[b];
    }
    // per-layer sums: warp per tree row
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
    if (L > 0) {
        for (int b = gw; b < B; b += nw) {
            if (status && status[b]) continue;
            const int32_t *row = union_count + (size_t)b * L;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int l = lane + 32 * c;
                if (l < L) acc[c] += (unsigned long long)__ldg(row + l);
            }
        }
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int l = lane + 32 * c;
            if (l < L && acc[c]) {
                atomicAdd(&sh[6 + N + l], acc[c]);
                su += acc[c];
            }
        }
    }
    // warp-reduce the scalars, one shared atomic per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nt += __shfl_xor_sync(0xffffffffu, nt, o);
        sk += __shfl_xor_sync(0xffffffffu, sk, o);
        sn += __shfl_xor_sync(0xffffffffu, sn, o);
        su += __shfl_xor_sync(0xffffffffu, su, o);
        sbad += __shfl_xor_sync(0xffffffffu, sbad, o);
        de += __shfl_xor_sync(0xffffffffu, de, o);
        du += __shfl_xor_sync(0xffffffffu, du, o);
    }
    if (lane == 0) {
        atomicAdd(&sh[0], nt);
        atomicAdd(&sh[1], sk);
        atomicAdd(&sh[2], sn);
        atomicAdd(&sh[3], su);
        atomicAdd(&sh[4], sbad);
        atomicAdd(&sd[0], de);
        atomicAdd(&sd[1], du);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += blockDim.x)
        if (sh[i]) atomicAdd(&stats[i], sh[i]);
    if (threadIdx.x < 2) atomicAdd(&dstats[threadIdx.x], sd[threadIdx.x]);
}

}  // namespace evict

extern "C" evict_status_t evict_batch_stats(int32_t batch, int32_t max_nodes, int32_t num_layers,
                                            const int32_t *n_nodes, const int32_t *k_star,
                                            const float *e_hat, const float *utility,
                                            const int32_t *union_count, const uint32_t *status,
                                            int64_t *stats, double *dstats, void *stream)
{
    if (batch < 1 || max_nodes < 1 || max_nodes > EVICT_MAX_NODES || num_layers < 0 ||
        num_layers > EVICT_MAX_LAYERS)
        return EVICT_ERR_INVALID_ARG;
    if (!k_star || !e_hat || !utility || !stats || !dstats || (num_layers > 0 && !union_count))
        return EVICT_ERR_INVALID_ARG;
    const int sms = evict::dev_sms();
    if (sms <= 0) return EVICT_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int len = 6 + max_nodes + num_layers;
    if (cudaMemsetAsync(stats, 0, sizeof(int64_t) * len, s) != cudaSuccess) return EVICT_ERR_CUDA;
    if (cudaMemsetAsync(dstats, 0, sizeof(double) * 2, s) != cudaSuccess) return EVICT_ERR_CUDA;
    int blocks = (batch + 255) / 256;
    if (blocks > sms * 2) blocks = sms * 2;
    evict::k_stats<<<blocks, 256, sizeof(unsigned long long) * len, s>>>(
        batch, max_nodes, num_layers, n_nodes, k_star, e_hat, utility, union_count, status,
        reinterpret_cast<unsigned long long *>(stats), dstats);
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
