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
// tree (coalesced); histogram increments are warp-aggregated (__match_any_sync:
// one shared atomic per distinct bin per warp, not per tree).  Per-layer union
// sums: one warp per tree row with lane = layer (coalesced row reads), 4 rows in
// flight per warp, register accumulators, one atomic per layer per warp at the end.
__global__ void __launch_bounds__(256) k_stats(int B, int N, int L, const int32_t *n_nodes, const int32_t *k_star,
                                               const float *e_hat, const float *utility,
                                               const int32_t *union_count, const uint32_t *status,
                                               unsigned long long *stats, double *dstats)
{
    extern __shared__ unsigned long long sh[];  // [6 + N + L]
    const int len = 6 + N + L;
    for (int i = threadIdx.x; i < len; i += blockDim.x) sh[i] = 0ull;
    __shared__ double sd[2];
    if (threadIdx.x < 2) sd[threadIdx.x] = 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned long long nt = 0, sk = 0, sn = 0, su = 0, sbad = 0;
    double de = 0.0, du = 0.0;
    const int stride = gridDim.x * blockDim.x;
    for (int b0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); b0 < B; b0 += stride) {
        const int b = b0 + lane;                       // warp-uniform loop, lane-valid trees
        const bool in = b < B;
        const bool bad = in && status && status[b];
        const int k = (in && !bad) ? k_star[b] : 0;
        if (in) {
            nt++;
            if (bad) {
                sbad++;
            } else {
                sk += k;
                sn += n_nodes ? n_nodes[b] : N;
                de += e_hat[b];
                du += utility[b];
            }
        }
        // histogram bin 0 = errored trees, k otherwise; warp-aggregated
        const int bin = in ? (bad ? 0 : k) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (in && lane == __ffs(peers) - 1) atomicAdd(&sh[5 + bin], (unsigned long long)__popc(peers));
    }
    // per-layer sums: warp per tree row, 4 rows in flight
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
    if (L > 0) {
        for (int b = gw; b < B; b += 4 * nw) {
            int32_t v[4][4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int bu = b + u * nw;
                const bool ok = bu < B && !(status && status[bu]);
                const int32_t *row = union_count + (size_t)(ok ? bu : 0) * L;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const int l = lane + 32 * c;
                    v[u][c] = (ok && l < L) ? __ldg(row + l) : 0;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int c = 0; c < 4; c++) acc[c] += (unsigned long long)v[u][c];
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
    if (sms <= 0 || !evict::dev_supported()) return EVICT_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int len = 6 + max_nodes + num_layers;
    if (cudaMemsetAsync(stats, 0, sizeof(int64_t) * len, s) != cudaSuccess) return EVICT_ERR_CUDA;
    if (cudaMemsetAsync(dstats, 0, sizeof(double) * 2, s) != cudaSuccess) return EVICT_ERR_CUDA;
    int blocks = (batch + 255) / 256;
    if (blocks > sms * 8) blocks = sms * 8;   // 64 warps per SM of loads in flight
    evict::k_stats<<<blocks, 256, sizeof(unsigned long long) * len, s>>>(
        batch, max_nodes, num_layers, n_nodes, k_star, e_hat, utility, union_count, status,
        reinterpret_cast<unsigned long long *>(stats), dstats);
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
