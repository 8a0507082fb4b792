// gen_cuda.cu — device build of the seeded workload generator (evict_gen.h).
// Bit-identical to gen_host.c (see evict_gen.h); used by bench.py to create
// device-resident inputs (the C5 sweep's 23 GB of routing ids cannot be made
// on the host in reasonable time).  No method arithmetic lives here.
#include <cuda_runtime.h>
#include <stdint.h>

#include "evict_gen.h"

namespace {

__global__ void k_trees(uint64_t seed, uint64_t tree_base, int B, int steps, int topk, int N,
                        int m_lo, int m_hi, int32_t *parent, float *q, int32_t *n_nodes,
                        gen_tree_scratch *scratch, int nscratch)
{
    int tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= nscratch) return;
    gen_tree_scratch *s = scratch + tid;
    for (int b = tid; b < B; b += nscratch)
        n_nodes[b] = gen_tree(seed, tree_base + (uint64_t)b, steps, topk, N, m_lo, m_hi,
                              parent + (size_t)b * N, q + (size_t)b * N, s);
}

__global__ void k_routing(uint64_t seed, uint64_t tree_base, int B, int N, int L, int E, int K,
                          int sigma_q4, int id_bytes, void *out)
{
    size_t total = (size_t)B * N * L;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        int l = (int)(t % L);
        size_t bv = t / L;
        int v = (int)(bv % N);
        size_t b = bv / N;
        int32_t ids[GEN_MAX_K];
        gen_route(seed, tree_base + b, v, l, E, K, sigma_q4, ids);
        size_t o = t * K;
        if (id_bytes == 1) {
            uint8_t *p = (uint8_t *)out + o;
            for (int j = 0; j < K; j++) p[j] = (uint8_t)ids[j];
        } else {
            int32_t *p = (int32_t *)out + o;
            for (int j = 0; j < K; j++) p[j] = ids[j];
        }
    }
}

__global__ void k_hidden(uint64_t seed, uint64_t tree_base, int B, int N, int L, int d, int mode,
                         uint16_t *out)
{
    size_t total = (size_t)L * B * N * d;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        int i = (int)(t % d);
        size_t r = t / d;  // (l*B + b)*N + v
        int v = (int)(r % N);
        size_t lb = r / N;
        size_t b = lb % B;
        int l = (int)(lb / B);
        uint64_t key = ((tree_base + b) * 256u + (uint64_t)v) * 1024u + (uint64_t)l;
        out[t] = gen_bf16_value(seed, GEN_S_HID, key, (uint64_t)i, mode, 0);
    }
}

__global__ void k_wgate(uint64_t seed, int L, int E, int d, int mode, int scale_log2, uint16_t *out)
{
    size_t total = (size_t)L * E * d;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        int i = (int)(t % d);
        size_t le = t / d;
        out[t] = gen_bf16_value(seed, GEN_S_WG, (uint64_t)(le / E) * 1024u + (uint64_t)(le % E),
                                (uint64_t)i, mode, scale_log2);
    }
}

__global__ void k_ids_to_mask(const uint8_t *ids, size_t rows, int K, int EW, uint64_t *mask)
{
    for (size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x; r < rows;
         r += (size_t)gridDim.x * blockDim.x) {
        uint64_t m[4] = {0, 0, 0, 0};
        for (int j = 0; j < K; j++) {
            int e = ids[r * K + j];
            m[e >> 6] |= 1ull << (e & 63);
        }
        for (int w = 0; w < EW; w++) mask[r * EW + w] = m[w];
    }
}

}  // namespace

extern "C" {

// one-hot routing masks [rows][EW] from uint8 ids [rows][K] (input re-encoding)
int gen_ids_to_mask_cuda(const void *ids, size_t rows, int K, int EW, void *mask, cudaStream_t stream)
{
    k_ids_to_mask<<<148 * 16, 256, 0, stream>>>((const uint8_t *)ids, rows, K, EW, (uint64_t *)mask);
    return (int)cudaGetLastError();
}


int gen_cuda_abi_version(void) { return 1; }

// scratch: device buffer of nscratch * sizeof(gen_tree_scratch) bytes
size_t gen_tree_scratch_bytes(void) { return sizeof(gen_tree_scratch); }

int gen_trees_cuda(uint64_t seed, uint64_t tree_base, int B, int steps, int topk, int N,
                   int m_lo, int m_hi, int32_t *parent, float *q, int32_t *n_nodes,
                   void *scratch, int nscratch, cudaStream_t stream)
{
    int threads = 128;
    int blocks = (nscratch + threads - 1) / threads;
    k_trees<<<blocks, threads, 0, stream>>>(seed, tree_base, B, steps, topk, N, m_lo, m_hi, parent,
                                            q, n_nodes, (gen_tree_scratch *)scratch, nscratch);
    return (int)cudaGetLastError();
}

int gen_routing_cuda(uint64_t seed, uint64_t tree_base, int B, int N, int L, int E, int K,
                     int sigma_q4, int id_bytes, void *out, cudaStream_t stream)
{
    k_routing<<<148 * 16, 256, 0, stream>>>(seed, tree_base, B, N, L, E, K, sigma_q4, id_bytes, out);
    return (int)cudaGetLastError();
}

int gen_hidden_cuda(uint64_t seed, uint64_t tree_base, int B, int N, int L, int d, int mode,
                    uint16_t *out, cudaStream_t stream)
{
    k_hidden<<<148 * 16, 256, 0, stream>>>(seed, tree_base, B, N, L, d, mode, out);
    return (int)cudaGetLastError();
}

int gen_wgate_cuda(uint64_t seed, int L, int E, int d, int mode, int scale_log2, uint16_t *out,
                   cudaStream_t stream)
{
    k_wgate<<<148 * 16, 256, 0, stream>>>(seed, L, E, d, mode, scale_log2, out);
    return (int)cudaGetLastError();
}

}  // extern "C"
