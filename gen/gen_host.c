/* gen_host.c — host build of the seeded workload generator (evict_gen.h).
 * Compiled with gcc -O2 -ffp-contract=off -fno-fast-math so every fp64
 * operation is a single correctly-rounded IEEE operation, identical to the
 * __dmul_rn/__dadd_rn/__ddiv_rn the device build uses. */
#include <stdlib.h>
#include <string.h>

#include "evict_gen.h"

int gen_abi_version(void) { return 1; }

/* trees [tree_base, tree_base + B): parent/q [B][N], n_nodes [B] */
void gen_trees_host(uint64_t seed, uint64_t tree_base, int B, int steps, int topk, int N,
                    int m_lo, int m_hi, int32_t *parent, float *q, int32_t *n_nodes)
{
    gen_tree_scratch *s = (gen_tree_scratch *)malloc(sizeof(gen_tree_scratch));
    for (int b = 0; b < B; b++)
        n_nodes[b] = gen_tree(seed, tree_base + (uint64_t)b, steps, topk, N, m_lo, m_hi,
                              parent + (size_t)b * N, q + (size_t)b * N, s);
    free(s);
}

/* routing ids [B][N][L][K] as uint8 (id_bytes 1) or int32 (id_bytes 4) */
void gen_routing_host(uint64_t seed, uint64_t tree_base, int B, int N, int L, int E, int K,
                      int sigma_q4, int id_bytes, void *out)
{
    int32_t ids[GEN_MAX_K];
    for (int b = 0; b < B; b++)
        for (int v = 0; v < N; v++)
            for (int l = 0; l < L; l++) {
                gen_route(seed, tree_base + (uint64_t)b, v, l, E, K, sigma_q4, ids);
                size_t o = (((size_t)b * N + v) * L + l) * K;
                for (int j = 0; j < K; j++) {
                    if (id_bytes == 1) ((uint8_t *)out)[o + j] = (uint8_t)ids[j];
                    else ((int32_t *)out)[o + j] = ids[j];
                }
            }
}

/* hidden states [L][B*N][d] bf16 bits; row = b*N + v of trees tree_base.. */
void gen_hidden_host(uint64_t seed, uint64_t tree_base, int B, int N, int L, int d, int mode,
                     uint16_t *out)
{
    for (int l = 0; l < L; l++)
        for (int b = 0; b < B; b++)
            for (int v = 0; v < N; v++) {
                uint64_t key = ((tree_base + (uint64_t)b) * 256u + (uint64_t)v) * 1024u + (uint64_t)l;
                size_t o = (((size_t)l * B + b) * N + v) * d;
                for (int i = 0; i < d; i++)
                    out[o + i] = gen_bf16_value(seed, GEN_S_HID, key, (uint64_t)i, mode, 0);
            }
}

/* router weights [L][E][d] bf16 bits */
void gen_wgate_host(uint64_t seed, int L, int E, int d, int mode, int scale_log2, uint16_t *out)
{
    for (int l = 0; l < L; l++)
        for (int e = 0; e < E; e++)
            for (int i = 0; i < d; i++)
                out[((size_t)l * E + e) * d + i] =
                    gen_bf16_value(seed, GEN_S_WG, (uint64_t)l * 1024u + (uint64_t)e, (uint64_t)i,
                                   mode, scale_log2);
}
