/*
 * gids_minimal.c -- the C ABI driven from plain C (no Python, no torch):
 * a 6-node graph, one sampled batch, one served batch, tier counts printed.
 * This is what a binding in another host language wraps.
 *
 *   gcc -std=c11 -I include examples/gids_minimal.c \
 *       -L paper_2306_16384_b200 -lgids -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2306_16384_b200 -o gids_minimal && ./gids_minimal
 */
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "gids.h"

#define CK(x)                                                                    \
    do {                                                                         \
        int rc_ = (x);                                                           \
        if (rc_) {                                                               \
            fprintf(stderr, "%s -> %d: %s\n", #x, rc_, gids_last_error());       \
            return 1;                                                            \
        }                                                                        \
    } while (0)

int main(void) {
    /* in-neighbour CSC of 6 nodes (graph.py:46-71): sources ascending per node */
    const uint64_t indptr[7] = {0, 2, 4, 6, 8, 10, 12};
    const uint64_t indices[12] = {1, 2, 0, 3, 0, 4, 1, 5, 2, 5, 3, 4};
    const int dim = 4;
    float* table;  /* storage tier: pinned host rows, read zero-copy */
    if (cudaMallocHost((void**)&table, sizeof(float) * 6 * dim)) return 1;
    for (int i = 0; i < 6 * dim; i++) table[i] = (float)i;

    gids_config cfg = {0};
    cfg.num_nodes = 6;
    cfg.num_edges = 12;
    cfg.feature_dim = dim;
    cfg.device = 0;
    cfg.cache_lines = 3;
    cfg.policy = GIDS_POLICY_EXACT;
    cfg.ways = 32;
    cfg.window_depth = 2;
    cfg.n_layers = 2;
    cfg.fanouts[0] = 2;
    cfg.fanouts[1] = 2;
    cfg.max_seeds = 2;
    /* eviction stream: a PCG64 state (numpy default_rng words) */
    const uint64_t evict_rng[6] = {0x1234, 0x5678, 0x9abc, 0xdef1, 0, 0};
    const uint64_t sampler_rng[6] = {0x1111, 0x2222, 0x3333, 0x4445, 0, 0};

    gids_handle* h = NULL;
    CK(gids_create(&cfg, evict_rng, &h));
    CK(gids_load_graph(h, indptr, indices));
    CK(gids_set_backing(h, table, 6));
    CK(gids_set_constant_buffer(h, NULL, 0, NULL));

    const int64_t seeds[2] = {0, 3};
    CK(gids_sample(h, seeds, 2, sampler_rng, 0));
    int64_t layer_len[2], n_unique, draws, contribution;
    CK(gids_sample_sizes(h, layer_len, &n_unique, &draws, &contribution));
    int64_t *edges_dev, *unique_dev;
    float* rows_dev;
    if (cudaMalloc((void**)&edges_dev, sizeof(int64_t) * 2 * (layer_len[0] + layer_len[1]) + 16) ||
        cudaMalloc((void**)&unique_dev, sizeof(int64_t) * n_unique) ||
        cudaMalloc((void**)&rows_dev, sizeof(float) * n_unique * dim))
        return 1;
    CK(gids_sample_export(h, edges_dev, unique_dev, 0));
    CK(gids_serve(h, unique_dev, n_unique, 0, rows_dev, 0, 0));
    gids_tier_counts t;
    CK(gids_serve_counts(h, &t));
    if (cudaDeviceSynchronize()) return 1;
    printf("unique=%lld draws=%lld hits=%lld buffer=%lld storage=%lld bypasses=%lld\n",
           (long long)n_unique, (long long)draws, (long long)t.cache_hits,
           (long long)t.cpu_buffer_hits, (long long)t.storage, (long long)t.bypasses);
    CK(gids_destroy(h));
    return t.sampled == n_unique ? 0 : 1;
}
