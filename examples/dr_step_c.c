/*
 * dr_step_c.c -- the C-ABI of libdr.so used from plain C (no Python, no torch): create a context
 * for 4,096 envs with the paper's parameters, run 100 steps of the full pipeline on device
 * buffers, reset every 10th env half-way, read back the per-step stats, and print them.
 *
 *   gcc -std=c99 -O2 examples/dr_step_c.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1906_11633_b200 -ldr -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1906_11633_b200 \
 *       -o examples/dr_step_c
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "dr.h"

#define CHECK(x)                                                                       \
    do {                                                                               \
        int rc_ = (x);                                                                 \
        if (rc_ != DR_OK) {                                                            \
            fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, dr_last_error());       \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

int main(void)
{
    const int64_t n = 4096;
    dr_params p;
    float *act, *obs, *oa, *oo, *odt, *of;
    uint8_t* mask;
    double stats[DR_N_STATS];
    int t, i;
    float* h_act = (float*)malloc(sizeof(float) * n * DR_N_ACT);
    float* h_obs = (float*)malloc(sizeof(float) * n * DR_OBS_IN);
    uint8_t* h_mask = (uint8_t*)malloc((size_t)n);
    /* inputs: actions on the paper's 11-bin grid, fingertips near the palm, unit quaternions */
    srand(1906);
    for (i = 0; i < n * DR_N_ACT; ++i) h_act[i] = -1.0f + (2.0f * (float)(rand() % 11) + 1.0f) / 11.0f;
    for (i = 0; i < n; ++i) {
        int c;
        for (c = 0; c < 15; ++c) h_obs[i * DR_OBS_IN + c] = 0.02f * (float)(c % 5) + 0.001f * (float)(rand() % 10);
        for (c = 15; c < 18; ++c) h_obs[i * DR_OBS_IN + c] = 0.03f;
        for (c = 18; c < 26; ++c) h_obs[i * DR_OBS_IN + c] = (c == 18 || c == 22) ? 1.0f : 0.0f;
        h_mask[i] = (uint8_t)(i % 10 == 0);
    }
    cudaMalloc((void**)&act, sizeof(float) * n * DR_N_ACT);
    cudaMalloc((void**)&obs, sizeof(float) * n * DR_OBS_IN);
    cudaMalloc((void**)&oa, sizeof(float) * n * DR_N_ACT);
    cudaMalloc((void**)&oo, sizeof(float) * n * DR_OBS_OUT);
    cudaMalloc((void**)&odt, sizeof(float) * n * DR_N_SUBSTEPS);
    cudaMalloc((void**)&of, sizeof(float) * n * 3);
    cudaMalloc((void**)&mask, (size_t)n);
    cudaMemcpy(act, h_act, sizeof(float) * n * DR_N_ACT, cudaMemcpyHostToDevice);
    cudaMemcpy(obs, h_obs, sizeof(float) * n * DR_OBS_IN, cudaMemcpyHostToDevice);
    cudaMemcpy(mask, h_mask, (size_t)n, cudaMemcpyHostToDevice);

    CHECK(dr_params_default(&p));
    CHECK(dr_init(&p, n, 1906011633ull));
    for (t = 0; t < 100; ++t) {
        if (t == 50) CHECK(dr_reset(mask));
        CHECK(dr_step(act, obs, oa, oo, odt, of));
    }
    CHECK(dr_synchronize());
    cudaMemcpy(stats, dr_stats((int)((dr_step_index() - 1) % DR_STAT_SLOTS)), sizeof(stats), cudaMemcpyDeviceToHost);
    printf("steps %llu  envs %.0f  delayed %.0f  dropout starts %.0f  masked %.0f  occluded %.0f  held %.0f  "
           "force triggers %.0f  resets(last step) %.0f  mean dt_env %.6f s\n",
           (unsigned long long)dr_step_index(), stats[DR_S_ENVS], stats[DR_S_DELAYED], stats[DR_S_DROP_INIT],
           stats[DR_S_MASKED], stats[DR_S_OCCLUDED], stats[DR_S_HELD], stats[DR_S_FORCE_TRIG], stats[DR_S_RESETS],
           stats[DR_S_SUM_DT] / stats[DR_S_ENVS]);
    CHECK(dr_finalize());
    return (stats[DR_S_ENVS] == (double)n) ? 0 : 2;
}
