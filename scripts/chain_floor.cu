// chain_floor.cu -- the per-step latency floor of back-to-back small kernels on one B200, for
// config 2 (4,096 envs: 128 CTAs of the latency step kernel, 3.2 us per step).  Measurement tool,
// not part of the product path.  Each variant captures 100 launches of a 128-CTA x 256-thread
// kernel into a CUDA graph and replays it; us per launch = replay time / 100 (best of 20 replays).
//   plain        : ordinary stream order (a launch starts after the previous grid completes)
//   pdl_wait     : programmatic dependent launch, griddepcontrol.wait at the start (the next grid
//                  is resident early, runs after the previous grid's completion and flush)
//   chained      : the step kernels' protocol -- a ticket atomic gives the step index t, CTA c polls
//                  the same-index CTA of the previous launch (ld.acquire.gpu on ready[c] == t),
//                  triggers the next launch, writes, and publishes ready[c] = t + 1 (st.release.gpu
//                  after the CTA barrier); no griddepcontrol.wait
// each with work = 0 (no stores) or a config-2-sized store set: 32 envs x 60 words of state per CTA
// (the state planes the step rewrites: one read round trip, then the stores), coalesced, between the
// wait and the publish.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o chain_floor chain_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

constexpr int CTAS = 128, THREADS = 256, WORDS = 32 * 60;

__device__ __forceinline__ unsigned ld_acq(const unsigned* q) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(q) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(unsigned* q, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(q), "r"(v) : "memory");
}

// mode 0 plain, 1 pdl_wait, 2 chained
template <int MODE, int WORK>
__global__ void __launch_bounds__(THREADS) step_like(unsigned long long* ticket, unsigned* ready, float* state) {
    __shared__ unsigned s_t;
    if (MODE == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        const unsigned t = (unsigned)(atomicAdd(ticket, 1ull) / gridDim.x);
        if (MODE == 2)
            while (ld_acq(ready + blockIdx.x) != t) __nanosleep(64);
        s_t = t;
    }
    __syncthreads();
    if (MODE != 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const unsigned t = s_t;
    if (WORK) {   // one read round trip of the CTA's state (all loads issued together), then the stores
        float* __restrict__ S = state + (size_t)blockIdx.x * WORDS;
        constexpr int PER = (WORDS + THREADS - 1) / THREADS;
        float v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = threadIdx.x + k * THREADS;
            v[k] = i < WORDS ? __ldcg(S + i) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = threadIdx.x + k * THREADS;
            if (i < WORDS) S[i] = v[k] * 0.5f + (float)t;
        }
    }
    __syncthreads();
    if (MODE == 2 && threadIdx.x == 0) st_rel(ready + blockIdx.x, t + 1u);
}

template <int MODE, int WORK>
static double run(cudaStream_t s, unsigned long long* ticket, unsigned* ready, float* state) {
    CK(cudaMemsetAsync(ticket, 0, 8, s));
    CK(cudaMemsetAsync(ready, 0, CTAS * 4, s));
    CK(cudaStreamSynchronize(s));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < 100; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CTAS);
        cfg.blockDim = dim3(THREADS);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = MODE == 0 ? 0 : 1;
        CK(cudaLaunchKernelEx(&cfg, step_like<MODE, WORK>, ticket, ready, state));
    }
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int w = 0; w < 5; ++w) CK(cudaGraphLaunch(ge, s));
    float best = 1e30f;
    for (int r = 0; r < 20; ++r) {
        CK(cudaEventRecord(e0, s));
        CK(cudaGraphLaunch(ge, s));
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
    return best * 1e3 / 100.0;   // us per launch
}

int main() {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    unsigned long long* ticket;
    unsigned* ready;
    float* state;
    CK(cudaMalloc(&ticket, 8));
    CK(cudaMalloc(&ready, CTAS * 4));
    CK(cudaMalloc(&state, (size_t)CTAS * WORDS * 4));
    CK(cudaMemset(state, 0, (size_t)CTAS * WORDS * 4));
    printf("{\"probe\": \"chain_floor\", \"ctas\": %d, \"threads\": %d, \"us_per_launch\": {"
           "\"plain\": %.3f, \"plain_work\": %.3f, \"pdl_wait\": %.3f, \"pdl_wait_work\": %.3f, "
           "\"chained\": %.3f, \"chained_work\": %.3f}}\n",
           CTAS, THREADS, run<0, 0>(s, ticket, ready, state), run<0, 1>(s, ticket, ready, state),
           run<1, 0>(s, ticket, ready, state), run<1, 1>(s, ticket, ready, state),
           run<2, 0>(s, ticket, ready, state), run<2, 1>(s, ticket, ready, state));
    return 0;
}
