// bw_ceiling.cu -- HBM ceilings of the read/write mixes the libdr kernels run (measurement tool,
// not part of the product path).  MEASURED_PEAKS.json's hbm_gbs is torch's copy_ (a 50/50 mix);
// the vision augmentation reads 1 byte per 4 written (u8 in, fp32 out) and the step kernel reads
// 768 B per 460 B written, so each gets the best of a family of plain streaming
// kernels with its own mix as a second denominator.
//
// Kernel: item i of N moves RV 16-byte words in (plane j at in[j N + i]) and WV 16-byte words out
// (plane j at out[j N + i]) -- every access a coalesced 128-bit load / store; the stored values
// depend on the loaded ones (no dead loads).  Variants: grid (k x SMs CTAs of 256 threads,
// grid-stride, or one item per thread) x store policy (default / .cs streaming).  Each launch moves
// `bytes_per_launch`; a ring of input/output buffers keeps the working set above L2.  Time: CUDA
// events around `reps` back-to-back launches, best of 5 runs.  Output: one JSON line per mix.
//
// usage: bw_ceiling [GB per launch] [ring] [reps] [pdl 0|1]
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bw_ceiling bw_ceiling.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <string>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

template <int CS>
__device__ __forceinline__ void st16(uint4* p, uint4 v) {
    if (CS) asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    else asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// PDL (programmatic dependent launch, as the vision and step kernels use): the next launch may start
// once every CTA of this one has begun; each CTA waits for the previous grid before it exits (the
// ring's buffers are disjoint, so the early reads and writes are safe, as in dr_vision.cu's rule).
// Small grids let several launches be resident at once: the ring must exceed that depth (use >= 8)
// or concurrent launches share buffers through L2.
template <int RV, int WV, int CS, int PDL>
__global__ void __launch_bounds__(256) mix_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n,
                                                  uint32_t salt, uint32_t* sink) {
    if (PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint4 a = make_uint4(salt, salt, salt, salt);
        uint4 r[RV > 0 ? RV : 1];
#pragma unroll
        for (int j = 0; j < RV; ++j) r[j] = __ldcs(in + (size_t)j * n + i);
#pragma unroll
        for (int j = 0; j < RV; ++j) { a.x ^= r[j].x; a.y ^= r[j].y; a.z ^= r[j].z; a.w ^= r[j].w; }
        if (WV == 0) {
            if ((a.x ^ a.y ^ a.z ^ a.w) == 0x9E3779B9u) atomicAdd(sink, 1u);   // keeps the loads live
        }
#pragma unroll
        for (int j = 0; j < WV; ++j) st16<CS>(out + (size_t)j * n + i, make_uint4(a.x + j, a.y, a.z, a.w));
    }
    if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
}

static int g_pdl = 0;
template <int RV, int WV, int CS>
static void launch(int grid, const uint4* in, uint4* out, size_t n, uint32_t* sink) {
    if (!g_pdl) {
        mix_kernel<RV, WV, CS, 0><<<grid, 256>>>(in, out, n, 1u, sink);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, mix_kernel<RV, WV, CS, 1>, in, out, n, 1u, sink);
}

template <int RV, int WV>
static float run(int cs, int grid, const uint4* in, uint4* out, size_t n, uint32_t* sink) {
    if (cs) launch<RV, WV, 1>(grid, in, out, n, sink);
    else launch<RV, WV, 0>(grid, in, out, n, sink);
    return 0.f;
}

typedef float (*RunFn)(int, int, const uint4*, uint4*, size_t, uint32_t*);

int main(int argc, char** argv) {
    const double gb_launch = argc > 1 ? atof(argv[1]) : 1.0;   // GB moved per launch
    const int ring = argc > 2 ? atoi(argv[2]) : 2;
    const int reps = argc > 3 ? atoi(argv[3]) : 20;
    g_pdl = argc > 4 ? atoi(argv[4]) : 0;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    struct M { const char* name; int rv, wv; RunFn fn; };
    const M mixes[] = {
        {"copy_1r_1w", 1, 1, run<1, 1>},
        {"vision_1r_4w", 1, 4, run<1, 4>},
        {"step_5r_3w", 5, 3, run<5, 3>},
        {"read_only", 1, 0, run<1, 0>},
        {"write_only", 0, 1, run<0, 1>},
    };
    uint32_t* sink;
    CK(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (const M& m : mixes) {
        const size_t words = (size_t)(gb_launch * 1e9 / 16.0 / (m.rv + m.wv));
        const size_t n = words;
        std::vector<uint4*> ins(ring, nullptr), outs(ring, nullptr);
        for (int r = 0; r < ring; ++r) {
            if (m.rv) { CK(cudaMalloc(&ins[r], n * m.rv * 16)); CK(cudaMemset(ins[r], r + 1, n * m.rv * 16)); }
            if (m.wv) { CK(cudaMalloc(&outs[r], n * m.wv * 16)); }
        }
        const double bytes = (double)n * 16.0 * (m.rv + m.wv);
        double best_gbs = 0;
        char best_cfg[64] = "";
        const int grids_k[] = {2, 4, 8, 16, 0};   // 0: one item per thread
        for (int cs = 0; cs < 2; ++cs) {
            for (int gk : grids_k) {
                const int grid = gk ? gk * sms : (int)std::min<size_t>((n + 255) / 256, 0x7fffffff);
                for (int r = 0; r < ring; ++r) m.fn(cs, grid, ins[r], outs[r], n, sink);   // warm
                CK(cudaDeviceSynchronize());
                float best_ms = 1e30f;
                for (int run = 0; run < 5; ++run) {
                    CK(cudaEventRecord(e0));
                    for (int i = 0; i < reps; ++i) m.fn(cs, grid, ins[i % ring], outs[i % ring], n, sink);
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0, e1));
                    best_ms = std::min(best_ms, ms / reps);
                }
                CK(cudaGetLastError());
                const double gbs = bytes / (best_ms * 1e-3) / 1e9;
                printf("  %-13s cs=%d grid=%-6s %8.3f us  %7.1f GB/s\n", m.name, cs, gk ? std::to_string(gk).c_str() : "full",
                       best_ms * 1e3, gbs);
                if (gbs > best_gbs) {
                    best_gbs = gbs;
                    snprintf(best_cfg, sizeof best_cfg, "cs=%d grid=%s", cs, gk ? std::to_string(gk * sms).c_str() : "full");
                }
            }
        }
        printf("{\"mix\": \"%s\", \"pdl\": %d, \"read_16B\": %d, \"write_16B\": %d, \"bytes_per_launch\": %.0f, \"ring\": %d, "
               "\"best_gbs\": %.1f, \"best\": \"%s\"}\n", m.name, g_pdl, m.rv, m.wv, bytes, ring, best_gbs, best_cfg);
        fflush(stdout);
        for (int r = 0; r < ring; ++r) { cudaFree(ins[r]); cudaFree(outs[r]); }
    }
    return 0;
}
