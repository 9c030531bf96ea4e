// launch_gap.cu -- back-to-back PDL launches of a 1-CTA-per-SM kernel (like bitgemm_tc_kernel):
// how long after a CTA exits does the next grid's CTA start on the same SM, and when does the
// next grid's griddepcontrol.wait return (relative to the last CTA end of the previous grid)?
// Variants: V0 spin only; V1 + TMEM alloc/dealloc 512; V2 + 1-D bulk-copy stream of a 1 GiB
// buffer through a 13 x 16 KiB SMEM ring (HBM saturated); V3 = V2 + y-like global stores at the
// end; SM = dynamic SMEM bytes.  8 launches captured in a CUDA graph (PDL attribute, early
// trigger).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lg launch_gap.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ long long gt() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Rec { long long start, wait_done, end; int sm, pad; };

template <int V>
__global__ void __launch_bounds__(480, 1) k(Rec* rec, const uint8_t* src, size_t per_cta, float* ydump, int call) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[13];
    __shared__ uint32_t tb;
    const long long t0 = gt();
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0)
        for (int i = 0; i < 13; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
    if (V >= 1 && warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;");
    long long tw = 0;
    if (threadIdx.x == 0) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        tw = gt();
    }
    if (V >= 2 && threadIdx.x == 0) {
        // stream per_cta bytes in 16 KiB bulk copies through the 13-stage ring
        const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
        const int n = (int)(per_cta / 16384);
        for (int i = 0; i < n; ++i) {
            const int s = i % 13;
            if (i >= 13) {
                const uint32_t ph = ((i / 13) - 1) & 1;
                asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(&full[s])), "r"(ph) : "memory");
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(16384) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + s * 16384)),
                         "l"(base + (size_t)i * 16384), "r"(16384), "r"(su(&full[s])) : "memory");
        }
        for (int i = n; i < n + 13 && i >= 13; ++i) {
            const int s = i % 13;
            const uint32_t ph = ((i / 13) - 1) & 1;
            asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(&full[s])), "r"(ph) : "memory");
        }
    } else if (V < 2) {
        while (gt() - t0 < 20000) {}
    }
    __syncthreads();
    if (V >= 3 && threadIdx.x < 128) ydump[(size_t)blockIdx.x * 128 + threadIdx.x] = (float)call;
    if (threadIdx.x == 0) {
        unsigned s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        Rec r;
        r.start = t0;
        r.wait_done = tw;
        r.end = gt();
        r.sm = (int)s;
        rec[blockIdx.x] = r;
    }
    if (V >= 1 && warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int V>
void run(const char* name, int smem, const uint8_t* src, size_t per_cta, float* y) {
    const int calls = 8, G = 148;
    Rec* rec;
    cudaMalloc(&rec, sizeof(Rec) * G * calls);
    cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int c = 0; c < calls; ++c) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(480);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k<V>, rec + c * G, src + (size_t)(c & 1) * G * per_cta, per_cta, y, c);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int r = 0; r < 3; ++r) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaError_t err = cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<Rec> h(G * calls);
    cudaMemcpy(h.data(), rec, sizeof(Rec) * G * calls, cudaMemcpyDeviceToHost);
    std::vector<double> gap, wrel, dur;
    for (int c = 1; c < calls; ++c) {
        long long lastend = 0;
        std::vector<long long> endsm(1024, 0);
        for (int i = 0; i < G; ++i) {
            const Rec& r = h[(c - 1) * G + i];
            lastend = std::max(lastend, r.end);
            endsm[r.sm] = r.end;
        }
        for (int i = 0; i < G; ++i) {
            const Rec& r = h[c * G + i];
            gap.push_back((r.start - endsm[r.sm]) / 1000.0);
            if (r.wait_done) wrel.push_back((r.wait_done - lastend) / 1000.0);
            dur.push_back((r.end - r.start) / 1000.0);
        }
    }
    auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v.empty() ? 0.0 : v[v.size() / 2]; };
    auto mn = [](const std::vector<double>& v) { return v.empty() ? 0.0 : *std::min_element(v.begin(), v.end()); };
    auto mx = [](const std::vector<double>& v) { return v.empty() ? 0.0 : *std::max_element(v.begin(), v.end()); };
    printf("%-34s smem %6d: %7.2f us/call  start-prev_end(same SM) min %5.2f med %5.2f max %5.2f  wait-last_end min %5.2f med %5.2f max %5.2f  cta dur med %6.2f  %s\n",
           name, smem, ms * 1000.0 / (10 * calls), mn(gap), med(gap), mx(gap), mn(wrel), med(wrel), mx(wrel), med(dur),
           err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(rec);
}

int main() {
    const size_t per_cta = (size_t)16384 * 112;   // 1.75 MiB per CTA -> 265 MB per call (C5 L=8)
    uint8_t* src;
    cudaMalloc(&src, per_cta * 148 * 2);
    cudaMemset(src, 1, per_cta * 148 * 2);
    float* y;
    cudaMalloc(&y, 148 * 128 * 4);
    run<0>("V0 spin 20us", 225 * 1024, src, per_cta, y);
    run<0>("V0 spin 20us", 100 * 1024, src, per_cta, y);
    run<0>("V0 spin 20us", 16 * 1024, src, per_cta, y);
    run<1>("V1 spin + tmem", 225 * 1024, src, per_cta, y);
    run<2>("V2 tmem + stream 1.75MB/CTA", 225 * 1024, src, per_cta, y);
    run<3>("V3 V2 + y stores", 225 * 1024, src, per_cta, y);
    run<2>("V2 stream 0.44MB/CTA", 225 * 1024, src, per_cta / 4, y);
    return 0;
}
