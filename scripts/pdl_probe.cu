// pdl_probe.cu -- does griddepcontrol.wait in a PDL secondary wait for the primary grid's
// completion (and memory flush)?  Primary: 148 CTAs, CTA 0 runs 40 us longer and writes
// flag = 1 as its last act.  Secondary (launched with programmatic stream serialization):
// each CTA records when griddepcontrol.wait returned and whether it saw the flag.
// Run back to back on a stream and inside a captured CUDA graph.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long gt() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void primary(volatile int* flag, long long* tend, int trigger_early) {
    if (trigger_early) asm volatile("griddepcontrol.launch_dependents;");
    const long long t0 = gt();
    const long long dur = blockIdx.x == 0 ? 40000 : 2000;
    while (gt() - t0 < dur) {}
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *flag = 1;
        __threadfence();
        *tend = gt();
    }
}
__global__ void secondary(volatile int* flag, long long* out) {
    const long long t0 = gt();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const long long t1 = gt();
    if (threadIdx.x == 0) {
        out[blockIdx.x * 3 + 0] = t0;
        out[blockIdx.x * 3 + 1] = t1;
        out[blockIdx.x * 3 + 2] = *flag;
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) *flag = 0;   // reset for the next round (after all reads? best effort)
}

static void launch_pair(int* flag, long long* tend, long long* out, cudaStream_t s, int early) {
    primary<<<148, 128, 0, s>>>(flag, tend, early);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, secondary, (volatile int*)flag, out);
}

static void report(const char* tag, long long* d_out, long long* d_tend) {
    long long h[148 * 3], tend;
    cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(&tend, d_tend, sizeof tend, cudaMemcpyDeviceToHost);
    int stale = 0;
    long long mn = 1LL << 62, mx = -(1LL << 62), smin = 1LL << 62;
    for (int i = 0; i < 148; ++i) {
        stale += h[i * 3 + 2] == 0;
        mn = h[i * 3 + 1] - tend < mn ? h[i * 3 + 1] - tend : mn;
        mx = h[i * 3 + 1] - tend > mx ? h[i * 3 + 1] - tend : mx;
        smin = h[i * 3] - tend < smin ? h[i * 3] - tend : smin;
    }
    printf("%-28s secondary start min %+8.2f us, wait returned %+8.2f..%+8.2f us rel. primary end; stale flag %d/148\n",
           tag, smin / 1e3, mn / 1e3, mx / 1e3, stale);
}

int main() {
    int* flag;
    long long *tend, *out;
    cudaMalloc(&flag, 4);
    cudaMalloc(&tend, 8);
    cudaMalloc(&out, 148 * 3 * 8);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int early = 0; early < 2; ++early) {
        cudaMemset(flag, 0, 4);
        launch_pair(flag, tend, out, s, early);
        cudaStreamSynchronize(s);
        report(early ? "stream, early trigger" : "stream, no trigger", out, tend);
        cudaMemset(flag, 0, 4);
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        launch_pair(flag, tend, out, s, early);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        report(early ? "graph, early trigger" : "graph, no trigger", out, tend);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
