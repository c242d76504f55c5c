// Handoff gap of a PDL-chained kernel pair: stream launches vs the same chain captured in a CUDA graph, with and without
// the programmatic-serialization attribute. Kernel i stamps atomicMax(end[i]) when its CTAs finish and
// atomicMin(start[i]) when they pass griddepcontrol.wait; gap = start[i+1] - end[i] (globaltimer ns).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(unsigned long long* st, unsigned long long* en, int i, float* buf, int iters) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicMin(st + i, gt());
    float a = buf[blockIdx.x * blockDim.x + threadIdx.x];
    for (int j = 0; j < iters; ++j) a = a * 1.0001f + 0.5f;
    buf[blockIdx.x * blockDim.x + threadIdx.x] = a;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(en + i, gt());
}
int main() {
    const int N = 200, ctas = 296, thr = 256;
    unsigned long long *st, *en; float* buf;
    cudaMalloc(&st, N * 8); cudaMalloc(&en, N * 8); cudaMalloc(&buf, ctas * thr * 4);
    cudaMemset(buf, 0, ctas * thr * 4);
    cudaStream_t s; cudaStreamCreate(&s);
    auto launch = [&](int i, bool pdl) {
        cudaLaunchConfig_t cfg{}; cfg.gridDim = ctas; cfg.blockDim = thr; cfg.stream = s;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0; cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k, st, en, i, buf, 2000);
    };
    for (int mode = 0; mode < 4; ++mode) {  // 0 stream+PDL, 1 stream no PDL, 2 graph+PDL, 3 graph no PDL
        const bool pdl = (mode % 2) == 0, graph = mode >= 2;
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemsetAsync(st, 0xFF, N * 8, s); cudaMemsetAsync(en, 0, N * 8, s);
            cudaGraphExec_t ge = nullptr;
            if (graph) {
                cudaGraph_t g; cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                for (int i = 0; i < N; ++i) launch(i, pdl);
                cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0); cudaGraphLaunch(ge, s);
            } else {
                for (int i = 0; i < N; ++i) launch(i, pdl);
            }
            cudaStreamSynchronize(s);
            std::vector<unsigned long long> a(N), b(N);
            cudaMemcpy(a.data(), st, N * 8, cudaMemcpyDeviceToHost); cudaMemcpy(b.data(), en, N * 8, cudaMemcpyDeviceToHost);
            std::vector<double> gaps, durs;
            for (int i = 10; i < N; ++i) { gaps.push_back((double)(long long)(a[i] - b[i - 1]) / 1e3); durs.push_back((double)(b[i] - a[i]) / 1e3); }
            std::sort(gaps.begin(), gaps.end()); std::sort(durs.begin(), durs.end());
            if (rep == 1) printf("%-16s gap median %.2f us (p10 %.2f p90 %.2f), kernel %.2f us, total %.1f us per launch\n",
                   mode == 0 ? "stream+PDL" : mode == 1 ? "stream" : mode == 2 ? "graph+PDL" : "graph",
                   gaps[gaps.size() / 2], gaps[gaps.size() / 10], gaps[gaps.size() * 9 / 10], durs[durs.size() / 2],
                   (double)(b[N - 1] - a[10]) / 1e3 / (N - 10));
            if (ge) cudaGraphExecDestroy(ge);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
