// Per-SM throughput of the softmax building blocks on this GPU: MUFU.EX2, FFMA2 (packed f32x2), FFMA.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
template <int OP>
__global__ void k(float* out, int iters) {
    float a[8];
    uint64_t p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; asm("mov.b64 %0, {%1,%1};" : "=l"(p[i]) : "f"(a[i])); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(p[i]));
            if (OP == 2) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
            if (OP == 3) {  // fp32 pair -> bf16x2 (F2FP), fed back as the next input
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(a[i]));
                a[i] = __uint_as_float(r);
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) { float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[i])); s += a[i] + lo; }
    if (s == 1.2345f) *out = s;
}
int main() {
    float* o;
    cudaMalloc(&o, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[4] = {"MUFU.EX2 (f32)", "FFMA2 (f32x2)", "FFMA (f32)", "F2FP bf16x2"};
    for (int op = 0; op < 4; ++op)
        for (int warps : {2, 4, 8, 16}) {
            const int iters = 4096;
            auto kern = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
            kern<<<sms, warps * 32>>>(o, 16);
            cudaEventRecord(e0);
            kern<<<sms, warps * 32>>>(o, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            int clk;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            const double ops = (double)sms * warps * 32 * iters * 8 * (op == 1 ? 2 : 1);
            printf("%-16s %2d warps/SM: %.1f instr-lanes/clk/SM (at %.2f GHz nominal)\n", names[op], warps,
                   ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e6);
        }
    return 0;
}
