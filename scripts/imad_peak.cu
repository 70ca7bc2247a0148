// Integer-pipe throughput microbenchmark on B200 (the IMAD roofline denominator).
// Each thread runs 8 independent chains of one opcode; reports ops/cycle/SM and Gop/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(uint32_t* out, uint32_t iters, uint32_t seed) {
    uint32_t a[8], b = seed | 1, c = seed * 3 + 1;
    uint64_t w[8];
    double d[8];
    const double db = 1.0000001 + seed * 1e-9, dc = 0.5;
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 7 + i; w[i] = a[i]; d[i] = a[i]; }
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = a[i] * b + c;                  // IMAD
            if (OP == 1) a[i] = __umulhi(a[i], b) + c;         // IMAD.HI (+ add folded?)
            if (OP == 2) w[i] = (uint64_t)(uint32_t)w[i] * b + w[i];  // IMAD.WIDE.U32
            if (OP == 3) a[i] = a[i] + b + c;                  // IADD3
            if (OP == 4) a[i] = min(a[i] - b, a[i]);           // VIADDMNMX
            if (OP == 5) a[i] = (a[i] ^ b) & c;                // LOP3
            if (OP == 6) d[i] = fma(d[i], db, dc);             // DFMA
            if (OP == 7) { a[i] = a[i] * b + c; d[i] = fma(d[i], db, dc); }  // IMAD || DFMA (1 each)
            if (OP == 8) a[i] = (uint32_t)__double2uint_rz(d[i] + a[i]);    // DADD + F2I.U32.F64
            if (OP == 9) d[i] = fma((double)a[i], db, d[i]);   // I2F.F64.U32 + DFMA
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i] + (uint32_t)w[i] + (uint32_t)(w[i] >> 32) + (uint32_t)d[i];
    if (s == 0x12345678) out[0] = s;
}

template <int OP>
void run(const char* name, int sms, double ghz) {
    uint32_t* out;
    cudaMalloc(&out, 4);
    const uint32_t iters = 4096;
    const int blocks = sms * 8, threads = 256;
    k<OP><<<blocks, threads>>>(out, 16, 7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<blocks, threads>>>(out, iters, 7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 8;
    const double per_cyc_sm = ops / (ms * 1e-3) / (ghz * 1e9) / sms;
    printf("%-12s %8.1f Gop/s  %6.1f lane-ops/cycle/SM (at %.3f GHz)\n", name, ops / ms / 1e6, per_cyc_sm, ghz);
    cudaFree(out);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double ghz = clk_khz / 1e6;
    printf("%s, %d SMs, max clock %.3f GHz\n", p.name, p.multiProcessorCount, ghz);
    run<0>("IMAD", p.multiProcessorCount, ghz);
    run<1>("IMAD.HI", p.multiProcessorCount, ghz);
    run<2>("IMAD.WIDE", p.multiProcessorCount, ghz);
    run<3>("IADD3", p.multiProcessorCount, ghz);
    run<4>("VIADDMNMX", p.multiProcessorCount, ghz);
    run<5>("LOP3", p.multiProcessorCount, ghz);
    run<6>("DFMA", p.multiProcessorCount, ghz);
    run<7>("IMAD+DFMA", p.multiProcessorCount, ghz);
    run<8>("DADD+F2I", p.multiProcessorCount, ghz);
    run<9>("I2F+DFMA", p.multiProcessorCount, ghz);
    return 0;
}
