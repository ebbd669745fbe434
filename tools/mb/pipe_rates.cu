// throughput of IMAD.HI.U32 (64-bit addend) vs IMAD vs LOP3 vs LEA vs ISETP+SEL on sm_100a
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__constant__ uint32_t kc[8];
template <int MODE>
__global__ void k(uint32_t* out, uint32_t seed, int iters) {
    uint32_t a[8], acc[8];
#pragma unroll
    for (int i = 0; i < 8; i++) { a[i] = seed * (i + 1) + threadIdx.x; acc[i] = i; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE == 0) acc[i] = (uint32_t)(((uint64_t)a[i] * 0xFFFFFFFFull + (uint64_t)acc[i]) >> 32);           // IMAD.HI
            else if (MODE == 1) acc[i] = a[i] * kc[i] + acc[i];                                                  // IMAD (const bank)
            else if (MODE == 2) acc[i] = (acc[i] & a[i]) ^ (a[i] >> 3 | acc[i]);                                 // LOP3 (+SHF)
            else if (MODE == 3) acc[i] = acc[i] + (a[i] << 4);                                                   // LEA
            else if (MODE == 4) acc[i] += (a[i] <= acc[i]) ? 16u : 256u;                                         // ISETP + SEL + IADD
            else if (MODE == 5) { acc[i] = (uint32_t)(((uint64_t)a[i] * 0xFFFFFFFFull + (uint64_t)acc[i]) >> 32); acc[i] = acc[i] * kc[i] + a[i]; }  // IMAD.HI + IMAD
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, uint32_t* d) {
    const int iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<148 * 8, 256>>>(d, 12345, 16);
    cudaEventRecord(e0);
    k<MODE><<<148 * 8, 256>>>(d, 12345, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double winst = 148.0 * 8 * 8 * iters * 8;  // warp-level "statements"
    printf("%-22s %.3f ms  %.3f statements/cycle/SMSP (1965 MHz)\n", name, ms, winst / (ms * 1e-3 * 1.965e9 * 592));
}
int main() {
    uint32_t h[8] = {1, 16, 256, 4096, 65536, 1 << 20, 1 << 24, 1 << 28};
    cudaMemcpyToSymbol(kc, h, sizeof(h));
    uint32_t* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
    run<0>("IMAD.HI", d); run<1>("IMAD cbank", d); run<2>("LOP3+SHF", d); run<3>("LEA", d); run<4>("ISETP+SEL+IADD", d); run<5>("IMAD.HI+IMAD", d);
    return 0;
}
