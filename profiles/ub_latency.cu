// Dependent-latency microbenchmark on one warp (cycles per loop iteration): DADD, DMUL, I2F.F64, a
// dependent LDS, a table walk (LDS + 64-bit shift) and a stripped-down decoder step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ub_latency profiles/ub_latency.cu && ./ub_latency
// B200 (this round): 8.3 / 8.5 / 23.2 / 37.6 / 53.5 / 110.1 cycles.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double *out, long long *cyc, double delta, int n, const unsigned *lutg)
{
    __shared__ unsigned lut[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) lut[i] = lutg[i];
    __syncthreads();
    double r = out[threadIdx.x];
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, delta);
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) r = __dmul_rn(r, 1.0000001);
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
    // I2F.F64 -> DMUL -> DADD with loop-carried int through F2I? use int chain: m = (int)r & 7 ... keep simple: i2f chain via bits
    int m = (int)threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double d = (double)m; m = (int)__double2hiint(d) & 1023; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
    // LDS dependent chain
    unsigned idx = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) idx = lut[idx & 4095];
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
    // 64-bit shift + LDS + select chain like the walk
    unsigned long long buf = 0x123456789abcdef0ull ^ idx;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { unsigned e = lut[(unsigned)(buf >> 52)]; int l = (e & 7) + 1; buf = (buf << l) | (e >> 20); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
    // full step: walk + i2f + dmul + dadd + sts
    __shared__ double row[32 * 33];
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        unsigned e = lut[(unsigned)(buf >> 52)]; int l = (e & 7) + 1; buf = (buf << l) | (e >> 20);
        unsigned sym = e & 0xffff; unsigned zz = sym - 1u; int mm = (int)(zz >> 1) ^ -(int)(zz & 1u);
        double inc = __dmul_rn((double)mm, delta);
        if (sym > 1u) r = __dadd_rn(r, inc);
        row[threadIdx.x * 33 + (i & 31)] = r;
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
    out[threadIdx.x] = r + (double)m + (double)idx + (double)buf + row[threadIdx.x];
}
int main()
{
    double *out; long long *cyc; unsigned *lut;
    cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 64); cudaMalloc(&lut, 4096 * 4);
    unsigned h[4096]; for (int i = 0; i < 4096; ++i) h[i] = (i * 2654435761u) >> 8;
    cudaMemcpy(lut, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMemset(out, 0, 256);
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(out, cyc, 1e-3, n, lut);
    long long hc[8]; cudaMemcpy(hc, cyc, 48, cudaMemcpyDeviceToHost);
    const char *nm[] = {"DADD", "DMUL", "I2F.F64+hi", "LDS", "walk(LDS+shift)", "full step"};
    for (int i = 0; i < 6; ++i) printf("%-18s %.1f cycles/iter\n", nm[i], (double)hc[i] / n);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
