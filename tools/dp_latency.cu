// Micro-benchmark: dependent-chain latency of fp64 DMUL / DADD / DFMA and of
// an LDS->DFMA chain on the running GPU (clock64 per warp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dp_latency.cu -o /tmp/dp_latency
#include <cstdio>

__global__ void chains(double *out, long long *cyc, double a, double b, int n) {
    double x = a, y = b;
    __shared__ double s[64];
    s[threadIdx.x] = a;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; i++) x = x * b;  // DMUL chain
    long long t1 = clock64();
    for (int i = 0; i < n; i++) y = y + a;  // DADD chain
    long long t2 = clock64();
    double z = a;
    for (int i = 0; i < n; i++) z = __fma_rn(z, b, a);  // DFMA chain
    long long t3 = clock64();
    double w = a;
    for (int i = 0; i < n; i++) { w = __fma_rn(w, s[(threadIdx.x + (int)w) & 31], a); }  // LDS->DFMA
    long long t4 = clock64();
    out[threadIdx.x] = x + y + z + w;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
        cyc[3] = t4 - t3;
    }
}

int main() {
    double *out;
    long long *cyc, h[4];
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMalloc(&cyc, 4 * sizeof(long long));
    const int n = 4096;
    chains<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, n);
    chains<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, n);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: DMUL %.1f  DADD %.1f  DFMA %.1f  LDS+DFMA %.1f\n",
           (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n);
    return 0;
}
