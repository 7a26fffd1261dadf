// Exhaustive check of a branch-free float reciprocal against __frcp_rn over
// every positive normal float in a binade range.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false tools/check_rcpf.cu -o tools/check_rcpf.bin
#include <cstdio>
__device__ __forceinline__ float rcpf_fast(float d) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    const float e = __fmaf_rn(-d, r, 1.0f);
    return __fmaf_rn(r, e, r);
}
__device__ __forceinline__ float rcpf_fast2(float d) {  // two Newton steps
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    float e = __fmaf_rn(-d, r, 1.0f);
    r = __fmaf_rn(r, e, r);
    e = __fmaf_rn(-d, r, 1.0f);
    return __fmaf_rn(r, e, r);
}
__global__ void k(unsigned base, unsigned long long *bad1, unsigned long long *bad2, float *ex) {
    const unsigned u = base + blockIdx.x * blockDim.x + threadIdx.x;
    const float d = __uint_as_float(u);
    const float b = __frcp_rn(d);
    if (__float_as_uint(rcpf_fast(d)) != __float_as_uint(b)) { atomicAdd(bad1, 1ull); *ex = d; }
    if (__float_as_uint(rcpf_fast2(d)) != __float_as_uint(b)) atomicAdd(bad2, 1ull);
}
int main() {
    unsigned long long *b1, *b2; float *ex;
    cudaMallocManaged(&b1, 8); cudaMallocManaged(&b2, 8); cudaMallocManaged(&ex, 4);
    *b1 = *b2 = 0;
    // exponents -100 .. +100 : biased 27 .. 227
    const unsigned lo = 27u << 23, hi = 228u << 23;
    for (unsigned s = lo; s < hi; s += 1u << 24) k<<<(1 << 24) / 256, 256>>>(s, b1, b2, ex);
    cudaDeviceSynchronize();
    printf("one Newton step: %llu mismatches, two: %llu (of %u floats; example %.9g)\n", *b1, *b2, hi - lo, *ex);
}
