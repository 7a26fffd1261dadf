// bsq_check.cu -- device-side check of the quotient helpers (test seam).
//
// Every division of the step is the reference's IEEE x / d, computed from a
// correctly rounded reciprocal and a Markstein residual step (bsq_device.cuh).
// bsq_check_quotients runs one helper over host arrays so the tests can
// compare it bit for bit with numpy's x / d on chosen inputs -- subnormal
// numerators, zeros of both signs, infinities, NaN, and the divisor ranges
// each call site guarantees.
#include <cstdint>

#include "bsq_device.cuh"
#include "bsq_launch.h"

namespace bsq {

#if BSQ_INST_F64
__global__ void k_quot(int op, const double *x, const double *d, long n, double *out) {
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a = x[i], b = d[i];
    double q;
    switch (op) {
    case 0: q = div_static(a, b, rcp_rn(b)); break;      // static divisors (generic)
    case 1: q = div_pos(a, b, rcp_rn(b)); break;         // static divisors > 0 (stage, correct)
    case 2: q = div_rcp(a, b, rcp_rn(b)); break;         // per-cell divisor, library reciprocal
    case 3: q = div_rcp_pos(a, b, rcp_depth(b)); break;  // flux depths (FAST path)
    case 4: q = div_nonneg(a, b, -rcp_depth(b)); break;  // k_final depths
    case 5: q = div_static_pos(a, b, -rcp_rn(b)); break; // Thomas pivots > 0
    case 7: q = div_tiny_exact(a, b, rcp_rn(b)); break;  // tiny numerators, call-free
    default: q = a / b; break;                           // IEEE division
    }
    out[i] = q;
}

int check_quotients(int op, const double *x, const double *d, long n, double *out) {
    double *dx = nullptr, *dd = nullptr, *dq = nullptr;
    const size_t bytes = sizeof(double) * (size_t)n;
    if (cudaMalloc(&dx, bytes) || cudaMalloc(&dd, bytes) || cudaMalloc(&dq, bytes)) {
        cudaFree(dx), cudaFree(dd), cudaFree(dq);
        return 2;
    }
    cudaMemcpy(dx, x, bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(dd, d, bytes, cudaMemcpyHostToDevice);
    k_quot<<<(unsigned)((n + 255) / 256), 256>>>(op, dx, dd, n, dq);
    const cudaError_t e = cudaMemcpy(out, dq, bytes, cudaMemcpyDeviceToHost);
    cudaFree(dx), cudaFree(dd), cudaFree(dq);
    return e == cudaSuccess ? 0 : 2;
}
#endif

}  // namespace bsq
