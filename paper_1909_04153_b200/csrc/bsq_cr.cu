// bsq_cr.cu -- the reference's optional odd-even cyclic-reduction line
// solver (solver="cr": cyclic_reduction_batch, _kernels.py:384-451), one CTA
// per line, the line held in shared memory.
//
// Within one reduction level the reference updates the rows
// idx = 2s-1, 4s-1, ... from rows idx -/+ s, which that level does not
// modify; within one back-substitution level it fills rows s-1, 3s-1, ...
// from rows already solved at coarser levels.  Each level is therefore a
// data-parallel map over idx, and running it with one thread per idx (a
// barrier between levels) performs exactly the reference's operations:
// results are bitwise equal.  Divisions are by per-row values (IEEE `/`).
// A zero pivot records (atomicMin) the key of the error the reference would
// raise first -- solve phase, x before y, line, then reduction / core /
// back substitution -- so the host reports the same ZeroDivisionError.
#include <cstdint>
#include <cstdlib>

#include "bsq_device.cuh"
#include "bsq_launch.h"

namespace bsq {

#ifndef BSQ_CR_THREADS
#define BSQ_CR_THREADS 1024  // 512: 1.46, 256: 1.83, 1024: 1.42 ms per 4096^2 solve
#endif
constexpr int CR_THREADS = BSQ_CR_THREADS;

// Shared-memory slot of row i: the low 4 bits XOR-ed with bits 4-7 and 8-11.
// A level touches rows s-1, 3s-1, ... (stride 2s); plain indexing puts 16
// threads of a warp on one bank pair once 2s >= 16, this permutation keeps a
// half-warp's 8-byte accesses on distinct bank pairs for every stride up to
// 512 (a bijection within each block of 16 rows; placement only, so the
// arithmetic and its results are unchanged).
__device__ __forceinline__ int crs(int i) { return i ^ ((i >> 4) & 15) ^ ((i >> 8) & 15); }

// line l of direction xdir: element e at padded (GL+l, GL+e) (x) or
// (GL+e, GL+l) (y)
template <class T, bool XDIR>
__device__ void cr_line(const Consts<T> &C, const CrPtrs<T> &K, int line, T *sm, int n2) {
    const Layout L = C.L;
    const int n = XDIR ? L.nx : L.ny;
    // x overwrites r: a back-substitution level reads r only of the rows it
    // solves (and x of coarser rows), the core reads both r before writing
    T *a = sm, *b = sm + n2, *c = sm + 2 * n2, *r = sm + 3 * n2, *x = r;
    const T *A = XDIR ? K.ax : K.ay;
    const T *B = XDIR ? K.bx : K.by;
    const T *Cc = XDIR ? K.cx : K.cy;
    const T *R = XDIR ? K.rx : K.ry;
    auto off = [&](int e) -> long { return XDIR ? L.at(GL + line, GL + e) : L.at(GL + e, GL + line); };
    // the diagonals: padded layout in x, transposed (contiguous per line) in y
    auto coff = [&](int e) -> long { return XDIR ? off(e) : (long)line * L.ny + e; };
    // load + ghost folding (implicit.py:178-179 / :190-191), identity padding
#pragma unroll 4
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        if (i < n) {
            const long o = off(i), oc = coff(i);
            T rv = R[o];
            const T av = A[oc], cv = Cc[oc];
            if (i == 0) {
                const T g0 = XDIR ? K.gp[L.at(GL + line, GL - 1)] : K.gq[L.at(GL - 1, GL + line)];
                rv = rv - av * g0;
            }
            if (i == n - 1) {
                const T g1 = XDIR ? K.gp[L.at(GL + line, n + GL)] : K.gq[L.at(n + GL, GL + line)];
                rv = rv - cv * g1;
            }
            const int j = crs(i);
            a[j] = av;
            b[j] = B[oc];
            c[j] = cv;
            r[j] = rv;
        } else {
            const int j = crs(i);
            a[j] = T(0);
            b[j] = T(1);
            c[j] = T(0);
            r[j] = T(0);
        }
    }
    __syncthreads();
    unsigned kind = 3;  // 0 reduction, 1 core determinant, 2 back substitution
    // reduction (_kernels.py:414-434)
    for (int stride = 1; stride < n2 / 2; stride *= 2) {
        const int step = 2 * stride;
        for (int k = threadIdx.x; k < n2 / step; k += blockDim.x) {
            const int i0 = step * k + step - 1, ir0 = i0 + stride;
            const int idx = crs(i0), il = crs(i0 - stride);
            if (b[il] == T(0)) kind = 0;
            const T alpha = -a[idx] / b[il];
            T aa = alpha * a[il];
            T bb = b[idx] + alpha * c[il];
            T rr = r[idx] + alpha * r[il];
            T cc;
            if (ir0 < n2) {
                const int ir = crs(ir0);
                if (b[ir] == T(0)) kind = 0;
                const T beta = -c[idx] / b[ir];
                cc = beta * c[ir];
                bb = bb + beta * a[ir];
                rr = rr + beta * r[ir];
            } else {
                cc = T(0);
            }
            a[idx] = aa;
            b[idx] = bb;
            c[idx] = cc;
            r[idx] = rr;
        }
        __syncthreads();
    }
    // 2x2 core (_kernels.py:435-441)
    if (threadIdx.x == 0) {
        const int i1 = crs(n2 / 2 - 1), i2 = crs(n2 - 1);
        const T det = b[i1] * b[i2] - c[i1] * a[i2];
        if (det == T(0) && kind > 1) kind = 1;
        const T x1 = (r[i1] * b[i2] - c[i1] * r[i2]) / det;
        const T x2 = (b[i1] * r[i2] - a[i2] * r[i1]) / det;
        x[i1] = x1;
        x[i2] = x2;
    }
    __syncthreads();
    // back substitution (_kernels.py:442-449)
    for (int stride = n2 / 4; stride >= 1; stride /= 2) {
        const int step = 2 * stride;
        for (int k = threadIdx.x; k * step + stride - 1 < n2; k += blockDim.x) {
            const int i0 = step * k + stride - 1, idx = crs(i0);
            if (b[idx] == T(0) && kind > 2) kind = 2;
            const T lower = i0 - stride >= 0 ? x[crs(i0 - stride)] : T(0);
            x[idx] = (r[idx] - a[idx] * lower - c[idx] * x[crs(i0 + stride)]) / b[idx];
        }
        __syncthreads();
    }
    if (kind < 3)
        atomicMin(K.bad, K.key_base | (XDIR ? 0u : 1u << 30) | ((unsigned)line << 2) | kind);
    T *out = XDIR ? K.outx : K.outy;
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[off(i)] = x[crs(i)];
}

__device__ __forceinline__ void bulk_prefetch_l2(const void *p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <class T>
__global__ void __launch_bounds__(CR_THREADS) k_cr(Consts<T> C, CrPtrs<T> K, int nbx, int n2x,
                                                   int n2y, int ahead) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *sm = reinterpret_cast<T *>(smem_raw);
    // the line `ahead` CTAs later in launch order (about the next one this
    // SM runs): its contiguous operands towards L2 while this line reduces
    const int nl = (int)blockIdx.x + ahead;
    if (ahead > 0 && threadIdx.x < 4 && nl < (int)gridDim.x) {
        const Layout L = C.L;
        const int k = threadIdx.x;
        if (nl < nbx) {  // x line: a, b, c, r rows of the padded layout
            const T *src = k == 0 ? K.ax : k == 1 ? K.bx : k == 2 ? K.cx : K.rx;
            bulk_prefetch_l2(src + L.at(GL + nl, GL), (unsigned)(L.nx * sizeof(T)) & ~15u);
        } else if (k < 3) {  // y line: the transposed diagonals (r is strided)
            const T *src = k == 0 ? K.ay : k == 1 ? K.by : K.cy;
            bulk_prefetch_l2(src + (long)(nl - nbx) * L.ny, (unsigned)(L.ny * sizeof(T)) & ~15u);
        }
    }
    if ((int)blockIdx.x < nbx)
        cr_line<T, true>(C, K, blockIdx.x, sm, n2x);
    else
        cr_line<T, false>(C, K, blockIdx.x - nbx, sm, n2y);
}

static int pow2_at_least(int n) {
    int n2 = 1;
    while (n2 < n) n2 *= 2;
    return n2 < 2 ? 2 : n2;
}

#if BSQ_INST_F64
size_t cr_smem_bytes(int nx, int ny, int elem) {
    const int n2 = pow2_at_least(nx > ny ? nx : ny);
    return (size_t)4 * n2 * elem;
}
#endif

template <class T>
void launch_cr(const Consts<T> &C, const CrPtrs<T> &K, cudaStream_t st) {
    const int n2x = pow2_at_least(C.L.nx), n2y = pow2_at_least(C.L.ny);
    const size_t smem = cr_smem_bytes(C.L.nx, C.L.ny, sizeof(T));
    cudaFuncSetAttribute(k_cr<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // one thread per row of the first reduction level, at most 512 below
    // 4096-row lines (C1, 1024 rows: 512 threads 0.017 ms per solve, 1024:
    // 0.033; C2, 2048 rows: 512 0.054, 1024 0.109) and CR_THREADS from there
    // (4096^2: 512 1.46, 1024 1.42 ms)
    const int n2 = n2x > n2y ? n2x : n2y;
    const int cap = n2 >= 4096 ? CR_THREADS : 512;
    int threads = n2 / 2 < cap ? n2 / 2 : cap;
    threads = threads < 64 ? 64 : (threads + 31) / 32 * 32;
    // CTAs resident at once (one line per SM at 4096 rows): the prefetch
    // distance.  The occupancy depends on the line length, so per launch.
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cr<T>, threads, smem);
    // only when one line fills an SM (4096 rows: 1.245 -> 1.174 ms per
    // solve); with several lines per SM they hide each other's loads (1024
    // rows: 0.0676 -> 0.069 with the prefetch)
    int ahead = per <= 1 ? sms : 0;
    static const char *env_ahead = std::getenv("BSQ_CR_AHEAD");  // A/B: 0 disables
    if (env_ahead) ahead = std::atoi(env_ahead);
    k_cr<T><<<C.L.ny + C.L.nx, threads, smem, st>>>(C, K, C.L.ny, n2x, n2y, ahead);
}

#if BSQ_INST_F64
template void launch_cr<double>(const Consts<double> &, const CrPtrs<double> &, cudaStream_t);
#endif
#if BSQ_INST_F32
template void launch_cr<float>(const Consts<float> &, const CrPtrs<float> &, cudaStream_t);
#endif

}  // namespace bsq
