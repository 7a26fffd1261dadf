// bsq_solve.cu -- implicit momentum recovery: batched tridiagonal line
// solves for P (x rows) and Q (y columns), and the cross-correction RHS.
//
// Reference: implicit.solve_momentum (implicit.py:173-205) with
// thomas_batch (_kernels.py:360-381); the correction sweep of
// stepper.py:262-280.
#include <cstdint>

#include "bsq_device.cuh"
#include "bsq_launch.h"

namespace bsq {

// ---------------------------------------------------------------------------
// Warp-specialized pipelined line solve.
//
// A CTA owns 32 lines (x: 32 consecutive rows; y: 32 consecutive columns).
// Warp 0 is the consumer: lane l runs line l's Thomas recurrence entirely out
// of shared memory.  Warps 1..8 are producers: per chunk of SK elements each
// producer thread owns exactly four (line, element) items and issues all of
// their global loads before touching shared memory, so a chunk's 32 KB are in
// flight at once; the folded right-hand side is assembled on the way in.
// Chunks are double buffered: while the consumer sweeps chunk c, producers
// fill chunk c+1 and drain chunk c-1.
//
// The LU factors of the static operator are precomputed on the host with
// thomas_batch's own arithmetic (den_i = b_i - a_i cw_{i-1},
// cw_i = c_i / den_i), so the per-step forward sweep
// dw_i = (r_i - a_i dw_{i-1}) / den_i and back substitution
// x_i = dw_i - cw_i x_{i+1} reproduce thomas_batch bit for bit.  The division
// by the static pivot uses div_static (correctly rounded).  The forward
// sweep's dw is parked in the output array and overwritten by x.
constexpr int SK = 32;                 // chunk length (elements per line)
constexpr int SLD = SK + 1;            // padded smem row: conflict-free access
constexpr int SW = 9;                  // warps per CTA: 1 consumer + 8 producers
constexpr int NPROD = (SW - 1) * 32;   // producer threads
constexpr int ITEMS = 32 * SK / NPROD; // items per producer thread per chunk
constexpr int SBUF = 32 * SLD;
static_assert(ITEMS * NPROD == 32 * SK, "producer items must tile the chunk");

template <class T>
struct SolveSmem {
    T r[2][SBUF], a[2][SBUF], den[2][SBUF], rden[2][SBUF], out[2][SBUF];
};

template <bool XDIR>
__device__ __forceinline__ int tile_idx(int line, int k) {
    // x: [line][k]: a producer warp writes one row segment, the consumer
    //    reads a padded column (stride SLD: conflict-free)
    // y: [k][line]: both sides touch 32 consecutive doubles
    return XDIR ? line * SLD + k : k * SLD + line;
}

template <bool XDIR>
__device__ __forceinline__ void item_of(int it, int &ln, int &k) {
    // consecutive producer lanes -> consecutive global addresses
    if (XDIR) { ln = it >> 5; k = it & 31; } else { k = it >> 5; ln = it & 31; }
}

template <class T, bool XDIR>
__device__ void solve_lines(const Consts<T> &C, const SolvePtrs<T> &S, int line0, SolveSmem<T> &sm) {
    const Layout L = C.L;
    const int n = XDIR ? L.nx : L.ny;  // line length
    const int nlines = XDIR ? L.ny : L.nx;
    const int nc = (n + SK - 1) / SK;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ptid = threadIdx.x - 32;
    const T *__restrict__ rhs = XDIR ? S.rx : S.ry;
    const T *__restrict__ A = XDIR ? S.ax : S.ay;
    const T *__restrict__ DEN = XDIR ? S.denx : S.deny;
    const T *__restrict__ RDEN = XDIR ? S.rdenx : S.rdeny;
    const T *__restrict__ CW = XDIR ? S.cwx : S.cwy;
    const T *__restrict__ clast = XDIR ? S.cx_last : S.cy_last;
    T *out = XDIR ? S.outx : S.outy;

    auto offset = [&](int line, int e) -> long {
        return XDIR ? L.at(GL + line, GL + e) : L.at(GL + e, GL + line);
    };

    // producers: chunk c of r, a, den, rden into buffer b; drain chunk d of
    // out (d < 0: none).  All loads first, then the drain, then smem stores.
    auto fill_fwd = [&](int c, int b, int d, int bd) {
        T rv[ITEMS], av[ITEMS], dv[ITEMS], qv[ITEMS];
        long ov[ITEMS];
        bool okv[ITEMS];
#pragma unroll
        for (int u = 0; u < ITEMS; u++) {
            int ln, k;
            item_of<XDIR>(u * NPROD + ptid, ln, k);
            const int line = line0 + ln, e = c * SK + k;
            okv[u] = c < nc && line < nlines && e < n;
            ov[u] = okv[u] ? offset(line, e) : 0;
            rv[u] = okv[u] ? rhs[ov[u]] : T(0);
            av[u] = okv[u] ? A[ov[u]] : T(0);
            dv[u] = okv[u] ? DEN[ov[u]] : T(1);
            qv[u] = okv[u] ? RDEN[ov[u]] : T(1);
        }
        if (d >= 0) {
#pragma unroll
            for (int u = 0; u < ITEMS; u++) {
                int ln, k;
                item_of<XDIR>(u * NPROD + ptid, ln, k);
                const int line = line0 + ln, e = d * SK + k;
                if (line < nlines && e < n) out[offset(line, e)] = sm.out[bd][tile_idx<XDIR>(ln, k)];
            }
        }
        if (c >= nc) return;
#pragma unroll
        for (int u = 0; u < ITEMS; u++) {
            int ln, k;
            item_of<XDIR>(u * NPROD + ptid, ln, k);
            const int line = line0 + ln, e = c * SK + k;
            T r = rv[u];
            if (okv[u] && e == 0) {  // implicit.py:178 / :190 ghost folding
                const T g0 = XDIR ? S.gp[L.at(GL + line, GL - 1)] : S.gq[L.at(GL - 1, GL + line)];
                r = r - av[u] * g0;
            }
            if (okv[u] && e == n - 1) {
                const T g1 = XDIR ? S.gp[L.at(GL + line, n + GL)] : S.gq[L.at(n + GL, GL + line)];
                r = r - clast[line] * g1;
            }
            const int t = tile_idx<XDIR>(ln, k);
            sm.r[b][t] = r;
            sm.a[b][t] = av[u];
            sm.den[b][t] = dv[u];
            sm.rden[b][t] = qv[u];
        }
    };
    // producers: chunk c of (dw parked in out, cw) into buffer b; drain chunk d
    auto fill_bwd = [&](int c, int b, int d, int bd) {
        T dwv[ITEMS], cwv[ITEMS];
#pragma unroll
        for (int u = 0; u < ITEMS; u++) {
            int ln, k;
            item_of<XDIR>(u * NPROD + ptid, ln, k);
            const int line = line0 + ln, e = c * SK + k;
            const bool ok = c >= 0 && line < nlines && e < n;
            const long o = ok ? offset(line, e) : 0;
            dwv[u] = ok ? out[o] : T(0);
            cwv[u] = ok ? CW[o] : T(0);
        }
        if (d >= 0) {
#pragma unroll
            for (int u = 0; u < ITEMS; u++) {
                int ln, k;
                item_of<XDIR>(u * NPROD + ptid, ln, k);
                const int line = line0 + ln, e = d * SK + k;
                if (line < nlines && e < n) out[offset(line, e)] = sm.out[bd][tile_idx<XDIR>(ln, k)];
            }
        }
        if (c < 0) return;
#pragma unroll
        for (int u = 0; u < ITEMS; u++) {
            int ln, k;
            item_of<XDIR>(u * NPROD + ptid, ln, k);
            const int t = tile_idx<XDIR>(ln, k);
            sm.r[b][t] = dwv[u];
            sm.a[b][t] = cwv[u];
        }
    };

    // ---- forward sweep --------------------------------------------------------
    if (warp > 0) fill_fwd(0, 0, -1, 0);
    __syncthreads();
    T dw = T(0);
    for (int c = 0; c < nc; c++) {
        const int b = c & 1;
        if (warp == 0) {
            const int kmax = min(SK, n - c * SK);
            if (kmax == SK) {
#pragma unroll 8
                for (int k = 0; k < SK; k++) {
                    const int t = tile_idx<XDIR>(lane, k);
                    const T r = sm.r[b][t];
                    const T num = (c == 0 && k == 0) ? r : r - sm.a[b][t] * dw;
                    dw = div_static(num, sm.den[b][t], sm.rden[b][t]);
                    sm.out[b][t] = dw;
                }
            } else {
                for (int k = 0; k < kmax; k++) {
                    const int t = tile_idx<XDIR>(lane, k);
                    const T r = sm.r[b][t];
                    const T num = (c == 0 && k == 0) ? r : r - sm.a[b][t] * dw;
                    dw = div_static(num, sm.den[b][t], sm.rden[b][t]);
                    sm.out[b][t] = dw;
                }
            }
        } else {
            fill_fwd(c + 1, b ^ 1, c - 1, b ^ 1);
        }
        __syncthreads();
    }
    // drain the last forward chunk while loading the last chunk for the back sweep
    if (warp > 0) fill_bwd(-1, 0, nc - 1, (nc - 1) & 1);
    __syncthreads();

    // ---- back substitution (chunks in reverse) ---------------------------------
    if (warp > 0) fill_bwd(nc - 1, 0, -1, 0);
    __syncthreads();
    T xv = T(0);
    for (int s = 0; s < nc; s++) {
        const int c = nc - 1 - s, b = s & 1;
        if (warp == 0) {
            const int kmax = min(SK, n - c * SK);
            for (int k = kmax - 1; k >= 0; k--) {
                const int t = tile_idx<XDIR>(lane, k);
                xv = (s == 0 && k == kmax - 1) ? sm.r[b][t] : sm.r[b][t] - sm.a[b][t] * xv;
                sm.out[b][t] = xv;
            }
        } else {
            fill_bwd(c - 1, b ^ 1, s >= 1 ? c + 1 : -1, b ^ 1);
        }
        __syncthreads();
    }
    if (warp > 0) fill_bwd(-1, 0, 0, (nc - 1) & 1);
}

// Blocks [0, nbx) take x lines (rows -> P); blocks [nbx, ...) y lines (columns -> Q).
template <class T>
__global__ void __launch_bounds__(SW * 32, 2) k_solve_pipe(Consts<T> C, SolvePtrs<T> S, int nbx) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SolveSmem<T> &sm = *reinterpret_cast<SolveSmem<T> *>(smem_raw);
    if ((int)blockIdx.x < nbx)
        solve_lines<T, true>(C, S, blockIdx.x * 32, sm);
    else
        solve_lines<T, false>(C, S, (blockIdx.x - nbx) * 32, sm);
}

// ---------------------------------------------------------------------------
// Cross-correction right-hand sides (stepper.py:268-273):
//   us_corr = base_u + (F*(P1, Q1) - F*_n),  vs_corr = base_v + (G*(P1, Q1) - G*_n)
// written over us / vs.
template <class T>
__global__ void __launch_bounds__(256) k_correct(Consts<T> C, CorrectPtrs<T> K) {
    const Layout L = C.L;
    const int I = GL + blockIdx.x * 32 + threadIdx.x, J = GL + blockIdx.y * 8 + threadIdx.y;
    if (I >= L.nx + GL || J >= L.ny + GL) return;
    const long o = L.at(J, I);
    const T d = K.dep[o], dx_ = K.ddx[o], dy_ = K.ddy[o];
    const T fs = cross_f(C, K.q1, o, d, dx_, dy_);
    const T gs = cross_g(C, K.p1, o, d, dx_, dy_);
    K.us[o] = K.bu[o] + (fs - K.fs[o]);
    K.vs[o] = K.bv[o] + (gs - K.gs[o]);
}

// ---------------------------------------------------------------------------
// launchers

template <class T>
void launch_solve(const Consts<T> &C, const SolvePtrs<T> &S, cudaStream_t st) {
    const int nbx = (C.L.ny + 31) / 32, nby = (C.L.nx + 31) / 32;
    const size_t smem = sizeof(SolveSmem<T>);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_solve_pipe<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set = true;
    }
    k_solve_pipe<T><<<nbx + nby, SW * 32, smem, st>>>(C, S, nbx);
}

template <class T>
void launch_correct(const Consts<T> &C, const CorrectPtrs<T> &K, cudaStream_t st) {
    dim3 grid((C.L.nx + 31) / 32, (C.L.ny + 7) / 8);
    k_correct<T><<<grid, dim3(32, 8), 0, st>>>(C, K);
}

template void launch_solve<double>(const Consts<double> &, const SolvePtrs<double> &, cudaStream_t);
template void launch_correct<double>(const Consts<double> &, const CorrectPtrs<double> &,
                                     cudaStream_t);

}  // namespace bsq
