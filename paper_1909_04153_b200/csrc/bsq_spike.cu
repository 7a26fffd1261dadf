// bsq_spike.cu -- partitioned (SPIKE) coupling of y-strip column solves
// (BSQ_Y_SPIKE, include/bsq.h).
//
// Rank s holds rows [s n, (s+1) n) of every column's tridiagonal system.  Its
// block A_s is factored alone; y_s = A_s^-1 r_s is the local solve (the
// ordinary strip solve with zero coupling), and the static spikes
//   v_s = A_s^-1 (a_first e_first),  w_s = A_s^-1 (c_last e_last)
// carry the couplings to the last row of block s-1 and the first row of
// block s+1.  The exact solution is
//   x_s = y_s - v_s b_{s-1} - w_s t_{s+1}
// with b_s = x_s[last], t_s = x_s[first].  Taking the last row of block s and
// the first row of block s+1 gives, for z_s = (b_s, t_{s+1}), s = 0..G-2, a
// block-tridiagonal system with 2x2 blocks:
//   b_s     + W_s^L t_{s+1} + V_s^L b_{s-1}     = Y_s^L
//   t_{s+1} + V_{s+1}^F b_s + W_{s+1}^F t_{s+2} = Y_{s+1}^F
// (F/L = first/last row values; b_{-1} = t_G = 0).  Every rank solves it per
// column (block Thomas, fp64, G-1 <= 63 blocks) and applies its own
// correction.
#include <cstdint>

#include "bsq_device.cuh"
#include "bsq_launch.h"

namespace bsq {

constexpr int SPIKE_GMAX = 64;

// table: G x 4 x nx (v_first, v_last, w_first, w_last); yb: G x 2 x nx
// (y_first, y_last); out bt: 2 x nx (b_{rank-1}, t_{rank+1}), 0 where absent
template <class T>
__global__ void k_spike_reduce(int nx, int G, int rank, const double *table, const T *yb, T *bt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nx) return;
    auto VF = [&](int s) { return table[((long)s * 4 + 0) * nx + i]; };
    auto VL = [&](int s) { return table[((long)s * 4 + 1) * nx + i]; };
    auto WF = [&](int s) { return table[((long)s * 4 + 2) * nx + i]; };
    auto WL = [&](int s) { return table[((long)s * 4 + 3) * nx + i]; };
    auto YF = [&](int s) { return double(yb[((long)s * 2 + 0) * nx + i]); };
    auto YL = [&](int s) { return double(yb[((long)s * 2 + 1) * nx + i]); };
    // forward elimination: D'_s = D_s - L_s D'_{s-1}^-1 U_{s-1}, with
    // D_s = [[1, WL_s], [VF_{s+1}, 1]], L_s = [[VL_s, 0], [0, 0]],
    // U_s = [[0, 0], [0, WF_{s+1}]]; only D'_s[0][0] and r'_s[0] change.
    double d00[SPIKE_GMAX], d01[SPIKE_GMAX], d10[SPIKE_GMAX], d11[SPIKE_GMAX];
    double r0[SPIKE_GMAX], r1[SPIKE_GMAX];
    const int nb = G - 1;
    for (int s = 0; s < nb; s++) {
        d00[s] = 1.0;
        d01[s] = WL(s);
        d10[s] = VF(s + 1);
        d11[s] = 1.0;
        r0[s] = YL(s);
        r1[s] = YF(s + 1);
        if (s > 0) {
            // M = L_s D'^-1_{s-1}: row 0 = VL_s * (row 0 of D'^-1_{s-1})
            const double det = d00[s - 1] * d11[s - 1] - d01[s - 1] * d10[s - 1];
            const double i00 = d11[s - 1] / det, i01 = -d01[s - 1] / det;
            const double m0 = VL(s) * i00, m1 = VL(s) * i01;
            // U_{s-1} = [[0,0],[0, WF_s]]: M U_{s-1} = [[0, m1 WF_s], [0, 0]]
            d01[s] -= m1 * WF(s);
            r0[s] -= m0 * r0[s - 1] + m1 * r1[s - 1];
        }
    }
    // back substitution: z_s = D'^-1_s (r'_s - U_s z_{s+1})
    double b_prev = 0.0, t_next = 0.0, zt_next = 0.0;  // zt_next = t_{s+2} of z_{s+1}
    for (int s = nb - 1; s >= 0; s--) {
        const double q0 = r0[s], q1 = r1[s] - (s + 1 < nb ? WF(s + 1) * zt_next : 0.0);
        const double det = d00[s] * d11[s] - d01[s] * d10[s];
        const double b = (d11[s] * q0 - d01[s] * q1) / det;
        const double t = (d00[s] * q1 - d10[s] * q0) / det;
        zt_next = t;
        if (s == rank - 1) b_prev = b;  // b_{rank-1}
        if (s == rank) t_next = t;      // t_{rank+1}
    }
    bt[i] = T(b_prev);
    bt[nx + i] = T(t_next);
}

// x = (y - v b_prev) - w t_next over rows [j0, j1) of the strip, in place.
// v is negligible from row jv on and w below row jw (|spike| < 2^-64
// everywhere there, SPIKE_TINY in bsq_api.cu): those terms are dropped.
template <class T>
__global__ void k_spike_fix(Consts<T> C, T *x, const T *v, const T *w, const T *bt, int south,
                            int north, int j0, int j1, int jv, int jw) {
    const Layout L = C.L;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = j0 + blockIdx.y * blockDim.y + threadIdx.y;
    if (i >= L.nx || j >= j1) return;
    const long o = L.at(GL + j, GL + i);
    T r = x[o];
    if (south && j < jv) r = r - v[o] * bt[i];
    if (north && j >= jw) r = r - w[o] * bt[L.nx + i];
    x[o] = r;
}

template <class T>
void launch_spike(const Consts<T> &C, int G, int rank, const double *table, const T *yb, T *bt,
                  T *x, const T *v, const T *w, int south, int north, cudaStream_t st,
                  int apply, int jv, int jw) {
    k_spike_reduce<T><<<(C.L.nx + 127) / 128, 128, 0, st>>>(C.L.nx, G, rank, table, yb, bt);
    if (!apply) return;
    const int ny = C.L.ny;
    if (!south) jv = 0;
    if (!north) jw = ny;
    auto rows = [&](int j0, int j1) {
        if (j1 <= j0) return;
        dim3 blk(32, 8), grd((C.L.nx + 31) / 32, (j1 - j0 + 7) / 8);
        k_spike_fix<T><<<grd, blk, 0, st>>>(C, x, v, w, bt, south, north, j0, j1, jv, jw);
    };
    if (jv < jw) {  // two bands near the interfaces, the rows between untouched
        rows(0, jv);
        rows(jw, ny);
    } else {
        rows(0, ny);
    }
}

#if BSQ_INST_F64
template void launch_spike<double>(const Consts<double> &, int, int, const double *,
                                   const double *, double *, double *, const double *,
                                   const double *, int, int, cudaStream_t, int, int, int);
#endif
#if BSQ_INST_F32
template void launch_spike<float>(const Consts<float> &, int, int, const double *, const float *,
                                  float *, float *, const float *, const float *, int, int,
                                  cudaStream_t, int, int, int);
#endif

}  // namespace bsq
