// bsq_kernels.cu -- sm_100a kernels of one adaptive-AB3 Boussinesq step.
//
// One step (stepper.py:225-305) is five device passes over the pitched
// fields (see DESIGN.md for the HBM budget of each):
//
//   k_ghost   ghost strips at t          (boundary.py:316-323)
//   k_stage   faces + central-upwind fluxes + FV rates + dispersive terms +
//             cross groups + U*/V* + Euler/AB3/VFD predictor, one fused
//             smem-tiled stencil pass (dispersion.py:67-149, stepper.py:109-132)
//   k_ghost   ghost strips of the predicted state at t+dt (stepper.py:252-254)
//   k_solve   x-line (P) and y-line (Q) tridiagonal solves, pre-factored
//             Thomas (implicit.py:173-205, _kernels.py:360-381); phase 2 folds
//             the cross-correction RHS (stepper.py:262-280) into its loads
//   k_final   clamp + film cutoff + sponge + blow-up/non-finite scan + CFL
//             extrema, with a deterministic last-block reduction
//             (stepper.py:281-305, boundary.py:264-300, _kernels.py:324-353)
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "bsq_device.cuh"
#include "bsq_launch.h"

namespace bsq {

// ---------------------------------------------------------------------------
// ghost strips

template <class T>
__device__ __forceinline__ T ns_value(const Consts<T> &C, const DevParams *P, int which, int f,
                                      int J, int I, const T *src) {
    // value the N or S fill writes at ghost row J, column I (boundary.py:206-261)
    const int nyt = C.L.ny + 4;
    const int side = J < GL ? SIDE_S : SIDE_N;
    if (C.side_kind[side] == KIND_MAKER) {
        double gw = which ? P->gw_n[side] : P->gw_t[side];
        double gf = which ? P->gf_n[side] : P->gf_t[side];
        if (f == 0) return T(gw);
        if (f == 1) return T(0);
        return side == SIDE_S ? T(gf) : T(-gf);
    }
    int Jm = side == SIDE_S ? (J == GL - 1 ? GL : GL + 1) : (J == nyt - GL ? nyt - GL - 1 : nyt - GL - 2);
    T s = f == 2 ? T(-1) : T(1);
    return s * src[C.L.at(Jm, I)];
}

// One thread per ghost cell.  Threads [0, 4*nyt) cover the E/W strips over
// all rows (they own the corners: fill order N, S, E, W); threads
// [4*nyt, 4*nyt + 4*nx) the N/S strips over interior columns.  Corner values
// compose the N/S rule at the mirror column, so no ordering between threads
// is needed.  src_w/src_p/src_q give the interior the mirrors read (for the
// t+dt fill: predicted w, old P/Q -- stepper.py:252-254).
template <class T>
__global__ void k_ghost(Consts<T> C, const DevParams *__restrict__ P, int which, const T *src_w,
                        const T *src_p, const T *src_q, T *dst_w, T *dst_p, T *dst_q) {
    const int nx = C.L.nx, ny = C.L.ny, nxt = nx + 4, nyt = ny + 4;
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    const T *src[3] = {src_w, src_p, src_q};
    T *dst[3] = {dst_w, dst_p, dst_q};
    if (k < 4 * nyt) {
        int J = k >> 2;
        int c = k & 3;  // 0,1 -> west cols 0,1; 2,3 -> east cols nxt-2, nxt-1
        int I = c < 2 ? c : nxt - 4 + c;
        int side = c < 2 ? SIDE_W : SIDE_E;
        bool interior_row = J >= GL && J < nyt - GL;
        if (C.side_kind[side] == KIND_MAKER) {
            double gw = which ? P->gw_n[side] : P->gw_t[side];
            double gf = which ? P->gf_n[side] : P->gf_t[side];
            dst_w[C.L.at(J, I)] = T(gw);
            dst_p[C.L.at(J, I)] = side == SIDE_W ? T(gf) : T(-gf);
            dst_q[C.L.at(J, I)] = T(0);
            return;
        }
        int Im = side == SIDE_W ? (I == GL - 1 ? GL : GL + 1) : (I == nxt - GL ? nxt - GL - 1 : nxt - GL - 2);
#pragma unroll
        for (int f = 0; f < 3; f++) {
            T cur = interior_row ? src[f][C.L.at(J, Im)] : ns_value(C, P, which, f, J, Im, src[f]);
            T s = f == 1 ? T(-1) : T(1);  // P is the wall-normal flux on E/W
            dst[f][C.L.at(J, I)] = s * cur;
        }
        return;
    }
    k -= 4 * nyt;
    if (k < 4 * nx) {
        int I = GL + (k >> 2);
        int r = k & 3;
        int J = r < 2 ? r : nyt - 4 + r;
#pragma unroll
        for (int f = 0; f < 3; f++) dst[f][C.L.at(J, I)] = ns_value(C, P, which, f, J, I, src[f]);
    }
}

// ---------------------------------------------------------------------------
// fused stage + predictor

constexpr int TX = 32, TY = 8;
constexpr int HX = TX + 4, HY = TY + 4;

template <class T>
__global__ void __launch_bounds__(TX *TY) k_stage(Consts<T> C, const DevParams *__restrict__ P,
                                                  StagePtrs<T> A, int predict) {
    __shared__ T s_w[HY][HX], s_p[HY][HX], s_q[HY][HX], s_eta[HY][HX];
    __shared__ T s_bfx[TY][TX + 3], s_bfy[TY + 3][TX];
    __shared__ T s_fx[3][TY][TX + 1], s_fy[3][TY + 1][TX];

    const Layout L = C.L;
    const int nx = L.nx, ny = L.ny, nxt = nx + 4, nyt = ny + 4;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int I0 = GL + blockIdx.x * TX, J0 = GL + blockIdx.y * TY;

    // tile + 2-cell halo of w, P, Q and eta = (w - bed_eff) - depth (dispersion.py:87)
    for (int k = tid; k < HY * HX; k += TX * TY) {
        int y = k / HX, x = k - y * HX;
        int J = J0 - 2 + y, I = I0 - 2 + x;
        T w = 0, p = 0, q = 0, e = 0;
        if (J < nyt && I < nxt) {
            long o = L.at(J, I);
            w = A.w[o];
            p = A.p[o];
            q = A.q[o];
            e = (w - A.be[o]) - A.dep[o];
        }
        s_w[y][x] = w;
        s_p[y][x] = p;
        s_q[y][x] = q;
        s_eta[y][x] = e;
    }
    for (int k = tid; k < TY * (TX + 3); k += TX * TY) {
        int y = k / (TX + 3), x = k - y * (TX + 3);
        int J = J0 + y, I = I0 - 2 + x;
        s_bfx[y][x] = (J < nyt && I <= nx + 2) ? A.bfx[L.at(J, I)] : T(0);
    }
    for (int k = tid; k < (TY + 3) * TX; k += TX * TY) {
        int y = k / TX, x = k - y * TX;
        int J = J0 - 2 + y, I = I0 + x;
        s_bfy[y][x] = (J <= ny + 2 && I < nxt) ? A.bfy[L.at(J, I)] : T(0);
    }
    __syncthreads();

    // x interfaces: between smem columns xi+1 (left cell) and xi+2 (right)
    for (int k = tid; k < TY * (TX + 1); k += TX * TY) {
        int r = k / (TX + 1), xi = k - r * (TX + 1);
        int y = r + 2;
        Faces<T> fl = cell_faces(s_w[y][xi], s_w[y][xi + 1], s_w[y][xi + 2], s_p[y][xi],
                                 s_p[y][xi + 1], s_p[y][xi + 2], s_q[y][xi], s_q[y][xi + 1],
                                 s_q[y][xi + 2], s_bfx[r][xi + 1], s_bfx[r][xi], C.theta);
        Faces<T> fr = cell_faces(s_w[y][xi + 1], s_w[y][xi + 2], s_w[y][xi + 3], s_p[y][xi + 1],
                                 s_p[y][xi + 2], s_p[y][xi + 3], s_q[y][xi + 1], s_q[y][xi + 2],
                                 s_q[y][xi + 3], s_bfx[r][xi + 2], s_bfx[r][xi + 1], C.theta);
        T f1, f2, f3;
        cu_flux(fl.whi, fr.wlo, fl.phi, fr.plo, fl.qhi, fr.qlo, s_bfx[r][xi + 1], C.g, C.h_eps,
                f1, f2, f3);
        s_fx[0][r][xi] = f1;
        s_fx[1][r][xi] = f2;
        s_fx[2][r][xi] = f3;
    }
    // y interfaces: between smem rows yi+1 (south cell) and yi+2 (north)
    for (int k = tid; k < (TY + 1) * TX; k += TX * TY) {
        int yi = k / TX, c = k - yi * TX;
        int x = c + 2;
        Faces<T> fs = cell_faces(s_w[yi][x], s_w[yi + 1][x], s_w[yi + 2][x], s_p[yi][x],
                                 s_p[yi + 1][x], s_p[yi + 2][x], s_q[yi][x], s_q[yi + 1][x],
                                 s_q[yi + 2][x], s_bfy[yi + 1][c], s_bfy[yi][c], C.theta);
        Faces<T> fn = cell_faces(s_w[yi + 1][x], s_w[yi + 2][x], s_w[yi + 3][x], s_p[yi + 1][x],
                                 s_p[yi + 2][x], s_p[yi + 3][x], s_q[yi + 1][x], s_q[yi + 2][x],
                                 s_q[yi + 3][x], s_bfy[yi + 2][c], s_bfy[yi + 1][c], C.theta);
        T f1, fq, fp;
        // normal momentum is Q, tangential is P: fy2 = P flux, fy3 = Q flux
        cu_flux(fs.whi, fn.wlo, fs.qhi, fn.qlo, fs.phi, fn.plo, s_bfy[yi + 1][c], C.g, C.h_eps,
                f1, fq, fp);
        s_fy[0][yi][c] = f1;
        s_fy[1][yi][c] = fp;
        s_fy[2][yi][c] = fq;
    }
    __syncthreads();

    const int J = J0 + ty, I = I0 + tx;
    if (J >= ny + GL || I >= nx + GL) return;
    const int y = ty + 2, x = tx + 2;
    const long o = L.at(J, I);
    const T wc = s_w[y][x], pc = s_p[y][x], qc = s_q[y][x];

    // fv_rates (_kernels.py:226-251)
    T rw = -(s_fx[0][ty][tx + 1] - s_fx[0][ty][tx]) * C.inv_dx -
           (s_fy[0][ty + 1][tx] - s_fy[0][ty][tx]) * C.inv_dy;
    T be_ = s_bfx[ty][tx + 2], bw_ = s_bfx[ty][tx + 1];
    T bn_ = s_bfy[ty + 2][tx], bs_ = s_bfy[ty + 1][tx];
    T src_x = -C.g * (wc - T(0.5) * (be_ + bw_)) * (be_ - bw_) * C.inv_dx;
    T src_y = -C.g * (wc - T(0.5) * (bn_ + bs_)) * (bn_ - bs_) * C.inv_dy;
    T h = wc - A.be[o];
    if (h < T(0)) h = T(0);
    T hstar = h > C.h_eps ? h : C.h_eps;
    T fric = T(0);
    if (C.c_f > T(0)) fric = C.c_f * sqrt(pc * pc + qc * qc) / (hstar * hstar);
    T rp = -(s_fx[1][ty][tx + 1] - s_fx[1][ty][tx]) * C.inv_dx -
           (s_fy[1][ty + 1][tx] - s_fy[1][ty][tx]) * C.inv_dy + src_x - fric * pc;
    T rq = -(s_fx[2][ty][tx + 1] - s_fx[2][ty][tx]) * C.inv_dx -
           (s_fy[2][ty + 1][tx] - s_fy[2][ty][tx]) * C.inv_dy + src_y - fric * qc;

    const T d = A.dep[o], dx_ = A.ddx[o], dy_ = A.ddy[o];
    T fs_, gs_;
    // dispersive_rates (_kernels.py:262-288)
    if (d > T(0)) {
        const T ec = s_eta[y][x];
        T e_xx = (s_eta[y][x + 1] - T(2) * ec + s_eta[y][x - 1]) * C.inv_dx2;
        T e_yy = (s_eta[y + 1][x] - T(2) * ec + s_eta[y - 1][x]) * C.inv_dy2;
        T e_xy = (s_eta[y + 1][x + 1] - s_eta[y + 1][x - 1] - s_eta[y - 1][x + 1] +
                  s_eta[y - 1][x - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
        T e_xxx = (s_eta[y][x + 2] - T(2) * s_eta[y][x + 1] + T(2) * s_eta[y][x - 1] -
                   s_eta[y][x - 2]) * T(0.5) * C.inv_dx * C.inv_dx2;
        T e_yyy = (s_eta[y + 2][x] - T(2) * s_eta[y + 1][x] + T(2) * s_eta[y - 1][x] -
                   s_eta[y - 2][x]) * T(0.5) * C.inv_dy * C.inv_dy2;
        T e_xyy = ((s_eta[y + 1][x + 1] - T(2) * s_eta[y][x + 1] + s_eta[y - 1][x + 1]) -
                   (s_eta[y + 1][x - 1] - T(2) * s_eta[y][x - 1] + s_eta[y - 1][x - 1])) *
                  T(0.5) * C.inv_dx * C.inv_dy2;
        T e_xxy = ((s_eta[y + 1][x + 1] - T(2) * s_eta[y + 1][x] + s_eta[y + 1][x - 1]) -
                   (s_eta[y - 1][x + 1] - T(2) * s_eta[y - 1][x] + s_eta[y - 1][x - 1])) *
                  T(0.5) * C.inv_dy * C.inv_dx2;
        T gd2 = C.g * d * d;
        T gd3 = gd2 * d;
        rp += C.b_disp * gd3 * (e_xxx + e_xyy) +
              C.b_disp * gd2 * (dx_ * (T(2) * e_xx + e_yy) + dy_ * e_xy);
        rq += C.b_disp * gd3 * (e_yyy + e_xxy) +
              C.b_disp * gd2 * (dy_ * (T(2) * e_yy + e_xx) + dx_ * e_xy);
        // cross_rates (_kernels.py:310-321)
        T q_x = (s_q[y][x + 1] - s_q[y][x - 1]) * T(0.5) * C.inv_dx;
        T q_y = (s_q[y + 1][x] - s_q[y - 1][x]) * T(0.5) * C.inv_dy;
        T q_xy = (s_q[y + 1][x + 1] - s_q[y + 1][x - 1] - s_q[y - 1][x + 1] + s_q[y - 1][x - 1]) *
                 T(0.25) * C.inv_dx * C.inv_dy;
        T p_x = (s_p[y][x + 1] - s_p[y][x - 1]) * T(0.5) * C.inv_dx;
        T p_y = (s_p[y + 1][x] - s_p[y - 1][x]) * T(0.5) * C.inv_dy;
        T p_xy = (s_p[y + 1][x + 1] - s_p[y + 1][x - 1] - s_p[y - 1][x + 1] + s_p[y - 1][x - 1]) *
                 T(0.25) * C.inv_dx * C.inv_dy;
        T sixth = div_static(d, C.six, C.r_six);
        T d2 = C.bp13 * d * d;
        fs_ = sixth * (dx_ * q_y + dy_ * q_x) + d2 * q_xy;
        gs_ = sixth * (dx_ * p_y + dy_ * p_x) + d2 * p_xy;
    } else {
        fs_ = T(0);
        gs_ = T(0);
    }

    // non-finite stage values (dispersion.py:92-98): first row-major cell
    const unsigned long long lin = (unsigned long long)(J - GL) * nx + (I - GL);
    if (!isfinite(rw)) atomicMin(&A.bad[0], lin);
    if (!isfinite(rp)) atomicMin(&A.bad[1], lin);
    if (!isfinite(rq)) atomicMin(&A.bad[2], lin);
    if (!isfinite(fs_)) atomicMin(&A.bad[3], lin);
    if (!isfinite(gs_)) atomicMin(&A.bad[4], lin);

    A.h0[0][o] = rw;
    A.h0[1][o] = rp;
    A.h0[2][o] = rq;
    A.h0[3][o] = fs_;
    A.h0[4][o] = gs_;
    if (!predict) return;

    // U*, V* (dispersion.py:131-148): divisions by grid constants
    T p_x = div_static(s_p[y][x + 1] - s_p[y][x - 1], C.two_dx, C.r_two_dx);
    T p_xx = div_static(s_p[y][x + 1] - T(2) * pc + s_p[y][x - 1], C.dx2, C.r_dx2);
    T ustar = pc - div_static(d * dx_, C.three, C.r_three) * p_x - C.bp13 * d * d * p_xx;
    T q_y = div_static(s_q[y + 1][x] - s_q[y - 1][x], C.two_dy, C.r_two_dy);
    T q_yy = div_static(s_q[y + 1][x] - T(2) * qc + s_q[y - 1][x], C.dy2, C.r_dy2);
    T vstar = qc - div_static(d * dy_, C.three, C.r_three) * q_y - C.bp13 * d * d * q_yy;

    // predictor (stepper.py:239-250, 109-132; multistep.py:139-153)
    T wn, bu, bv, us, vs;
    if (P->euler) {
        const T dt = T(P->dt);
        wn = wc + dt * rw;
        bu = ustar + dt * rp;
        bv = vstar + dt * rq;
        us = bu;
        vs = bv;
    } else {
        const T wc0 = T(P->wc), wp1 = T(P->wp), wp2 = T(P->wp2);
        const T s0 = T(P->sc), s1 = T(P->sp), s2 = T(P->sp2);
        wn = wc + (wc0 * rw + wp1 * A.h1[0][o] + wp2 * A.h2[0][o]);
        bu = ustar + (wc0 * rp + wp1 * A.h1[1][o] + wp2 * A.h2[1][o]);
        bv = vstar + (wc0 * rq + wp1 * A.h1[2][o] + wp2 * A.h2[2][o]);
        us = bu + (s0 * fs_ + s1 * A.h1[3][o] + s2 * A.h2[3][o]);
        vs = bv + (s0 * gs_ + s1 * A.h1[4][o] + s2 * A.h2[4][o]);
    }
    A.wn[o] = wn;
    A.bu[o] = bu;
    A.bv[o] = bv;
    A.us[o] = us;
    A.vs[o] = vs;
}

// ---------------------------------------------------------------------------
// tridiagonal line solves (pre-factored Thomas)

// F* at one cell from the solved Q (cross_rates sp, _kernels.py:305-320)
template <class T>
__device__ __forceinline__ T cross_f(const Consts<T> &C, const T *q, long o, T d, T dx_, T dy_) {
    if (d <= T(0)) return T(0);
    const long N = o + C.L.pitch, S = o - C.L.pitch;
    T q_x = (q[o + 1] - q[o - 1]) * T(0.5) * C.inv_dx;
    T q_y = (q[N] - q[S]) * T(0.5) * C.inv_dy;
    T q_xy = (q[N + 1] - q[N - 1] - q[S + 1] + q[S - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
    T sixth = div_static(d, C.six, C.r_six);
    T d2 = C.bp13 * d * d;
    return sixth * (dx_ * q_y + dy_ * q_x) + d2 * q_xy;
}

// G* from the solved P (cross_rates sq)
template <class T>
__device__ __forceinline__ T cross_g(const Consts<T> &C, const T *p, long o, T d, T dx_, T dy_) {
    if (d <= T(0)) return T(0);
    const long N = o + C.L.pitch, S = o - C.L.pitch;
    T p_x = (p[o + 1] - p[o - 1]) * T(0.5) * C.inv_dx;
    T p_y = (p[N] - p[S]) * T(0.5) * C.inv_dy;
    T p_xy = (p[N + 1] - p[N - 1] - p[S + 1] + p[S - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
    T sixth = div_static(d, C.six, C.r_six);
    T d2 = C.bp13 * d * d;
    return sixth * (dx_ * p_y + dy_ * p_x) + d2 * p_xy;
}

// Warp-specialized pipelined line solve.
//
// A CTA owns 32 lines (x: 32 consecutive rows; y: 32 consecutive columns).
// Warp 0 is the consumer: lane l runs line l's Thomas recurrence entirely
// out of shared memory.  Warps 1..7 are producers: per chunk of SK elements
// they stream the inputs with coalesced loads (a row segment for x, a
// 32-column row slice for y), assemble the folded right-hand side -- for
// phase 2 including the cross-correction F*(P1,Q1) stencil -- and write the
// consumer's results back.  Chunks are double buffered: while the consumer
// sweeps chunk c, producers fill chunk c+1 and drain chunk c-1.
//
// The LU factors of the static operator are precomputed on the host with
// thomas_batch's own arithmetic (den_i = b_i - a_i cw_{i-1},
// cw_i = c_i / den_i), so the per-step forward sweep
// dw_i = (r_i - a_i dw_{i-1}) / den_i and back substitution
// x_i = dw_i - cw_i x_{i+1} reproduce thomas_batch bit for bit.  The forward
// sweep's dw is parked in the output array and overwritten by x.
constexpr int SK = 32;           // chunk length (elements per line)
constexpr int SLD = SK + 1;      // padded smem row: conflict-free column access
constexpr int SW = 8;            // warps per CTA (1 consumer + 7 producers)
constexpr int SBUF = 32 * SLD;   // one [32][SLD] tile

template <class T>
struct SolveSmem {
    T r[2][SBUF], a[2][SBUF], den[2][SBUF], rden[2][SBUF], out[2][SBUF];
};

template <class T, bool XDIR>
__device__ __forceinline__ int tile_idx(int line, int k) {
    // x: [line][k] so a producer warp writes one row segment contiguously and
    //    the consumer reads a column (padded stride: conflict-free)
    // y: [k][line] so both sides touch 32 consecutive doubles
    return XDIR ? line * SLD + k : k * SLD + line;
}

template <class T, bool XDIR>
__device__ __forceinline__ long line_off(const Layout &L, int line, int k) {
    return XDIR ? L.at(GL + line, GL + k) : L.at(GL + k, GL + line);
}

template <class T, bool XDIR, int PHASE>
__device__ void solve_lines(const Consts<T> &C, const SolvePtrs<T> &S, int line0, SolveSmem<T> &sm) {
    const Layout L = C.L;
    const int n = XDIR ? L.nx : L.ny;           // line length
    const int nlines = XDIR ? L.ny : L.nx;
    const int nc = (n + SK - 1) / SK;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ptid = threadIdx.x - 32, np = (SW - 1) * 32;
    const T *rhs = XDIR ? S.rx : S.ry;
    const T *A = XDIR ? S.ax : S.ay;
    const T *DEN = XDIR ? S.denx : S.deny;
    const T *RDEN = XDIR ? S.rdenx : S.rdeny;
    const T *CW = XDIR ? S.cwx : S.cwy;
    const T *clast = XDIR ? S.cx_last : S.cy_last;
    T *out = XDIR ? S.outx : S.outy;

    // item -> (line, k) so consecutive producer lanes touch consecutive addresses
    auto item = [&](int it, int &ln, int &k) {
        if (XDIR) { ln = it >> 5; k = it & 31; } else { k = it >> 5; ln = it & 31; }
    };

    auto fill_fwd = [&](int c, int b) {
        for (int it = ptid; it < 32 * SK; it += np) {
            int ln, k;
            item(it, ln, k);
            const int line = line0 + ln, e = c * SK + k;
            const int t = tile_idx<T, XDIR>(ln, k);
            if (line >= nlines || e >= n) {
                sm.r[b][t] = T(0); sm.a[b][t] = T(0); sm.den[b][t] = T(1); sm.rden[b][t] = T(1);
                continue;
            }
            const long o = line_off<T, XDIR>(L, line, e);
            T r;
            if (PHASE == 1) {
                r = rhs[o];
            } else {  // us_corr = base + (F*(P1, Q1) - F*_n)   (stepper.py:272-273)
                T cr = XDIR ? cross_f(C, S.q1, o, S.dep[o], S.ddx[o], S.ddy[o])
                            : cross_g(C, S.p1, o, S.dep[o], S.ddx[o], S.ddy[o]);
                r = rhs[o] + (cr - (XDIR ? S.fs[o] : S.gs[o]));
            }
            const T a = A[o];
            if (e == 0) {  // implicit.py:178 / :190 ghost folding
                const T g0 = XDIR ? S.gp[L.at(GL + line, GL - 1)] : S.gq[L.at(GL - 1, GL + line)];
                r = r - a * g0;
            }
            if (e == n - 1) {
                const T g1 = XDIR ? S.gp[L.at(GL + line, n + GL)] : S.gq[L.at(n + GL, GL + line)];
                r = r - clast[line] * g1;
            }
            sm.r[b][t] = r;
            sm.a[b][t] = a;
            sm.den[b][t] = DEN[o];
            sm.rden[b][t] = RDEN[o];
        }
    };
    auto drain = [&](int c, int b) {  // out tile -> global
        for (int it = ptid; it < 32 * SK; it += np) {
            int ln, k;
            item(it, ln, k);
            const int line = line0 + ln, e = c * SK + k;
            if (line < nlines && e < n) out[line_off<T, XDIR>(L, line, e)] = sm.out[b][tile_idx<T, XDIR>(ln, k)];
        }
    };
    auto fill_bwd = [&](int c, int b) {  // dw (parked in out) and cw
        for (int it = ptid; it < 32 * SK; it += np) {
            int ln, k;
            item(it, ln, k);
            const int line = line0 + ln, e = c * SK + k;
            const int t = tile_idx<T, XDIR>(ln, k);
            if (line >= nlines || e >= n) {
                sm.r[b][t] = T(0); sm.a[b][t] = T(0);
                continue;
            }
            const long o = line_off<T, XDIR>(L, line, e);
            sm.r[b][t] = out[o];
            sm.a[b][t] = CW[o];
        }
    };

    // ---- forward sweep -------------------------------------------------------
    if (warp > 0) fill_fwd(0, 0);
    __syncthreads();
    T dw = T(0);
    for (int c = 0; c < nc; c++) {
        const int b = c & 1;
        if (warp == 0) {
            const int kmax = min(SK, n - c * SK);
            for (int k = 0; k < kmax; k++) {
                const int t = tile_idx<T, XDIR>(lane, k);
                const T r = sm.r[b][t];
                const T num = (c == 0 && k == 0) ? r : r - sm.a[b][t] * dw;
                dw = div_static(num, sm.den[b][t], sm.rden[b][t]);
                sm.out[b][t] = dw;
            }
        } else {
            if (c + 1 < nc) fill_fwd(c + 1, b ^ 1);
            if (c >= 1) drain(c - 1, b ^ 1);
        }
        __syncthreads();
    }
    if (warp > 0) drain(nc - 1, (nc - 1) & 1);
    __syncthreads();

    // ---- back substitution (chunks in reverse) -------------------------------
    if (warp > 0) fill_bwd(nc - 1, 0);
    __syncthreads();
    T xv = T(0);
    for (int s = 0; s < nc; s++) {
        const int c = nc - 1 - s, b = s & 1;
        if (warp == 0) {
            const int kmax = min(SK, n - c * SK);
            for (int k = kmax - 1; k >= 0; k--) {
                const int t = tile_idx<T, XDIR>(lane, k);
                xv = (s == 0 && k == kmax - 1) ? sm.r[b][t] : sm.r[b][t] - sm.a[b][t] * xv;
                sm.out[b][t] = xv;
            }
        } else {
            if (s + 1 < nc) fill_bwd(c - 1, b ^ 1);
            if (s >= 1) drain(c + 1, b ^ 1);
        }
        __syncthreads();
    }
    if (warp > 0) drain(0, (nc - 1) & 1);
}

// Blocks [0, nbx) take x lines (rows -> P); blocks [nbx, ...) y lines (columns -> Q).
template <class T, int PHASE>
__global__ void __launch_bounds__(SW * 32, 2) k_solve_pipe(Consts<T> C, SolvePtrs<T> S, int nbx) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SolveSmem<T> &sm = *reinterpret_cast<SolveSmem<T> *>(smem_raw);
    if ((int)blockIdx.x < nbx)
        solve_lines<T, true, PHASE>(C, S, blockIdx.x * 32, sm);
    else
        solve_lines<T, false, PHASE>(C, S, (blockIdx.x - nbx) * 32, sm);
}

// Reference single-thread-per-line variant (kept for A/B timing; not launched
// by the step).
template <class T>
__global__ void __launch_bounds__(64) k_solve(Consts<T> C, SolvePtrs<T> S, int phase, int nbx) {
    const Layout L = C.L;
    const int nx = L.nx, ny = L.ny;
    const bool xdir = (int)blockIdx.x < nbx;
    const int line = (xdir ? blockIdx.x : blockIdx.x - nbx) * blockDim.x + threadIdx.x;
    if (xdir) {
        if (line >= ny) return;
        const int J = GL + line;
        const T gw = S.gp[L.at(J, GL - 1)], ge = S.gp[L.at(J, nx + GL)];
        T dw = 0;
        for (int i = 0; i < nx; i++) {
            const long o = L.at(J, GL + i);
            T r;
            if (phase == 1) {
                r = S.rx[o];
            } else {  // us_corr = base_u + (F*(P1, Q1) - F*_n)   (stepper.py:272)
                r = S.rx[o] + (cross_f(C, S.q1, o, S.dep[o], S.ddx[o], S.ddy[o]) - S.fs[o]);
            }
            if (i == 0) r = r - S.ax[o] * gw;                       // implicit.py:178
            if (i == nx - 1) r = r - S.cx_last[line] * ge;           // implicit.py:179
            T num = i == 0 ? r : r - S.ax[o] * dw;
            dw = div_static(num, S.denx[o], S.rdenx[o]);
            S.scrx[o] = dw;
        }
        T xv = dw;
        S.outx[L.at(J, GL + nx - 1)] = xv;
        for (int i = nx - 2; i >= 0; i--) {
            const long o = L.at(J, GL + i);
            xv = S.scrx[o] - S.cwx[o] * xv;
            S.outx[o] = xv;
        }
    } else {
        if (line >= nx) return;
        const int I = GL + line;
        const T gs = S.gq[L.at(GL - 1, I)], gn = S.gq[L.at(ny + GL, I)];
        T dw = 0;
        for (int j = 0; j < ny; j++) {
            const long o = L.at(GL + j, I);
            T r;
            if (phase == 1) {
                r = S.ry[o];
            } else {
                r = S.ry[o] + (cross_g(C, S.p1, o, S.dep[o], S.ddx[o], S.ddy[o]) - S.gs[o]);
            }
            if (j == 0) r = r - S.ay[o] * gs;
            if (j == ny - 1) r = r - S.cy_last[line] * gn;
            T num = j == 0 ? r : r - S.ay[o] * dw;
            dw = div_static(num, S.deny[o], S.rdeny[o]);
            S.scry[o] = dw;
        }
        T xv = dw;
        S.outy[L.at(GL + ny - 1, I)] = xv;
        for (int j = ny - 2; j >= 0; j--) {
            const long o = L.at(GL + j, I);
            xv = S.scry[o] - S.cwy[o] * xv;
            S.outy[o] = xv;
        }
    }
}

// ---------------------------------------------------------------------------
// finalize: clamp, momenta, film, sponge, blow-up, extrema, reductions

constexpr int FX = 32, FY = 8, FT = FX * FY;

template <class T>
__global__ void __launch_bounds__(FT) k_final(Consts<T> C, FinalPtrs<T> F) {
    __shared__ double r_rate[FT], r_speed[FT], r_depth[FT], r_dev[FT], r_clamp[FT];
    __shared__ int r_nan[FT];
    __shared__ bool am_last;
    const Layout L = C.L;
    const int nx = L.nx, ny = L.ny;
    const int tid = threadIdx.y * FX + threadIdx.x;
    const int I = GL + blockIdx.x * FX + threadIdx.x, J = GL + blockIdx.y * FY + threadIdx.y;
    double m_rate = 0, m_speed = 0, m_depth = 0, m_dev = 0, clamp = 0;
    int dev_nan = 0;
    if (I < nx + GL && J < ny + GL) {
        const long o = L.at(J, I);
        const T be = F.be[o];
        T w = F.w[o];
        // clamp and volume tally (stepper.py:281-285); np.maximum keeps NaN
        T def = be - w;
        if (def > T(0) || def != def) clamp = double(def);
        w = (w >= be || w != w) ? w : be;
        T p = F.pin[o], q = F.qin[o];
        // film cutoff (stepper.py:288-292)
        if (C.h_dry > T(0) && (w - be) < C.h_dry) {
            p = T(0);
            q = T(0);
        }
        const T rest = C.ws > be ? C.ws : be;  // np.maximum(ws, bed_eff)
        // sponge bands in side order N, S, E, W (boundary.py:264-300)
#pragma unroll
        for (int side = 0; side < 4; side++) {
            if (C.side_kind[side] != KIND_SPONGE || C.sponge_len[side] == 0) continue;
            int k = (side == SIDE_E || side == SIDE_W) ? (I - GL) - C.sponge_lo[side]
                                                       : (J - GL) - C.sponge_lo[side];
            if (k < 0 || k >= C.sponge_len[side]) continue;
            const T fac = F.fac[side][k];
            w = rest + (w - rest) * fac;
            p = p * fac;
            q = q * fac;
        }
        F.w[o] = w;
        F.pout[o] = p;
        F.qout[o] = q;
        // blow-up deviation (stepper.py:295)
        T dv = w - rest;
        dv = dv < T(0) ? -dv : dv;
        if (dv != dv) dev_nan = 1; else m_dev = double(dv);
        const unsigned long long lin = (unsigned long long)(J - GL) * nx + (I - GL);
        if (!isfinite(w)) atomicMin(&F.res->state_bad[0], lin);
        if (!isfinite(p)) atomicMin(&F.res->state_bad[1], lin);
        if (!isfinite(q)) atomicMin(&F.res->state_bad[2], lin);
        // speed_extrema (_kernels.py:337-352)
        T h = w - be;
        if (h < T(0)) h = T(0);
        T hstar = h > C.h_eps ? h : C.h_eps;
        T c = sqrt(C.g * h);
        T su = fabs(p) / hstar + c;
        T sv = fabs(q) / hstar + c;
        T rate = nb_max(su * C.inv_dx, sv * C.inv_dy);
        m_depth = double(h);
        m_speed = double(nb_max(su, sv));
        m_rate = double(rate);
        if (!(m_speed > 0)) m_speed = 0;  // the serial scan skips NaN
        if (!(m_rate > 0)) m_rate = 0;
        if (!(m_depth > 0)) m_depth = 0;
    }
    r_rate[tid] = m_rate;
    r_speed[tid] = m_speed;
    r_depth[tid] = m_depth;
    r_dev[tid] = m_dev;
    r_clamp[tid] = clamp;
    r_nan[tid] = dev_nan;
    __syncthreads();
    for (int s = FT / 2; s > 0; s >>= 1) {
        if (tid < s) {
            r_rate[tid] = fmax(r_rate[tid], r_rate[tid + s]);
            r_speed[tid] = fmax(r_speed[tid], r_speed[tid + s]);
            r_depth[tid] = fmax(r_depth[tid], r_depth[tid + s]);
            r_dev[tid] = fmax(r_dev[tid], r_dev[tid + s]);
            r_clamp[tid] = r_clamp[tid] + r_clamp[tid + s];
            r_nan[tid] |= r_nan[tid + s];
        }
        __syncthreads();
    }
    const int nblk = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
    if (tid == 0) {
        Partial pt;
        pt.max_rate = r_rate[0];
        pt.max_speed = r_speed[0];
        pt.max_depth = r_depth[0];
        pt.max_dev = r_dev[0];
        pt.clamped = r_clamp[0];
        pt.dev_nan = r_nan[0];
        pt.pad_ = 0;
        F.part[bid] = pt;
        __threadfence();
        unsigned int prev = atomicAdd(F.counter, 1u);
        am_last = prev == (unsigned int)(nblk - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    // last block: fixed-order reduction of the partials (deterministic)
    double a = 0, b = 0, c = 0, d = 0, e = 0;
    int n = 0;
    for (int k = tid; k < nblk; k += FT) {
        const volatile Partial *pp = (const volatile Partial *)&F.part[k];
        a = fmax(a, pp->max_rate);
        b = fmax(b, pp->max_speed);
        c = fmax(c, pp->max_depth);
        d = fmax(d, pp->max_dev);
        e = e + pp->clamped;
        n |= pp->dev_nan;
    }
    r_rate[tid] = a;
    r_speed[tid] = b;
    r_depth[tid] = c;
    r_dev[tid] = d;
    r_clamp[tid] = e;
    r_nan[tid] = n;
    __syncthreads();
    for (int s = FT / 2; s > 0; s >>= 1) {
        if (tid < s) {
            r_rate[tid] = fmax(r_rate[tid], r_rate[tid + s]);
            r_speed[tid] = fmax(r_speed[tid], r_speed[tid + s]);
            r_depth[tid] = fmax(r_depth[tid], r_depth[tid + s]);
            r_dev[tid] = fmax(r_dev[tid], r_dev[tid + s]);
            r_clamp[tid] = r_clamp[tid] + r_clamp[tid + s];
            r_nan[tid] |= r_nan[tid + s];
        }
        __syncthreads();
    }
    if (tid == 0) {
        F.res->max_rate = r_rate[0];
        F.res->max_speed = r_speed[0];
        F.res->max_depth = r_depth[0];
        F.res->max_dev = r_nan[0] ? (double)NAN : r_dev[0];
        F.res->clamped = r_clamp[0];
        *F.counter = 0u;
    }
}

// speed extrema of an arbitrary state (construction-time extrema,
// stepper.py:210): reuses k_final's reduction tail with no state update.
template <class T>
__global__ void __launch_bounds__(FT) k_extrema(Consts<T> C, const T *w, const T *p, const T *q,
                                                const T *be, Partial *part) {
    __shared__ double r_rate[FT], r_speed[FT], r_depth[FT];
    const Layout L = C.L;
    const int tid = threadIdx.y * FX + threadIdx.x;
    const int I = GL + blockIdx.x * FX + threadIdx.x, J = GL + blockIdx.y * FY + threadIdx.y;
    double mr = 0, ms = 0, md = 0;
    if (I < L.nx + GL && J < L.ny + GL) {
        const long o = L.at(J, I);
        T h = w[o] - be[o];
        if (h < T(0)) h = T(0);
        T hstar = h > C.h_eps ? h : C.h_eps;
        T c = sqrt(C.g * h);
        T su = fabs(p[o]) / hstar + c;
        T sv = fabs(q[o]) / hstar + c;
        mr = double(nb_max(su * C.inv_dx, sv * C.inv_dy));
        ms = double(nb_max(su, sv));
        md = double(h);
        if (!(mr > 0)) mr = 0;
        if (!(ms > 0)) ms = 0;
        if (!(md > 0)) md = 0;
    }
    r_rate[tid] = mr;
    r_speed[tid] = ms;
    r_depth[tid] = md;
    __syncthreads();
    for (int s = FT / 2; s > 0; s >>= 1) {
        if (tid < s) {
            r_rate[tid] = fmax(r_rate[tid], r_rate[tid + s]);
            r_speed[tid] = fmax(r_speed[tid], r_speed[tid + s]);
            r_depth[tid] = fmax(r_depth[tid], r_depth[tid + s]);
        }
        __syncthreads();
    }
    if (tid == 0) {
        Partial pt{};
        pt.max_rate = r_rate[0];
        pt.max_speed = r_speed[0];
        pt.max_depth = r_depth[0];
        part[blockIdx.y * gridDim.x + blockIdx.x] = pt;
    }
}

// ---------------------------------------------------------------------------
// launchers

template <class T>
void launch_ghost(const Consts<T> &C, const DevParams *P, int which, const T *sw, const T *sp,
                  const T *sq, T *dw, T *dp, T *dq, cudaStream_t st) {
    int n = 4 * (C.L.ny + 4) + 4 * C.L.nx;
    k_ghost<T><<<(n + 127) / 128, 128, 0, st>>>(C, P, which, sw, sp, sq, dw, dp, dq);
}

template <class T>
void launch_stage(const Consts<T> &C, const DevParams *P, const StagePtrs<T> &A, int predict,
                  cudaStream_t st) {
    dim3 grid((C.L.nx + TX - 1) / TX, (C.L.ny + TY - 1) / TY);
    k_stage<T><<<grid, dim3(TX, TY), 0, st>>>(C, P, A, predict);
}

template <class T>
void launch_solve(const Consts<T> &C, const SolvePtrs<T> &S, int phase, cudaStream_t st) {
    const int nbx = (C.L.ny + 31) / 32, nby = (C.L.nx + 31) / 32;
    const size_t smem = sizeof(SolveSmem<T>);
    static bool attr_set[2] = {false, false};
    if (phase == 1) {
        if (!attr_set[0]) {
            cudaFuncSetAttribute(k_solve_pipe<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr_set[0] = true;
        }
        k_solve_pipe<T, 1><<<nbx + nby, SW * 32, smem, st>>>(C, S, nbx);
    } else {
        if (!attr_set[1]) {
            cudaFuncSetAttribute(k_solve_pipe<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr_set[1] = true;
        }
        k_solve_pipe<T, 2><<<nbx + nby, SW * 32, smem, st>>>(C, S, nbx);
    }
}

template <class T>
void launch_solve_simple(const Consts<T> &C, const SolvePtrs<T> &S, int phase, cudaStream_t st) {
    const int bs = 64;
    int nbx = (C.L.ny + bs - 1) / bs, nby = (C.L.nx + bs - 1) / bs;
    k_solve<T><<<nbx + nby, bs, 0, st>>>(C, S, phase, nbx);
}

template <class T>
void launch_final(const Consts<T> &C, const FinalPtrs<T> &F, cudaStream_t st) {
    dim3 grid((C.L.nx + FX - 1) / FX, (C.L.ny + FY - 1) / FY);
    k_final<T><<<grid, dim3(FX, FY), 0, st>>>(C, F);
}

int final_blocks(int nx, int ny) { return ((nx + FX - 1) / FX) * ((ny + FY - 1) / FY); }

template <class T>
void launch_extrema(const Consts<T> &C, const T *w, const T *p, const T *q, const T *be,
                    Partial *part, cudaStream_t st) {
    dim3 grid((C.L.nx + FX - 1) / FX, (C.L.ny + FY - 1) / FY);
    k_extrema<T><<<grid, dim3(FX, FY), 0, st>>>(C, w, p, q, be, part);
}

template void launch_ghost<double>(const Consts<double> &, const DevParams *, int, const double *,
                                   const double *, const double *, double *, double *, double *,
                                   cudaStream_t);
template void launch_stage<double>(const Consts<double> &, const DevParams *,
                                   const StagePtrs<double> &, int, cudaStream_t);
template void launch_solve<double>(const Consts<double> &, const SolvePtrs<double> &, int,
                                   cudaStream_t);
template void launch_final<double>(const Consts<double> &, const FinalPtrs<double> &,
                                   cudaStream_t);
template void launch_extrema<double>(const Consts<double> &, const double *, const double *,
                                     const double *, const double *, Partial *, cudaStream_t);

}  // namespace bsq
