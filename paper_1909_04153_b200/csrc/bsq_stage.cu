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

template void launch_ghost<double>(const Consts<double> &, const DevParams *, int, const double *,
                                   const double *, const double *, double *, double *, double *,
                                   cudaStream_t);
template void launch_stage<double>(const Consts<double> &, const DevParams *,
                                   const StagePtrs<double> &, int, cudaStream_t);

}  // namespace bsq
