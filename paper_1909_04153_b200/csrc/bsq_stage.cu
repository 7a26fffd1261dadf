// bsq_stage.cu -- the fused stage kernel: everything a step evaluates on the
// state at t_n, in one pass over HBM.
//
// Per interior cell this computes the reference's
//   faces_x/faces_y  (_kernels.py:29-103)   limited faces + positivity shift
//   flux_x/flux_y    (_kernels.py:106-212)  central-upwind fluxes, wet/dry
//   fv_rates         (_kernels.py:215-251)  divergence, bed source, friction
//   eta + dispersive_rates (dispersion.py:87, _kernels.py:254-288)
//   cross_rates      (_kernels.py:291-321)  F*, G*
//   compute_ustar_vstar (dispersion.py:120-149)
//   Euler / AB3 predictor (stepper.py:239-250, 109-132; multistep.py:139-153)
// and writes the new stage level, the predicted w, U*, V* and the
// quadrature bases.  Faces and fluxes never leave registers.
//
// Column walk.  A CTA covers 32 columns x (NW*R) rows; w, P, Q and eta of the
// tile plus a 2-cell halo are staged in shared memory once (the only
// barrier).  Lane l of warp k owns column I0+l and walks rows
// J0+k*R .. J0+k*R+R-1 upwards:
//   y direction: the faces of row J+1 and the flux through the J|J+1 face
//     are computed once and carried to the next row, where they are the
//     south face/flux -- every y interface is evaluated exactly once;
//   x direction: each lane evaluates its own cell's faces and the flux
//     through its west face; the west neighbour's east face and the east
//     neighbour's west flux arrive by warp shuffle.  The tile's edge cells
//     (column I0-1's east face, and the flux through the tile's east edge)
//     are batched for all R rows in one pre-pass on R lanes.
// Every interface flux is a function of the same face values as in the
// reference, so the result is bitwise the reference's.
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "bsq_device.cuh"
#include "bsq_launch.h"

namespace bsq {

constexpr int SW_ = 32;          // columns per CTA (one per lane)
#ifndef BSQ_CW_WARPS
#define BSQ_CW_WARPS 4
#endif
#ifndef BSQ_CW_ROWS
#define BSQ_CW_ROWS 4
#endif
constexpr int SNW = BSQ_CW_WARPS;  // warps per CTA
constexpr int SR = BSQ_CW_ROWS;    // rows per warp
constexpr int STY = SNW * SR;    // rows per CTA
constexpr int SHX = SW_ + 4, SHY = STY + 4;
constexpr unsigned FULL = 0xffffffffu;
static_assert(SR <= 16, "edge pre-pass uses lanes 0..SR-1 and 16..16+SR-1");

// per-cell inputs a row consumes after its flux work, landed by cp.async
enum { CI_BE, CI_D, CI_DX, CI_DY, CI_H1, CI_H2 = CI_H1 + 5, CI_N = CI_H2 + 5 };

template <class T>
struct StageSmem {
    T w[SHY][SHX], p[SHY][SHX], q[SHY][SHX], eta[SHY][SHX];
    T cin[SNW][CI_N][SW_];  // this row's cell inputs, per warp
};

__device__ __forceinline__ void cp_async_elem(void *dst, const void *src, int bytes) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <class T>
__device__ __forceinline__ T shfl_idx(T v, int src) { return __shfl_sync(FULL, v, src); }
template <class T>
__device__ __forceinline__ T shfl_up1(T v) { return __shfl_up_sync(FULL, v, 1); }
template <class T>
__device__ __forceinline__ T shfl_dn1(T v) { return __shfl_down_sync(FULL, v, 1); }

template <class T>
__global__ void __launch_bounds__(SW_ *SNW, 4) k_stage(Consts<T> C, const DevParams *__restrict__ P,
                                                   StagePtrs<T> A, int predict, int row0) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    StageSmem<T> &S = *reinterpret_cast<StageSmem<T> *>(smem_raw);
    pdl_trigger();
    pdl_wait();
    const Layout L = C.L;
    const int nx = L.nx, ny = L.ny, nxt = nx + 4, nyt = ny + 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int I0 = GL + blockIdx.x * SW_, J0 = GL + row0 + blockIdx.y * STY;

    // ---- tile + 2-cell halo; eta = (w - bed_eff) - depth (dispersion.py:87) ----
    // batches of LB items per thread, all loads of a batch in flight together
    constexpr int NTH = SW_ * SNW, NIT = (SHY * SHX + NTH - 1) / NTH, LB = 4;
#pragma unroll 1
    for (int b = 0; b < NIT; b += LB) {
        T vw[LB], vp[LB], vq[LB], vb[LB], vd[LB];
#pragma unroll
        for (int u = 0; u < LB; u++) {
            const int k = threadIdx.x + (b + u) * NTH;
            const int y = k / SHX, x = k - y * SHX;
            const int J = J0 - 2 + y, I = I0 - 2 + x;
            const bool in = k < SHY * SHX && J < nyt && I < nxt;
            const long o = in ? L.at(J, I) : L.at(GL, GL);
            vw[u] = A.w[o];
            vp[u] = A.p[o];
            vq[u] = A.q[o];
            vb[u] = A.be[o];
            vd[u] = A.dep[o];
        }
#pragma unroll
        for (int u = 0; u < LB; u++) {
            const int k = threadIdx.x + (b + u) * NTH;
            if (k >= SHY * SHX) continue;
            const int y = k / SHX, x = k - y * SHX;
            const int J = J0 - 2 + y, I = I0 - 2 + x;
            const bool in = J < nyt && I < nxt;
            S.w[y][x] = in ? vw[u] : T(0);
            S.p[y][x] = in ? vp[u] : T(0);
            S.q[y][x] = in ? vq[u] : T(0);
            S.eta[y][x] = in ? (vw[u] - vb[u]) - vd[u] : T(0);
        }
    }
    __syncthreads();

    const int I = I0 + lane, x = lane + 2;  // this lane's column (padded / smem)
    const int jw = J0 + warp * SR;          // first row of this warp
    const T g = C.g, hg = C.half_g, h_eps = C.h_eps, theta = C.theta;
    // bed on face (J, col) -- clamped to the array for out-of-grid lanes
    auto bfx_at = [&](int J, int col) -> T {
        return (J < nyt && col <= nx + 2) ? A.bfx[L.at(J, col)] : T(0);
    };
    auto bfy_at = [&](int J, int col) -> T {
        return (J <= ny + 2 && col < nxt) ? A.bfy[L.at(J, col)] : T(0);
    };
    // x faces of the cell at smem (yy, xx), face beds bhi (east), blo (west)
    auto xfaces = [&](int yy, int xx, T bhi, T blo) {
        return cell_faces(S.w[yy][xx - 1], S.w[yy][xx], S.w[yy][xx + 1], S.p[yy][xx - 1],
                          S.p[yy][xx], S.p[yy][xx + 1], S.q[yy][xx - 1], S.q[yy][xx],
                          S.q[yy][xx + 1], bhi, blo, theta);
    };
    auto yfaces = [&](int yy, int xx, T bhi, T blo) {
        return cell_faces(S.w[yy - 1][xx], S.w[yy][xx], S.w[yy + 1][xx], S.p[yy - 1][xx],
                          S.p[yy][xx], S.p[yy + 1][xx], S.q[yy - 1][xx], S.q[yy][xx],
                          S.q[yy + 1][xx], bhi, blo, theta);
    };

    // ---- x edge pre-pass (lanes 0..SR-1: one row each) --------------------------
    // east face of column I0-1, and the flux through the tile's east edge
    // (between columns I0+31 and I0+32), for rows jw .. jw+SR-1
    T e_w = 0, e_p = 0, e_q = 0, fe1 = 0, fe2 = 0, fe3 = 0;
    if (lane < SR) {
        const int J = jw + lane, yy = J - (J0 - 2);
        const Faces<T> fw = xfaces(yy, 1, bfx_at(J, I0 - 1), bfx_at(J, I0 - 2));
        e_w = fw.whi;
        e_p = fw.phi;
        e_q = fw.qhi;
        const T b31 = bfx_at(J, I0 + 31);
        const Faces<T> fl = xfaces(yy, SW_ + 1, b31, bfx_at(J, I0 + 30));
        const Faces<T> fr = xfaces(yy, SW_ + 2, bfx_at(J, I0 + 32), b31);
        cu_flux_rcp(fl.whi, fr.wlo, fl.phi, fr.plo, fl.qhi, fr.qlo, b31, g, hg, h_eps, fe1, fe2, fe3);
    }

    // ---- y pre-pass: faces of rows jw-1 and jw, flux through their face ---------
    T bfy_s = bfy_at(jw - 1, I);  // bed on the south face of the current row
    T bfy_n = bfy_at(jw, I);
    Faces<T> yc;  // y faces of the current row (only the north face is used)
    T fs1, fs2, fs3;
    {
        const int yy = jw - (J0 - 2);
        const Faces<T> ys = yfaces(yy - 1, x, bfy_s, bfy_at(jw - 2, I));
        yc = yfaces(yy, x, bfy_n, bfy_s);
        T fq, fp;  // normal momentum is Q, tangential is P: fy2 = P flux, fy3 = Q flux
        cu_flux_rcp(ys.whi, yc.wlo, ys.qhi, yc.qlo, ys.phi, yc.plo, bfy_s, g, hg, h_eps, fs1, fq, fp);
        fs2 = fp;
        fs3 = fq;
    }

    T bfx_e = bfx_at(jw, I);  // prefetch row jw's face beds
    const bool ab3 = predict && !P->euler;
    for (int r = 0; r < SR; r++) {
        const int J = jw + r, yy = J - (J0 - 2);
        const bool cell = J < ny + GL && I < nx + GL;
        // this row's per-cell inputs go straight to shared memory (cp.async):
        // in flight during the flux work, holding no registers
        const long o = cell ? L.at(J, I) : L.at(GL, GL);
        T(*ci)[SW_] = S.cin[warp];
        cp_async_elem(&ci[CI_BE][lane], A.be + o, sizeof(T));
        cp_async_elem(&ci[CI_D][lane], A.dep + o, sizeof(T));
        cp_async_elem(&ci[CI_DX][lane], A.ddx + o, sizeof(T));
        cp_async_elem(&ci[CI_DY][lane], A.ddy + o, sizeof(T));
        if (ab3) {
#pragma unroll
            for (int f = 0; f < 5; f++) {
                cp_async_elem(&ci[CI_H1 + f][lane], A.h1[f] + o, sizeof(T));
                cp_async_elem(&ci[CI_H2 + f][lane], A.h2[f] + o, sizeof(T));
            }
        }
        cp_async_commit();
        const T bfy_nn = bfy_at(J + 1, I);
        // -- x: own faces, the west flux, the east flux from the east lane --
        const T bx_e = bfx_e;                       // bed_face_x[J][I]
        T bx_w = shfl_up1(bx_e);                    // bed_face_x[J][I-1]
        if (lane == 0) bx_w = bfx_at(J, I0 - 1);
        if (r + 1 < SR) bfx_e = bfx_at(J + 1, I);
        const Faces<T> xf = xfaces(yy, x, bx_e, bx_w);
        T lw = shfl_up1(xf.whi), lp = shfl_up1(xf.phi), lq = shfl_up1(xf.qhi);
        const T ew = shfl_idx(e_w, r), ep = shfl_idx(e_p, r), eq = shfl_idx(e_q, r);
        if (lane == 0) {
            lw = ew;
            lp = ep;
            lq = eq;
        }
        T fw1, fw2, fw3;  // flux through the west face of this cell
        cu_flux_rcp(lw, xf.wlo, lp, xf.plo, lq, xf.qlo, bx_w, g, hg, h_eps, fw1, fw2, fw3);
        T fe_1 = shfl_dn1(fw1), fe_2 = shfl_dn1(fw2), fe_3 = shfl_dn1(fw3);
        const T g1 = shfl_idx(fe1, r), g2 = shfl_idx(fe2, r), g3 = shfl_idx(fe3, r);
        if (lane == SW_ - 1) {
            fe_1 = g1;
            fe_2 = g2;
            fe_3 = g3;
        }
        // -- y: faces of row J+1, flux through the J|J+1 face (carried north) --
        const Faces<T> yn = yfaces(yy + 1, x, bfy_nn, bfy_n);
        T fn1, fnq, fnp;
        cu_flux_rcp(yc.whi, yn.wlo, yc.qhi, yn.qlo, yc.phi, yn.plo, bfy_n, g, hg, h_eps, fn1, fnq, fnp);
        const T fn2 = fnp, fn3 = fnq;

        cp_async_wait_all();  // this lane's cell inputs have landed
        if (cell) {
            const T wc = S.w[yy][x], pc = S.p[yy][x], qc = S.q[yy][x];
            if (A.maxw) A.maxw[o] = np_maximum(A.maxw[o], wc);  // MaxSurfaceTracker fold
            const T c_be = ci[CI_BE][lane], c_d = ci[CI_D][lane];
            const T c_dx = ci[CI_DX][lane], c_dy = ci[CI_DY][lane];
            // fv_rates (_kernels.py:230-251)
            T rw = -(fe_1 - fw1) * C.inv_dx - (fn1 - fs1) * C.inv_dy;
            const T src_x = -g * (wc - T(0.5) * (bx_e + bx_w)) * (bx_e - bx_w) * C.inv_dx;
            const T src_y = -g * (wc - T(0.5) * (bfy_n + bfy_s)) * (bfy_n - bfy_s) * C.inv_dy;
            T h = wc - c_be;
            h = floor0(h);
            const T hstar = floor_eps(h, h_eps);
            T fric = T(0);
            if (C.c_f > T(0)) fric = C.c_f * sqrt(pc * pc + qc * qc) / (hstar * hstar);
            T rp = -(fe_2 - fw2) * C.inv_dx - (fn2 - fs2) * C.inv_dy + src_x - fric * pc;
            T rq = -(fe_3 - fw3) * C.inv_dx - (fn3 - fs3) * C.inv_dy + src_y - fric * qc;

            const T d = c_d, dx_ = c_dx, dy_ = c_dy;
            T fs_ = T(0), gs_ = T(0);
            if (d > T(0)) {
                // dispersive_rates (_kernels.py:269-288)
                const T(*E)[SHX] = S.eta;
                const T ec = E[yy][x];
                const T e_xx = (E[yy][x + 1] - T(2) * ec + E[yy][x - 1]) * C.inv_dx2;
                const T e_yy = (E[yy + 1][x] - T(2) * ec + E[yy - 1][x]) * C.inv_dy2;
                const T e_xy = (E[yy + 1][x + 1] - E[yy + 1][x - 1] - E[yy - 1][x + 1] +
                                E[yy - 1][x - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
                const T e_xxx = (E[yy][x + 2] - T(2) * E[yy][x + 1] + T(2) * E[yy][x - 1] -
                                 E[yy][x - 2]) * T(0.5) * C.inv_dx * C.inv_dx2;
                const T e_yyy = (E[yy + 2][x] - T(2) * E[yy + 1][x] + T(2) * E[yy - 1][x] -
                                 E[yy - 2][x]) * T(0.5) * C.inv_dy * C.inv_dy2;
                const T e_xyy = ((E[yy + 1][x + 1] - T(2) * E[yy][x + 1] + E[yy - 1][x + 1]) -
                                 (E[yy + 1][x - 1] - T(2) * E[yy][x - 1] + E[yy - 1][x - 1])) *
                                T(0.5) * C.inv_dx * C.inv_dy2;
                const T e_xxy = ((E[yy + 1][x + 1] - T(2) * E[yy + 1][x] + E[yy + 1][x - 1]) -
                                 (E[yy - 1][x + 1] - T(2) * E[yy - 1][x] + E[yy - 1][x - 1])) *
                                T(0.5) * C.inv_dy * C.inv_dx2;
                const T gd2 = g * d * d;
                const T gd3 = gd2 * d;
                rp += C.b_disp * gd3 * (e_xxx + e_xyy) +
                      C.b_disp * gd2 * (dx_ * (T(2) * e_xx + e_yy) + dy_ * e_xy);
                rq += C.b_disp * gd3 * (e_yyy + e_xxy) +
                      C.b_disp * gd2 * (dy_ * (T(2) * e_yy + e_xx) + dx_ * e_xy);
                // cross_rates (_kernels.py:310-321)
                const T(*Q)[SHX] = S.q;
                const T(*Pp)[SHX] = S.p;
                const T q_x = (Q[yy][x + 1] - Q[yy][x - 1]) * T(0.5) * C.inv_dx;
                const T q_y = (Q[yy + 1][x] - Q[yy - 1][x]) * T(0.5) * C.inv_dy;
                const T q_xy = (Q[yy + 1][x + 1] - Q[yy + 1][x - 1] - Q[yy - 1][x + 1] +
                                Q[yy - 1][x - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
                const T p_x = (Pp[yy][x + 1] - Pp[yy][x - 1]) * T(0.5) * C.inv_dx;
                const T p_y = (Pp[yy + 1][x] - Pp[yy - 1][x]) * T(0.5) * C.inv_dy;
                const T p_xy = (Pp[yy + 1][x + 1] - Pp[yy + 1][x - 1] - Pp[yy - 1][x + 1] +
                                Pp[yy - 1][x - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
                const T sixth = div_pos(d, C.six, C.r_six);
                const T d2 = C.bp13 * d * d;
                fs_ = sixth * (dx_ * q_y + dy_ * q_x) + d2 * q_xy;
                gs_ = sixth * (dx_ * p_y + dy_ * p_x) + d2 * p_xy;
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

            if (predict) {
                // U*, V* (dispersion.py:131-148): divisions by grid constants
                const T pe = S.p[yy][x + 1], pw = S.p[yy][x - 1];
                const T qn = S.q[yy + 1][x], qs = S.q[yy - 1][x];
                const T p_x = div_pos(pe - pw, C.two_dx, C.r_two_dx);
                const T p_xx = div_pos(pe - T(2) * pc + pw, C.dx2, C.r_dx2);
                const T ustar =
                    pc - div_pos(d * dx_, C.three, C.r_three) * p_x - C.bp13 * d * d * p_xx;
                const T q_y = div_pos(qn - qs, C.two_dy, C.r_two_dy);
                const T q_yy = div_pos(qn - T(2) * qc + qs, C.dy2, C.r_dy2);
                const T vstar =
                    qc - div_pos(d * dy_, C.three, C.r_three) * q_y - C.bp13 * d * d * q_yy;
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
                    const T(*h1v)[SW_] = &ci[CI_H1];
                    const T(*h2v)[SW_] = &ci[CI_H2];
                    wn = wc + (wc0 * rw + wp1 * h1v[0][lane] + wp2 * h2v[0][lane]);
                    bu = ustar + (wc0 * rp + wp1 * h1v[1][lane] + wp2 * h2v[1][lane]);
                    bv = vstar + (wc0 * rq + wp1 * h1v[2][lane] + wp2 * h2v[2][lane]);
                    us = bu + (s0 * fs_ + s1 * h1v[3][lane] + s2 * h2v[3][lane]);
                    vs = bv + (s0 * gs_ + s1 * h1v[4][lane] + s2 * h2v[4][lane]);
                }
                A.wn[o] = wn;
                A.bu[o] = bu;
                A.bv[o] = bv;
                A.us[o] = us;
                A.vs[o] = vs;
            }
        }
        // carry north: this row's north face/flux is the next row's south
        yc = yn;
        fs1 = fn1;
        fs2 = fn2;
        fs3 = fn3;
        bfy_s = bfy_n;
        bfy_n = bfy_nn;
    }
}

template <class T>
void launch_stage_tiled(const Consts<T> &C, const DevParams *P, const StagePtrs<T> &A, int predict,
                        cudaStream_t st, const StageMaps *M, int row0, int nrows);

// Both precisions run the tiled variant (bsq_stage_tiled.cu; fp64: 64
// registers, 32 warps per SM -- the column walk below needs 128 fp64
// registers and loses on latency hiding, 1.317 vs 1.114 ms at 4096^2; fp32:
// 0.473 vs 0.593 ms for the column walk once the fp32 boxes start on 16-B
// boundaries).  BSQ_F32_TILED=0 selects the fp32 column walk (A/B only).
template <class T>
void launch_stage(const Consts<T> &C, const DevParams *P, const StagePtrs<T> &A, int predict,
                  cudaStream_t st, const StageMaps *M, int row0, int nrows) {
    static_assert(STAGE_BAND % STY == 0 && STAGE_BAND % STAGE_TY == 0, "band of whole tiles");
    if (nrows < 0) nrows = C.L.ny - row0;
    if (nrows <= 0) return;
    static const bool f32_tiled = [] {
        const char *e = std::getenv("BSQ_F32_TILED");
        return !(e && e[0] == '0');
    }();
    if (sizeof(T) == 8 || f32_tiled) {
        launch_stage_tiled(C, P, A, predict, st, M, row0, nrows);
    } else {
        const size_t smem = sizeof(StageSmem<T>);
        static bool attr_set = false;
        if (!attr_set) {
            cudaFuncSetAttribute(k_stage<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            attr_set = true;
        }
        dim3 grid((C.L.nx + SW_ - 1) / SW_, (nrows + STY - 1) / STY);
        launch_k(k_stage<T>, grid, dim3(SW_ * SNW), smem, st, C, P, A, predict, row0);
    }
}

#if BSQ_INST_F64
template void launch_stage<double>(const Consts<double> &, const DevParams *,
                                   const StagePtrs<double> &, int, cudaStream_t, const StageMaps *,
                                   int, int);
#endif
#if BSQ_INST_F32
template void launch_stage<float>(const Consts<float> &, const DevParams *,
                                  const StagePtrs<float> &, int, cudaStream_t, const StageMaps *,
                                  int, int);
#endif

}  // namespace bsq
