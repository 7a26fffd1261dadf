// bsq_ghost.cu -- ghost-strip fill (boundary policies) for the Boussinesq step.
//
// A step launches, in order (see DESIGN.md for the HBM budget of each):
//   k_ghost      ghost strips at t                       (boundary.py:316-323)
//   k_stage      fused stage set + predictor             (bsq_stage_tiled.cu / bsq_stage.cu)
//   k_ghost      strips of the predicted state at t+dt   (stepper.py:252-254)
//   k_solve_tma  first x/y line solves                   (bsq_solve.cu)
//   k_correct    cross-correction right-hand sides       (bsq_correct.cu)
//   k_solve_tma  second x/y line solves
//   k_final      clamp, film, sponge, checks, extrema    (bsq_final.cu)
// and, when the next stage is queued early, k_frame (save of this state's
// ghost frame) + the next step's k_ghost and k_stage.
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
// index of ghost cell (J, I) in k_frame's buffer (rows 0, 1, ny+2, ny+3 over
// the padded width, then columns 0, 1, nx+2, nx+3 over the interior rows)
__device__ __forceinline__ long frame_index(int nx, int ny, int J, int I) {
    const int W = nx + 4;
    if (J < GL || J >= ny + GL) return (long)(J < GL ? J : J - ny) * W + I;
    return 4L * W + (long)(I < GL ? I : I - nx) * ny + (J - GL);
}

template <class T>
__global__ void k_ghost(Consts<T> C, const DevParams *__restrict__ P, int which, const T *src_w,
                        const T *src_p, const T *src_q, T *dst_w, T *dst_p, T *dst_q, T *save) {
    pdl_trigger();
    pdl_wait();
    const int nx = C.L.nx, ny = C.L.ny, nxt = nx + 4, nyt = ny + 4;
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    const T *src[3] = {src_w, src_p, src_q};
    T *dst[3] = {dst_w, dst_p, dst_q};
    const long nframe = 4L * nxt + 4L * ny;
    // the frame save: every frame cell is written by exactly one thread, which
    // reads its old value first
    // every read of a thread (its sources, and the old ghost values the frame
    // save keeps) is issued before its first store: the compiler cannot reorder
    // them itself (src and dst may be the same arrays), and serialized they
    // made the fill three memory round trips long
    auto write3 = [&](int J, int I, const T (&v)[3]) {
        const long o = C.L.at(J, I);
        if (save) {
            T old[3];
#pragma unroll
            for (int f = 0; f < 3; f++) old[f] = dst[f][o];
            const long fi = frame_index(nx, ny, J, I);
#pragma unroll
            for (int f = 0; f < 3; f++) save[f * nframe + fi] = old[f];
        }
#pragma unroll
        for (int f = 0; f < 3; f++) dst[f][o] = v[f];
    };
    if (k < 4 * nyt) {
        int J = k >> 2;
        int c = k & 3;  // 0,1 -> west cols 0,1; 2,3 -> east cols nxt-2, nxt-1
        int I = c < 2 ? c : nxt - 4 + c;
        int side = c < 2 ? SIDE_W : SIDE_E;
        bool interior_row = J >= GL && J < nyt - GL;
        // a strip's halo rows (internal N/S side) belong to the neighbour rank
        if (!interior_row && C.side_kind[J < GL ? SIDE_S : SIDE_N] == KIND_INTERNAL) return;
        if (C.side_kind[side] == KIND_MAKER) {
            double gw = which ? P->gw_n[side] : P->gw_t[side];
            double gf = which ? P->gf_n[side] : P->gf_t[side];
            const T v[3] = {T(gw), side == SIDE_W ? T(gf) : T(-gf), T(0)};
            write3(J, I, v);
            return;
        }
        int Im = side == SIDE_W ? (I == GL - 1 ? GL : GL + 1) : (I == nxt - GL ? nxt - GL - 1 : nxt - GL - 2);
        T v[3];
#pragma unroll
        for (int f = 0; f < 3; f++) {
            T cur = interior_row ? src[f][C.L.at(J, Im)] : ns_value(C, P, which, f, J, Im, src[f]);
            v[f] = (f == 1 ? T(-1) : T(1)) * cur;  // P is the wall-normal flux on E/W
        }
        write3(J, I, v);
        return;
    }
    k -= 4 * nyt;
    if (k < 4 * nx) {
        int I = GL + (k >> 2);
        int r = k & 3;
        int J = r < 2 ? r : nyt - 4 + r;
        if (C.side_kind[J < GL ? SIDE_S : SIDE_N] == KIND_INTERNAL) return;
        T v[3];
#pragma unroll
        for (int f = 0; f < 3; f++) v[f] = ns_value(C, P, which, f, J, I, src[f]);
        write3(J, I, v);
    }
}

// The 2-cell ghost frame of (w, p, q): rows 0, 1, ny+2, ny+3 over the padded
// width, then columns 0, 1, nx+2, nx+3 over the interior rows.  save = 1
// copies frame -> buf, 0 copies buf -> frame.  Used to keep a state's
// user-visible ghosts while a queued next stage runs on ghosts at t_{n+1}.
template <class T>
__global__ void k_frame(Consts<T> C, T *w, T *p, T *q, T *buf, int save) {
    const Layout L = C.L;
    const int W = L.nx + 4, nrow = 4 * W, n = nrow + 4 * L.ny;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int J, I;
    if (k < nrow) {
        const int r = k / W;
        J = r < 2 ? r : L.ny + r;  // 0, 1, ny+2, ny+3
        I = k - r * W;
    } else {
        const int kk = k - nrow, c = kk / L.ny;
        J = GL + (kk - c * L.ny);
        I = c < 2 ? c : L.nx + c;  // 0, 1, nx+2, nx+3
    }
    const long o = L.at(J, I);
    T *f[3] = {w, p, q};
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (save)
            buf[(long)a * n + k] = f[a][o];
        else
            f[a][o] = buf[(long)a * n + k];
    }
}

template <class T>
void launch_frame(const Consts<T> &C, T *w, T *p, T *q, T *buf, int save, cudaStream_t st) {
    const int n = 4 * (C.L.nx + 4) + 4 * C.L.ny;
    k_frame<T><<<(n + 255) / 256, 256, 0, st>>>(C, w, p, q, buf, save);
}

#if BSQ_INST_F64
size_t frame_elems(int nx, int ny) { return 3 * ((size_t)4 * (nx + 4) + (size_t)4 * ny); }
#endif

#if BSQ_INST_F64
template void launch_frame<double>(const Consts<double> &, double *, double *, double *, double *,
                                   int, cudaStream_t);
#endif
#if BSQ_INST_F32
template void launch_frame<float>(const Consts<float> &, float *, float *, float *, float *, int,
                                  cudaStream_t);
#endif

template <class T>
void launch_ghost(const Consts<T> &C, const DevParams *P, int which, const T *sw, const T *sp,
                  const T *sq, T *dw, T *dp, T *dq, cudaStream_t st, T *save) {
    int n = 4 * (C.L.ny + 4) + 4 * C.L.nx;
    launch_k(k_ghost<T>, dim3((n + 127) / 128), dim3(128), 0, st, C, P, which, sw, sp, sq, dw, dp, dq,
             save);
}

#if BSQ_INST_F64
template void launch_ghost<double>(const Consts<double> &, const DevParams *, int, const double *,
                                   const double *, const double *, double *, double *, double *,
                                   cudaStream_t, double *);
#endif
#if BSQ_INST_F32
template void launch_ghost<float>(const Consts<float> &, const DevParams *, int, const float *,
                                  const float *, const float *, float *, float *, float *,
                                  cudaStream_t, float *);
#endif

}  // namespace bsq
