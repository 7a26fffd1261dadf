// bsq_correct.cu -- cross-correction right-hand sides of the second solve.
#include <cstdint>

#include "bsq_device.cuh"
#include "bsq_launch.h"

namespace bsq {

// ---------------------------------------------------------------------------
// Cross-correction right-hand sides (stepper.py:268-273):
//   us_corr = base_u + (F*(P1, Q1) - F*_n),  vs_corr = base_v + (G*(P1, Q1) - G*_n)
// written over us / vs.
// Each thread owns CR consecutive cells of one column (2 in fp64, 4 in fp32:
// 0.140 -> 0.135 ms; 8 rows 0.203 ms); the 3-column window
// of P1 and Q1 over rows J-1 .. J+CR is loaded once and shared, and every
// load is issued before any arithmetic: the kernel is a pure stream.
#ifndef BSQ_CORRECT_CR32
#define BSQ_CORRECT_CR32 4
#endif
#ifndef BSQ_CORRECT_CR64
#define BSQ_CORRECT_CR64 2
#endif
template <class T>
__host__ __device__ constexpr int cr_rows() { return sizeof(T) == 8 ? BSQ_CORRECT_CR64 : BSQ_CORRECT_CR32; }

// EXACT: some depth is under Markstein's exact range (Consts::exact, host-checked)
template <class T, bool EXACT>
__global__ void __launch_bounds__(256) k_correct(Consts<T> C, CorrectPtrs<T> K) {
    constexpr int CR = cr_rows<T>();
    pdl_trigger();
    pdl_wait();
    const Layout L = C.L;
    const int I = GL + blockIdx.x * 32 + threadIdx.x;
    const int J0 = GL + (blockIdx.y * 8 + threadIdx.y) * CR;
    const long pitch = L.pitch;
    if (I >= L.nx + GL || J0 >= L.ny + GL) return;
    T d[CR], dx_[CR], dy_[CR], bu[CR], bv[CR], fs[CR], gs[CR], qw[CR + 2][3], pw[CR + 2][3];
    const long o0 = L.at(J0, I);
#pragma unroll
    for (int r = 0; r < CR + 2; r++)  // rows J0-1 .. J0+CR (rows up to ny+2 exist)
#pragma unroll
        for (int b = 0; b < 3; b++) {
            const long o = o0 + (r - 1) * pitch + (b - 1);
            const bool in = J0 + r - 1 <= L.ny + GL;
            qw[r][b] = in ? K.q1[o] : T(0);
            pw[r][b] = in ? K.p1[o] : T(0);
        }
#pragma unroll
    for (int k = 0; k < CR; k++) {
        const long o = o0 + k * pitch;
        const bool in = J0 + k < L.ny + GL;
        d[k] = in ? K.dep[o] : T(0);
        dx_[k] = in ? K.ddx[o] : T(0);
        dy_[k] = in ? K.ddy[o] : T(0);
        bu[k] = in ? K.bu[o] : T(0);
        bv[k] = in ? K.bv[o] : T(0);
        fs[k] = in ? K.fs[o] : T(0);
        gs[k] = in ? K.gs[o] : T(0);
    }
#pragma unroll
    for (int k = 0; k < CR; k++) {
        if (J0 + k >= L.ny + GL) continue;
        T f = T(0), g = T(0);
        if (d[k] > T(0)) {  // cross_rates (_kernels.py:310-321) on the solved P1, Q1
            // window row k = J-1, k+1 = J, k+2 = J+1; column 0 = I-1, 1 = I, 2 = I+1
            const T *qs = qw[k], *qc = qw[k + 1], *qn = qw[k + 2];
            const T *ps = pw[k], *pc = pw[k + 1], *pn = pw[k + 2];
            T q_x = (qc[2] - qc[0]) * T(0.5) * C.inv_dx;
            T q_y = (qn[1] - qs[1]) * T(0.5) * C.inv_dy;
            T q_xy = (qn[2] - qn[0] - qs[2] + qs[0]) * T(0.25) * C.inv_dx * C.inv_dy;
            T p_x = (pc[2] - pc[0]) * T(0.5) * C.inv_dx;
            T p_y = (pn[1] - ps[1]) * T(0.5) * C.inv_dy;
            T p_xy = (pn[2] - pn[0] - ps[2] + ps[0]) * T(0.25) * C.inv_dx * C.inv_dy;
            T sixth = div_pos(d[k], C.six, C.r_six);
            if (EXACT && tiny_nz(d[k], TINY_NUM)) sixth = div_tiny_exact(d[k], C.six, C.r_six);
            T d2 = C.bp13 * d[k] * d[k];
            f = sixth * (dx_[k] * q_y + dy_[k] * q_x) + d2 * q_xy;
            g = sixth * (dx_[k] * p_y + dy_[k] * p_x) + d2 * p_xy;
        }
        K.us[o0 + k * pitch] = bu[k] + (f - fs[k]);
        K.vs[o0 + k * pitch] = bv[k] + (g - gs[k]);
    }
}

// fp32: two adjacent columns per thread (8-byte loads and stores: the 4-byte
// kernel above is load-instruction bound in fp32 -- long-scoreboard 6.0 and
// lg-throttle 1.9 stalls per issue).  The 3-column window of a column pair
// is the pair's float2 plus the float2s either side (L1 hits).  Same
// operations per cell as k_correct.
#ifndef BSQ_CORRECT2_CR
#define BSQ_CORRECT2_CR 4  // rows per thread (1 / 2 / 4: 0.126 / 0.130 / 0.123 ms)
#endif
static __global__ void __launch_bounds__(256) k_correct_f32x2(Consts<float> C, CorrectPtrs<float> K) {
    constexpr int CR = BSQ_CORRECT2_CR;
    pdl_trigger();
    pdl_wait();
    const Layout L = C.L;
    const int I = GL + (blockIdx.x * 32 + threadIdx.x) * 2;  // first of the pair (even offset)
    const int J0 = GL + (blockIdx.y * 8 + threadIdx.y) * CR;
    const long pitch = L.pitch;
    if (I >= L.nx + GL || J0 >= L.ny + GL) return;
    const bool two = I + 1 < L.nx + GL;
    // window columns I-2 .. I+3 of rows J0-1 .. J0+CR, as three float2
    float qw[CR + 2][6], pw[CR + 2][6];
    const long o0 = L.at(J0, I);
#pragma unroll
    for (int r = 0; r < CR + 2; r++) {
        const bool in = J0 + r - 1 <= L.ny + GL;
#pragma unroll
        for (int b = 0; b < 3; b++) {
            const long o = o0 + (r - 1) * pitch + 2 * (b - 1);
            const float2 q = in ? *reinterpret_cast<const float2 *>(K.q1 + o) : make_float2(0.f, 0.f);
            const float2 pp = in ? *reinterpret_cast<const float2 *>(K.p1 + o) : make_float2(0.f, 0.f);
            qw[r][2 * b] = q.x, qw[r][2 * b + 1] = q.y;
            pw[r][2 * b] = pp.x, pw[r][2 * b + 1] = pp.y;
        }
    }
    float2 d[CR], dx_[CR], dy_[CR], bu[CR], bv[CR], fs[CR], gs[CR];
#pragma unroll
    for (int k = 0; k < CR; k++) {
        const long o = o0 + k * pitch;
        const bool in = J0 + k < L.ny + GL;
        const float2 z = make_float2(0.f, 0.f);
        d[k] = in ? *reinterpret_cast<const float2 *>(K.dep + o) : z;
        dx_[k] = in ? *reinterpret_cast<const float2 *>(K.ddx + o) : z;
        dy_[k] = in ? *reinterpret_cast<const float2 *>(K.ddy + o) : z;
        bu[k] = in ? *reinterpret_cast<const float2 *>(K.bu + o) : z;
        bv[k] = in ? *reinterpret_cast<const float2 *>(K.bv + o) : z;
        fs[k] = in ? *reinterpret_cast<const float2 *>(K.fs + o) : z;
        gs[k] = in ? *reinterpret_cast<const float2 *>(K.gs + o) : z;
    }
    auto cell = [&](int k, int c, float dk, float dxk, float dyk) -> float2 {
        // window row k = J-1, k+1 = J, k+2 = J+1; column c-1, c, c+1 (c = 2 or 3)
        float f = 0.f, g = 0.f;
        if (dk > 0.f) {
            const float *qs = qw[k], *qc = qw[k + 1], *qn = qw[k + 2];
            const float *ps = pw[k], *pc = pw[k + 1], *pn = pw[k + 2];
            const float q_x = (qc[c + 1] - qc[c - 1]) * 0.5f * C.inv_dx;
            const float q_y = (qn[c] - qs[c]) * 0.5f * C.inv_dy;
            const float q_xy = (qn[c + 1] - qn[c - 1] - qs[c + 1] + qs[c - 1]) * 0.25f * C.inv_dx * C.inv_dy;
            const float p_x = (pc[c + 1] - pc[c - 1]) * 0.5f * C.inv_dx;
            const float p_y = (pn[c] - ps[c]) * 0.5f * C.inv_dy;
            const float p_xy = (pn[c + 1] - pn[c - 1] - ps[c + 1] + ps[c - 1]) * 0.25f * C.inv_dx * C.inv_dy;
            const float sixth = div_pos(dk, C.six, C.r_six);
            const float d2 = C.bp13 * dk * dk;
            f = sixth * (dxk * q_y + dyk * q_x) + d2 * q_xy;
            g = sixth * (dxk * p_y + dyk * p_x) + d2 * p_xy;
        }
        return make_float2(f, g);
    };
#pragma unroll
    for (int k = 0; k < CR; k++) {
        if (J0 + k >= L.ny + GL) continue;
        const float2 a = cell(k, 2, d[k].x, dx_[k].x, dy_[k].x);
        const float2 b = cell(k, 3, d[k].y, dx_[k].y, dy_[k].y);
        const long o = o0 + k * pitch;
        const float2 u = make_float2(bu[k].x + (a.x - fs[k].x), bu[k].y + (b.x - fs[k].y));
        const float2 v = make_float2(bv[k].x + (a.y - gs[k].x), bv[k].y + (b.y - gs[k].y));
        if (two) {
            *reinterpret_cast<float2 *>(K.us + o) = u;
            *reinterpret_cast<float2 *>(K.vs + o) = v;
        } else {
            K.us[o] = u.x;
            K.vs[o] = v.x;
        }
    }
}

// ---------------------------------------------------------------------------
// launchers

// A row band runs as a grid of nrows rows whose arrays start row0 rows down
// (same kernel, no extra operand: an extra parameter cost 10 registers)
template <class T>
void launch_correct(const Consts<T> &C, const CorrectPtrs<T> &K, cudaStream_t st, int row0,
                    int nrows) {
    constexpr int CR = cr_rows<T>();
    static_assert(STAGE_BAND % (8 * CR) == 0, "band of whole blocks");
    if (nrows < 0) nrows = C.L.ny - row0;
    if (nrows <= 0) return;
    Consts<T> Cb = C;
    CorrectPtrs<T> Kb = K;
    if (row0 > 0) {
        const long sh = (long)row0 * C.L.pitch;
        Cb.L.ny = nrows;
        Kb.bu += sh, Kb.bv += sh, Kb.fs += sh, Kb.gs += sh, Kb.p1 += sh, Kb.q1 += sh;
        Kb.dep += sh, Kb.ddx += sh, Kb.ddy += sh, Kb.us += sh, Kb.vs += sh;
    } else {
        Cb.L.ny = nrows;
    }
#if !defined(BSQ_CORRECT_F32_SCALAR)
    if constexpr (sizeof(T) == 4) {  // fp32 (no exact branch: a tolerance contract)
        constexpr int CR2 = BSQ_CORRECT2_CR;
        dim3 grid2((C.L.nx + 63) / 64, (nrows + 8 * CR2 - 1) / (8 * CR2));  // 64 x (8*CR2) cells
        launch_k(k_correct_f32x2, grid2, dim3(32, 8), 0, st, Cb, Kb);
        return;
    }
#endif
    dim3 grid((C.L.nx + 31) / 32, (nrows + 8 * CR - 1) / (8 * CR));  // 32 x (8*CR) cells
    launch_k(Cb.exact ? k_correct<T, true> : k_correct<T, false>, grid, dim3(32, 8), 0, st, Cb, Kb);
}

#if BSQ_INST_F64
template void launch_correct<double>(const Consts<double> &, const CorrectPtrs<double> &,
                                     cudaStream_t, int, int);
#endif
#if BSQ_INST_F32
template void launch_correct<float>(const Consts<float> &, const CorrectPtrs<float> &,
                                    cudaStream_t, int, int);
#endif

}  // namespace bsq
