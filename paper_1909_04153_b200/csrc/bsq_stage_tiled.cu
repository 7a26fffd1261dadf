// bsq_stage_tiled.cu -- tiled variant of the fused stage kernel: everything a step evaluates on the
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
// quadrature bases.  Faces and fluxes live only in shared memory.
//
// CTA = 32 x 8 cells, warp ty = tile row ty.  Three CTA barriers:
//   A  load w, P, Q, bed_eff, depth for the tile and a 2-cell halo, and the
//      face beds, by TMA (one mbarrier)
//   B  faces of every cell once: x faces for columns -1..32, y faces for
//      rows -1..8 of the tile (the reference evaluates each face once too),
//      eta over the halo box                                     | barrier
//   C  fluxes of the 33 x 8 x-interfaces and 32 x 9 y-interfaces, each
//      stored over the east/north faces it alone consumed         | barrier
//   D  per-cell rates, dispersive terms, cross groups, U*/V*, predictor
// Phases B and C map items to (warp, lane) directly -- row ty, column lane --
// in three rounds, so no warp mixes item kinds and no index needs a divide.
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "bsq_device.cuh"
#include "bsq_launch.h"
#include "bsq_tma.cuh"

namespace bsq {

#ifndef BSQ_STAGE_AHEAD
#define BSQ_STAGE_AHEAD 222  // fp64: L2-prefetch the phase-A boxes of the tile this many CTAs
                             // ahead (1.5 x 148 SMs; 74/148/185/222/259/296/592: step
                             // -0.003/-0.017/-0.016/-0.025/-0.015/-0.021/-0.018 ms)
#endif
#ifndef BSQ_STAGE_MINB
#define BSQ_STAGE_MINB 4  // CTAs per SM the register budget is sized for (64 regs)
#endif
#ifndef BSQ_STAGE_MINB32
#define BSQ_STAGE_MINB32 6  // fp32: 40 registers, 6 CTAs per SM (47 / 5: 0.4705 -> 0.4515 ms)
#endif

namespace tiled {
constexpr int TX = STAGE_TX, TY = STAGE_TY, NT = TX * TY;
constexpr int HX = TX + 4, HY = TY + 4;       // tile + 2-cell halo
constexpr int FXW = TX + 2, FYH = TY + 2;     // cells with x faces per row / rows with y faces
constexpr int NXF = TY * FXW, NYF = FYH * TX; // face items
constexpr int NXI = TY * (TX + 1), NYI = (TY + 1) * TX;  // interface items
constexpr int NFL = NXI + NYI;
constexpr int FL_PASSES = (NFL + NT - 1) / NT;

// TMA tile loads need the box origin on a 16-byte boundary along x (measured:
// tools/tma_box_probe.cu, an "illegal instruction" otherwise) and box widths
// of 16-byte multiples.  The halo box starts at padded column I0 - 2: 16-B
// aligned in fp64 (xo = 14), 8 B off in fp32 (xo = 30), where the boxes start
// XS = 2 columns further west and are 40 wide; smem column c of the tile's
// view is box column c + XS.
template <class T>
struct Box {
    static constexpr int XS = sizeof(T) == 8 ? 0 : 2;
    static constexpr int W = sizeof(T) == 8 ? HX : HX + 4;  // loaded width (bed_face_x too:
                                                            // one column more than used)
};

template <class T>
struct StageSmem {
    static constexpr int W = Box<T>::W;
    // TMA destinations: 128-byte aligned each
    alignas(128) T w[HY][W];
    alignas(128) T p[HY][W];
    alignas(128) T q[HY][W];
    alignas(128) T be[HY][W];
    alignas(128) T dep[HY][W];
    alignas(128) T eta[HY][W];
    alignas(128) T bfx[TY][W];    // bed_face_x for columns -2..TX
    alignas(128) T bfy[TY + 3][TX];  // bed_face_y for rows -2..TY
    alignas(8) uint64_t bar;
    struct {  // phase B/C faces (hi = east/north, lo = west/south; w, P, Q);
              // phase C/D fluxes over the hi faces (flux v in hi array v)
        T xhi[3][TY][FXW], xlo[3][TY][FXW];
        T yhi[3][FYH][TX], ylo[3][FYH][TX];
    } f;
};


template <class T>
constexpr int stage_minb() { return sizeof(T) == 8 ? BSQ_STAGE_MINB : BSQ_STAGE_MINB32; }

template <class T, bool FR>
__global__ void __launch_bounds__(NT, stage_minb<T>()) k_stage(Consts<T> C, const DevParams *__restrict__ P,
                                                 const __grid_constant__ StagePtrs<T> A, int predict,
                                                 const __grid_constant__ StageMaps M, int row0) {
    // the TMA destinations need 128-B alignment: the kernel has no static
    // smem, so the dynamic window starts at the CTA's smem base (checked)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    StageSmem<T> &S = *reinterpret_cast<StageSmem<T> *>(smem_raw);
    if (threadIdx.x == 0 && threadIdx.y == 0 && (smem_u32(smem_raw) & 127u) != 0) __trap();
    pdl_trigger();
    pdl_wait();
    const Layout L = C.L;
    const int nx = L.nx, ny = L.ny;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int I0 = GL + blockIdx.x * TX, J0 = GL + row0 + blockIdx.y * TY;

    // ---- A: tile + halo, by TMA ------------------------------------------------
    // One thread issues seven 2-D bulk tensor copies (w, P, Q, bed_eff, depth
    // over the tile + 2-cell halo; the two face-bed boxes); out-of-grid cells
    // arrive zero-filled, as the reference's padding needs none of them.
    if (tid == 0) {
        mbar_init(&S.bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    constexpr int XS = Box<T>::XS, BW = Box<T>::W;
    if (tid == 0) {
        // halo box origin: padded column I0 - 2 - XS (+ xo: the maps start at
        // the pitched row), padded row J0 - 2
        const int x0 = L.xo + I0 - GL - XS, y0 = J0 - GL;
        mbar_expect_tx(&S.bar, (unsigned)sizeof(T) * (5 * HY * BW + TY * BW + (TY + 3) * TX));
        tma_load_2d(&S.w[0][0], &M.w, x0, y0, &S.bar);
        tma_load_2d(&S.p[0][0], &M.p, x0, y0, &S.bar);
        tma_load_2d(&S.q[0][0], &M.q, x0, y0, &S.bar);
        tma_load_2d(&S.be[0][0], &M.be, x0, y0, &S.bar);
        tma_load_2d(&S.dep[0][0], &M.dep, x0, y0, &S.bar);
        tma_load_2d(&S.bfx[0][0], &M.bfx, x0, J0, &S.bar);
        tma_load_2d(&S.bfy[0][0], &M.bfy, L.xo + I0, y0, &S.bar);
    }
    // the tile's views: column 0 = padded column I0 - 2
    T(*const Sw)[BW] = reinterpret_cast<T(*)[BW]>(&S.w[0][XS]);
    T(*const Sp)[BW] = reinterpret_cast<T(*)[BW]>(&S.p[0][XS]);
    T(*const Sq)[BW] = reinterpret_cast<T(*)[BW]>(&S.q[0][XS]);
    T(*const Sbe)[BW] = reinterpret_cast<T(*)[BW]>(&S.be[0][XS]);
    T(*const Sdep)[BW] = reinterpret_cast<T(*)[BW]>(&S.dep[0][XS]);
    T(*const Seta)[BW] = reinterpret_cast<T(*)[BW]>(&S.eta[0][XS]);
    T(*const Sbfx)[BW] = reinterpret_cast<T(*)[BW]>(&S.bfx[0][XS]);
    // phase D's per-cell inputs that phase A does not read: start them towards
    // L2 now (no registers held), so phase D's loads hit on chip
#ifndef BSQ_STAGE_LANE_PREFETCH
    if (tid == 0) {  // the TMA unit fetches the 32 x 8 boxes
        const int na = (predict && !P->euler) ? 12 : 2;
        for (int k = 0; k < na; k++) tma_prefetch_2d(&M.pf[k], L.xo + I0 - GL + 2, J0);
        // the phase-A boxes of the tile AHEAD CTAs later in launch order (its
        // CTA starts a fraction of a wave after this one ends): into L2 now,
        // so its tile loads do not wait on DRAM -- the wait for them was the
        // kernel's top stall (15 % of warp samples on the mbarrier poll).
        // fp64 only: fp32 measured 0.4688 -> 0.4709 ms with it.
        constexpr int AHEAD = sizeof(T) == 8 ? BSQ_STAGE_AHEAD : 0;
        const int nbx = gridDim.x, b = blockIdx.y * nbx + blockIdx.x + AHEAD;
        if (AHEAD > 0 && b < nbx * (int)gridDim.y) {
            const int I1 = GL + (b % nbx) * TX, J1 = GL + row0 + (b / nbx) * TY;
            const int x1 = L.xo + I1 - GL - XS, y1 = J1 - GL;
            tma_prefetch_2d(&M.w, x1, y1);
            tma_prefetch_2d(&M.p, x1, y1);
            tma_prefetch_2d(&M.q, x1, y1);
            tma_prefetch_2d(&M.be, x1, y1);
            tma_prefetch_2d(&M.dep, x1, y1);
            tma_prefetch_2d(&M.bfx, x1, J1);
            tma_prefetch_2d(&M.bfy, L.xo + I1, y1);
        }
    }
#else
    {
        // lane k < 24 of warp ty: array k >> 1 (ddx, ddy, h1[0..4], h2[0..4]),
        // 128-B line k & 1 of the warp's 256-B tile row
        constexpr int LINE = 128 / sizeof(T);
        const int Jc = J0 + ty, Ic = I0 + (tx & 1) * LINE;
        const int na = (predict && !P->euler) ? 12 : 2;
        if (tx < 2 * na && Jc < ny + GL && Ic < nx + GL) {
            const int k = tx >> 1;
            prefetch_l2(A.pf[k] + L.at(Jc, Ic));  // one indexed constant load
        }
    }
#endif
#if defined(BSQ_STAGE_SPIN)
    mbar_wait(&S.bar, 0);
#else
    mbar_wait_park(&S.bar, 0);
#endif
    // ---- B: faces, once per cell, + eta -----------------------------------------
    // Warp ty, lane tx (2-D map: no div/mod, no warp covering two kinds):
    //   round 0  x faces of tile row ty, face columns 0..31
    //   round 1  y faces of face row ty (0..7)
    //   round 2  warps 0,1: y face rows 8, 9; warp 2: x face columns 32, 33 of
    //            the 8 rows (16 lanes); warps 3..7: eta over the halo box
    auto xface = [&](int r, int c) {  // x faces of cell (row r, column c-1)
        const int y = r + 2, x = c + 1;
        const Faces<T> f = cell_faces(Sw[y][x - 1], Sw[y][x], Sw[y][x + 1], Sp[y][x - 1],
                                      Sp[y][x], Sp[y][x + 1], Sq[y][x - 1], Sq[y][x],
                                      Sq[y][x + 1], Sbfx[r][c + 1], Sbfx[r][c], C.theta);
        S.f.xhi[0][r][c] = f.whi;
        S.f.xlo[0][r][c] = f.wlo;
        S.f.xhi[1][r][c] = f.phi;
        S.f.xlo[1][r][c] = f.plo;
        S.f.xhi[2][r][c] = f.qhi;
        S.f.xlo[2][r][c] = f.qlo;
    };
    auto yface = [&](int r, int c) {  // y faces of cell (row r-1, column c)
        const int y = r + 1, x = c + 2;
        const Faces<T> f = cell_faces(Sw[y - 1][x], Sw[y][x], Sw[y + 1][x], Sp[y - 1][x],
                                      Sp[y][x], Sp[y + 1][x], Sq[y - 1][x], Sq[y][x],
                                      Sq[y + 1][x], S.bfy[r + 1][c], S.bfy[r][c], C.theta);
        S.f.yhi[0][r][c] = f.whi;
        S.f.ylo[0][r][c] = f.wlo;
        S.f.yhi[1][r][c] = f.phi;
        S.f.ylo[1][r][c] = f.plo;
        S.f.yhi[2][r][c] = f.qhi;
        S.f.ylo[2][r][c] = f.qlo;
    };
    static_assert(TX == 32 && TY >= 4 && TY <= 16, "2-D item maps: warp = tile row, 32 columns");
    bool tiny = false;
    xface(ty, tx);
    yface(ty, tx);
    if (ty < 2) {
        yface(TY + ty, tx);
    } else if (ty == 2) {
        if (tx < 2 * TY) xface(tx >> 1, TX + (tx & 1));
    } else {
        // eta = (w - bed_eff) - depth over the halo box (dispersion.py:87);
        // the same warps look for tiny momenta in the box (0 < |P|,|Q| <
        // 2^-400), which could put a numerator under Markstein's exact range
        for (int k = tid - 3 * TX; k < HY * BW; k += NT - 3 * TX) {
            (&S.eta[0][0])[k] = ((&S.w[0][0])[k] - (&S.be[0][0])[k]) - (&S.dep[0][0])[k];
            tiny |= tiny_nz((&S.p[0][0])[k], TINY_IN) | tiny_nz((&S.q[0][0])[k], TINY_IN);
        }
    }
    // the tile divides exactly (IEEE) if any input was tiny: rare, warp-uniform
    const bool exact = __syncthreads_or(tiny | C.exact) != 0;

    // phases C and D, instantiated twice: the Markstein quotients, or (a tile
    // with tiny inputs, never on ordinary data) IEEE divisions throughout
    auto phase_cd = [&](auto ex_tag) {
    constexpr bool EX = decltype(ex_tag)::value;
    // ---- C: fluxes, written over the faces they consume --------------------------
    //   round 0  x interfaces of row ty, 0..31;  round 1  y interface row ty
    //   round 2  warp 0: y interface row 8; warp 1: x interface 32 of the 8 rows
    // Interface (r, xi) reads the east ("hi") faces of column xi and the west
    // ("lo") faces of column xi+1.  Column xi's hi faces feed no other
    // interface, so the thread that consumed them stores the three fluxes in
    // their place (flux v -> hi array v): no barrier and no registers held
    // between computing and storing.  Same for y with row yi's north faces.
    auto xflux = [&](int r, int xi) {
        T f1, f2, f3;
        cu_flux_rcp<FR, EX>(S.f.xhi[0][r][xi], S.f.xlo[0][r][xi + 1], S.f.xhi[1][r][xi],
                    S.f.xlo[1][r][xi + 1], S.f.xhi[2][r][xi], S.f.xlo[2][r][xi + 1],
                    Sbfx[r][xi + 1], C.g, C.half_g, C.h_eps, f1, f2, f3);
        S.f.xhi[0][r][xi] = f1;
        S.f.xhi[1][r][xi] = f2;
        S.f.xhi[2][r][xi] = f3;
    };
    auto yflux = [&](int yi, int c) {  // south cell = face row yi; normal = Q
        T f1, fq, fp;
        cu_flux_rcp<FR, EX>(S.f.yhi[0][yi][c], S.f.ylo[0][yi + 1][c], S.f.yhi[2][yi][c],
                    S.f.ylo[2][yi + 1][c], S.f.yhi[1][yi][c], S.f.ylo[1][yi + 1][c],
                    S.bfy[yi + 1][c], C.g, C.half_g, C.h_eps, f1, fq, fp);
        S.f.yhi[0][yi][c] = f1;
        S.f.yhi[1][yi][c] = fp;  // fy2 carries P
        S.f.yhi[2][yi][c] = fq;  // fy3 carries Q
    };
    xflux(ty, tx);
    yflux(ty, tx);
    if (ty == 0) yflux(TY, tx);
    else if (ty == 1 && tx < TY) xflux(tx, TX);
    __syncthreads();
    // phase D's view of the fluxes
#define FX(v, r, xi) S.f.xhi[v][r][xi]
#define FY(v, yi, c) S.f.yhi[v][yi][c]

    // ---- D: per cell ----------------------------------------------------------------
    const int J = J0 + ty, I = I0 + tx;
    if (J >= ny + GL || I >= nx + GL) return;
    const int y = ty + 2, x = tx + 2;
    const long o = L.at(J, I);
    const T wc = Sw[y][x], pc = Sp[y][x], qc = Sq[y][x];
    if (A.maxw) A.maxw[o] = np_maximum(A.maxw[o], wc);  // MaxSurfaceTracker fold
    const T be_ = Sbfx[ty][tx + 2], bw_ = Sbfx[ty][tx + 1];
    const T bn_ = S.bfy[ty + 2][tx], bs_ = S.bfy[ty + 1][tx];

    // fv_rates (_kernels.py:230-251)
    T rw = -(FX(0, ty, tx + 1) - FX(0, ty, tx)) * C.inv_dx -
           (FY(0, ty + 1, tx) - FY(0, ty, tx)) * C.inv_dy;
    const T src_x = -C.g * (wc - T(0.5) * (be_ + bw_)) * (be_ - bw_) * C.inv_dx;
    const T src_y = -C.g * (wc - T(0.5) * (bn_ + bs_)) * (bn_ - bs_) * C.inv_dy;
    T h = wc - Sbe[y][x];
    h = floor0(h);
    const T hstar = floor_eps(h, C.h_eps);
    T fric = T(0);
    if (C.c_f > T(0)) {  // c_f sqrt(P^2 + Q^2) / h*^2, the quotient via RN(1/h*^2) (div_rcp)
        const T h2 = hstar * hstar;
        const T num = C.c_f * sqrt(pc * pc + qc * qc);
        fric = qx<EX>(div_rcp(num, h2, rcp_rn(h2)), num, h2);
    }
    T rp = -(FX(1, ty, tx + 1) - FX(1, ty, tx)) * C.inv_dx -
           (FY(1, ty + 1, tx) - FY(1, ty, tx)) * C.inv_dy + src_x - fric * pc;
    T rq = -(FX(2, ty, tx + 1) - FX(2, ty, tx)) * C.inv_dx -
           (FY(2, ty + 1, tx) - FY(2, ty, tx)) * C.inv_dy + src_y - fric * qc;

    const T d = Sdep[y][x], dx_ = A.ddx[o], dy_ = A.ddy[o];
    T fs_, gs_;
    if (d > T(0)) {
        // dispersive_rates (_kernels.py:269-288)
        const T ec = Seta[y][x];
        const T e_xx = (Seta[y][x + 1] - T(2) * ec + Seta[y][x - 1]) * C.inv_dx2;
        const T e_yy = (Seta[y + 1][x] - T(2) * ec + Seta[y - 1][x]) * C.inv_dy2;
        const T e_xy = (Seta[y + 1][x + 1] - Seta[y + 1][x - 1] - Seta[y - 1][x + 1] +
                        Seta[y - 1][x - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
        const T e_xxx = (Seta[y][x + 2] - T(2) * Seta[y][x + 1] + T(2) * Seta[y][x - 1] -
                         Seta[y][x - 2]) * T(0.5) * C.inv_dx * C.inv_dx2;
        const T e_yyy = (Seta[y + 2][x] - T(2) * Seta[y + 1][x] + T(2) * Seta[y - 1][x] -
                         Seta[y - 2][x]) * T(0.5) * C.inv_dy * C.inv_dy2;
        const T e_xyy = ((Seta[y + 1][x + 1] - T(2) * Seta[y][x + 1] + Seta[y - 1][x + 1]) -
                         (Seta[y + 1][x - 1] - T(2) * Seta[y][x - 1] + Seta[y - 1][x - 1])) *
                        T(0.5) * C.inv_dx * C.inv_dy2;
        const T e_xxy = ((Seta[y + 1][x + 1] - T(2) * Seta[y + 1][x] + Seta[y + 1][x - 1]) -
                         (Seta[y - 1][x + 1] - T(2) * Seta[y - 1][x] + Seta[y - 1][x - 1])) *
                        T(0.5) * C.inv_dy * C.inv_dx2;
        const T gd2 = C.g * d * d;
        const T gd3 = gd2 * d;
        rp += C.b_disp * gd3 * (e_xxx + e_xyy) +
              C.b_disp * gd2 * (dx_ * (T(2) * e_xx + e_yy) + dy_ * e_xy);
        rq += C.b_disp * gd3 * (e_yyy + e_xxy) +
              C.b_disp * gd2 * (dy_ * (T(2) * e_yy + e_xx) + dx_ * e_xy);
        // cross_rates (_kernels.py:310-321)
        const T q_x = (Sq[y][x + 1] - Sq[y][x - 1]) * T(0.5) * C.inv_dx;
        const T q_y = (Sq[y + 1][x] - Sq[y - 1][x]) * T(0.5) * C.inv_dy;
        const T q_xy = (Sq[y + 1][x + 1] - Sq[y + 1][x - 1] - Sq[y - 1][x + 1] +
                        Sq[y - 1][x - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
        const T p_x = (Sp[y][x + 1] - Sp[y][x - 1]) * T(0.5) * C.inv_dx;
        const T p_y = (Sp[y + 1][x] - Sp[y - 1][x]) * T(0.5) * C.inv_dy;
        const T p_xy = (Sp[y + 1][x + 1] - Sp[y + 1][x - 1] - Sp[y - 1][x + 1] +
                        Sp[y - 1][x - 1]) * T(0.25) * C.inv_dx * C.inv_dy;
        const T sixth = qx<EX>(div_pos(d, C.six, C.r_six), d, C.six);
        const T d2 = C.bp13 * d * d;
        fs_ = sixth * (dx_ * q_y + dy_ * q_x) + d2 * q_xy;
        gs_ = sixth * (dx_ * p_y + dy_ * p_x) + d2 * p_xy;
    } else {
        fs_ = T(0);
        gs_ = T(0);
    }

    // non-finite stage values (dispersion.py:92-98): first row-major cell
    const unsigned long long lin = (unsigned long long)(J - GL) * nx + (I - GL);
    if (!(isfinite(rw) & isfinite(rp) & isfinite(rq) & isfinite(fs_) & isfinite(gs_))) {
        if (!isfinite(rw)) atomicMin(&A.bad[0], lin);
        if (!isfinite(rp)) atomicMin(&A.bad[1], lin);
        if (!isfinite(rq)) atomicMin(&A.bad[2], lin);
        if (!isfinite(fs_)) atomicMin(&A.bad[3], lin);
        if (!isfinite(gs_)) atomicMin(&A.bad[4], lin);
    }

    A.h0[0][o] = rw;
    A.h0[1][o] = rp;
    A.h0[2][o] = rq;
    A.h0[3][o] = fs_;
    A.h0[4][o] = gs_;
    if (!predict) return;

    // U*, V* (dispersion.py:131-148): divisions by grid constants
    const T pdx = Sp[y][x + 1] - Sp[y][x - 1], pdxx = Sp[y][x + 1] - T(2) * pc + Sp[y][x - 1];
    const T p_x = qx<EX>(div_pos(pdx, C.two_dx, C.r_two_dx), pdx, C.two_dx);
    const T p_xx = qx<EX>(div_pos(pdxx, C.dx2, C.r_dx2), pdxx, C.dx2);
    const T ddx3 = d * dx_;
    const T ustar = pc - qx<EX>(div_pos(ddx3, C.three, C.r_three), ddx3, C.three) * p_x - C.bp13 * d * d * p_xx;
    const T qdy = Sq[y + 1][x] - Sq[y - 1][x], qdyy = Sq[y + 1][x] - T(2) * qc + Sq[y - 1][x];
    const T q_y = qx<EX>(div_pos(qdy, C.two_dy, C.r_two_dy), qdy, C.two_dy);
    const T q_yy = qx<EX>(div_pos(qdyy, C.dy2, C.r_dy2), qdyy, C.dy2);
    const T ddy3 = d * dy_;
    const T vstar = qc - qx<EX>(div_pos(ddy3, C.three, C.r_three), ddy3, C.three) * q_y - C.bp13 * d * d * q_yy;

    // predictor (stepper.py:239-250, 109-132; multistep.py:139-153)
    T wn, bu, bv, us, vs;
    if (P->euler) {
        const T dt = par<T>(P->dt, P->f_dt);
        wn = wc + dt * rw;
        bu = ustar + dt * rp;
        bv = vstar + dt * rq;
        us = bu;
        vs = bv;
    } else {
        const T wc0 = par<T>(P->wc, P->f_wc), wp1 = par<T>(P->wp, P->f_wp), wp2 = par<T>(P->wp2, P->f_wp2);
        const T s0 = par<T>(P->sc, P->f_sc), s1 = par<T>(P->sp, P->f_sp), s2 = par<T>(P->sp2, P->f_sp2);
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
    };
    if (exact) phase_cd(std::true_type{});
    else phase_cd(std::false_type{});
}

}  // namespace tiled

template <class T, bool FR>
static void launch_tiled(const Consts<T> &C, const DevParams *P, const StagePtrs<T> &A, int predict,
                         cudaStream_t st, const StageMaps *M, int row0, int nrows) {
    const size_t smem = sizeof(tiled::StageSmem<T>);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(tiled::k_stage<T, FR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr_set = true;
    }
    StagePtrs<T> Ap = A;
    Ap.pf[0] = A.ddx;
    Ap.pf[1] = A.ddy;
    for (int k = 0; k < 5; k++) {
        Ap.pf[2 + k] = A.h1[k];
        Ap.pf[7 + k] = A.h2[k];
    }
    dim3 grid((C.L.nx + tiled::TX - 1) / tiled::TX, (nrows + tiled::TY - 1) / tiled::TY);
    launch_k(tiled::k_stage<T, FR>, grid, dim3(tiled::TX, tiled::TY), smem, st, C, P, Ap, predict,
             *M, row0);
}

template <class T>
void launch_stage_tiled(const Consts<T> &C, const DevParams *P, const StagePtrs<T> &A, int predict,
                        cudaStream_t st, const StageMaps *M, int row0, int nrows) {
    if (flux_fast_rcp_ok(C.h_eps))
        launch_tiled<T, true>(C, P, A, predict, st, M, row0, nrows);
    else
        launch_tiled<T, false>(C, P, A, predict, st, M, row0, nrows);
}

#if BSQ_INST_F64
template void launch_stage_tiled<double>(const Consts<double> &, const DevParams *,
                                         const StagePtrs<double> &, int, cudaStream_t,
                                         const StageMaps *, int, int);
#endif
#if BSQ_INST_F32
template void launch_stage_tiled<float>(const Consts<float> &, const DevParams *,
                                        const StagePtrs<float> &, int, cudaStream_t,
                                        const StageMaps *, int, int);
#endif

}  // namespace bsq
