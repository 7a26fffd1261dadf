// bsq_launch.h -- kernel argument bundles and launchers (host-visible).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "bsq_device.cuh"

namespace bsq {

// whether the step's kernels are launched as programmatic dependents of
// their predecessors (BSQ_PDL=1; off by default, bsq_api.cu)
bool pdl_on();
// device check of the quotient helpers (bsq_check.cu; host arrays)
int check_quotients(int op, const double *x, const double *d, long n, double *out);

// <<<g, b, smem, st>>> with the programmatic-stream-serialization attribute
// when pdl_on(): the kernel must call pdl_wait() before reading what earlier
// work on the stream wrote
template <typename... KArgs, typename... Args>
inline void launch_k(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st,
                     Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

template <class T>
struct StagePtrs {
    const T *w, *p, *q;             // committed state, ghost-filled at t
    const T *be, *dep, *ddx, *ddy;  // static fields
    const T *bfx, *bfy;
    T *h0[5];                       // new stage set e, f, g, fstar, gstar
    const T *h1[5], *h2[5];         // previous two levels (AB3 only)
    T *wn;                          // predicted w -> pending state's w
    T *bu, *bv, *us, *vs;           // quadrature bases and predicted U*, V*
    unsigned long long *bad;        // [5] first non-finite stage cell
    T *maxw;                        // running max of w to fold this state into, or null
    const T *pf[12];                // phase-D inputs to prefetch: ddx, ddy, h1[0..4], h2[0..4]
};

template <class T>
struct SolvePtrs {
    const T *gp, *gq;               // arrays holding the P / Q ghost values to fold
    const T *cx_last, *cy_last;     // c_{n-1} of every x / y line (ghost folding)
    // y-strip sharding: the y lines continue across ranks (exact pipelined Thomas)
    int south_int, north_int;       // internal sides: no folding there
    const T *dw_in;                 // forward: dw of the row below (south rank), per column
    T *dw_out;                      // forward: dw of this strip's last row
    const T *x_in;                  // backward: x of the row above (north rank)
    T *x_out;                       // backward: x of this strip's first row
    int exact;                      // divide exactly (EXD): exact_tiny requested
};

// which parts of the line solves a launch runs
enum SolveMode { SOLVE_FULL = 0, SOLVE_X_YFWD = 1, SOLVE_YBWD = 2 };

// TMA descriptors of the solve's operands, interior region of each pitched
// array.  x maps: box {EK, 32} (elements along x, 32 rows), 128-B swizzle;
// y maps: box {32, EK} (32 columns, elements along y).  `out` is the solved
// field (also the forward sweep's dw scratch).
struct SolveMaps {
    CUtensorMap x_rhs, x_a, x_den, x_rden, x_cw, x_out;
    CUtensorMap y_rhs, y_a, y_den, y_rden, y_cw, y_out;
    // the x-direction arrays themselves (padded layout), for the warp-per-line
    // path of few long x lines (bsq_solve.cu solve_xline_warp)
    const void *xp_rhs, *xp_a, *xp_den, *xp_rden, *xp_cw;
    void *xp_out;
};

// solver="cr": the reference's odd-even cyclic reduction (bsq_cr.cu)
template <class T>
struct CrPtrs {
    const T *ax, *bx, *cx, *ay, *by, *cy;  // the operator's diagonals (x: padded layout;
                                           // y: transposed, column i's row j at i*ny + j)
    const T *rx, *ry;                      // right-hand sides (ghosts folded in-kernel)
    const T *gp, *gq;                      // ghost sources, as SolvePtrs
    T *outx, *outy;
    unsigned int *bad;                     // min error key (0xFFFFFFFF: none)
    unsigned int key_base;                 // (solve phase - 1) << 31
};

template <class T>
struct CorrectPtrs {
    const T *bu, *bv, *fs, *gs;     // quadrature bases and stored F*_n, G*_n
    const T *p1, *q1;               // first-solve momenta with ghosts
    const T *dep, *ddx, *ddy;
    T *us, *vs;                     // corrected right-hand sides
};

template <class T>
struct FinalPtrs {
    T *w;                           // predicted w in, final w out (pending state)
    const T *pin, *qin;             // solved momenta
    T *pout, *qout;                 // pending state's P, Q
    const T *be;
    const T *fac[4];                // sponge factors per side
    Partial *part;
    unsigned int *counter;
    DevResult *res;
    const long long *goff;          // gauge cells (element offsets), gathered by the last CTA
    int ng;
    T *gval;                        // ng x (w, P, Q) of the new state
    const DevParams *P;             // this step's parameters (controller inputs)
    DevParams *pnext;               // speculation: the next step's ghost/stage parameters
    // BSQ_Y_SPIKE: the second solve's coupling correction, applied on load
    // (q - v b_prev - w t_next, k_spike_fix's operations) instead of a pass
    const T *spv, *spw, *spbt;      // null: no correction pending
    int sp_south, sp_north;
    int sp_jv, sp_jw;               // rows [0, sp_jv) take v, rows [sp_jw, ny) take w
};

// save != nullptr: each ghost cell's previous value goes to save first, in
// k_frame's layout (the frame save fused into the fill)
template <class T>
void launch_ghost(const Consts<T> &C, const DevParams *P, int which, const T *sw, const T *sp,
                  const T *sq, T *dw, T *dp, T *dq, cudaStream_t st, T *save = nullptr);
// stage tile (fp64 tiled kernel): STAGE_TX x STAGE_TY cells per CTA
#ifndef BSQ_STAGE_TY
#define BSQ_STAGE_TY 8
#endif
constexpr int STAGE_TX = 32, STAGE_TY = BSQ_STAGE_TY;

// TMA descriptors of the stage tile loads (padded arrays; boxes of the
// tile + 2-cell halo, (TX+4) x (TY+4) cells, and of the face beds)
struct StageMaps {
    CUtensorMap w, p, q, be, dep, bfx, bfy;
    CUtensorMap pf[12];  // 32 x 8 interior boxes of StagePtrs::pf (L2 prefetch by the TMA unit)
};

template <class T>
void launch_frame(const Consts<T> &C, T *w, T *p, T *q, T *buf, int save, cudaStream_t st);
size_t frame_elems(int nx, int ny);
// rows [row0, row0 + nrows) of the interior (nrows < 0: to the last row);
// row0 a multiple of STAGE_BAND
constexpr int STAGE_BAND = 32;
template <class T>
void launch_stage(const Consts<T> &C, const DevParams *P, const StagePtrs<T> &A, int predict,
                  cudaStream_t st, const StageMaps *M = nullptr, int row0 = 0, int nrows = -1);
// pivot properties of a factored operator (launch_solve's `pivots`)
enum { PIV_POSITIVE = 1, PIV_RDEN_INRANGE = 2 };
template <class T>
void launch_solve(const Consts<T> &C, const SolveMaps &M, const SolvePtrs<T> &S, int pivots,
                  cudaStream_t st, int mode = SOLVE_FULL);
int solve_chunk_elems(int elem_bytes);
template <class T>
void launch_cr(const Consts<T> &C, const CrPtrs<T> &K, cudaStream_t st);
size_t cr_smem_bytes(int nx, int ny, int elem);
// rows [row0, row0 + nrows) (nrows < 0: to the last row); row0 a multiple of STAGE_BAND
template <class T>
void launch_correct(const Consts<T> &C, const CorrectPtrs<T> &K, cudaStream_t st, int row0 = 0,
                    int nrows = -1);
template <class T>
void launch_final(const Consts<T> &C, const FinalPtrs<T> &F, cudaStream_t st);
// a strip's device controller on the rank-reduced max rate (res->max_rate)
void launch_spec_next(const DevParams *P, DevResult *res, DevParams *N, cudaStream_t st);
template <class T>
void launch_extrema(const Consts<T> &C, const T *w, const T *p, const T *q, const T *be,
                    Partial *part, cudaStream_t st);
int final_blocks(int nx, int ny);
int final_rows(int nx, int ny);  // k_final grid rows: row partials + counters
// BSQ_Y_SPIKE: per-column coupling system + in-place correction of a strip's Q
// apply = 0: only the per-column coupling values bt (k_final applies them)
template <class T>
void launch_spike(const Consts<T> &C, int G, int rank, const double *table, const T *yb, T *bt,
                  T *x, const T *v, const T *w, int south, int north, cudaStream_t st,
                  int apply, int jv, int jw);
// observers: gauge gather and the running max of w
template <class T>
void launch_gather(const T *w, const T *p, const T *q, const long long *goff, int ng, T *gval,
                   cudaStream_t st);
template <class T>
void launch_fold_max(const Consts<T> &C, const T *w, T *maxw, cudaStream_t st);

}  // namespace bsq
