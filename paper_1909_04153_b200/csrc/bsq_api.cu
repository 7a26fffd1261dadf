// bsq_api.cu -- the C ABI (include/bsq.h): context, workspace carving, the
// static LU precompute, host<->device I/O and the per-step launch sequence.
//
// The engine is templated on the device real type: BSQ_FP64 is the bitwise
// parity build; BSQ_FP32 stores and computes in float (north_star's fp32
// mode), converting at the host boundary so the ABI stays float64.
//
// Host arithmetic (coefficients, Thomas pivots) is plain IEEE binary64 with
// contraction disabled (-ffp-contract=off), so it reproduces the reference's
// numpy/numba values bit for bit (implicit.py:84-119, _kernels.py:360-378).
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <type_traits>
#include <vector>

#include <cudaTypedefs.h>

#include <nvtx3/nvToolsExt.h>

#ifndef BSQ_SPIKE2_IN_FINAL
#define BSQ_SPIKE2_IN_FINAL 0
#endif

#include "../../include/bsq.h"
#include "bsq_launch.h"

// NVTX ranges around the entry points (header-only NVTX v3: a no-op unless a
// profiler is attached), so an nsys / ncu timeline shows which call a
// kernel belongs to
namespace {
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
const char *phase_name(int ph) {
    static const char *names[] = {"bsq_phase:ghost",         "bsq_phase:stage",
                                  "bsq_phase:solve1_fwd",    "bsq_phase:solve1_bwd",
                                  "bsq_phase:correct",       "bsq_phase:solve2_fwd",
                                  "bsq_phase:solve2_bwd",    "bsq_phase:final",
                                  "bsq_phase:stage_inner",   "bsq_phase:stage_edge",
                                  "bsq_phase:correct_inner", "bsq_phase:correct_edge"};
    return (ph >= 0 && ph < (int)(sizeof(names) / sizeof(names[0]))) ? names[ph] : "bsq_phase";
}
}  // namespace

using namespace bsq;

bool bsq::pdl_on() {
    static const int on = [] {
        // off by default: measured 1.848 -> 1.860 ms per step with it on (the
        // early-resident CTAs of the next kernel take slots from the tail)
        const char *e = std::getenv("BSQ_PDL");
        return (e && e[0] == '1') ? 1 : 0;
    }();
    return on != 0;
}

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CU(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(BSQ_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));  \
    } while (0)

namespace {

constexpr int kMaxEv = 16;

enum Arr {
    A_W0, A_P0, A_Q0, A_W1, A_P1, A_Q1,
    A_BE, A_DEP, A_DDX, A_DDY, A_BFX, A_BFY,
    A_AX, A_DENX, A_RDENX, A_CWX, A_AY, A_DENY, A_RDENY, A_CWY,
    A_BU, A_BV, A_US, A_VS, A_P2, A_Q2,
    A_BX, A_CX, A_BY, A_CY,  // diagonals for solver="cr" (y ones transposed: [column][row])
    A_AYT,                   // solver="cr": the y sub-diagonal transposed
    A_SPV, A_SPW,            // BSQ_Y_SPIKE: south / north coupling spikes
    A_W2,                    // third w buffer: the speculative next stage writes here
    A_HIST0,  // 4 slots x 5 fields follow
    A_COUNT = A_HIST0 + 20
};

enum Small { S_CXL, S_CYL, S_FAC, S_PAR, S_RES, S_PART, S_CNT, S_DWIN, S_DWOUT, S_XIN, S_XOUT,
             S_SPBT, S_PAR2, S_FRAME, S_COUNT };

bool spike_mode(const bsq_desc *d) {
    return d->y_coupling == BSQ_Y_SPIKE && (d->south_internal || d->north_internal);
}

// arrays a context does not use take no memory
bool array_used(const bsq_desc *d, int k) {
    if (k >= A_BX && k <= A_AYT) return d->solver == BSQ_CR;
    if (k == A_SPV || k == A_SPW) return spike_mode(d);
    return true;
}

template <class T>
Layout make_layout(const bsq_desc *d) {
    Layout L;
    L.nx = d->nx;
    L.ny = d->ny;
    const int line = 128 / (int)sizeof(T);  // elements per 128 B
    L.xo = line - GL;
    const int need = L.xo + d->nx + 4;
    L.pitch = (need + line - 1) / line * line;
    return L;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

template <class T>
size_t layout_bytes(const bsq_desc *d, size_t offs[A_COUNT + S_COUNT], int *fac_stride) {
    const Layout L = make_layout<T>(d);
    size_t off = 0;
    const size_t one = align256((size_t)L.elems() * sizeof(T));
    for (int k = 0; k < A_COUNT; k++) {
        offs[k] = off;
        if (array_used(d, k)) off += one;
    }
    int fs = d->nx > d->ny ? d->nx : d->ny;
    fs = (fs + 31) / 32 * 32;
    *fac_stride = fs;
    const size_t small[S_COUNT] = {sizeof(T) * d->ny, sizeof(T) * d->nx, sizeof(T) * 4 * fs,
                                   sizeof(DevParams), sizeof(DevResult),
                                   sizeof(Partial) * (size_t)(final_blocks(d->nx, d->ny) +
                                                              final_rows(d->nx, d->ny)),
                                   sizeof(unsigned int) * (size_t)(1 + final_rows(d->nx, d->ny)),
                                   sizeof(T) * d->nx, sizeof(T) * d->nx, sizeof(T) * d->nx,
                                   sizeof(T) * d->nx, sizeof(T) * 2 * d->nx, sizeof(DevParams),
                                   sizeof(T) * frame_elems(d->nx, d->ny)};
    for (int k = 0; k < S_COUNT; k++) {
        offs[A_COUNT + k] = off;
        off += align256(small[k]);
    }
    return off;
}

int check_desc(const bsq_desc *d) {
    if (!d) return fail(BSQ_ERR_BAD_ARG, "null descriptor");
    if (d->nx < 5 || d->ny < 5) return fail(BSQ_ERR_BAD_ARG, "grid needs at least 5x5 cells");
    if (d->precision != BSQ_FP64 && d->precision != BSQ_FP32)
        return fail(BSQ_ERR_BAD_ARG, "precision must be BSQ_FP64 or BSQ_FP32");
    if (d->solver != BSQ_THOMAS && d->solver != BSQ_CR)
        return fail(BSQ_ERR_BAD_ARG, "solver must be BSQ_THOMAS or BSQ_CR");
    if (d->solver == BSQ_CR) {
        if (d->south_internal || d->north_internal)
            return fail(BSQ_ERR_BAD_ARG, "solver=cr is not sharded (use the Thomas pipeline)");
        const int eb = d->precision == BSQ_FP64 ? 8 : 4;
        if (cr_smem_bytes(d->nx, d->ny, eb) > 227 * 1024)
            return fail(BSQ_ERR_BAD_ARG, "solver=cr holds a line in shared memory: lines up to "
                                         "4096 (fp64) / 8192 (fp32) cells");
    }
    if (!(d->dx > 0 && d->dy > 0)) return fail(BSQ_ERR_BAD_ARG, "cell sizes must be positive");
    if (d->y_coupling != BSQ_Y_PIPELINE && d->y_coupling != BSQ_Y_SPIKE)
        return fail(BSQ_ERR_BAD_ARG, "y_coupling must be BSQ_Y_PIPELINE or BSQ_Y_SPIKE");
    if (d->south_internal || d->north_internal) {
        if (d->row0 < 0 || d->row0 + d->ny > d->ny_global)
            return fail(BSQ_ERR_BAD_ARG, "strip rows outside the global grid");
        if ((d->south_internal != 0) != (d->row0 > 0) ||
            (d->north_internal != 0) != (d->row0 + d->ny < d->ny_global))
            return fail(BSQ_ERR_BAD_ARG, "internal sides must face other strips");
    }
    for (int s = 0; s < 4; s++) {
        if (d->side_kind[s] < 0 || d->side_kind[s] > 2) return fail(BSQ_ERR_BAD_ARG, "bad side kind");
        const int n = (s == SIDE_E || s == SIDE_W) ? d->nx : d->ny;
        if (d->sponge_len[s] < 0 || d->sponge_lo[s] < 0 || d->sponge_lo[s] + d->sponge_len[s] > n)
            return fail(BSQ_ERR_BAD_ARG, "sponge band outside the grid");
    }
    return BSQ_OK;
}

// implicit.py:84-90 -- _coefficients(d, slope, delta, bp13)
void coefficients(double d, double slope, double delta2, double six_delta, double bp13, double *a,
                  double *b, double *cc) {
    double curv = bp13 * d * d / delta2;
    double drift = d * slope / six_delta;
    *a = drift - curv;
    *b = 1.0 + 2.0 * curv;
    *cc = -drift - curv;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    return encode;
}

}  // namespace

// ---------------------------------------------------------------------------
// the engine

struct EngineBase {
    virtual ~EngineBase() {}
};

template <class T>
struct Engine : EngineBase {
    static constexpr bool F64 = std::is_same<T, double>::value;
    bsq_desc d;
    Layout L;
    Consts<T> C;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    T *arr[A_COUNT];
    T *cx_last = nullptr, *cy_last = nullptr, *fac[4];
    T *dw_in = nullptr, *dw_out = nullptr, *x_in = nullptr, *x_out = nullptr;  // strip boundaries
    std::vector<double> cw_tail;   // cw of the strip's last row per column (next strip's cw_south)
    size_t offs[A_COUNT + S_COUNT];
    char *base = nullptr;
    DevParams *dparams = nullptr;
    DevResult *dres = nullptr;
    bool solve_exact = false;  // the line solves divide exactly (EXD): exact_tiny
    Partial *part = nullptr;
    unsigned int *counter = nullptr;
    DevParams *hparams = nullptr;  // pinned
    DevResult *hres = nullptr;     // pinned
    T *hfac = nullptr;             // pinned, 4 x fac_stride
    T *hstage = nullptr;           // pinned conversion staging (fp32 only): one padded field
    int fac_stride = 0, nfinal = 0;
    int cur = 0, head = 3, nlev = 0, pend_slot = 0;
    // w has three buffers (committed, pending, spare) so the next step's
    // stage can run before this step is committed; P and Q ping-pong
    int wc_ = 0, wp_ = 1;
    // speculation: dpar[pk] is this step's parameter block, dpar[pk ^ 1] the
    // next step's as k_final's controller writes it
    DevParams *dpar[2] = {nullptr, nullptr};
    int pk = 0;
    bool spec_pending = false;   // next step's ghost + stage are queued
    bool spec_commit = false;    // ... and the step they follow was committed
    bool spec_used = false;      // this step runs on them
    int spec_lo = 0, spec_hi = 0;  // rows of the queued stage (a strip queues its inner rows)
    bool final_split = false;    // BSQ_PH_FINAL_LAUNCH ran: the max rate was rank-reduced
    bsq_step_params last_p{};    // parameters of the step that queued them
    const bsq_step_params *cur_p = nullptr;  // the step in progress (bsq_step's argument)
    SpecNext spec_h{};           // their scheme parameters (device controller)
    // ghosts: the queued stage applies the next step's ghosts at t to the new
    // state, whose user-visible ghosts are the reference's (applied at t+dt
    // before the solves); those are saved and put back only if the state is
    // read before the next step (which then re-applies the ghosts at t)
    T *frame_w = nullptr, *frame_p = nullptr, *frame_q = nullptr;  // overwritten frame
    bool frame_restored = false;
    cudaEvent_t ev_res = nullptr;
    // overlapped state download (fp64): a copy stream reads the committed
    // state right after the step's result while the queued stage runs, and
    // the host patches the ghost frame from the saved copy
    cudaStream_t st_io = nullptr;
    cudaEvent_t ev_frame = nullptr;  // the frame save of the queued stage is done
    T *hframe = nullptr;             // pinned host copy of the saved frame
    cudaEvent_t ev_pre[kMaxEv] = {};
    const char *pre_name[kMaxEv] = {};
    int npre = 0;
    long long step_launches = 0;  // kernels queued by the current / last bsq_step
    bool pending = false, singular = false, pos_pivots = true, timing = false;
    bool rden_inrange = true;  // every pivot's exponent in [-1000, 1000]: RN(1/den) on chip
    int piv_flags() const {
        return (pos_pivots ? PIV_POSITIVE : 0) | (rden_inrange ? PIV_RDEN_INRANGE : 0);
    }
    cudaEvent_t ev[kMaxEv] = {};
    const char *ev_name[kMaxEv] = {};
    int nev = 0, last_n = 0;
    float last_ms[kMaxEv] = {};
    // observers: gauge cells gathered by k_final's last CTA,
    // and the running max of w folded by the next stage kernel
    long long *d_goff = nullptr;
    T *d_gval = nullptr, *h_gstage = nullptr;  // device / pinned staging, ng x 3
    std::vector<double> g_pend, g_com;  // samples of the pending / committed state
    int ng = 0;
    bool g_fresh = false;   // g_com holds the committed state's values
    T *maxw = nullptr;      // padded layout, interior used
    bool fold_req = false;  // fold the committed state into maxw at the next stage
    bool spike_fix_pending = false;  // k_final applies the second solve's spike correction
    // strips: rows [lo, hi) of the stage / the correction read no halo row, so
    // they run while the halo is in flight (BSQ_PH_*_INNER), the rest after
    bool stage_inner = false, correct_inner = false;
    void inner_rows(int reach, int &lo, int &hi) const {
        lo = d.south_internal ? STAGE_BAND : 0;
        hi = d.north_internal ? (d.ny - reach) / STAGE_BAND * STAGE_BAND : d.ny;
    }
    SolveMaps maps;                  // TMA descriptors (out slots patched per launch)
    CUtensorMap map_xout[3], map_yout[3];  // pending P/Q of state 0, state 1; P2/Q2

    static constexpr int kW[3] = {A_W0, A_W1, A_W2};
    T *W(int s) { return arr[kW[s == cur ? wc_ : wp_]]; }  // W(cur) committed, W(1-cur) pending
    T *Wspare() { return arr[kW[3 - wc_ - wp_]]; }
    T *Pp(int s) { return arr[s ? A_P1 : A_P0]; }
    T *Qq(int s) { return arr[s ? A_Q1 : A_Q0]; }
    T *H(int slot, int f) { return arr[A_HIST0 + slot * 5 + f]; }

    ~Engine() override {
        if (st) cudaStreamSynchronize(st);
        for (int k = 0; k < kMaxEv; k++) {
            if (ev[k]) cudaEventDestroy(ev[k]);
            if (ev_pre[k]) cudaEventDestroy(ev_pre[k]);
        }
        if (ev_res) cudaEventDestroy(ev_res);
        if (ev_frame) cudaEventDestroy(ev_frame);
        if (st_io) cudaStreamDestroy(st_io);
        if (hframe) cudaFreeHost(hframe);
        if (hparams) cudaFreeHost(hparams);
        if (hres) cudaFreeHost(hres);
        if (hfac) cudaFreeHost(hfac);
        if (hstage) cudaFreeHost(hstage);
        if (h_gstage) cudaFreeHost(h_gstage);
        if (d_goff) cudaFree(d_goff);
        if (d_gval) cudaFree(d_gval);
        if (maxw) cudaFree(maxw);
        if (d_sptab) cudaFree(d_sptab);
        if (own_stream && st) cudaStreamDestroy(st);
    }

    // -- host <-> device copies (float64 host arrays) --------------------------
    // rows x cols host block (host pitch `hpitch` elements) -> device at
    // element offset `dst_off`; fp32 converts through pinned staging.
    int upload(T *dst, long dst_off, const double *src, int rows, int cols, int hpitch) {
        if constexpr (F64) {
            CU(cudaMemcpy2DAsync(dst + dst_off, sizeof(T) * L.pitch, src, sizeof(double) * hpitch,
                                 sizeof(double) * cols, rows, cudaMemcpyHostToDevice, st));
        } else {
            CU(cudaStreamSynchronize(st));  // staging is reused
            for (long r = 0; r < rows; r++)
                for (long k = 0; k < cols; k++) hstage[r * cols + k] = T(src[r * hpitch + k]);
            CU(cudaMemcpy2DAsync(dst + dst_off, sizeof(T) * L.pitch, hstage, sizeof(T) * cols,
                                 sizeof(T) * cols, rows, cudaMemcpyHostToDevice, st));
            CU(cudaStreamSynchronize(st));
        }
        return BSQ_OK;
    }
    int download(double *dst, const T *src, long src_off, int rows, int cols) {
        if constexpr (F64) {
            CU(cudaMemcpy2DAsync(dst, sizeof(double) * cols, src + src_off, sizeof(T) * L.pitch,
                                 sizeof(T) * cols, rows, cudaMemcpyDeviceToHost, st));
        } else {
            CU(cudaMemcpy2DAsync(hstage, sizeof(T) * cols, src + src_off, sizeof(T) * L.pitch,
                                 sizeof(T) * cols, rows, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            for (long k = 0; k < (long)rows * cols; k++) dst[k] = double(hstage[k]);
        }
        return BSQ_OK;
    }
    int upload_padded(T *dst, const double *src, int rows, int cols) {
        return upload(dst, L.xo, src, rows, cols, cols);
    }
    int download_padded(double *dst, const T *src, int rows, int cols) {
        return download(dst, src, L.xo, rows, cols);
    }
    int upload_interior(T *dst, const double *src) {
        return upload(dst, L.at(GL, GL), src, L.ny, L.nx, L.nx);
    }
    int download_interior(double *dst, const T *src) {
        return download(dst, src, L.at(GL, GL), L.ny, L.nx);
    }

    // -- setup ---------------------------------------------------------------
    void set_consts() {
        const bsq_desc *p = &d;
        C.L = L;
        C.g = T(p->g);
        C.half_g = T(0.5) * C.g;
        C.h_eps = T(p->h_eps);
        C.theta = T(p->theta);
        C.c_f = T(p->c_f);
        C.b_disp = T(p->b_disp);
        C.bp13 = T(p->bp13);
        C.h_dry = T(p->h_dry);
        C.ws = T(p->ws);
        // derived exactly as the reference derives them (_kernels.py:224-261),
        // in the working precision
        C.inv_dx = T(1) / T(p->dx);
        C.inv_dy = T(1) / T(p->dy);
        C.inv_dx2 = C.inv_dx * C.inv_dx;
        C.inv_dy2 = C.inv_dy * C.inv_dy;
        C.two_dx = T(2) * T(p->dx);
        C.two_dy = T(2) * T(p->dy);
        C.r_two_dx = T(1) / C.two_dx;
        C.r_two_dy = T(1) / C.two_dy;
        C.dx2 = T(p->dx2);
        C.dy2 = T(p->dy2);
        C.r_dx2 = T(1) / C.dx2;
        C.r_dy2 = T(1) / C.dy2;
        C.three = T(3);
        C.r_three = T(1) / T(3);
        C.six = T(6);
        C.r_six = T(1) / T(6);
        for (int s = 0; s < 4; s++) {
            C.side_kind[s] = p->side_kind[s];
            C.sponge_lo[s] = p->sponge_lo[s];
            C.sponge_len[s] = p->sponge_len[s];
        }
        if (p->south_internal) C.side_kind[SIDE_S] = KIND_INTERNAL;
        if (p->north_internal) C.side_kind[SIDE_N] = KIND_INTERNAL;
        C.cross = p->cross_correction;
    }

    // Whether a static numerator of the stage / correction quotients --
    // depth (d / 6), d * d_x and d * d_y (/ 3) -- lies under the Markstein
    // exact range (0 < |x| < 2^-960): then every tile divides exactly.
    bool static_tiny(const bsq_static *f) const {
        const long nxt = d.nx + 4;
        auto tiny = [](double v) { return v != 0.0 && std::fabs(v) < TINY_NUM; };
        for (int j = 2; j < d.ny + 2; j++)
            for (int i = 2; i < d.nx + 2; i++) {
                const long o = j * nxt + i;
                const double dd = f->depth[o];
                if (tiny(dd) || tiny(dd * f->depth_dx[o]) || tiny(dd * f->depth_dy[o])) return true;
            }
        return false;
    }

    // Pre-factor every x row and y column of the static implicit operator
    // with thomas_batch's own recurrence (_kernels.py:368-378) in float64,
    // then store sub-diagonal, pivot, -RN(1/pivot) and cw in the working
    // precision (the reciprocal is rounded from the stored pivot).
    int factor_lines(const bsq_static *f) {
        const int nx = d.nx, ny = d.ny, nxt = nx + 4;
        const long E = L.elems();
        std::vector<T> ax(E, T(0)), denx(E, T(1)), rdenx(E, T(-1)), cwx(E, T(0));
        std::vector<T> bxv(E, T(1)), cxv(E, T(0)), byv(E, T(1)), cyv(E, T(0));  // for "cr"
        // "cr" y lines read their diagonals contiguously: column i's element j
        // at i * ny + j (the right-hand side and the result stay in the
        // padded layout)
        std::vector<T> ayt(d.solver == BSQ_CR ? E : 0, T(0));
        std::vector<T> ay(E, T(0)), deny(E, T(1)), rdeny(E, T(-1)), cwy(E, T(0));
        std::vector<T> cxl(ny), cyl(nx);
        const double six_dx = 6.0 * d.dx, six_dy = 6.0 * d.dy;
        bool sing = false, pos = true, inrange = true;
        auto put = [&](std::vector<T> &A, std::vector<T> &D, std::vector<T> &R,
                       std::vector<T> &CW, long o, double a, double den, double cw) {
            A[o] = T(a);
            const T dT = T(den);
            D[o] = dT;
            R[o] = -(T(1) / dT);  // negated (div_static_pos)
            CW[o] = T(cw);
            if (!(dT > T(0))) pos = false;
            if (den == 0.0) sing = true;
            // rcp_rn_inrange's verified domain: |exponent| <= 1000 (fp64), 100 (fp32)
            const double ad = std::fabs(double(dT)), lim = F64 ? 0x1p1000 : 0x1p100;
            if (!(ad >= 1.0 / lim && ad <= lim)) inrange = false;
        };
        for (int j = 0; j < ny; j++) {  // x rows
            double cw_prev = 0.0;
            for (int i = 0; i < nx; i++) {
                const long h = (long)(j + GL) * nxt + i + GL;
                double a, b, cc;
                coefficients(f->depth[h], f->depth_dx[h], d.dx2, six_dx, d.bp13, &a, &b, &cc);
                const double den = i == 0 ? b : b - a * cw_prev;
                const double cw = cc / den;
                put(ax, denx, rdenx, cwx, L.at(j + GL, i + GL), a, den, cw);
                bxv[L.at(j + GL, i + GL)] = T(b);
                cxv[L.at(j + GL, i + GL)] = T(cc);
                cw_prev = cw;
                if (i == nx - 1) cxl[j] = T(cc);
            }
        }
        // y columns; a strip with an internal south side continues the global
        // column's recurrence from the south strip's last cw
        const bool spike = spike_mode(&d);
        if (d.south_internal && !spike && !f->cw_south)
            return fail(BSQ_ERR_BAD_ARG, "strip with an internal south side needs cw_south");
        cw_tail.assign(nx, 0.0);
        for (int i = 0; i < nx; i++) {
            const bool cont = d.south_internal != 0 && !spike;  // spike: each block alone
            double cw_prev = cont ? f->cw_south[i] : 0.0;
            for (int j = 0; j < ny; j++) {
                const long h = (long)(j + GL) * nxt + i + GL;
                double a, b, cc;
                coefficients(f->depth[h], f->depth_dy[h], d.dy2, six_dy, d.bp13, &a, &b, &cc);
                const double den = (j == 0 && !cont) ? b : b - a * cw_prev;
                const double cw = cc / den;
                put(ay, deny, rdeny, cwy, L.at(j + GL, i + GL), a, den, cw);
                if (d.solver == BSQ_CR) {
                    const long t = (long)i * ny + j;
                    ayt[t] = T(a);
                    byv[t] = T(b);
                    cyv[t] = T(cc);
                }
                cw_prev = cw;
                if (j == ny - 1) cyl[i] = T(cc);
            }
            cw_tail[i] = cw_prev;
        }
        singular = sing;
        pos_pivots = pos;
        rden_inrange = inrange;
        if (spike) make_spikes(ay, deny, cwy, cyl);
        const size_t B = sizeof(T) * E;
        const std::vector<T> *src[13] = {&ax, &denx, &rdenx, &cwx, &ay, &deny, &rdeny, &cwy,
                                         &bxv, &cxv, &byv, &cyv, &ayt};
        const int dst[13] = {A_AX, A_DENX, A_RDENX, A_CWX, A_AY, A_DENY, A_RDENY, A_CWY,
                             A_BX, A_CX, A_BY, A_CY, A_AYT};
        for (int k = 0; k < (d.solver == BSQ_CR ? 13 : 8); k++)
            CU(cudaMemcpyAsync(arr[dst[k]], src[k]->data(), B, cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(cx_last, cxl.data(), sizeof(T) * ny, cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(cy_last, cyl.data(), sizeof(T) * nx, cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));  // host vectors go out of scope
        return BSQ_OK;
    }

    // BSQ_Y_SPIKE: v = A^-1 (a_first e_first), w = A^-1 (c_last e_last) for
    // every column of this strip's block, with the block's own LU factors
    // (thomas_batch's recurrence on a unit right-hand side)
    std::vector<double> sp_coef;  // 4 x nx: v_first, v_last, w_first, w_last
    // rows [0, sp_jv) carry the south spike v and rows [sp_jw, ny) the north
    // spike w at magnitudes >= SPIKE_TINY; beyond them the corrections
    // (|v b|, |w t| < 2^-64 of the interface values) are dropped
    static constexpr double SPIKE_TINY = 0x1p-64;
    int sp_jv = 0, sp_jw = 0;
    void make_spikes(const std::vector<T> &ay, const std::vector<T> &deny,
                     const std::vector<T> &cwy, const std::vector<T> &cyl) {
        const int nx = d.nx, ny = d.ny;
        const long E = L.elems();
        std::vector<T> vv(E, T(0)), ww(E, T(0));
        std::vector<double> col(ny);
        sp_coef.assign(4 * (size_t)nx, 0.0);
        sp_jv = 0;
        sp_jw = ny;
        for (int i = 0; i < nx; i++) {
            auto at = [&](int j) { return L.at(j + GL, i + GL); };
            if (d.south_internal) {
                double dw = double(ay[at(0)]) / double(deny[at(0)]);
                col[0] = dw;
                for (int j = 1; j < ny; j++) {
                    dw = (0.0 - double(ay[at(j)]) * dw) / double(deny[at(j)]);
                    col[j] = dw;
                }
                for (int j = ny - 2; j >= 0; j--) col[j] = col[j] - double(cwy[at(j)]) * col[j + 1];
                for (int j = 0; j < ny; j++) vv[at(j)] = T(col[j]);
                for (int j = ny - 1; j >= sp_jv; j--)
                    if (!(std::fabs(double(T(col[j]))) < SPIKE_TINY)) {  // NaN counts as large
                        sp_jv = j + 1;
                        break;
                    }
                sp_coef[0 * (size_t)nx + i] = double(T(col[0]));
                sp_coef[1 * (size_t)nx + i] = double(T(col[ny - 1]));
            }
            if (d.north_internal) {
                col[ny - 1] = double(cyl[i]) / double(deny[at(ny - 1)]);
                for (int j = ny - 2; j >= 0; j--) col[j] = 0.0 - double(cwy[at(j)]) * col[j + 1];
                for (int j = 0; j < ny; j++) ww[at(j)] = T(col[j]);
                for (int j = 0; j < sp_jw; j++)
                    if (!(std::fabs(double(T(col[j]))) < SPIKE_TINY)) {
                        sp_jw = j;
                        break;
                    }
                sp_coef[2 * (size_t)nx + i] = double(T(col[0]));
                sp_coef[3 * (size_t)nx + i] = double(T(col[ny - 1]));
            }
        }
        if (std::getenv("BSQ_SPIKE_VERBOSE"))
            std::fprintf(stderr, "bsq spike cut-offs: v rows [0, %d), w rows [%d, %d)\n",
                         d.south_internal ? sp_jv : 0, d.north_internal ? sp_jw : ny, ny);
        cudaMemcpyAsync(arr[A_SPV], vv.data(), sizeof(T) * E, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(arr[A_SPW], ww.data(), sizeof(T) * E, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
    }

    double *d_sptab = nullptr;  // G x 4 x nx, all ranks' spike coefficients
    int sp_G = 0, sp_rank = 0;

    int set_spike_table(const double *table, int G, int rank) {
        if (!spike_mode(&d)) return fail(BSQ_ERR_BAD_ARG, "context is not a spike-coupled strip");
        if (!table || G < 2 || G > 64 || rank < 0 || rank >= G)
            return fail(BSQ_ERR_BAD_ARG, "bad spike table (2 <= ranks <= 64)");
        if ((rank > 0) != (d.south_internal != 0) || (rank < G - 1) != (d.north_internal != 0))
            return fail(BSQ_ERR_BAD_ARG, "rank does not match the strip's internal sides");
        if (d_sptab) cudaFree(d_sptab);
        d_sptab = nullptr;
        CU(cudaMalloc(&d_sptab, sizeof(double) * 4 * (size_t)G * d.nx));
        CU(cudaMemcpyAsync(d_sptab, table, sizeof(double) * 4 * (size_t)G * d.nx,
                           cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
        sp_G = G;
        sp_rank = rank;
        return BSQ_OK;
    }

    int spike_fix(int solve, const void *ybound) {
        if (!d_sptab) return fail(BSQ_ERR_BAD_ARG, "spike table not set");
        if ((solve != 1 && solve != 2) || !ybound) return fail(BSQ_ERR_BAD_ARG, "bad spike_fix args");
        T *x = Qq(1 - cur);  // both solves land in the pending Q
        T *bt = (T *)(base + offs[A_COUNT + S_SPBT]);
        // BSQ_SPIKE2_IN_FINAL: the second solve's correction applied by
        // k_final as it loads Q (same operations as k_spike_fix).  Off: with
        // the cut-off rows the pass covers only the rows near the interfaces
        // (≈47 % of a 4096-row strip), and k_final's spike instantiation
        // spills (0.190 vs 0.134 ms); the pass costs 0.033 ms.
        const bool in_final = solve == 2 && BSQ_SPIKE2_IN_FINAL;
        launch_spike(C, sp_G, sp_rank, d_sptab, (const T *)ybound, bt, x, arr[A_SPV], arr[A_SPW],
                     d.south_internal, d.north_internal, st, !in_final, sp_jv, sp_jw);
        spike_fix_pending = in_final;
        CU(cudaGetLastError());
        return BSQ_OK;
    }

    // TMA descriptor of the interior region of one pitched array
    int make_map(CUtensorMap *m, T *base, bool xdir) {
        auto encode = tensor_map_encoder();
        if (!encode) return fail(BSQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        const cuuint32_t ek = (cuuint32_t)solve_chunk_elems(sizeof(T));
        cuuint64_t dims[2] = {(cuuint64_t)L.nx, (cuuint64_t)L.ny};
        cuuint64_t strides[1] = {(cuuint64_t)L.pitch * sizeof(T)};
        cuuint32_t box[2] = {xdir ? ek : 32u, xdir ? 32u : ek};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(m, F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                            2, base + L.at(GL, GL), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            xdir ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(BSQ_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        return BSQ_OK;
    }

    // TMA descriptor of a padded array for `bc` x `br` boxes (the stage's tile
    // loads).  The map starts at the pitched row start (128-B aligned, as a
    // map base must be 16-B aligned and fp32's padded origin xo = 30 is not):
    // box x coordinates carry + xo, and `cols` padded columns follow xo.
    int make_map_box(CUtensorMap *m, T *base, int cols, int rows, int bc, int br) {
        auto encode = tensor_map_encoder();
        if (!encode) return fail(BSQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        cuuint64_t dims[2] = {(cuuint64_t)(L.xo + cols), (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)L.pitch * sizeof(T)};
        cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(m, F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                            2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(BSQ_ERR_CUDA, "cuTensorMapEncodeTiled (stage box) failed");
        return BSQ_OK;
    }

    // stage tile boxes: 36 x 12 (32 x 8 tile + 2-cell halo); fp32: 40 x 12,
    // starting two columns further west (box origins on 16-B boundaries:
    // bsq_stage_tiled.cu Box<T>)
    CUtensorMap smap_w[3], smap_p[2], smap_q[2], smap_be, smap_dep, smap_bfx, smap_bfy;
    int build_stage_maps() {
        const int nxt = d.nx + 4, nyt = d.ny + 4, TX = STAGE_TX, TY = STAGE_TY,
                  HX = TX + (F64 ? 4 : 8), HY = TY + 4;
        int rc;
        for (int k = 0; k < 3; k++)
            if ((rc = make_map_box(&smap_w[k], arr[kW[k]], nxt, nyt, HX, HY))) return rc;
        for (int k = 0; k < 2; k++)
            if ((rc = make_map_box(&smap_p[k], Pp(k), nxt, nyt, HX, HY)) ||
                (rc = make_map_box(&smap_q[k], Qq(k), nxt, nyt, HX, HY)))
                return rc;
        if ((rc = make_map_box(&smap_be, arr[A_BE], nxt, nyt, HX, HY)) ||
            (rc = make_map_box(&smap_dep, arr[A_DEP], nxt, nyt, HX, HY)) ||
            (rc = make_map_box(&smap_bfx, arr[A_BFX], nxt - 1, nyt, HX, TY)) ||
            (rc = make_map_box(&smap_bfy, arr[A_BFY], nxt, nyt - 1, TX, TY + 3)))
            return rc;
        return BSQ_OK;
    }
    // 32 x 8 tile boxes of the stage's phase-D inputs (static slopes and the
    // ring slots), built once per array
    std::vector<std::pair<const T *, CUtensorMap>> pf_cache;
    const CUtensorMap *pf_map(const T *a) {
        for (auto &e : pf_cache)
            if (e.first == a) return &e.second;
        CUtensorMap m;
        if (make_map_box(&m, const_cast<T *>(a), d.nx + 4, d.ny + 4, STAGE_TX, STAGE_TY)) return nullptr;
        pf_cache.emplace_back(a, m);
        return &pf_cache.back().second;
    }
    StageMaps stage_maps_for(const StagePtrs<T> &A) {
        StageMaps M = stage_maps_for(A.w, A.p, A.q);
        const T *src[12] = {A.ddx, A.ddy, A.h1[0], A.h1[1], A.h1[2], A.h1[3], A.h1[4],
                            A.h2[0], A.h2[1], A.h2[2], A.h2[3], A.h2[4]};
        for (int k = 0; k < 12; k++) {
            const CUtensorMap *m = src[k] ? pf_map(src[k]) : nullptr;
            if (m) M.pf[k] = *m;
            else std::memset(&M.pf[k], 0, sizeof(CUtensorMap));
        }
        return M;
    }
    StageMaps stage_maps_for(const T *w, const T *p, const T *q) {
        StageMaps M;
        for (int k = 0; k < 3; k++)
            if (arr[kW[k]] == w) M.w = smap_w[k];
        M.p = Pp(0) == p ? smap_p[0] : smap_p[1];
        M.q = Qq(0) == q ? smap_q[0] : smap_q[1];
        M.be = smap_be;
        M.dep = smap_dep;
        M.bfx = smap_bfx;
        M.bfy = smap_bfy;
        return M;
    }

    int build_maps() {
        SolveMaps &M = maps;
        M.xp_rhs = arr[A_US];
        M.xp_a = arr[A_AX];
        M.xp_den = arr[A_DENX];
        M.xp_rden = arr[A_RDENX];
        M.xp_cw = arr[A_CWX];
        int rc;
        if ((rc = build_stage_maps())) return rc;
        if ((rc = make_map(&M.x_rhs, arr[A_US], true)) || (rc = make_map(&M.x_a, arr[A_AX], true)) ||
            (rc = make_map(&M.x_den, arr[A_DENX], true)) ||
            (rc = make_map(&M.x_rden, arr[A_RDENX], true)) ||
            (rc = make_map(&M.x_cw, arr[A_CWX], true)) ||
            (rc = make_map(&M.y_rhs, arr[A_VS], false)) || (rc = make_map(&M.y_a, arr[A_AY], false)) ||
            (rc = make_map(&M.y_den, arr[A_DENY], false)) ||
            (rc = make_map(&M.y_rden, arr[A_RDENY], false)) ||
            (rc = make_map(&M.y_cw, arr[A_CWY], false)) || (rc = make_map(&map_xout[0], Pp(0), true)) ||
            (rc = make_map(&map_xout[1], Pp(1), true)) || (rc = make_map(&map_xout[2], arr[A_P2], true)) ||
            (rc = make_map(&map_yout[0], Qq(0), false)) || (rc = make_map(&map_yout[1], Qq(1), false)) ||
            (rc = make_map(&map_yout[2], arr[A_Q2], false)))
            return rc;
        return BSQ_OK;
    }

    int create(const bsq_desc *desc, const bsq_static *f, void *workspace, size_t bytes, void *stream) {
        d = *desc;
        L = make_layout<T>(desc);
        const size_t need = layout_bytes<T>(desc, offs, &fac_stride);
        if (bytes < need) return fail(BSQ_ERR_BAD_ARG, "workspace too small");
        if (((uintptr_t)workspace & 255) != 0) return fail(BSQ_ERR_BAD_ARG, "workspace not 256-B aligned");
        nfinal = final_blocks(desc->nx, desc->ny);
        base = (char *)workspace;
        for (int k = 0; k < A_COUNT; k++) arr[k] = (T *)(base + offs[k]);
        dw_in = (T *)(base + offs[A_COUNT + S_DWIN]);
        dw_out = (T *)(base + offs[A_COUNT + S_DWOUT]);
        x_in = (T *)(base + offs[A_COUNT + S_XIN]);
        x_out = (T *)(base + offs[A_COUNT + S_XOUT]);
        cx_last = (T *)(base + offs[A_COUNT + S_CXL]);
        cy_last = (T *)(base + offs[A_COUNT + S_CYL]);
        for (int s = 0; s < 4; s++) fac[s] = (T *)(base + offs[A_COUNT + S_FAC]) + s * fac_stride;
        dpar[0] = (DevParams *)(base + offs[A_COUNT + S_PAR]);
        dpar[1] = (DevParams *)(base + offs[A_COUNT + S_PAR2]);
        dparams = dpar[0];
        dres = (DevResult *)(base + offs[A_COUNT + S_RES]);
        part = (Partial *)(base + offs[A_COUNT + S_PART]);
        counter = (unsigned int *)(base + offs[A_COUNT + S_CNT]);
        if (stream) {
            st = (cudaStream_t)stream;
        } else {
            CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            own_stream = true;
        }
        CU(cudaMallocHost(&hparams, sizeof(DevParams)));
        CU(cudaMallocHost(&hres, sizeof(DevResult)));
        CU(cudaMallocHost(&hfac, sizeof(T) * 4 * fac_stride));
        if (!F64) CU(cudaMallocHost(&hstage, sizeof(T) * (size_t)(d.ny + 4) * (d.nx + 4)));
        for (int k = 0; k < kMaxEv; k++) {
            CU(cudaEventCreate(&ev[k]));
            CU(cudaEventCreate(&ev_pre[k]));
        }
        CU(cudaEventCreateWithFlags(&ev_res, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&ev_frame, cudaEventDisableTiming));
        if (F64) {  // the overlapped state download (download_beside_spec)
            CU(cudaStreamCreateWithFlags(&st_io, cudaStreamNonBlocking));
            CU(cudaMallocHost(&hframe, sizeof(T) * frame_elems(d.nx, d.ny)));
        }
        set_consts();
        C.exact = F64 && static_tiny(f) ? 1 : 0;
        solve_exact = F64 && d.exact_tiny != 0;
        C.exact_final = solve_exact ? 1 : 0;
        const int nx = d.nx, ny = d.ny;
        CU(cudaMemsetAsync(workspace, 0, need, st));  // ghost cells of scratch arrays stay defined
        int rc;
        if ((rc = upload_padded(arr[A_BE], f->bed_eff, ny + 4, nx + 4)) ||
            (rc = upload_padded(arr[A_DEP], f->depth, ny + 4, nx + 4)) ||
            (rc = upload_padded(arr[A_DDX], f->depth_dx, ny + 4, nx + 4)) ||
            (rc = upload_padded(arr[A_DDY], f->depth_dy, ny + 4, nx + 4)) ||
            (rc = upload_padded(arr[A_BFX], f->bed_face_x, ny + 4, nx + 3)) ||
            (rc = upload_padded(arr[A_BFY], f->bed_face_y, ny + 3, nx + 4)) ||
            (rc = factor_lines(f)) || (rc = build_maps()))
            return rc;
        CU(cudaMemsetAsync(counter, 0, sizeof(unsigned int) * (1 + final_rows(nx, ny)), st));
        CU(cudaStreamSynchronize(st));
        return BSQ_OK;
    }

    // -- state ----------------------------------------------------------------
    int upload_state(const double *w, const double *p, const double *q) {
        const int s = cur, ny = d.ny, nx = d.nx;
        int rc;
        if ((rc = upload_padded(W(s), w, ny + 4, nx + 4)) ||
            (rc = upload_padded(Pp(s), p, ny + 4, nx + 4)) ||
            (rc = upload_padded(Qq(s), q, ny + 4, nx + 4)))
            return rc;
        CU(cudaStreamSynchronize(st));
        pending = false;
        g_fresh = false;
        spec_pending = false;
        frame_w = frame_p = frame_q = nullptr;
        return BSQ_OK;
    }
    T *frame_buf() { return (T *)(base + offs[A_COUNT + S_FRAME]); }

    // a state about to be read shows the ghosts the reference leaves on it
    void unframe(T *w, T *p, T *q) {
        if (frame_w && frame_w == w && frame_p == p && frame_q == q) {
            launch_frame(C, w, p, q, frame_buf(), 0, st);
            frame_w = frame_p = frame_q = nullptr;
            frame_restored = true;
        }
    }

    int download_state(int which, double *w, double *p, double *q) {
        if (which == 1 && !pending) return fail(BSQ_ERR_BAD_ARG, "no pending step");
        const int s = which == 1 ? 1 - cur : cur, ny = d.ny, nx = d.nx;
        if (F64 && frame_w && frame_w == W(s) && frame_p == Pp(s) && frame_q == Qq(s))
            return download_beside_spec(s, w, p, q);
        unframe(W(s), Pp(s), Qq(s));
        int rc;
        if ((rc = download_padded(w, W(s), ny + 4, nx + 4)) ||
            (rc = download_padded(p, Pp(s), ny + 4, nx + 4)) ||
            (rc = download_padded(q, Qq(s), ny + 4, nx + 4)))
            return rc;
        CU(cudaStreamSynchronize(st));
        return BSQ_OK;
    }
    // The queued stage of the next step only rewrites this state's ghost
    // frame (saved first): copy the state on st_io as soon as the step's
    // result is in, beside the queued work, and put the saved frame into the
    // host arrays.  The device keeps the frame the queued stage needs.
    int download_beside_spec(int s, double *w, double *p, double *q) {
        const int ny = d.ny, nx = d.nx, W_ = nx + 4, nrow = 4 * W_, n = nrow + 4 * ny;
        CU(cudaStreamWaitEvent(st_io, ev_res, 0));
        double *dst[3] = {w, p, q};
        const T *src[3] = {W(s), Pp(s), Qq(s)};
        for (int a = 0; a < 3; a++)
            CU(cudaMemcpy2DAsync(dst[a], sizeof(double) * W_, src[a] + L.xo, sizeof(T) * L.pitch,
                                 sizeof(T) * W_, ny + 4, cudaMemcpyDeviceToHost, st_io));
        CU(cudaStreamWaitEvent(st_io, ev_frame, 0));
        CU(cudaMemcpyAsync(hframe, frame_buf(), sizeof(T) * 3 * (size_t)n, cudaMemcpyDeviceToHost,
                           st_io));
        CU(cudaStreamSynchronize(st_io));
        // k_frame's order: rows 0, 1, ny+2, ny+3, then columns 0, 1, nx+2, nx+3
        for (int a = 0; a < 3; a++) {
            const T *f = hframe + (size_t)a * n;
            for (int r = 0; r < 4; r++) {
                const long J = r < 2 ? r : ny + r;
                for (int i = 0; i < W_; i++) dst[a][J * W_ + i] = double(f[r * W_ + i]);
            }
            for (int c = 0; c < 4; c++) {
                const long I = c < 2 ? c : nx + c;
                for (int j = 0; j < ny; j++)
                    dst[a][(long)(GL + j) * W_ + I] = double(f[nrow + c * ny + j]);
            }
        }
        return BSQ_OK;
    }
    int download_history(int level, int field, double *out) {
        if (field < 0 || field > 4 || level < 0 || level >= nlev)
            return fail(BSQ_ERR_BAD_ARG, "bad history level/field");
        int rc;
        if ((rc = download_interior(out, H((head - level + 4) % 4, field)))) return rc;
        CU(cudaStreamSynchronize(st));
        return BSQ_OK;
    }

    // -- step ---------------------------------------------------------------------
    void ev_mark(const char *name) {
        if (!timing || nev >= kMaxEv) return;
        ev_name[nev] = name;
        cudaEventRecord(ev[nev++], st);
    }

    int stage_params(const bsq_step_params *p) {
        DevParams &h = *hparams;
        h.t = p->t;
        h.dt = p->dt;
        h.euler = p->euler;
        h.wc = p->wc;
        h.wp = p->wp;
        h.wp2 = p->wp2;
        h.sc = p->sc;
        h.sp = p->sp;
        h.sp2 = p->sp2;
        h.f_dt = (float)h.dt, h.f_wc = (float)h.wc, h.f_wp = (float)h.wp, h.f_wp2 = (float)h.wp2;
        h.f_sc = (float)h.sc, h.f_sp = (float)h.sp, h.f_sp2 = (float)h.sp2, h.f_pad_ = 0.f;
        h.spec = p->spec ? 1 : 0;
        h.adaptive = p->adaptive;
        h.step_index = p->step_index;
        h.cfl_target = p->cfl_target;
        h.alpha = p->alpha;
        h.dt_min = p->dt_min;
        h.dt_max = p->dt_max;
        h.dt_init = p->dt_init;
        h.chain = p->chain;
        h.dt_fixed = p->dt_fixed;
        h.dt_prev = p->dt_prev;
        for (int s = 0; s < 4; s++) {
            h.gw_t[s] = d.ws + p->maker_eta_t[s];  // boundary.py:240 w_val = ws + eta
            h.gf_t[s] = p->maker_flux_t[s];
            h.gw_n[s] = d.ws + p->maker_eta_n[s];
            h.gf_n[s] = p->maker_flux_n[s];
        }
        CU(cudaMemcpyAsync(dparams, hparams, sizeof(DevParams), cudaMemcpyHostToDevice, st));
        bool any = false;
        for (int s = 0; s < 4; s++) {
            const int n = d.sponge_len[s];
            if (n > 0) {
                if (!p->sponge_fac[s]) return fail(BSQ_ERR_BAD_ARG, "missing sponge factors");
                T *dst = hfac + (size_t)s * fac_stride;
                for (int k = 0; k < n; k++) dst[k] = T(p->sponge_fac[s][k]);
                any = true;
            }
        }
        if (any)
            CU(cudaMemcpyAsync(fac[0], hfac, sizeof(T) * 4 * fac_stride, cudaMemcpyHostToDevice, st));
        return BSQ_OK;
    }

    StagePtrs<T> stage_ptrs(int slot) {
        StagePtrs<T> A = stage_ptrs_on(W(cur), Pp(cur), Qq(cur), slot, head, (head + 3) % 4, W(1 - cur));
        A.maxw = fold_req ? maxw : nullptr;
        return A;
    }

    // the stage of the state (w, p, q) whose newest / middle stage levels are
    // ring slots s1 / s2, writing slot `slot` and the predicted w into wn
    StagePtrs<T> stage_ptrs_on(T *w, T *p, T *q, int slot, int s1, int s2, T *wn) {
        StagePtrs<T> A;
        A.w = w;
        A.p = p;
        A.q = q;
        A.be = arr[A_BE];
        A.dep = arr[A_DEP];
        A.ddx = arr[A_DDX];
        A.ddy = arr[A_DDY];
        A.bfx = arr[A_BFX];
        A.bfy = arr[A_BFY];
        for (int f = 0; f < 5; f++) {
            A.h0[f] = H(slot, f);
            A.h1[f] = H(s1, f);
            A.h2[f] = H(s2, f);
        }
        A.wn = wn;
        A.bu = arr[A_BU];
        A.bv = arr[A_BV];
        A.us = arr[A_US];
        A.vs = arr[A_VS];
        A.bad = dres->stage_bad;
        A.maxw = nullptr;
        return A;
    }

    static bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

    // the queued ghost + stage are this step's: the previous step was
    // committed and every input they consumed equals this step's
    bool spec_matches(const bsq_step_params *p) const {
        if (!(spec_pending && spec_commit && spec_h.valid && p->spec)) return false;
        if (!same_bits(p->dt, spec_h.dt) || (p->euler != 0) != (spec_h.euler != 0)) return false;
        if (!p->euler &&
            !(same_bits(p->wc, spec_h.wc) && same_bits(p->wp, spec_h.wp) &&
              same_bits(p->wp2, spec_h.wp2) && same_bits(p->sc, spec_h.sc) &&
              same_bits(p->sp, spec_h.sp) && same_bits(p->sp2, spec_h.sp2)))
            return false;
        for (int s = 0; s < 4; s++)
            if (!same_bits(p->maker_eta_t[s], last_p.maker_eta_n[s]) ||
                !same_bits(p->maker_flux_t[s], last_p.maker_flux_n[s]))
                return false;
        return true;
    }

    SolvePtrs<T> solve_ptrs(int nxt_state) {
        SolvePtrs<T> S;
        S.exact = solve_exact;
        S.gp = Pp(nxt_state);
        S.gq = Qq(nxt_state);
        S.cx_last = cx_last;
        S.cy_last = cy_last;
        S.south_int = d.south_internal;
        S.north_int = d.north_internal;
        S.dw_in = dw_in;
        S.dw_out = dw_out;
        S.x_in = x_in;
        S.x_out = x_out;
        return S;
    }

    // phase 1 solves U*, V* into the pending state's P, Q; phase 2 solves the
    // corrected right-hand sides (written over us / vs) into P2, Q2
    // Both solves write the pending state's P, Q (the second overwrites the
    // first once the cross terms have read it); `scratch` sends a second solve
    // to P2 / Q2 instead (the bsq_solve_momentum seam)
    const SolveMaps &solve_maps(int phase, int nxt_state, bool scratch = false) {
        const int k = (phase == 2 && scratch) ? 2 : nxt_state;
        maps.x_out = map_xout[k];
        maps.y_out = map_yout[k];
        maps.xp_out = k == 2 ? arr[A_P2] : Pp(k);
        return maps;
    }

    CorrectPtrs<T> correct_ptrs(int slot, int nxt_state) {
        CorrectPtrs<T> K;
        K.bu = arr[A_BU];
        K.bv = arr[A_BV];
        K.fs = H(slot, 3);
        K.gs = H(slot, 4);
        K.p1 = Pp(nxt_state);
        K.q1 = Qq(nxt_state);
        K.dep = arr[A_DEP];
        K.ddx = arr[A_DDX];
        K.ddy = arr[A_DDY];
        K.us = arr[A_US];
        K.vs = arr[A_VS];
        return K;
    }

    void fill_result(bsq_step_result *r) {
        const DevResult &h = *hres;
        r->max_rate = h.max_rate;
        r->max_speed = h.max_speed;
        r->max_depth = h.max_depth;
        r->max_dev = h.max_dev;
        r->clamped = h.clamped;
        for (int k = 0; k < 5; k++) r->stage_bad[k] = h.stage_bad[k] == ~0ull ? -1 : (int64_t)h.stage_bad[k];
        for (int k = 0; k < 3; k++) r->state_bad[k] = h.state_bad[k] == ~0ull ? -1 : (int64_t)h.state_bad[k];
    }

    bool strip() const { return d.south_internal || d.north_internal; }

    // The TMA unit bounds its tensor stores in 16-byte units of the inner
    // dimension: when a row's nx elements end inside a unit (odd nx in fp64,
    // nx % 4 != 0 in fp32) the solve's stores into the pending P / Q also
    // write their first east ghost column.  The ghosts at t+dt are read
    // afterwards (cross terms, second-solve folding), so re-apply them: same
    // kernel, same inputs as the stage phase's fill.
    bool tma_tail_clobbers() const { return (d.nx * (int)sizeof(T)) % 16 != 0; }
    void reghost_after_tma(int nxt) {
        if (!tma_tail_clobbers()) return;
        ++step_launches;
        launch_ghost(C, dparams, 1, W(nxt), Pp(cur), Qq(cur), W(nxt), Pp(nxt), Qq(nxt), st);
    }

    // One phase of the step (include/bsq.h BSQ_PH_*).  For a whole grid the
    // y-line solves run complete inside the *F phases and the *B phases are
    // empty; for a strip they split at the rank boundary exchange.
    int phase(int ph, const bsq_step_params *p, bsq_step_result *r) {
        const int nxt = 1 - cur;
        const int slot = (head + 1) % 4;
        const bool piped = strip() && !spike_mode(&d);  // rank-pipelined y recurrence
        const int fwd_mode = piped ? SOLVE_X_YFWD : SOLVE_FULL;
        switch (ph) {
        case BSQ_PH_GHOST: {
            cur_p = p;
            step_launches = 0;
            // a step abandoned after bsq_spike_fix(2) (e.g. a failed exchange)
            // must not hand its coupling correction to this step's k_final
            spike_fix_pending = false;
            spec_used = spec_matches(p);
            spec_pending = false;
            if (spec_used) {  // the stage already ran (on dpar[pk ^ 1])
                pk ^= 1;
                dparams = dpar[pk];
                int rc = stage_params(p);  // the rest of this step's parameters
                if (rc) return rc;
                nev = npre;
                for (int k = 0; k < npre; k++) {
                    std::swap(ev[k], ev_pre[k]);
                    ev_name[k] = pre_name[k];
                }
                // the committed state carries the ghosts at t (the reference
                // applies them in place) -- unless a read put the old ones back
                if (frame_restored) {
                    ++step_launches;
                    launch_ghost(C, dparams, 0, W(cur), Pp(cur), Qq(cur), W(cur), Pp(cur), Qq(cur),
                                 st);
                }
                frame_w = frame_p = frame_q = nullptr;
                frame_restored = false;
                break;
            }
            int rc = stage_params(p);
            if (rc) return rc;
            CU(cudaMemsetAsync(dres, 0xFF, sizeof(DevResult), st));
            nev = 0;
            ev_mark("start");
            ++step_launches;
            launch_ghost(C, dparams, 0, W(cur), Pp(cur), Qq(cur), W(cur), Pp(cur), Qq(cur), st);
            ev_mark("ghost_t");
            // the ghosts at t are in place now, as in the reference: a frame
            // saved for a rejected speculation is stale from here on
            frame_w = frame_p = frame_q = nullptr;
            frame_restored = false;
            break;
        }
        case BSQ_PH_STAGE:
            if (!spec_used) {
                ++step_launches;
                const StagePtrs<T> A = stage_ptrs(slot);
                const StageMaps sm = stage_maps_for(A);
                launch_stage(C, dparams, A, 1, st, &sm);
                fold_req = false;
                ev_mark("stage");
            } else {
                stage_rest(slot);
            }
            ++step_launches;
            launch_ghost(C, dparams, 1, W(nxt), Pp(cur), Qq(cur), W(nxt), Pp(nxt), Qq(nxt), st);
            ev_mark("ghost_n");
            break;
        case BSQ_PH_SOLVE1F:
            ++step_launches;
            if (d.solver == BSQ_CR) {
                launch_cr(C, cr_ptrs(1, nxt), st);
            } else {
                launch_solve(C, solve_maps(1, nxt), solve_ptrs(nxt), piv_flags(), st, fwd_mode);
                reghost_after_tma(nxt);
            }
            ev_mark("solve1");
            break;
        case BSQ_PH_SOLVE1B:
            if (piped) {
                ++step_launches;
                launch_solve(C, solve_maps(1, nxt), solve_ptrs(nxt), piv_flags(), st, SOLVE_YBWD);
                reghost_after_tma(nxt);
                ev_mark("solve1b");
            }
            break;
        case BSQ_PH_CORRECT:
            if (d.cross_correction) {
                ++step_launches;
                launch_correct(C, correct_ptrs(slot, nxt), st);
                ev_mark("correct");
            }
            break;
        case BSQ_PH_STAGE_INNER: {
            // the stage reads rows J-2 .. J+2: rows >= 2 away from an internal
            // side need none of the halo rows being exchanged
            int lo, hi;
            inner_rows(2, lo, hi);
            stage_inner = !spec_used && hi > lo;
            if (stage_inner) {
                ++step_launches;
                const StagePtrs<T> A = stage_ptrs(slot);
                const StageMaps sm = stage_maps_for(A);
                launch_stage(C, dparams, A, 1, st, &sm, lo, hi - lo);
            }
            break;
        }
        case BSQ_PH_STAGE_EDGE: {
            if (!spec_used) {
                const StagePtrs<T> A = stage_ptrs(slot);
                const StageMaps sm = stage_maps_for(A);
                if (stage_inner) {
                    int lo, hi;
                    inner_rows(2, lo, hi);
                    step_launches += (lo > 0) + (hi < d.ny);
                    launch_stage(C, dparams, A, 1, st, &sm, 0, lo);
                    launch_stage(C, dparams, A, 1, st, &sm, hi, d.ny - hi);
                } else {
                    ++step_launches;
                    launch_stage(C, dparams, A, 1, st, &sm);
                }
                fold_req = false;
                ev_mark("stage");
            } else {
                stage_rest(slot);
            }
            stage_inner = false;
            ++step_launches;
            launch_ghost(C, dparams, 1, W(nxt), Pp(cur), Qq(cur), W(nxt), Pp(nxt), Qq(nxt), st);
            ev_mark("ghost_n");
            break;
        }
        case BSQ_PH_CORRECT_INNER: {
            // the correction reads rows J-1 .. J+1 of the first-solve momenta
            int lo, hi;
            inner_rows(1, lo, hi);
            correct_inner = d.cross_correction && hi > lo;
            if (correct_inner) {
                ++step_launches;
                launch_correct(C, correct_ptrs(slot, nxt), st, lo, hi - lo);
            }
            break;
        }
        case BSQ_PH_CORRECT_EDGE:
            if (d.cross_correction) {
                if (correct_inner) {
                    int lo, hi;
                    inner_rows(1, lo, hi);
                    step_launches += (lo > 0) + (hi < d.ny);
                    launch_correct(C, correct_ptrs(slot, nxt), st, 0, lo);
                    launch_correct(C, correct_ptrs(slot, nxt), st, hi, d.ny - hi);
                } else {
                    ++step_launches;
                    launch_correct(C, correct_ptrs(slot, nxt), st);
                }
                ev_mark("correct");
            }
            correct_inner = false;
            break;
        case BSQ_PH_SOLVE2F:
            if (d.cross_correction) {
                ++step_launches;
                if (d.solver == BSQ_CR)
                    launch_cr(C, cr_ptrs(2, nxt), st);
                else {
                    launch_solve(C, solve_maps(2, nxt), solve_ptrs(nxt), piv_flags(), st, fwd_mode);
                    reghost_after_tma(nxt);
                }
                ev_mark("solve2");
            }
            break;
        case BSQ_PH_SOLVE2B:
            if (d.cross_correction && piped) {
                ++step_launches;
                launch_solve(C, solve_maps(2, nxt), solve_ptrs(nxt), piv_flags(), st, SOLVE_YBWD);
                reghost_after_tma(nxt);
                ev_mark("solve2b");
            }
            break;
        case BSQ_PH_FINAL_LAUNCH:
            final_kernel(slot, nxt);
            final_split = true;
            break;
        case BSQ_PH_FINAL:
            return finish(r, slot, nxt);
        default:
            return fail(BSQ_ERR_BAD_ARG, "unknown phase");
        }
        CU(cudaGetLastError());
        return BSQ_OK;
    }

    int step(const bsq_step_params *p, bsq_step_result *r) {
        for (int ph = BSQ_PH_GHOST; ph <= BSQ_PH_FINAL; ph++) {
            const int rc = phase(ph, p, r);
            if (rc) return rc;
        }
        return BSQ_OK;
    }

    // the rows of a speculated stage's step that the queued stage did not run
    // (a strip queues only the rows that read no halo row)
    void stage_rest(int slot) {
        if (spec_lo <= 0 && spec_hi >= d.ny) return;
        const StagePtrs<T> A = stage_ptrs(slot);
        const StageMaps sm = stage_maps_for(A);
        if (spec_lo > 0) {
            ++step_launches;
            launch_stage(C, dparams, A, 1, st, &sm, 0, spec_lo);
        }
        if (spec_hi < d.ny) {
            ++step_launches;
            launch_stage(C, dparams, A, 1, st, &sm, spec_hi, d.ny - spec_hi);
        }
        ev_mark("stage");
    }

    // k_final: the single-grid controller (spec_next in its last CTA) unless
    // this is a strip, whose rate must first be reduced over the ranks
    void final_kernel(int slot, int nxt) {
        FinalPtrs<T> F;
        F.w = W(nxt);
        F.pin = Pp(nxt);  // the last solve's result, in place
        F.qin = Qq(nxt);
        F.pout = Pp(nxt);
        F.qout = Qq(nxt);
        F.be = arr[A_BE];
        for (int s = 0; s < 4; s++) F.fac[s] = fac[s];
        F.part = part;
        F.counter = counter;
        F.res = dres;
        F.goff = d_goff;
        F.ng = ng;
        F.gval = d_gval;
        F.spbt = spike_fix_pending ? (const T *)(base + offs[A_COUNT + S_SPBT]) : nullptr;
        F.spv = arr[A_SPV];
        F.spw = arr[A_SPW];
        F.sp_south = d.south_internal;
        F.sp_north = d.north_internal;
        F.sp_jv = sp_jv;
        F.sp_jw = sp_jw;
        spike_fix_pending = false;
        F.P = dparams;
        F.pnext = (hparams->spec && !strip() && !fold_req) ? dpar[pk ^ 1] : nullptr;
        ++step_launches;
        launch_final(C, F, st);
        ev_mark("final");
    }

    int finish(bsq_step_result *r, int slot, int nxt) {
        if (!final_split) final_kernel(slot, nxt);
        // a strip speculates only when the host reduced the rate in between
        const bool spec = hparams->spec && !fold_req && (!strip() || final_split);
        final_split = false;
        if (spec && strip()) {
            ++step_launches;
            launch_spec_next(dparams, dres, dpar[pk ^ 1], st);
        }
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
        if (ng)
            CU(cudaMemcpyAsync(h_gstage, d_gval, sizeof(T) * 3 * ng, cudaMemcpyDeviceToHost, st));
        CU(cudaEventRecord(ev_res, st));
        if (spec) {
            // the next step's ghost at t and stage, on this step's new state,
            // behind the result copy: they overlap the host's turn-around
            last_p = *cur_p;
            CU(cudaMemsetAsync(dres, 0xFF, sizeof(DevResult), st));
            DevParams *pn = dpar[pk ^ 1];
            npre = 0;
            auto pre = [&](const char *nm) {
                if (!timing || npre >= kMaxEv) return;
                pre_name[npre] = nm;
                cudaEventRecord(ev_pre[npre++], st);
            };
            // the new state keeps the ghosts the reference leaves on it
            // (applied at t+dt before the solves); the queued stage needs the
            // ones at t_{n+1}: save, apply, run, restore
            pre("start");
            // ghosts at t_{n+1}, saving the frame they overwrite on the way
            ++step_launches;
            launch_ghost(C, pn, 0, W(nxt), Pp(nxt), Qq(nxt), W(nxt), Pp(nxt), Qq(nxt), st,
                         frame_buf());
            CU(cudaEventRecord(ev_frame, st));
            frame_w = W(nxt), frame_p = Pp(nxt), frame_q = Qq(nxt);
            frame_restored = false;
            pre("ghost_t");
            const StagePtrs<T> A = stage_ptrs_on(W(nxt), Pp(nxt), Qq(nxt), (slot + 1) % 4, slot, head,
                                                 Wspare());
            const StageMaps sm = stage_maps_for(A);
            // a strip: the rows that read no halo row (the next step's
            // exchange has not happened); the edge rows run in that step
            if (strip()) inner_rows(2, spec_lo, spec_hi);
            else spec_lo = 0, spec_hi = d.ny;
            if (spec_hi > spec_lo) {
                ++step_launches;
                launch_stage(C, pn, A, 1, st, &sm, spec_lo, spec_hi - spec_lo);
            } else {
                spec_lo = spec_hi = 0;  // nothing queued: the next step runs every row
            }
            pre("stage");
            CU(cudaGetLastError());
            spec_pending = true;
            spec_commit = false;
        }
        CU(cudaEventSynchronize(ev_res));
        spec_h = hres->next;
        if (!spec) spec_h.valid = 0;
        for (int k = 0; k < 3 * ng; k++) g_pend[k] = double(h_gstage[k]);
        if (timing) {
            last_n = nev - 1;
            for (int k = 1; k < nev; k++) cudaEventElapsedTime(&last_ms[k - 1], ev[k - 1], ev[k]);
        }
        fill_result(r);
        pend_slot = slot;
        pending = true;
        bool stage_err = false;
        for (int k = 0; k < 5; k++) stage_err |= r->stage_bad[k] >= 0;
        if (stage_err) return BSQ_OK;  // the stage error is raised first (dispersion.py:92-98)
        if (d.solver == BSQ_CR && hres->cr_bad != 0xFFFFFFFFu) {
            return fail(BSQ_ERR_SINGULAR, cr_message(hres->cr_bad));
        }
        if (d.solver != BSQ_CR && singular)
            return fail(BSQ_ERR_SINGULAR, "singular tridiagonal system: zero pivot");
        return BSQ_OK;
    }

    // the ZeroDivisionError text of cyclic_reduction_batch (_kernels.py:419-446)
    static const char *cr_message(unsigned key) {
        static const char *msg[3] = {"singular tridiagonal system in reduction",
                                     "singular tridiagonal system: zero core determinant",
                                     "singular tridiagonal system in back substitution"};
        return msg[(key & 3u) < 3u ? (key & 3u) : 0];
    }

    CrPtrs<T> cr_ptrs(int phase, int nxt_state, bool scratch = false) {
        CrPtrs<T> K;
        K.ax = arr[A_AX];
        K.bx = arr[A_BX];
        K.cx = arr[A_CX];
        K.ay = arr[A_AYT];  // transposed, as by / cy
        K.by = arr[A_BY];
        K.cy = arr[A_CY];
        K.rx = arr[A_US];
        K.ry = arr[A_VS];
        K.gp = Pp(nxt_state);
        K.gq = Qq(nxt_state);
        K.outx = (phase == 2 && scratch) ? arr[A_P2] : Pp(nxt_state);
        K.outy = (phase == 2 && scratch) ? arr[A_Q2] : Qq(nxt_state);
        K.bad = &dres->cr_bad;
        K.key_base = phase == 1 ? 0u : 1u << 31;
        return K;
    }

    int array_layout(int which, size_t *off, int *pitch, int *xo, int *eb) {
        const T *ptr = nullptr;
        switch (which) {
        case BSQ_ARR_W: unframe(W(cur), Pp(cur), Qq(cur)); ptr = W(cur); break;
        case BSQ_ARR_P: unframe(W(cur), Pp(cur), Qq(cur)); ptr = Pp(cur); break;
        case BSQ_ARR_Q: unframe(W(cur), Pp(cur), Qq(cur)); ptr = Qq(cur); break;
        case BSQ_ARR_W_NEW: ptr = W(1 - cur); break;
        case BSQ_ARR_P_NEW: ptr = Pp(1 - cur); break;
        case BSQ_ARR_Q_NEW: ptr = Qq(1 - cur); break;
        case BSQ_ARR_DW_IN: ptr = dw_in; break;
        case BSQ_ARR_DW_OUT: ptr = dw_out; break;
        case BSQ_ARR_X_IN: ptr = x_in; break;
        case BSQ_ARR_X_OUT: ptr = x_out; break;
        case BSQ_ARR_Q2: ptr = arr[A_Q2]; break;
        case BSQ_ARR_RESULT:  // DevResult: max_rate (a double) first
            static_assert(offsetof(DevResult, max_rate) == 0, "max_rate leads DevResult");
            *off = (size_t)((const char *)dres - base);
            *pitch = 1;
            *xo = 0;
            *eb = (int)sizeof(double);
            return BSQ_OK;
        default: return fail(BSQ_ERR_BAD_ARG, "unknown array id");
        }
        *off = (size_t)((const char *)ptr - base);
        *pitch = L.pitch;
        *xo = L.xo;
        *eb = (int)sizeof(T);
        return BSQ_OK;
    }

    int commit() {
        if (!pending) return fail(BSQ_ERR_BAD_ARG, "no pending step to commit");
        cur = 1 - cur;
        const int old_wc = wc_;
        wc_ = wp_;
        wp_ = 3 - old_wc - wc_;  // the spare: where a queued next stage wrote w
        head = pend_slot;
        if (nlev < 3) nlev++;
        pending = false;
        if (spec_pending) spec_commit = true;
        g_com = g_pend;
        g_fresh = ng > 0;
        return BSQ_OK;
    }

    // -- observers ----------------------------------------------------------------------
    int set_gauges(const int *rows, const int *cols, int n) {
        if (n < 0 || (n > 0 && (!rows || !cols))) return fail(BSQ_ERR_BAD_ARG, "bad gauge list");
        std::vector<long long> off(n);
        for (int k = 0; k < n; k++) {
            if (rows[k] < GL || rows[k] >= d.ny + GL || cols[k] < GL || cols[k] >= d.nx + GL)
                return fail(BSQ_ERR_BAD_ARG, "gauge cell outside the interior");
            off[k] = L.at(rows[k], cols[k]);
        }
        CU(cudaStreamSynchronize(st));
        if (d_goff) cudaFree(d_goff);
        if (d_gval) cudaFree(d_gval);
        if (h_gstage) cudaFreeHost(h_gstage);
        d_goff = nullptr;
        d_gval = nullptr;
        h_gstage = nullptr;
        ng = n;
        g_pend.assign(3 * (size_t)n, 0.0);
        g_com.assign(3 * (size_t)n, 0.0);
        g_fresh = false;
        if (n == 0) return BSQ_OK;
        CU(cudaMalloc(&d_goff, sizeof(long long) * n));
        CU(cudaMalloc(&d_gval, sizeof(T) * 3 * n));
        CU(cudaMallocHost(&h_gstage, sizeof(T) * 3 * n));
        CU(cudaMemcpyAsync(d_goff, off.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
        return BSQ_OK;
    }

    // (w, P, Q) at every gauge cell of the committed state: the last step's
    // k_final sample when it is current, else one gather launch
    int gauge_values(double *out) {
        if (!ng) return BSQ_OK;
        if (!g_fresh) {
            launch_gather(W(cur), Pp(cur), Qq(cur), d_goff, ng, d_gval, st);
            CU(cudaGetLastError());
            CU(cudaMemcpyAsync(h_gstage, d_gval, sizeof(T) * 3 * ng, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            for (int k = 0; k < 3 * ng; k++) g_com[k] = double(h_gstage[k]);
            g_fresh = true;
        }
        std::memcpy(out, g_com.data(), sizeof(double) * 3 * ng);
        return BSQ_OK;
    }

    int max_tracker(int op) {
        switch (op) {
        case BSQ_MAX_OFF:
            CU(cudaStreamSynchronize(st));
            if (maxw) cudaFree(maxw);
            maxw = nullptr;
            fold_req = false;
            return BSQ_OK;
        case BSQ_MAX_RESET: {
            if (!maxw) CU(cudaMalloc(&maxw, sizeof(T) * (size_t)L.elems()));
            const T ninf = -std::numeric_limits<T>::infinity();
            std::vector<T> h((size_t)L.elems(), ninf);
            CU(cudaMemcpyAsync(maxw, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, st));
            CU(cudaStreamSynchronize(st));
            fold_req = false;
            return BSQ_OK;
        }
        case BSQ_MAX_FOLD:
            if (!maxw) return fail(BSQ_ERR_BAD_ARG, "max tracker not enabled");
            if (spec_pending) {  // the next stage is already queued: fold now
                launch_fold_max(C, W(cur), maxw, st);
                CU(cudaGetLastError());
                return BSQ_OK;
            }
            fold_req = true;  // the next stage kernel folds the committed state
            return BSQ_OK;
        case BSQ_MAX_FLUSH:
            if (!maxw) return fail(BSQ_ERR_BAD_ARG, "max tracker not enabled");
            if (fold_req) {
                launch_fold_max(C, W(cur), maxw, st);
                CU(cudaGetLastError());
                fold_req = false;
            }
            return BSQ_OK;
        default:
            return fail(BSQ_ERR_BAD_ARG, "unknown max-tracker op");
        }
    }

    int download_max(double *out) {
        if (!maxw) return fail(BSQ_ERR_BAD_ARG, "max tracker not enabled");
        int rc;
        if ((rc = max_tracker(BSQ_MAX_FLUSH)) || (rc = download_interior(out, maxw))) return rc;
        CU(cudaStreamSynchronize(st));
        return BSQ_OK;
    }

    // -- kernel-level seams ----------------------------------------------------------
    int stage_rates(double *outs[5]) {
        spec_pending = false;
        CU(cudaMemsetAsync(dres, 0xFF, sizeof(DevResult), st));
        const int slot = (head + 1) % 4;
        const StagePtrs<T> A = stage_ptrs(slot);
        const StageMaps sm = stage_maps_for(A);
        launch_stage(C, dparams, A, 0, st, &sm);
        fold_req = false;
        CU(cudaGetLastError());
        int rc;
        for (int k = 0; k < 5; k++)
            if ((rc = download_interior(outs[k], H(slot, k)))) return rc;
        CU(cudaStreamSynchronize(st));
        pending = false;
        return BSQ_OK;
    }

    int solve_momentum(const double *us, const double *vs, const double *pgw, const double *pge,
                       const double *qgs, const double *qgn, double *pout, double *qout) {
        if (d.solver != BSQ_CR && singular)
            return fail(BSQ_ERR_SINGULAR, "singular tridiagonal system: zero pivot");
        spec_pending = false;
        const int nxt = 1 - cur, nx = d.nx, ny = d.ny;
        int rc;
        if ((rc = upload_interior(arr[A_US], us)) || (rc = upload_interior(arr[A_VS], vs)))
            return rc;
        // ghost vectors into the scratch state's ghost column / row
        if ((rc = upload(Pp(nxt), L.at(GL, GL - 1), pgw, ny, 1, 1)) ||
            (rc = upload(Pp(nxt), L.at(GL, nx + GL), pge, ny, 1, 1)) ||
            (rc = upload(Qq(nxt), L.at(GL - 1, GL), qgs, 1, nx, nx)) ||
            (rc = upload(Qq(nxt), L.at(ny + GL, GL), qgn, 1, nx, nx)))
            return rc;
        if (d.solver == BSQ_CR) {
            CU(cudaMemsetAsync(&dres->cr_bad, 0xFF, sizeof(unsigned int), st));
            launch_cr(C, cr_ptrs(2, nxt, true), st);  // into P2 / Q2
        } else {
            launch_solve(C, solve_maps(2, nxt, true), solve_ptrs(nxt), piv_flags(), st);
        }
        CU(cudaGetLastError());
        if ((rc = download_interior(pout, arr[A_P2])) || (rc = download_interior(qout, arr[A_Q2])))
            return rc;
        CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        pending = false;
        if (d.solver == BSQ_CR && hres->cr_bad != 0xFFFFFFFFu)
            return fail(BSQ_ERR_SINGULAR, cr_message(hres->cr_bad));
        return BSQ_OK;
    }

    int speed_extrema(double *out3) {
        const int s = cur;
        launch_extrema(C, W(s), Pp(s), Qq(s), arr[A_BE], part, st);
        CU(cudaGetLastError());
        std::vector<Partial> h(nfinal);
        CU(cudaMemcpyAsync(h.data(), part, sizeof(Partial) * nfinal, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        double a = 0, b = 0, dd = 0;
        for (const Partial &pt : h) {
            a = pt.max_rate > a ? pt.max_rate : a;
            b = pt.max_speed > b ? pt.max_speed : b;
            dd = pt.max_depth > dd ? pt.max_depth : dd;
        }
        out3[0] = a;
        out3[1] = b;
        out3[2] = dd;
        return BSQ_OK;
    }

    int fill_ghosts(const double *eta, const double *flux) {
        spec_pending = false;
        frame_w = frame_p = frame_q = nullptr;
        DevParams &h = *hparams;
        for (int s = 0; s < 4; s++) {
            h.gw_t[s] = d.ws + eta[s];
            h.gf_t[s] = flux[s];
        }
        CU(cudaMemcpyAsync(dparams, hparams, sizeof(DevParams), cudaMemcpyHostToDevice, st));
        const int s = cur;
        launch_ghost(C, dparams, 0, W(s), Pp(s), Qq(s), W(s), Pp(s), Qq(s), st);
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(st));
        return BSQ_OK;
    }
};

struct bsq_ctx {
    int prec;
    Engine<double> *e64;
    Engine<float> *e32;
};

// run `expr` on the context's engine, whichever precision it is
#define ENGINE(c, expr)                                       \
    ((c)->prec == BSQ_FP64 ? ([&](Engine<double> *e) { return expr; })((c)->e64) \
                           : ([&](Engine<float> *e) { return expr; })((c)->e32))

extern "C" {

const char *bsq_last_error(void) { return g_err.c_str(); }

int bsq_device_count(int *count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(BSQ_ERR_NO_DEVICE, cudaGetErrorString(e));
    }
    *count = n;
    return BSQ_OK;
}

size_t bsq_workspace_bytes(const bsq_desc *desc) {
    if (check_desc(desc) != BSQ_OK) return 0;
    size_t offs[A_COUNT + S_COUNT];
    int fs;
    return desc->precision == BSQ_FP64 ? layout_bytes<double>(desc, offs, &fs)
                                       : layout_bytes<float>(desc, offs, &fs);
}

int bsq_create(const bsq_desc *desc, const bsq_static *f, void *workspace, size_t bytes,
               void *stream, bsq_ctx **out) {
    int rc = check_desc(desc);
    if (rc) return rc;
    if (!f || !out || !workspace) return fail(BSQ_ERR_BAD_ARG, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(BSQ_ERR_NO_DEVICE, "no CUDA device");
    bsq_ctx *c = new bsq_ctx{desc->precision, nullptr, nullptr};
    if (c->prec == BSQ_FP64) {
        c->e64 = new Engine<double>();
        rc = c->e64->create(desc, f, workspace, bytes, stream);
    } else {
        c->e32 = new Engine<float>();
        rc = c->e32->create(desc, f, workspace, bytes, stream);
    }
    if (rc) {
        std::string keep = g_err;
        bsq_destroy(c);
        return fail(rc, keep);
    }
    *out = c;
    return BSQ_OK;
}

int bsq_destroy(bsq_ctx *c) {
    if (!c) return BSQ_OK;
    delete c->e64;
    delete c->e32;
    delete c;
    return BSQ_OK;
}

int bsq_upload_state(bsq_ctx *c, const double *w, const double *p, const double *q) {
    if (!c || !w || !p || !q) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->upload_state(w, p, q));
}

int bsq_download_state(bsq_ctx *c, int which, double *w, double *p, double *q) {
    if (!c || !w || !p || !q) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->download_state(which, w, p, q));
}

int bsq_download_history(bsq_ctx *c, int level, int field, double *out) {
    if (!c || !out) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->download_history(level, field, out));
}

int bsq_step(bsq_ctx *c, const bsq_step_params *p, bsq_step_result *r) {
    NvtxRange nv("bsq_step");
    if (!c || !p || !r) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->step(p, r));
}

int bsq_commit(bsq_ctx *c) {
    if (!c) return fail(BSQ_ERR_BAD_ARG, "null ctx");
    return ENGINE(c, e->commit());
}

int bsq_phase(bsq_ctx *c, int phase, const bsq_step_params *p, bsq_step_result *r) {
    NvtxRange nv(phase_name(phase));
    if (!c || (phase == BSQ_PH_GHOST && !p) || (phase == BSQ_PH_FINAL && !r))
        return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->phase(phase, p, r));
}

int bsq_factor_tail(bsq_ctx *c, double *cw_north) {
    if (!c || !cw_north) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, ([&] {
        for (size_t k = 0; k < e->cw_tail.size(); k++) cw_north[k] = e->cw_tail[k];
        return (int)BSQ_OK;
    })());
}

int bsq_array_layout(bsq_ctx *c, int array, size_t *off, int *pitch, int *xo, int *eb) {
    if (!c || !off || !pitch || !xo || !eb) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->array_layout(array, off, pitch, xo, eb));
}

int bsq_pivot_flags(bsq_ctx *c, int *all_positive, int *singular) {
    if (!c || !all_positive || !singular) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, (*all_positive = e->pos_pivots ? 1 : 0, *singular = e->singular ? 1 : 0,
                      (int)BSQ_OK));
}

int bsq_stage_rates(bsq_ctx *c, double *e_, double *f, double *g, double *fs, double *gs) {
    if (!c || !e_ || !f || !g || !fs || !gs) return fail(BSQ_ERR_BAD_ARG, "null argument");
    double *outs[5] = {e_, f, g, fs, gs};
    return ENGINE(c, e->stage_rates(outs));
}

int bsq_solve_momentum(bsq_ctx *c, const double *us, const double *vs, const double *pgw,
                       const double *pge, const double *qgs, const double *qgn, double *pout,
                       double *qout) {
    if (!c || !us || !vs || !pgw || !pge || !qgs || !qgn || !pout || !qout)
        return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->solve_momentum(us, vs, pgw, pge, qgs, qgn, pout, qout));
}

int bsq_speed_extrema(bsq_ctx *c, double *out3) {
    if (!c || !out3) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->speed_extrema(out3));
}

int bsq_fill_ghosts(bsq_ctx *c, const double *eta, const double *flux) {
    if (!c || !eta || !flux) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->fill_ghosts(eta, flux));
}

int bsq_spike_coeffs(bsq_ctx *c, double *out) {
    if (!c || !out) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, ([&] {
        if (!spike_mode(&e->d)) return fail(BSQ_ERR_BAD_ARG, "context is not a spike-coupled strip");
        std::memcpy(out, e->sp_coef.data(), sizeof(double) * e->sp_coef.size());
        return (int)BSQ_OK;
    })());
}

int bsq_set_spike_table(bsq_ctx *c, const double *table, int nranks, int rank) {
    if (!c) return fail(BSQ_ERR_BAD_ARG, "null ctx");
    return ENGINE(c, e->set_spike_table(table, nranks, rank));
}

int bsq_spike_fix(bsq_ctx *c, int solve, const void *ybound) {
    if (!c) return fail(BSQ_ERR_BAD_ARG, "null ctx");
    return ENGINE(c, e->spike_fix(solve, ybound));
}

int bsq_set_gauges(bsq_ctx *c, const int *rows, const int *cols, int n) {
    if (!c) return fail(BSQ_ERR_BAD_ARG, "null ctx");
    return ENGINE(c, e->set_gauges(rows, cols, n));
}

int bsq_gauge_values(bsq_ctx *c, double *out) {
    if (!c || !out) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->gauge_values(out));
}

int bsq_max_tracker(bsq_ctx *c, int op) {
    if (!c) return fail(BSQ_ERR_BAD_ARG, "null ctx");
    return ENGINE(c, e->max_tracker(op));
}

int bsq_download_max(bsq_ctx *c, double *out) {
    if (!c || !out) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, e->download_max(out));
}

int bsq_set_timing(bsq_ctx *c, int enable) {
    if (!c) return fail(BSQ_ERR_BAD_ARG, "null ctx");
    return ENGINE(c, (e->timing = enable != 0, BSQ_OK));
}

int bsq_kernel_times(bsq_ctx *c, int max_n, float *ms, const char **names, int *n_out) {
    if (!c || !n_out) return fail(BSQ_ERR_BAD_ARG, "null argument");
    return ENGINE(c, ([&] {
        const int n = e->last_n < max_n ? e->last_n : max_n;
        for (int k = 0; k < n; k++) {
            if (ms) ms[k] = e->last_ms[k];
            if (names) names[k] = e->ev_name[k + 1];
        }
        *n_out = n;
        return (int)BSQ_OK;
    })());
}

int bsq_check_quotients(int op, const double *x, const double *d, long n, double *out) {
    if (!x || !d || !out || n < 0 || op < 0 || op > 7) return fail(BSQ_ERR_BAD_ARG, "bad arguments");
    if (n == 0) return BSQ_OK;
    return check_quotients(op, x, d, n, out) ? fail(BSQ_ERR_CUDA, "quotient check failed") : BSQ_OK;
}

int bsq_kernels_per_step(bsq_ctx *c) {
    if (!c) return 0;
    return ENGINE(c, (int)(e->step_launches ? e->step_launches : (e->d.cross_correction ? 7 : 5)));
}

}  // extern "C"
