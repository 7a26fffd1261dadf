// bsq_api.cu -- the C ABI (include/bsq.h): context, workspace carving, the
// static LU precompute, host<->device I/O and the per-step launch sequence.
//
// Host arithmetic here (coefficients, Thomas pivots) is plain IEEE binary64
// with contraction disabled (-ffp-contract=off), so it reproduces the
// reference's numpy/numba values bit for bit (implicit.py:84-119,
// _kernels.py:360-378).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/bsq.h"
#include "bsq_launch.h"

using namespace bsq;

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CU(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(BSQ_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

namespace {

constexpr int kMaxEv = 16;

enum Arr {
    A_W0, A_P0, A_Q0, A_W1, A_P1, A_Q1,
    A_BE, A_DEP, A_DDX, A_DDY, A_BFX, A_BFY,
    A_AX, A_DENX, A_RDENX, A_CWX, A_AY, A_DENY, A_RDENY, A_CWY,
    A_BU, A_BV, A_US, A_VS, A_P2, A_Q2,
    A_HIST0,  // 4 slots x 5 fields follow
    A_COUNT = A_HIST0 + 20
};

}  // namespace

struct bsq_ctx {
    bsq_desc d;
    Layout L;
    Consts<double> C;
    cudaStream_t st;
    bool own_stream;
    double *arr[A_COUNT];
    double *cx_last, *cy_last, *fac[4];
    DevParams *dparams;
    DevResult *dres;
    Partial *part;
    unsigned int *counter;
    DevParams *hparams;  // pinned
    DevResult *hres;     // pinned
    double *hfac;        // pinned, 4 x fac_stride
    int fac_stride;
    int nfinal;
    int cur;        // committed state buffer (0/1)
    int head;       // ring slot of the newest committed stage set
    int nlev;
    int pend_slot;
    bool pending;
    bool singular;
    bool pos_pivots;  // every Thomas pivot > 0: select-free division in the solves
    bool timing;
    cudaEvent_t ev[kMaxEv];
    const char *ev_name[kMaxEv];
    int nev;
    float last_ms[kMaxEv];
    int last_n;
    SolveMaps maps;                    // TMA descriptors (out slots patched per launch)
    CUtensorMap x_out[3], y_out[3];    // pending P/Q of state 0, state 1; P2/Q2

    double *W(int s) { return arr[s ? A_W1 : A_W0]; }
    double *Pp(int s) { return arr[s ? A_P1 : A_P0]; }
    double *Qq(int s) { return arr[s ? A_Q1 : A_Q0]; }
    double *H(int slot, int f) { return arr[A_HIST0 + slot * 5 + f]; }
};

extern "C" {
static int build_maps(bsq_ctx *c);
}

static Layout make_layout(const bsq_desc *d) {
    Layout L;
    L.nx = d->nx;
    L.ny = d->ny;
    const int line = 128 / (int)sizeof(double);  // elements per 128 B
    L.xo = line - GL;
    int need = L.xo + d->nx + 4;
    L.pitch = (need + line - 1) / line * line;
    return L;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t layout_bytes(const bsq_desc *d, size_t offs[], int *fac_stride) {
    Layout L = make_layout(d);
    size_t off = 0;
    size_t one = align256((size_t)L.elems() * sizeof(double));
    for (int k = 0; k < A_COUNT; k++) {
        offs[k] = off;
        off += one;
    }
    int fs = (d->nx > d->ny ? d->nx : d->ny);
    fs = (fs + 31) / 32 * 32;
    *fac_stride = fs;
    offs[A_COUNT + 0] = off;  // cx_last
    off += align256(sizeof(double) * d->ny);
    offs[A_COUNT + 1] = off;  // cy_last
    off += align256(sizeof(double) * d->nx);
    offs[A_COUNT + 2] = off;  // fac
    off += align256(sizeof(double) * 4 * fs);
    offs[A_COUNT + 3] = off;  // params
    off += align256(sizeof(DevParams));
    offs[A_COUNT + 4] = off;  // result
    off += align256(sizeof(DevResult));
    offs[A_COUNT + 5] = off;  // partials
    off += align256(sizeof(Partial) * (size_t)final_blocks(d->nx, d->ny));
    offs[A_COUNT + 6] = off;  // counter
    off += 256;
    return off;
}

static int check_desc(const bsq_desc *d) {
    if (!d) return fail(BSQ_ERR_BAD_ARG, "null descriptor");
    if (d->nx < 5 || d->ny < 5) return fail(BSQ_ERR_BAD_ARG, "grid needs at least 5x5 cells");
    if (d->precision != BSQ_FP64) return fail(BSQ_ERR_BAD_ARG, "only BSQ_FP64 is built");
    if (d->solver != BSQ_THOMAS) return fail(BSQ_ERR_BAD_ARG, "only the Thomas solver is built");
    if (!(d->dx > 0 && d->dy > 0)) return fail(BSQ_ERR_BAD_ARG, "cell sizes must be positive");
    for (int s = 0; s < 4; s++) {
        if (d->side_kind[s] < 0 || d->side_kind[s] > 2) return fail(BSQ_ERR_BAD_ARG, "bad side kind");
        int n = (s == SIDE_E || s == SIDE_W) ? d->nx : d->ny;
        if (d->sponge_len[s] < 0 || d->sponge_lo[s] < 0 || d->sponge_lo[s] + d->sponge_len[s] > n)
            return fail(BSQ_ERR_BAD_ARG, "sponge band outside the grid");
    }
    return BSQ_OK;
}

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
    size_t offs[A_COUNT + 8];
    int fs;
    return layout_bytes(desc, offs, &fs);
}

// host pitched staging helpers ------------------------------------------------

static int upload_padded(bsq_ctx *c, double *dst, const double *src, int rows, int cols) {
    CU(cudaMemcpy2DAsync(dst + c->L.xo, sizeof(double) * c->L.pitch, src, sizeof(double) * cols,
                         sizeof(double) * cols, rows, cudaMemcpyHostToDevice, c->st));
    return BSQ_OK;
}

static int download_padded(bsq_ctx *c, double *dst, const double *src, int rows, int cols) {
    CU(cudaMemcpy2DAsync(dst, sizeof(double) * cols, src + c->L.xo, sizeof(double) * c->L.pitch,
                         sizeof(double) * cols, rows, cudaMemcpyDeviceToHost, c->st));
    return BSQ_OK;
}

static int download_interior(bsq_ctx *c, double *dst, const double *src) {
    CU(cudaMemcpy2DAsync(dst, sizeof(double) * c->L.nx, src + c->L.at(GL, GL),
                         sizeof(double) * c->L.pitch, sizeof(double) * c->L.nx, c->L.ny,
                         cudaMemcpyDeviceToHost, c->st));
    return BSQ_OK;
}

static int upload_interior(bsq_ctx *c, double *dst, const double *src) {
    CU(cudaMemcpy2DAsync(dst + c->L.at(GL, GL), sizeof(double) * c->L.pitch, src,
                         sizeof(double) * c->L.nx, sizeof(double) * c->L.nx, c->L.ny,
                         cudaMemcpyHostToDevice, c->st));
    return BSQ_OK;
}

// implicit.py:84-90 -- _coefficients(d, slope, delta, bp13)
static void coefficients(double d, double slope, double delta2, double six_delta, double bp13,
                         double *a, double *b, double *cc) {
    double curv = bp13 * d * d / delta2;
    double drift = d * slope / six_delta;
    *a = drift - curv;
    *b = 1.0 + 2.0 * curv;
    *cc = -drift - curv;
}

// Pre-factor every x row and y column of the static implicit operator with
// thomas_batch's own recurrence (_kernels.py:368-378) and upload
// sub-diagonal, pivot, RN(1/pivot) and cw.
static int factor_lines(bsq_ctx *c, const bsq_static *f) {
    const int nx = c->d.nx, ny = c->d.ny, nxt = nx + 4;
    const Layout &L = c->L;
    const long E = L.elems();
    std::vector<double> ax(E, 0.0), denx(E, 1.0), rdenx(E, 1.0), cwx(E, 0.0);
    std::vector<double> ay(E, 0.0), deny(E, 1.0), rdeny(E, 1.0), cwy(E, 0.0);
    std::vector<double> cxl(ny), cyl(nx);
    const double six_dx = 6.0 * c->d.dx, six_dy = 6.0 * c->d.dy;
    bool singular = false, pos = true;
    for (int j = 0; j < ny; j++) {  // x rows
        double cw_prev = 0.0;
        for (int i = 0; i < nx; i++) {
            long h = (long)(j + GL) * nxt + i + GL;
            long o = L.at(j + GL, i + GL);
            double a, b, cc;
            coefficients(f->depth[h], f->depth_dx[h], c->d.dx2, six_dx, c->d.bp13, &a, &b, &cc);
            double den = i == 0 ? b : b - a * cw_prev;
            if (den == 0.0) singular = true;
            double cw = cc / den;
            ax[o] = a;
            denx[o] = den;
            rdenx[o] = -(1.0 / den);  // stored negated (div_static_pos)
            if (!(den > 0.0)) pos = false;
            cwx[o] = cw;
            cw_prev = cw;
            if (i == nx - 1) cxl[j] = cc;
        }
    }
    for (int i = 0; i < nx; i++) {  // y columns
        double cw_prev = 0.0;
        for (int j = 0; j < ny; j++) {
            long h = (long)(j + GL) * nxt + i + GL;
            long o = L.at(j + GL, i + GL);
            double a, b, cc;
            coefficients(f->depth[h], f->depth_dy[h], c->d.dy2, six_dy, c->d.bp13, &a, &b, &cc);
            double den = j == 0 ? b : b - a * cw_prev;
            if (den == 0.0) singular = true;
            double cw = cc / den;
            ay[o] = a;
            deny[o] = den;
            rdeny[o] = -(1.0 / den);
            if (!(den > 0.0)) pos = false;
            cwy[o] = cw;
            cw_prev = cw;
            if (j == ny - 1) cyl[i] = cc;
        }
    }
    c->singular = singular;
    c->pos_pivots = pos;
    const size_t B = sizeof(double) * E;
    CU(cudaMemcpyAsync(c->arr[A_AX], ax.data(), B, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->arr[A_DENX], denx.data(), B, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->arr[A_RDENX], rdenx.data(), B, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->arr[A_CWX], cwx.data(), B, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->arr[A_AY], ay.data(), B, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->arr[A_DENY], deny.data(), B, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->arr[A_RDENY], rdeny.data(), B, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->arr[A_CWY], cwy.data(), B, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->cx_last, cxl.data(), sizeof(double) * ny, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->cy_last, cyl.data(), sizeof(double) * nx, cudaMemcpyHostToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));  // host vectors go out of scope
    return BSQ_OK;
}

int bsq_create(const bsq_desc *desc, const bsq_static *f, void *workspace, size_t bytes,
               void *stream, bsq_ctx **out) {
    int rc = check_desc(desc);
    if (rc) return rc;
    if (!f || !out || !workspace) return fail(BSQ_ERR_BAD_ARG, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(BSQ_ERR_NO_DEVICE, "no CUDA device");
    size_t offs[A_COUNT + 8];
    int fs;
    size_t need = layout_bytes(desc, offs, &fs);
    if (bytes < need) return fail(BSQ_ERR_BAD_ARG, "workspace too small");
    if (((uintptr_t)workspace & 255) != 0) return fail(BSQ_ERR_BAD_ARG, "workspace not 256-B aligned");

    bsq_ctx *c = new bsq_ctx();
    memset(c, 0, sizeof(*c));
    c->d = *desc;
    c->L = make_layout(desc);
    c->fac_stride = fs;
    c->nfinal = final_blocks(desc->nx, desc->ny);
    char *base = (char *)workspace;
    for (int k = 0; k < A_COUNT; k++) c->arr[k] = (double *)(base + offs[k]);
    c->cx_last = (double *)(base + offs[A_COUNT + 0]);
    c->cy_last = (double *)(base + offs[A_COUNT + 1]);
    for (int s = 0; s < 4; s++) c->fac[s] = (double *)(base + offs[A_COUNT + 2]) + s * fs;
    c->dparams = (DevParams *)(base + offs[A_COUNT + 3]);
    c->dres = (DevResult *)(base + offs[A_COUNT + 4]);
    c->part = (Partial *)(base + offs[A_COUNT + 5]);
    c->counter = (unsigned int *)(base + offs[A_COUNT + 6]);
    if (stream) {
        c->st = (cudaStream_t)stream;
        c->own_stream = false;
    } else {
        if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) {
            delete c;
            return fail(BSQ_ERR_CUDA, "stream create failed");
        }
        c->own_stream = true;
    }
    if (cudaMallocHost(&c->hparams, sizeof(DevParams)) != cudaSuccess ||
        cudaMallocHost(&c->hres, sizeof(DevResult)) != cudaSuccess ||
        cudaMallocHost(&c->hfac, sizeof(double) * 4 * fs) != cudaSuccess) {
        bsq_destroy(c);
        return fail(BSQ_ERR_CUDA, "pinned staging allocation failed");
    }
    for (int k = 0; k < kMaxEv; k++) cudaEventCreate(&c->ev[k]);

    // constants, each derived as the reference derives it
    Consts<double> &C = c->C;
    C.L = c->L;
    C.g = desc->g;
    C.h_eps = desc->h_eps;
    C.theta = desc->theta;
    C.c_f = desc->c_f;
    C.b_disp = desc->b_disp;
    C.bp13 = desc->bp13;
    C.h_dry = desc->h_dry;
    C.ws = desc->ws;
    C.inv_dx = 1.0 / desc->dx;
    C.inv_dy = 1.0 / desc->dy;
    C.inv_dx2 = C.inv_dx * C.inv_dx;
    C.inv_dy2 = C.inv_dy * C.inv_dy;
    C.two_dx = 2.0 * desc->dx;
    C.two_dy = 2.0 * desc->dy;
    C.r_two_dx = 1.0 / C.two_dx;
    C.r_two_dy = 1.0 / C.two_dy;
    C.dx2 = desc->dx2;
    C.dy2 = desc->dy2;
    C.r_dx2 = 1.0 / desc->dx2;
    C.r_dy2 = 1.0 / desc->dy2;
    C.three = 3.0;
    C.r_three = 1.0 / 3.0;
    C.six = 6.0;
    C.r_six = 1.0 / 6.0;
    for (int s = 0; s < 4; s++) {
        C.side_kind[s] = desc->side_kind[s];
        C.sponge_lo[s] = desc->sponge_lo[s];
        C.sponge_len[s] = desc->sponge_len[s];
    }
    C.cross = desc->cross_correction;

    const int nx = desc->nx, ny = desc->ny;
    // zero everything once (ghost cells of scratch arrays stay defined)
    if (cudaMemsetAsync(workspace, 0, need, c->st) != cudaSuccess) {
        bsq_destroy(c);
        return fail(BSQ_ERR_CUDA, "workspace clear failed");
    }
    if ((rc = upload_padded(c, c->arr[A_BE], f->bed_eff, ny + 4, nx + 4)) ||
        (rc = upload_padded(c, c->arr[A_DEP], f->depth, ny + 4, nx + 4)) ||
        (rc = upload_padded(c, c->arr[A_DDX], f->depth_dx, ny + 4, nx + 4)) ||
        (rc = upload_padded(c, c->arr[A_DDY], f->depth_dy, ny + 4, nx + 4)) ||
        (rc = upload_padded(c, c->arr[A_BFX], f->bed_face_x, ny + 4, nx + 3)) ||
        (rc = upload_padded(c, c->arr[A_BFY], f->bed_face_y, ny + 3, nx + 4)) ||
        (rc = factor_lines(c, f)) || (rc = build_maps(c))) {
        std::string keep = g_err;
        bsq_destroy(c);
        return fail(rc, keep);
    }
    if (cudaMemsetAsync(c->counter, 0, sizeof(unsigned int), c->st) != cudaSuccess ||
        cudaStreamSynchronize(c->st) != cudaSuccess) {
        bsq_destroy(c);
        return fail(BSQ_ERR_CUDA, "setup failed");
    }
    c->cur = 0;
    c->head = 3;
    c->nlev = 0;
    *out = c;
    return BSQ_OK;
}

int bsq_destroy(bsq_ctx *c) {
    if (!c) return BSQ_OK;
    if (c->st) cudaStreamSynchronize(c->st);
    for (int k = 0; k < kMaxEv; k++)
        if (c->ev[k]) cudaEventDestroy(c->ev[k]);
    if (c->hparams) cudaFreeHost(c->hparams);
    if (c->hres) cudaFreeHost(c->hres);
    if (c->hfac) cudaFreeHost(c->hfac);
    if (c->own_stream && c->st) cudaStreamDestroy(c->st);
    delete c;
    return BSQ_OK;
}

int bsq_upload_state(bsq_ctx *c, const double *w, const double *p, const double *q) {
    if (!c || !w || !p || !q) return fail(BSQ_ERR_BAD_ARG, "null argument");
    int rc;
    int s = c->cur, ny = c->d.ny, nx = c->d.nx;
    if ((rc = upload_padded(c, c->W(s), w, ny + 4, nx + 4)) ||
        (rc = upload_padded(c, c->Pp(s), p, ny + 4, nx + 4)) ||
        (rc = upload_padded(c, c->Qq(s), q, ny + 4, nx + 4)))
        return rc;
    CU(cudaStreamSynchronize(c->st));
    c->pending = false;
    return BSQ_OK;
}

int bsq_download_state(bsq_ctx *c, int which, double *w, double *p, double *q) {
    if (!c || !w || !p || !q) return fail(BSQ_ERR_BAD_ARG, "null argument");
    if (which == 1 && !c->pending) return fail(BSQ_ERR_BAD_ARG, "no pending step");
    int s = which == 1 ? 1 - c->cur : c->cur, ny = c->d.ny, nx = c->d.nx, rc;
    if ((rc = download_padded(c, w, c->W(s), ny + 4, nx + 4)) ||
        (rc = download_padded(c, p, c->Pp(s), ny + 4, nx + 4)) ||
        (rc = download_padded(c, q, c->Qq(s), ny + 4, nx + 4)))
        return rc;
    CU(cudaStreamSynchronize(c->st));
    return BSQ_OK;
}

int bsq_download_history(bsq_ctx *c, int level, int field, double *out) {
    if (!c || !out || field < 0 || field > 4 || level < 0 || level >= c->nlev)
        return fail(BSQ_ERR_BAD_ARG, "bad history level/field");
    int slot = (c->head - level + 4) % 4, rc;
    if ((rc = download_interior(c, out, c->H(slot, field)))) return rc;
    CU(cudaStreamSynchronize(c->st));
    return BSQ_OK;
}

// ---------------------------------------------------------------------------

static void ev_mark(bsq_ctx *c, const char *name) {
    if (!c->timing || c->nev >= kMaxEv) return;
    c->ev_name[c->nev] = name;
    cudaEventRecord(c->ev[c->nev++], c->st);
}

static int stage_params(bsq_ctx *c, const bsq_step_params *p) {
    DevParams &h = *c->hparams;
    h.t = p->t;
    h.dt = p->dt;
    h.euler = p->euler;
    h.wc = p->wc;
    h.wp = p->wp;
    h.wp2 = p->wp2;
    h.sc = p->sc;
    h.sp = p->sp;
    h.sp2 = p->sp2;
    for (int s = 0; s < 4; s++) {
        h.gw_t[s] = c->d.ws + p->maker_eta_t[s];  // boundary.py:240 w_val = ws + eta
        h.gf_t[s] = p->maker_flux_t[s];
        h.gw_n[s] = c->d.ws + p->maker_eta_n[s];
        h.gf_n[s] = p->maker_flux_n[s];
    }
    CU(cudaMemcpyAsync(c->dparams, c->hparams, sizeof(DevParams), cudaMemcpyHostToDevice, c->st));
    bool any = false;
    for (int s = 0; s < 4; s++) {
        int n = c->d.sponge_len[s];
        if (c->d.side_kind[s] == BSQ_SPONGE && n > 0) {
            if (!p->sponge_fac[s]) return fail(BSQ_ERR_BAD_ARG, "missing sponge factors");
            memcpy(c->hfac + (size_t)s * c->fac_stride, p->sponge_fac[s], sizeof(double) * n);
            any = true;
        }
    }
    if (any)
        CU(cudaMemcpyAsync(c->fac[0], c->hfac, sizeof(double) * 4 * c->fac_stride,
                           cudaMemcpyHostToDevice, c->st));
    return BSQ_OK;
}

static StagePtrs<double> stage_ptrs(bsq_ctx *c, int slot) {
    StagePtrs<double> A;
    int s = c->cur;
    A.w = c->W(s);
    A.p = c->Pp(s);
    A.q = c->Qq(s);
    A.be = c->arr[A_BE];
    A.dep = c->arr[A_DEP];
    A.ddx = c->arr[A_DDX];
    A.ddy = c->arr[A_DDY];
    A.bfx = c->arr[A_BFX];
    A.bfy = c->arr[A_BFY];
    int s1 = c->head, s2 = (c->head + 3) % 4;
    for (int f = 0; f < 5; f++) {
        A.h0[f] = c->H(slot, f);
        A.h1[f] = c->H(s1, f);
        A.h2[f] = c->H(s2, f);
    }
    A.wn = c->W(1 - s);
    A.bu = c->arr[A_BU];
    A.bv = c->arr[A_BV];
    A.us = c->arr[A_US];
    A.vs = c->arr[A_VS];
    A.bad = c->dres->stage_bad;
    return A;
}

// phase 1 solves U*, V* into the pending state's P, Q; phase 2 solves the
// corrected right-hand sides (written over us / vs) into P2, Q2.
static SolvePtrs<double> solve_ptrs(bsq_ctx *c, int nxt_state) {
    SolvePtrs<double> S;
    S.gp = c->Pp(nxt_state);
    S.gq = c->Qq(nxt_state);
    S.cx_last = c->cx_last;
    S.cy_last = c->cy_last;
    return S;
}

static const SolveMaps &solve_maps(bsq_ctx *c, int phase, int nxt_state) {
    SolveMaps &M = c->maps;
    const int k = phase == 1 ? nxt_state : 2;  // out: pending P/Q, or P2/Q2
    M.x_out = c->x_out[k];
    M.y_out = c->y_out[k];
    return M;
}

// TMA descriptor of the interior region of one pitched array
static int make_map(CUtensorMap *m, double *base, const Layout &L, bool xdir) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return fail(BSQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint32_t ek = (cuuint32_t)solve_chunk_elems(sizeof(double));
    cuuint64_t dims[2] = {(cuuint64_t)L.nx, (cuuint64_t)L.ny};
    cuuint64_t strides[1] = {(cuuint64_t)L.pitch * sizeof(double)};
    cuuint32_t box[2] = {xdir ? ek : 32u, xdir ? 32u : ek};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base + L.at(GL, GL), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        xdir ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(BSQ_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return BSQ_OK;
}

static int build_maps(bsq_ctx *c) {
    const Layout &L = c->L;
    SolveMaps &M = c->maps;
    int rc;
    if ((rc = make_map(&M.x_rhs, c->arr[A_US], L, true)) ||
        (rc = make_map(&M.x_a, c->arr[A_AX], L, true)) ||
        (rc = make_map(&M.x_den, c->arr[A_DENX], L, true)) ||
        (rc = make_map(&M.x_rden, c->arr[A_RDENX], L, true)) ||
        (rc = make_map(&M.x_cw, c->arr[A_CWX], L, true)) ||
        (rc = make_map(&M.y_rhs, c->arr[A_VS], L, false)) ||
        (rc = make_map(&M.y_a, c->arr[A_AY], L, false)) ||
        (rc = make_map(&M.y_den, c->arr[A_DENY], L, false)) ||
        (rc = make_map(&M.y_rden, c->arr[A_RDENY], L, false)) ||
        (rc = make_map(&M.y_cw, c->arr[A_CWY], L, false)) ||
        (rc = make_map(&c->x_out[0], c->Pp(0), L, true)) ||
        (rc = make_map(&c->x_out[1], c->Pp(1), L, true)) ||
        (rc = make_map(&c->x_out[2], c->arr[A_P2], L, true)) ||
        (rc = make_map(&c->y_out[0], c->Qq(0), L, false)) ||
        (rc = make_map(&c->y_out[1], c->Qq(1), L, false)) ||
        (rc = make_map(&c->y_out[2], c->arr[A_Q2], L, false)))
        return rc;
    return BSQ_OK;
}

static CorrectPtrs<double> correct_ptrs(bsq_ctx *c, int slot, int nxt_state) {
    CorrectPtrs<double> K;
    K.bu = c->arr[A_BU];
    K.bv = c->arr[A_BV];
    K.fs = c->H(slot, 3);
    K.gs = c->H(slot, 4);
    K.p1 = c->Pp(nxt_state);
    K.q1 = c->Qq(nxt_state);
    K.dep = c->arr[A_DEP];
    K.ddx = c->arr[A_DDX];
    K.ddy = c->arr[A_DDY];
    K.us = c->arr[A_US];
    K.vs = c->arr[A_VS];
    return K;
}

static void fill_result(bsq_ctx *c, bsq_step_result *r) {
    const DevResult &h = *c->hres;
    r->max_rate = h.max_rate;
    r->max_speed = h.max_speed;
    r->max_depth = h.max_depth;
    r->max_dev = h.max_dev;
    r->clamped = h.clamped;
    for (int k = 0; k < 5; k++)
        r->stage_bad[k] = h.stage_bad[k] == ~0ull ? -1 : (int64_t)h.stage_bad[k];
    for (int k = 0; k < 3; k++)
        r->state_bad[k] = h.state_bad[k] == ~0ull ? -1 : (int64_t)h.state_bad[k];
}

int bsq_step(bsq_ctx *c, const bsq_step_params *p, bsq_step_result *r) {
    if (!c || !p || !r) return fail(BSQ_ERR_BAD_ARG, "null argument");
    int rc = stage_params(c, p);
    if (rc) return rc;
    CU(cudaMemsetAsync(c->dres, 0xFF, sizeof(DevResult), c->st));
    const int cur = c->cur, nxt = 1 - cur;
    const int slot = (c->head + 1) % 4;
    c->nev = 0;
    ev_mark(c, "start");
    launch_ghost(c->C, c->dparams, 0, c->W(cur), c->Pp(cur), c->Qq(cur), c->W(cur), c->Pp(cur),
                 c->Qq(cur), c->st);
    ev_mark(c, "ghost_t");
    launch_stage(c->C, c->dparams, stage_ptrs(c, slot), 1, c->st);
    ev_mark(c, "stage");
    launch_ghost(c->C, c->dparams, 1, c->W(nxt), c->Pp(cur), c->Qq(cur), c->W(nxt), c->Pp(nxt),
                 c->Qq(nxt), c->st);
    ev_mark(c, "ghost_n");
    launch_solve(c->C, solve_maps(c, 1, nxt), solve_ptrs(c, nxt), c->pos_pivots, c->st);
    ev_mark(c, "solve1");
    if (c->d.cross_correction) {
        launch_correct(c->C, correct_ptrs(c, slot, nxt), c->st);
        ev_mark(c, "correct");
        launch_solve(c->C, solve_maps(c, 2, nxt), solve_ptrs(c, nxt), c->pos_pivots, c->st);
        ev_mark(c, "solve2");
    }
    FinalPtrs<double> F;
    F.w = c->W(nxt);
    F.pin = c->d.cross_correction ? c->arr[A_P2] : c->Pp(nxt);
    F.qin = c->d.cross_correction ? c->arr[A_Q2] : c->Qq(nxt);
    F.pout = c->Pp(nxt);
    F.qout = c->Qq(nxt);
    F.be = c->arr[A_BE];
    for (int s = 0; s < 4; s++) F.fac[s] = c->fac[s];
    F.part = c->part;
    F.counter = c->counter;
    F.res = c->dres;
    launch_final(c->C, F, c->st);
    ev_mark(c, "final");
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(c->hres, c->dres, sizeof(DevResult), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    if (c->timing) {
        c->last_n = c->nev - 1;
        for (int k = 1; k < c->nev; k++) cudaEventElapsedTime(&c->last_ms[k - 1], c->ev[k - 1], c->ev[k]);
    }
    fill_result(c, r);
    c->pend_slot = slot;
    c->pending = true;
    bool stage_err = false;
    for (int k = 0; k < 5; k++) stage_err |= r->stage_bad[k] >= 0;
    if (c->singular && !stage_err)
        return fail(BSQ_ERR_SINGULAR, "singular tridiagonal system: zero pivot");
    return BSQ_OK;
}

int bsq_commit(bsq_ctx *c) {
    if (!c || !c->pending) return fail(BSQ_ERR_BAD_ARG, "no pending step to commit");
    c->cur = 1 - c->cur;
    c->head = c->pend_slot;
    if (c->nlev < 3) c->nlev++;
    c->pending = false;
    return BSQ_OK;
}

int bsq_stage_rates(bsq_ctx *c, double *e, double *f, double *g, double *fs, double *gs) {
    if (!c || !e || !f || !g || !fs || !gs) return fail(BSQ_ERR_BAD_ARG, "null argument");
    CU(cudaMemsetAsync(c->dres, 0xFF, sizeof(DevResult), c->st));
    int slot = (c->head + 1) % 4, rc;
    launch_stage(c->C, c->dparams, stage_ptrs(c, slot), 0, c->st);
    CU(cudaGetLastError());
    double *outs[5] = {e, f, g, fs, gs};
    for (int k = 0; k < 5; k++)
        if ((rc = download_interior(c, outs[k], c->H(slot, k)))) return rc;
    CU(cudaStreamSynchronize(c->st));
    c->pending = false;
    return BSQ_OK;
}

int bsq_solve_momentum(bsq_ctx *c, const double *us, const double *vs, const double *pgw,
                       const double *pge, const double *qgs, const double *qgn, double *pout,
                       double *qout) {
    if (!c || !us || !vs || !pgw || !pge || !qgs || !qgn || !pout || !qout)
        return fail(BSQ_ERR_BAD_ARG, "null argument");
    if (c->singular) return fail(BSQ_ERR_SINGULAR, "singular tridiagonal system: zero pivot");
    int rc;
    const int nxt = 1 - c->cur, nx = c->d.nx, ny = c->d.ny;
    const Layout &L = c->L;
    if ((rc = upload_interior(c, c->arr[A_US], us)) || (rc = upload_interior(c, c->arr[A_VS], vs)))
        return rc;
    // ghost vectors into the scratch state's ghost column / row
    CU(cudaMemcpy2DAsync(c->Pp(nxt) + L.at(GL, GL - 1), sizeof(double) * L.pitch, pgw,
                         sizeof(double), sizeof(double), ny, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpy2DAsync(c->Pp(nxt) + L.at(GL, nx + GL), sizeof(double) * L.pitch, pge,
                         sizeof(double), sizeof(double), ny, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->Qq(nxt) + L.at(GL - 1, GL), qgs, sizeof(double) * nx,
                       cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->Qq(nxt) + L.at(ny + GL, GL), qgn, sizeof(double) * nx,
                       cudaMemcpyHostToDevice, c->st));
    launch_solve(c->C, solve_maps(c, 2, nxt), solve_ptrs(c, nxt), c->pos_pivots, c->st);  // into P2 / Q2
    CU(cudaGetLastError());
    if ((rc = download_interior(c, pout, c->arr[A_P2])) ||
        (rc = download_interior(c, qout, c->arr[A_Q2])))
        return rc;
    CU(cudaStreamSynchronize(c->st));
    c->pending = false;
    return BSQ_OK;
}

int bsq_speed_extrema(bsq_ctx *c, double *out3) {
    if (!c || !out3) return fail(BSQ_ERR_BAD_ARG, "null argument");
    int s = c->cur;
    launch_extrema(c->C, c->W(s), c->Pp(s), c->Qq(s), c->arr[A_BE], c->part, c->st);
    CU(cudaGetLastError());
    std::vector<Partial> h(c->nfinal);
    CU(cudaMemcpyAsync(h.data(), c->part, sizeof(Partial) * c->nfinal, cudaMemcpyDeviceToHost,
                       c->st));
    CU(cudaStreamSynchronize(c->st));
    double a = 0, b = 0, d = 0;
    for (const Partial &pt : h) {
        a = pt.max_rate > a ? pt.max_rate : a;
        b = pt.max_speed > b ? pt.max_speed : b;
        d = pt.max_depth > d ? pt.max_depth : d;
    }
    out3[0] = a;
    out3[1] = b;
    out3[2] = d;
    return BSQ_OK;
}

int bsq_fill_ghosts(bsq_ctx *c, const double *eta, const double *flux) {
    if (!c || !eta || !flux) return fail(BSQ_ERR_BAD_ARG, "null argument");
    DevParams &h = *c->hparams;
    for (int s = 0; s < 4; s++) {
        h.gw_t[s] = c->d.ws + eta[s];
        h.gf_t[s] = flux[s];
    }
    CU(cudaMemcpyAsync(c->dparams, c->hparams, sizeof(DevParams), cudaMemcpyHostToDevice, c->st));
    int s = c->cur;
    launch_ghost(c->C, c->dparams, 0, c->W(s), c->Pp(s), c->Qq(s), c->W(s), c->Pp(s), c->Qq(s),
                 c->st);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(c->st));
    return BSQ_OK;
}

int bsq_set_timing(bsq_ctx *c, int enable) {
    if (!c) return fail(BSQ_ERR_BAD_ARG, "null ctx");
    c->timing = enable != 0;
    return BSQ_OK;
}

int bsq_kernel_times(bsq_ctx *c, int max_n, float *ms, const char **names, int *n_out) {
    if (!c || !n_out) return fail(BSQ_ERR_BAD_ARG, "null argument");
    int n = c->last_n < max_n ? c->last_n : max_n;
    for (int k = 0; k < n; k++) {
        if (ms) ms[k] = c->last_ms[k];
        if (names) names[k] = c->ev_name[k + 1];
    }
    *n_out = n;
    return BSQ_OK;
}

int bsq_kernels_per_step(bsq_ctx *c) {
    if (!c) return 0;
    return c->d.cross_correction ? 7 : 5;
}

}  // extern "C"
