/*
 * bsq.h -- C ABI of the B200-native adaptive-AB3 Boussinesq step.
 *
 * The library replaces the per-step compute of the reference solver's step
 * loop, boussim.stepper.Simulator._advance
 * (/root/reference/pkg/src/boussim/stepper.py:225-325), and the numba
 * kernels it calls (/root/reference/pkg/src/boussim/_kernels.py:20-451).
 * The host (paper_1909_04153_b200/stepper.py, a drop-in for
 * boussim.stepper.Simulator) keeps the controller and evaluates the handful
 * of fp64 scalars per step; everything per cell runs in sm_100a kernels.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Host arrays are float64, row-major,
 *     in the reference's padded layout: fields (ny+4) x (nx+4),
 *     bed_face_x (ny+4) x (nx+3), bed_face_y (ny+3) x (nx+4); interior
 *     arrays ny x nx (grid.py:1-20).
 *   - Device memory is owned by the caller: bsq_workspace_bytes() says how
 *     much, bsq_create() carves its buffers out of that one allocation (the
 *     Python host passes a torch-owned CUDA tensor).  Outside the workspace
 *     the library makes only these small or opt-in allocations of its own:
 *     the step parameter / result blocks and reduction partials, the SPIKE
 *     table (G x 4 x nx, bsq_set_spike_table), the gauge buffers
 *     (bsq_set_gauges) and the running-max field (one padded array, only
 *     after BSQ_MAX_RESET); all are freed by bsq_destroy.
 *   - All device work runs on the stream given to bsq_create (NULL: the
 *     library creates a non-blocking stream).  Calls that return host
 *     results synchronize that stream before returning.
 *   - Side order everywhere is north, south, east, west (boundary.py:25).
 *   - Every entry point returns a bsq_status; bsq_last_error() describes
 *     the most recent failure on the calling thread.
 */
#ifndef BSQ_H
#define BSQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BSQ_OK = 0,
    BSQ_ERR_BAD_ARG = 1,  /* -> ValueError */
    BSQ_ERR_CUDA = 2,     /* -> RuntimeError */
    BSQ_ERR_SINGULAR = 3, /* -> ZeroDivisionError (_kernels.py:369-376) */
    BSQ_ERR_NO_DEVICE = 4,
    BSQ_ERR_NCCL = 5
} bsq_status;

enum { BSQ_SIDE_NORTH = 0, BSQ_SIDE_SOUTH = 1, BSQ_SIDE_EAST = 2, BSQ_SIDE_WEST = 3 };
enum { BSQ_WALL = 0, BSQ_MAKER = 1, BSQ_SPONGE = 2 }; /* sponge ghosts mirror like a wall */
enum { BSQ_FP64 = 0, BSQ_FP32 = 1 };
enum { BSQ_THOMAS = 0, BSQ_CR = 1 };
/* How a y-strip's column solves couple to the neighbouring strips:
 *   BSQ_Y_PIPELINE  the global column's Thomas recurrence continues across
 *                   ranks (dw / x boundary vectors, phases *F then *B): bitwise
 *                   equal to one grid, but the sweeps serialize over ranks;
 *   BSQ_Y_SPIKE     every strip factors and solves its block alone, then a
 *                   partitioned (SPIKE) correction with precomputed spikes
 *                   couples the blocks through a 2(G-1)-unknown system per
 *                   column (bsq_spike_*): ranks run concurrently; equal to
 *                   the one-grid solution to rounding (~1e-15 relative). */
enum { BSQ_Y_PIPELINE = 0, BSQ_Y_SPIKE = 1 };

/* Grid, physics and scheme constants.  Derived constants are passed in,
 * computed by the host exactly as the reference's Python computes them
 * (e.g. dx2 = dx**2, bp13 = b_disp + 1.0/3.0), so the device never
 * re-derives a value that could round differently. */
typedef struct {
    int32_t nx, ny;            /* interior cells */
    int32_t precision;         /* BSQ_FP64 (bitwise parity) or BSQ_FP32 */
    int32_t solver;            /* BSQ_THOMAS */
    int32_t side_kind[4];      /* BSQ_WALL / BSQ_MAKER / BSQ_SPONGE per side */
    int32_t cross_correction;  /* re-solve with exact cross increment (stepper.py:262-280) */
    int32_t sponge_lo[4];      /* first band cell index (col for E/W, row for N/S) */
    int32_t sponge_len[4];     /* band length, 0 = none */
    double dx, dy, dx2, dy2;
    double g, b_disp, bp13, c_f, theta, h_eps, h_dry, ws;
    /* y-strip sharding (one context per rank; all zero for a whole grid).
     * The context holds interior rows [row0, row0+ny) of a global grid; an
     * internal side has no boundary policy: its two ghost rows are the
     * neighbour's interior rows, exchanged by the host between phases. */
    int32_t south_internal, north_internal;
    int32_t row0, ny_global;
    int32_t y_coupling;        /* BSQ_Y_PIPELINE or BSQ_Y_SPIKE (strips only) */
    /* 1: every quotient exact for numerators under 2^-960 as well (the line
     * solves and k_final divide with the IEEE division; see bsq_device.cuh
     * "Tiny numerators"); 0: Markstein quotients there, which can miss IEEE
     * by an ulp for such numerators (the stage is exact either way) */
    int32_t exact_tiny;
} bsq_desc;

/* Static fields (host pointers, reference layout; copied at create).  For a
 * strip, rows are the strip's interior plus 2 rows of the global array on
 * each side (bed_face_y: ny+3 rows starting at the strip's padded row 0). */
typedef struct {
    const double *bed_eff, *depth, *depth_dx, *depth_dy; /* (ny+4) x (nx+4) */
    const double *bed_face_x;                            /* (ny+4) x (nx+3) */
    const double *bed_face_y;                            /* (ny+3) x (nx+4) */
    const double *cw_south; /* strip with internal south: cw of the row below, per column (nx) */
} bsq_static;

/* Per-step host scalars (stepper.py:239-254; multistep.py:118-228;
 * boundary.py:190-199, 264-300). */
typedef struct {
    double t, dt;
    int32_t euler;            /* 1: bootstrap step (step_index < 3) */
    int32_t reserved;
    double wc, wp, wp2;       /* ab3_weights, ratio_policy="clamp" */
    double sc, sp, sp2;       /* increment_weights */
    double maker_eta_t[4], maker_flux_t[4]; /* maker_surface_flux at t     */
    double maker_eta_n[4], maker_flux_n[4]; /* maker_surface_flux at t+dt */
    const double *sponge_fac[4];            /* host, sponge_len[s] factors exp(-lambda dt) */
    /* Speculation (whole grids; 0 = off).  With the controller state below,
     * bsq_step queues the NEXT step's ghost and stage kernels right behind
     * this step's finalize, with dt and weights from a device copy of the
     * controller (stepper.py:304-312, multistep.py:31-228), so they overlap
     * the host's turn-around.  The next bsq_step uses them only if this step
     * was committed and its own dt, scheme, weights and maker values at t
     * equal the speculated ones bit for bit; otherwise it relaunches them. */
    int32_t spec;
    int32_t adaptive;          /* TimeController.mode == "adaptive" */
    int64_t step_index;        /* this step's index (before the increment) */
    double cfl_target, alpha, dt_min, dt_max, dt_init;
    double chain;              /* lazy-EMA chain before this step's update */
    double dt_fixed;           /* controller dt in "fixed" mode */
    double dt_prev;            /* the previous step's dt */
} bsq_step_params;

/* Per-step device reductions, returned to the host. */
typedef struct {
    double max_rate, max_speed, max_depth; /* speed_extrema of the new state (_kernels.py:324-353) */
    double max_dev;                        /* max |w - max(ws, bed_eff)|; NaN if w non-finite */
    double clamped;                        /* sum max(bed_eff - w_pred, 0) over the interior */
    int64_t stage_bad[5]; /* first row-major interior index of a non-finite e,f,g,fstar,gstar, or -1 */
    int64_t state_bad[3]; /* same for w, P, Q of the new state */
} bsq_step_result;

typedef struct bsq_ctx bsq_ctx;

/* -- lifecycle ---------------------------------------------------------- */
size_t bsq_workspace_bytes(const bsq_desc *desc);
int bsq_create(const bsq_desc *desc, const bsq_static *fields, void *workspace, size_t bytes,
               void *stream, bsq_ctx **out);
int bsq_destroy(bsq_ctx *ctx);
const char *bsq_last_error(void);
int bsq_device_count(int *count);

/* -- state / history I/O (host buffers, reference layout) ------------------ */
int bsq_upload_state(bsq_ctx *ctx, const double *w, const double *p, const double *q);
/* which: 0 = committed state, 1 = pending new state of the last bsq_step */
int bsq_download_state(bsq_ctx *ctx, int which, double *w, double *p, double *q);
/* level 0 = newest committed stage set; field 0..4 = e, f, g, fstar, gstar */
int bsq_download_history(bsq_ctx *ctx, int level, int field, double *out);

/* -- the step ----------------------------------------------------------- */
/* Runs stepper.py:233-305 on the device into pending buffers and returns
 * the reductions the host controller needs.  Nothing is committed. */
int bsq_step(bsq_ctx *ctx, const bsq_step_params *params, bsq_step_result *result);
/* Accept the pending step: state <- new state, history ring advances. */
int bsq_commit(bsq_ctx *ctx);

/* -- kernel-level seams (per-kernel parity tests) -------------------------- */
/* stage set E,F,G,F*,G* of the committed state as it is (no ghost fill) */
int bsq_stage_rates(bsq_ctx *ctx, double *e, double *f, double *g, double *fstar,
                    double *gstar);
/* implicit.solve_momentum (implicit.py:197-205) with the device solver */
int bsq_solve_momentum(bsq_ctx *ctx, const double *ustar, const double *vstar,
                       const double *pg_west, const double *pg_east, const double *qg_south,
                       const double *qg_north, double *p_out, double *q_out);
/* hydro.speed_extrema of the committed state: {max_rate, max_speed, max_depth} */
int bsq_speed_extrema(bsq_ctx *ctx, double *out3);
/* Boundaries.apply_ghosts on the committed state with maker values */
int bsq_fill_ghosts(bsq_ctx *ctx, const double *maker_eta, const double *maker_flux);

/* -- y-strip sharding: phased step and device layout ------------------------ */
/* A sharded step is bsq_step split at its exchange points; the host moves
 * halo rows and the y-line boundary vectors between phases on the context's
 * stream (NCCL send/recv, or device copies when ranks are emulated):
 *   BSQ_PH_GHOST   upload params, ghost strips at t (physical sides only)
 *     -> exchange 2 rows of w, P, Q with each neighbour
 *   BSQ_PH_STAGE   stage kernel + predicted-state ghosts at t+dt
 *   BSQ_PH_SOLVE1F x lines (complete) + y lines forward sweep
 *     (needs dw_in from the south rank; produces dw_out for the north rank)
 *   BSQ_PH_SOLVE1B y lines back substitution (x_in from the north rank;
 *     produces x_out for the south rank)
 *     -> exchange 1 row of the pending P, Q with each neighbour
 *   BSQ_PH_CORRECT cross-correction right-hand sides
 *   BSQ_PH_SOLVE2F, BSQ_PH_SOLVE2B  second solve, as above
 *   BSQ_PH_FINAL   finalize + reductions -> result (local; the host reduces
 *                  across ranks), synchronizes the stream
 * Speculation on strips (params->spec): call BSQ_PH_FINAL_LAUNCH first (the
 * finalize kernel alone), all-reduce (max) the first double of BSQ_ARR_RESULT
 * -- the strip's max CFL rate -- over the ranks on the context's stream, then
 * BSQ_PH_FINAL: the device controller turns the global rate into the next
 * step's parameters and queues its ghosts at t and the stage's inner rows
 * behind the result copy; the next step verifies them bit for bit (as
 * bsq_step does) and runs only the stage's edge rows. */
enum {
    BSQ_PH_GHOST = 0, BSQ_PH_STAGE = 1, BSQ_PH_SOLVE1F = 2, BSQ_PH_SOLVE1B = 3,
    BSQ_PH_CORRECT = 4, BSQ_PH_SOLVE2F = 5, BSQ_PH_SOLVE2B = 6, BSQ_PH_FINAL = 7,
    /* BSQ_PH_STAGE / BSQ_PH_CORRECT split around their halo exchange: the
     * INNER phase runs the rows that read no halo row (queue it while the
     * halo is in flight), the EDGE phase the rest once the halo is in place
     * (and, for the stage, the predicted-state ghosts) */
    BSQ_PH_STAGE_INNER = 8, BSQ_PH_STAGE_EDGE = 9, BSQ_PH_CORRECT_INNER = 10,
    BSQ_PH_CORRECT_EDGE = 11, BSQ_PH_FINAL_LAUNCH = 12
};
int bsq_phase(bsq_ctx *ctx, int phase, const bsq_step_params *params, bsq_step_result *result);
/* cw of this strip's last row, per column (nx): the next strip's cw_south */
int bsq_factor_tail(bsq_ctx *ctx, double *cw_north);
/* Device placement of a named array inside the workspace (byte offset from
 * the workspace base, row pitch and padded-column offset in elements, element
 * size).  The committed/pending state buffers swap every commit. */
enum {
    BSQ_ARR_W = 0, BSQ_ARR_P = 1, BSQ_ARR_Q = 2,                /* committed state */
    BSQ_ARR_W_NEW = 3, BSQ_ARR_P_NEW = 4, BSQ_ARR_Q_NEW = 5,    /* pending state */
    BSQ_ARR_DW_IN = 6, BSQ_ARR_DW_OUT = 7, BSQ_ARR_X_IN = 8, BSQ_ARR_X_OUT = 9, /* nx vectors */
    BSQ_ARR_Q2 = 10, /* scratch Q of the bsq_solve_momentum seam (the step itself solves
                        both times into BSQ_ARR_Q_NEW) */
    BSQ_ARR_RESULT = 11  /* the step's device result; its first double is the max CFL
                            rate (speculation on strips, see BSQ_PH_FINAL_LAUNCH) */
};
int bsq_array_layout(bsq_ctx *ctx, int array, size_t *byte_offset, int *pitch, int *xo,
                     int *elem_bytes);
/* whether every Thomas pivot of this context is > 0, and whether one is 0
 * (a sharded run raises if any rank is singular) */
int bsq_pivot_flags(bsq_ctx *ctx, int *all_positive, int *singular);

/* -- y-strips with BSQ_Y_SPIKE --------------------------------------------
 * Setup: every rank's 4 x nx spike boundary coefficients (bsq_spike_coeffs:
 * v[first], v[last], w[first], w[last] per column, where v / w solve the
 * strip's block against its south / north coupling column) are gathered into
 * a G x 4 x nx table, in rank order, and given to every rank.
 * Per solve (after BSQ_PH_SOLVE1F or BSQ_PH_SOLVE2F): gather every rank's
 * first and last solved row of Q (BSQ_ARR_Q_NEW: both solves land in the
 * pending Q) into a device array G x 2 x nx of the context's precision, then
 * bsq_spike_fix(solve, ...) solves the coupling system per column and
 * corrects Q in place on the library stream, on the rows where the strip's
 * spikes are not negligible (|v|, |w| >= 2^-64 at setup: the rows near the
 * internal sides; elsewhere the dropped terms are below 2^-64 of the
 * interface values).  A build with -DBSQ_SPIKE2_IN_FINAL=1 defers solve 2's
 * correction into BSQ_PH_FINAL (k_final applies it as it loads Q; the
 * pending Q is then the coupled solution only after BSQ_PH_FINAL, and a new
 * BSQ_PH_GHOST drops a correction that never reached it). */
int bsq_spike_coeffs(bsq_ctx *ctx, double *out);
int bsq_set_spike_table(bsq_ctx *ctx, const double *table, int nranks, int rank);
int bsq_spike_fix(bsq_ctx *ctx, int solve, const void *ybound_device);

/* -- per-step observers on device ----------------------------
 * Replace the host observers of the reference run loop (cli.py:635-649),
 * which read the whole host state after every step:
 *   GaugeRecorder.record (scenario.py:184-202) reads w, P, Q at a few cells;
 *   MaxSurfaceTracker.update (scenario.py:297-299) folds interior w into a
 *   running np.maximum. */
/* Gauge cells, padded (row, col) of this context's grid (gauge_cell,
 * scenario.py:155-161); n = 0 clears.  Every step's k_final then samples
 * them in its last CTA and they come back with the step result. */
int bsq_set_gauges(bsq_ctx *ctx, const int *rows, const int *cols, int n);
/* n x 3 doubles (w, P, Q) at the gauges, committed state */
int bsq_gauge_values(bsq_ctx *ctx, double *out);
/* Running max of interior w (padded-layout device buffer owned by the ctx):
 *   BSQ_MAX_RESET  allocate if needed and fill with -inf
 *   BSQ_MAX_FOLD   fold the committed state (np.maximum, NaN propagates);
 *                  deferred: the next step's stage kernel does it in its
 *                  pass over w, at no extra HBM pass
 *   BSQ_MAX_FLUSH  run a pending fold now
 *   BSQ_MAX_OFF    free */
enum { BSQ_MAX_OFF = 0, BSQ_MAX_RESET = 1, BSQ_MAX_FOLD = 2, BSQ_MAX_FLUSH = 3 };
int bsq_max_tracker(bsq_ctx *ctx, int op);
/* ny x nx running max (flushes a pending fold first) */
int bsq_download_max(bsq_ctx *ctx, double *out);

/* -- artifact formatting (host only, no device needed) --------
 * Append `nrows` rows of `ncols` doubles (row stride `stride` elements) to
 * the file at `path` as the reference's ESRI-ASCII data block
 * (grid.py:262-267: " ".join(f"{v:.17g}"), one line per row, the north row
 * first when `north_first`).  Returns the bytes written, or -1. */
long long bsq_append_rows(const char *path, const double *values, long nrows, long ncols,
                          long stride, int north_first);

/* Wavemaker forcing at time t (boundary.py:190-199): comps is
 * n rows of (amplitude, omega, k, phase); out = (eta, normal flux), summed in
 * component order with libm sin -- bitwise the reference's math.sin sums.
 * Host only. */
int bsq_maker_sums(const double *comps, int n, double t, double *out);

/* -- timing support ------------------------------------------------------ */
/* When enabled, bsq_step brackets each kernel with CUDA events on the
 * library stream; bsq_kernel_times returns the last step's per-kernel
 * device times (ms) and names, in launch order. */
int bsq_set_timing(bsq_ctx *ctx, int enable);
int bsq_kernel_times(bsq_ctx *ctx, int max_n, float *ms, const char **names, int *n_out);
/* number of kernels the last bsq_step launched (with speculation this
 * includes the next step's queued ghost + stage, and excludes its own) */
int bsq_kernels_per_step(bsq_ctx *ctx);

/* -- test seam: the device quotient helpers on host arrays ----------------
 * out[i] = x[i] / d[i] as computed by helper `op` (bsq_check.cu): 0
 * div_static, 1 div_pos, 2 div_rcp, 3 div_rcp_pos, 4 div_nonneg, 5
 * div_static_pos, 6 the IEEE division, 7 div_tiny_exact (numerators under
 * 2^-960).  fp64. */
int bsq_check_quotients(int op, const double *x, const double *d, long n, double *out);

#ifdef __cplusplus
}
#endif
#endif /* BSQ_H */
