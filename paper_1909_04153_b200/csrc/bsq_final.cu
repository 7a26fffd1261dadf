// bsq_final.cu -- the post-solve pass of a step and the CFL reductions.
//
// Per interior cell, in the reference's order (stepper.py:281-305):
// clamp w >= bed_eff with the clamped-volume tally, install the solved
// momenta, film cutoff, sponge bands N, S, E, W (boundary.py:264-300), then
// the blow-up deviation, non-finite scan and speed extrema
// (_kernels.py:324-353) of the final state.  Reductions: registers -> warp
// shuffles -> CTA -> per-CTA partials -> the last CTA to finish reduces the
// partials in a fixed order, so results are run-to-run deterministic (max is
// order free; the clamped-volume sum has a fixed association).
#include <cmath>
#include <cstdint>

#include "bsq_device.cuh"
#include "bsq_launch.h"

namespace bsq {

__device__ __forceinline__ unsigned long long bits(double v) {
    return (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ unsigned long long bits(float v) { return __float_as_uint(v); }
__device__ __forceinline__ bool bits_nonzero(double v) { return bits(v) != 0ull; }

#ifndef BSQ_FINAL_F32_MULQ
#define BSQ_FINAL_F32_MULQ 1
#endif
#ifndef BSQ_FINAL_FR
#define BSQ_FINAL_FR 8
#endif
#ifndef BSQ_FINAL_FG
#define BSQ_FINAL_FG 4
#endif
constexpr int FX = 32, FY = 8, FR = BSQ_FINAL_FR;  // block 32 x 8 threads, FR rows per thread
constexpr int FG = BSQ_FINAL_FG;  // rows loaded per batch (all loads first, then the work)
constexpr int FT = FX * FY, FWARPS = FT / 32;
#ifndef BSQ_FINAL_MINB
#define BSQ_FINAL_MINB 3  // 80 registers, no spills (4: 64 with spills, 0.148 vs 0.133 ms)
#endif
#ifndef BSQ_FINAL_MINB32
#define BSQ_FINAL_MINB32 4  // fp32: 63 registers without spills (0.0982 -> 0.0971 ms)
#endif
template <class T>
constexpr int final_minb() { return sizeof(T) == 8 ? BSQ_FINAL_MINB : BSQ_FINAL_MINB32; }

struct Red {
    double rate, speed, depth, dev, clamp;
    int nan;
};

// per-thread accumulators in the kernel's precision: max is exact and the
// conversion to double monotone, so the maxima equal the fp64-accumulated ones.
// The clamped-volume tally too (fp64: the same double sum; fp32: a float sum
// over the thread's cells, converted once -- a per-cell double add and
// conversion ran on the fp64 pipe)
template <class T>
struct Acc {
    T rate, speed, depth, dev;
    T clamp;
    int nan;
};

// Warp max of non-negative, non-NaN values (the accumulators only ever take a
// value strictly greater than +0 or keep +0): their bit patterns order like
// the values, so redux.sync on the words does it -- high words first, then
// the low words of the lanes holding the top high word.
__device__ __forceinline__ double warp_max_nonneg(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    return __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
}
__device__ __forceinline__ float warp_max_nonneg(float v) {
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(v)));
}

// fixed-shape xor tree for the clamped-volume sum; skipped (+0) when the
// whole warp has nothing to add
__device__ __forceinline__ double warp_sum(double v) {
    if (!__any_sync(0xffffffffu, bits_nonzero(v))) return v;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

__device__ __forceinline__ void red_warp(Red &r) {
    r.rate = warp_max_nonneg(r.rate);
    r.speed = warp_max_nonneg(r.speed);
    r.depth = warp_max_nonneg(r.depth);
    r.dev = warp_max_nonneg(r.dev);
    r.clamp = warp_sum(r.clamp);
    r.nan = __any_sync(0xffffffffu, r.nan);
}

template <class T>
__device__ __forceinline__ Red red_warp(const Acc<T> &a) {
    Red r;
    r.rate = double(warp_max_nonneg(a.rate));
    r.speed = double(warp_max_nonneg(a.speed));
    r.depth = double(warp_max_nonneg(a.depth));
    r.dev = double(warp_max_nonneg(a.dev));
    r.clamp = warp_sum(double(a.clamp));
    r.nan = __any_sync(0xffffffffu, a.nan);
    return r;
}

// CTA-wide reduction of warp-reduced values; result valid in thread 0
__device__ __forceinline__ Red red_block_warped(Red r) {
    __shared__ Red s[FWARPS];
    const int tid = threadIdx.y * FX + threadIdx.x;
    __syncthreads();  // protect s against a previous use
    if ((tid & 31) == 0) s[tid >> 5] = r;
    __syncthreads();
    if (tid == 0) {
        Red t = s[0];
        for (int k = 1; k < FWARPS; k++) {
            t.rate = fmax(t.rate, s[k].rate);
            t.speed = fmax(t.speed, s[k].speed);
            t.depth = fmax(t.depth, s[k].depth);
            t.dev = fmax(t.dev, s[k].dev);
            t.clamp = t.clamp + s[k].clamp;
            t.nan |= s[k].nan;
        }
        r = t;
    }
    return r;
}

__device__ __forceinline__ Red red_block(Red r) {
    red_warp(r);
    return red_block_warped(r);
}

// speed_extrema contribution of one cell (_kernels.py:337-352); the serial
// scan's `if x > max` skips NaN, hence the !(x > 0) guards.
template <bool FAST = false, bool EXT = false, class T>
__device__ __forceinline__ void extrema_cell(const Consts<T> &C, T w, T p, T q, T be, Acc<T> &r) {
    // a dry, still cell (h = 0, P = Q = 0) contributes rate = speed = depth = 0,
    // which never raises a maximum: skip it (whole dry warps branch over)
    if (!(w - be > T(0)) && p == T(0) && q == T(0)) return;
    T h = w - be;
    h = floor0(h);
    const T hstar = floor_eps(h, C.h_eps);
    const T c = sqrt(C.g * h);
    // both quotients correctly rounded via one reciprocal (branch-free when
    // h_eps is in rcp_rn_inrange's range: bsq_device.cuh flux_fast_rcp_ok)
    const T nrh = -(FAST ? rcp_depth(hstar) : rcp_rn(hstar));
    T su, sv;
    if constexpr (sizeof(T) == 4 && BSQ_FINAL_F32_MULQ) {
        // fp32 (a tolerance contract): the speeds only feed the CFL maxima,
        // so the quotients are products with the reciprocal
        su = fabs(p) * -nrh + c;
        sv = fabs(q) * -nrh + c;
    } else {
        su = div_nonneg(fabs(p), hstar, nrh) + c;
        sv = div_nonneg(fabs(q), hstar, nrh) + c;
    }
    if (EXT && (tiny_nz(p, TINY_NUM) | tiny_nz(q, TINY_NUM))) {  // exact_tiny: under Markstein's range
        const T rh = -nrh;
        if (tiny_nz(p, TINY_NUM)) su = div_tiny_exact(fabs(p), hstar, rh) + c;
        if (tiny_nz(q, TINY_NUM)) sv = div_tiny_exact(fabs(q), hstar, rh) + c;
    }
    const T rate = nb_max(su * C.inv_dx, sv * C.inv_dy);
    const T speed = nb_max(su, sv);
    if (rate > r.rate) r.rate = rate;
    if (speed > r.speed) r.speed = speed;
    if (h > r.depth) r.depth = h;
}

__device__ __forceinline__ Partial to_partial(const Red &r) {
    Partial pt;
    pt.max_rate = r.rate;
    pt.max_speed = r.speed;
    pt.max_depth = r.depth;
    pt.max_dev = r.dev;
    pt.clamped = r.clamp;
    pt.dev_nan = r.nan;
    pt.pad_ = 0;
    return pt;
}

// fold n partials written by other CTAs: thread t takes t, t+FT, ... in
// order, then the block tree; result valid in thread 0
__device__ __forceinline__ Red fold_partials(const Partial *p, int n) {
    const int tid = threadIdx.y * FX + threadIdx.x;
    Red a{0, 0, 0, 0, 0, 0};
    for (int k = tid; k < n; k += FT) {
        const Partial *pp = p + k;
        a.rate = fmax(a.rate, __ldcg(&pp->max_rate));
        a.speed = fmax(a.speed, __ldcg(&pp->max_speed));
        a.depth = fmax(a.depth, __ldcg(&pp->max_depth));
        a.dev = fmax(a.dev, __ldcg(&pp->max_dev));
        a.clamp = a.clamp + __ldcg(&pp->clamped);
        a.nan |= __ldcg(&pp->dev_nan);
    }
    return red_block(a);
}

// Python's min / max of two floats: the first argument unless the second is
// strictly smaller / larger
__device__ __forceinline__ double py_min(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double py_max(double a, double b) { return b > a ? b : a; }

// The next step's scheme parameters from this step's max CFL rate: the host
// controller (stepper.py cfl_candidate / lazy_ema / dt update) and the
// clamped AB3 / VFD weights (multistep.py StepTriple.validated, ab3_weights,
// vfd_weights, increment_weights), same operations in the same order.  The
// host recomputes all of it and only uses the speculated stage if every
// value agrees bit for bit.
static __device__ void spec_next(const DevParams &P, double max_rate, DevParams &N, SpecNext &o) {
    double dt;
    if (P.adaptive) {
        const double cand = max_rate <= 0.0
                                ? P.dt_max
                                : py_min(py_max(P.cfl_target / max_rate, P.dt_min), P.dt_max);
        const double chain = cand <= P.chain ? cand : P.alpha * cand + (1.0 - P.alpha) * P.chain;
        dt = P.step_index + 1 >= 3 ? chain : P.dt_init;
    } else {
        dt = P.dt_fixed;
    }
    const int euler = P.step_index + 1 < 3;
    double w0 = 0, w1 = 0, w2 = 0, s0 = 0, s1 = 0, s2 = 0;
    if (!euler) {
        double a = P.dt, b = P.dt_prev;  // StepTriple(dt, dt_prev, dt_prev2), clamped
        const double r1 = dt / a, r2 = a / b;
        const double lo = 0.1 * (1.0 - 1e-12), hi = 10.0 * (1.0 + 1e-12);
        if (!(lo <= r1 && r1 <= hi && lo <= r2 && r2 <= hi)) {
            a = py_min(py_max(a, dt / 10.0), dt / 0.1);
            b = py_min(py_max(b, a / 10.0), a / 0.1);
        }
        if (dt == a && a == b) {
            w0 = (23.0 / 12.0) * dt;
            w1 = (-16.0 / 12.0) * dt;
            w2 = (5.0 / 12.0) * dt;
            s0 = 2.0;
            s1 = -3.0;
            s2 = 1.0;
        } else {
            w0 = (dt / 6.0) * (dt * (2.0 * dt + 6.0 * a + 3.0 * b) / (a * (a + b)) + 6.0);
            w1 = -(dt / 6.0) * (dt * (2.0 * dt + 3.0 * a + 3.0 * b) / (a * b));
            w2 = (dt / 6.0) * (dt * (2.0 * dt + 3.0 * a) / (b * (a + b)));
            double n0, n1, n2, m0, m1, m2, o0, o1, o2;
            if (a == b) {
                const double h = a;
                n0 = 1.5 / h, n1 = -2.0 / h, n2 = 0.5 / h;
                m0 = 0.5 / h, m1 = 0.0, m2 = -0.5 / h;
                o0 = -0.5 / h, o1 = 2.0 / h, o2 = -1.5 / h;
            } else {
                n0 = (2.0 * a + b) / (a * (a + b)), n1 = -(a + b) / (a * b), n2 = a / (b * (a + b));
                m0 = b / (a * (a + b)), m1 = (a - b) / (a * b), m2 = -a / (b * (a + b));
                o0 = -b / (a * (a + b)), o1 = (a + b) / (a * b), o2 = -(a + 2.0 * b) / (b * (a + b));
            }
            s0 = w0 * n0 + w1 * m0 + w2 * o0;
            s1 = w0 * n1 + w1 * m1 + w2 * o1;
            s2 = w0 * n2 + w1 * m2 + w2 * o2;
        }
    }
    N.t = P.t + P.dt;
    N.dt = dt;
    N.euler = euler;
    N.wc = w0, N.wp = w1, N.wp2 = w2, N.sc = s0, N.sp = s1, N.sp2 = s2;
    N.f_dt = (float)dt, N.f_wc = (float)w0, N.f_wp = (float)w1, N.f_wp2 = (float)w2;
    N.f_sc = (float)s0, N.f_sp = (float)s1, N.f_sp2 = (float)s2;
    for (int s = 0; s < 4; s++) {  // the next step's ghosts at t are this step's at t + dt
        N.gw_t[s] = P.gw_n[s];
        N.gf_t[s] = P.gf_n[s];
    }
    N.spec = 0;
    o.dt = dt;
    o.euler = euler;
    o.valid = 1;
    o.wc = w0, o.wp = w1, o.wp2 = w2, o.sc = s0, o.sp = s1, o.sp2 = s2;
}


// Persistent: a grid of (resident CTAs) walks the 32 x 64-cell tiles in a
// fixed grid-stride order and reduces once at the end (one block reduction,
// partial and counter per CTA instead of per tile: the per-tile barrier and
// atomic were the kernel's top stall after the loads).
template <class T, bool SPIKE, bool FAST, bool EXT>
__global__ void __launch_bounds__(FT, final_minb<T>()) k_final(Consts<T> C, FinalPtrs<T> F,
                                                              int tiles_x, int ntiles) {
    __shared__ bool am_last;
    pdl_trigger();
    pdl_wait();
    const Layout L = C.L;
    const int nx = L.nx, ny = L.ny;
    const bool sponges = (C.sponge_len[0] | C.sponge_len[1] | C.sponge_len[2] | C.sponge_len[3]) != 0;
    const long rstep = (long)FY * L.pitch;
    Acc<T> r{T(0), T(0), T(0), T(0), T(0), 0};
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int bx = tile % tiles_x, by = tile / tiles_x;
    const int I = GL + bx * FX + threadIdx.x;
    const int J0 = GL + by * FR * FY + threadIdx.y;
    const long o0 = L.at(J0, I);
    const bool iin = I < nx + GL;
#pragma unroll
    for (int k0 = 0; k0 < FR; k0 += FG) {
        // all loads of the batch first (pure stream), then the work
        T vbe[FG], vw[FG], vp[FG], vq[FG];
#pragma unroll
        for (int k = 0; k < FG; k++) {
            const bool in = iin && J0 + (k0 + k) * FY < ny + GL;
            const long o = in ? o0 + (k0 + k) * rstep : L.at(GL, GL);
            vbe[k] = F.be[o];
            vw[k] = F.w[o];
            vp[k] = F.pin[o];
            vq[k] = F.qin[o];
        }
        if (SPIKE) {  // the strip's coupling correction of the second solve (k_spike_fix)
#pragma unroll
            for (int k = 0; k < FG; k++) {
                const bool in = iin && J0 + (k0 + k) * FY < ny + GL;
                const long o = in ? o0 + (k0 + k) * rstep : L.at(GL, GL);
                const int ic = iin ? I - GL : 0;  // no read past the 2*nx bound rows
                const int jr = J0 + (k0 + k) * FY - GL;  // strip row (the spikes' cut-offs)
                T r = vq[k];
                if (F.sp_south && jr < F.sp_jv) r = r - F.spv[o] * F.spbt[ic];
                if (F.sp_north && jr >= F.sp_jw) r = r - F.spw[o] * F.spbt[nx + ic];
                vq[k] = r;
            }
        }
#pragma unroll
        for (int k = 0; k < FG; k++) {
            const int J = J0 + (k0 + k) * FY;
            if (!iin || J >= ny + GL) continue;
            const long o = o0 + (k0 + k) * rstep;
            const T be = vbe[k];
            T w = vw[k];
            T p = vp[k], q = vq[k];
            // clamp and volume tally (stepper.py:281-285); np.maximum keeps NaN
            const T def = be - w;
            if (def > T(0) || def != def) r.clamp = r.clamp + def;
            w = (w >= be || w != w) ? w : be;
            // film cutoff (stepper.py:288-292)
            if (C.h_dry > T(0) && (w - be) < C.h_dry) {
                p = T(0);
                q = T(0);
            }
            const T rest = C.ws > be ? C.ws : be;  // np.maximum(ws, bed_eff)
#pragma unroll
            for (int side = 0; side < 4 && sponges; side++) {  // sponge bands, order N, S, E, W
                // band in local coordinates (a strip may hold part of a N/S band)
                if (C.sponge_len[side] == 0) continue;
                const int kk = (side == SIDE_E || side == SIDE_W) ? (I - GL) - C.sponge_lo[side]
                                                                  : (J - GL) - C.sponge_lo[side];
                if (kk < 0 || kk >= C.sponge_len[side]) continue;
                const T fac = F.fac[side][kk];
                w = rest + (w - rest) * fac;
                p = p * fac;
                q = q * fac;
            }
            // the solves left P, Q in place and w* is already the pending w: store
            // only what the clamp, film cutoff or sponge changed (bit patterns
            // compared, so a zero's sign is kept exactly)
            if (bits(w) != bits(vw[k])) F.w[o] = w;
            if (F.pout != F.pin || bits(p) != bits(vp[k])) F.pout[o] = p;
            if (SPIKE || F.qout != F.qin || bits(q) != bits(vq[k])) F.qout[o] = q;
            T dv = w - rest;  // blow-up deviation (stepper.py:295)
            dv = dv < T(0) ? -dv : dv;
            if (dv != dv) r.nan = 1;
            else if (dv > r.dev) r.dev = dv;
            if (!(isfinite(w) & isfinite(p) & isfinite(q))) {
                const unsigned long long lin = (unsigned long long)(J - GL) * nx + (I - GL);
                if (!isfinite(w)) atomicMin(&F.res->state_bad[0], lin);
                if (!isfinite(p)) atomicMin(&F.res->state_bad[1], lin);
                if (!isfinite(q)) atomicMin(&F.res->state_bad[2], lin);
            }
            extrema_cell<FAST, EXT>(C, w, p, q, be, r);
        }
    }
    }  // tiles
    Red rr = red_block_warped(red_warp(r));
    const int tid = threadIdx.y * FX + threadIdx.x;
    // Deterministic fold: every CTA writes its partial; the last one to finish
    // folds them in CTA order (one round of parallel L2 loads -- ld.cg: written
    // by other CTAs before their fence + counter increment -- and a block
    // reduction).  The grid-stride tile order is fixed for a given grid, so
    // the clamped-volume sum is the same every run.
    if (tid == 0) {
        F.part[blockIdx.x] = to_partial(rr);
        __threadfence();
        const unsigned int prev = atomicAdd(&F.counter[0], 1u);
        am_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    const Red a = fold_partials(F.part, gridDim.x);
    // gauge cells of the new state (scenario.py:184-202 reads w, P, Q there);
    // other CTAs wrote them: read through L2
    for (int g = tid; g < F.ng; g += FT) {
        const long long o = F.goff[g];
        F.gval[3 * g] = __ldcg(F.w + o);
        F.gval[3 * g + 1] = __ldcg(F.pout + o);
        F.gval[3 * g + 2] = __ldcg(F.qout + o);
    }
    if (tid == 0) {
        F.res->max_rate = a.rate;
        F.res->max_speed = a.speed;
        F.res->max_depth = a.depth;
        F.res->max_dev = a.nan ? (double)NAN : a.dev;
        F.res->clamped = a.clamp;
        F.counter[0] = 0u;
        if (F.pnext && F.P->spec) spec_next(*F.P, a.rate, *F.pnext, F.res->next);
    }
}

// The device controller for a y-strip: the same spec_next as k_final's last
// CTA, on the max rate the host has all-reduced over the ranks in place
// (res->max_rate) -- k_final alone only sees the strip's own maximum.
#if BSQ_INST_F64
static __global__ void k_spec_next(const DevParams *P, DevResult *res, DevParams *N) {
    if (threadIdx.x == 0 && P->spec) spec_next(*P, res->max_rate, *N, res->next);
}
void launch_spec_next(const DevParams *P, DevResult *res, DevParams *N, cudaStream_t st) {
    k_spec_next<<<1, 32, 0, st>>>(P, res, N);
}
#endif

// speed_extrema of a committed state (construction time, stepper.py:210)
template <class T>
__global__ void __launch_bounds__(FT) k_extrema(Consts<T> C, const T *w, const T *p, const T *q,
                                                const T *be, Partial *part) {
    const Layout L = C.L;
    const int I = GL + blockIdx.x * FX + threadIdx.x;
    Acc<T> a{T(0), T(0), T(0), T(0), T(0), 0};
    for (int k = 0; k < FR; k++) {
        const int J = GL + blockIdx.y * FR * FY + k * FY + threadIdx.y;
        if (I >= L.nx + GL || J >= L.ny + GL) continue;
        const long o = L.at(J, I);
        extrema_cell(C, w[o], p[o], q[o], be[o], a);
    }
    const Red r = red_block_warped(red_warp(a));
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        Partial pt{};
        pt.max_rate = r.rate;
        pt.max_speed = r.speed;
        pt.max_depth = r.depth;
        part[blockIdx.y * gridDim.x + blockIdx.x] = pt;
    }
}

// gauge gather outside a step (initial record, after a state upload)
template <class T>
__global__ void k_gather(const T *w, const T *p, const T *q, const long long *goff, int ng,
                         T *gval) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ng) return;
    const long long o = goff[g];
    gval[3 * g] = w[o];
    gval[3 * g + 1] = p[o];
    gval[3 * g + 2] = q[o];
}

// MaxSurfaceTracker.update (scenario.py:297-299): np.maximum(max_w, w) over
// the interior, numpy's NaN-propagating rule; the stage kernel folds the same
// way when a fold is pending, this is the stand-alone flush
template <class T>
__global__ void k_fold_max(Consts<T> C, const T *w, T *maxw) {
    const Layout L = C.L;
    const int I = GL + blockIdx.x * blockDim.x + threadIdx.x;
    const int J = GL + blockIdx.y;
    if (I >= L.nx + GL) return;
    const long o = L.at(J, I);
    maxw[o] = np_maximum(maxw[o], w[o]);
}

static dim3 final_grid(int nx, int ny) { return dim3((nx + FX - 1) / FX, (ny + FY * FR - 1) / (FY * FR)); }

#if BSQ_INST_F64
int final_blocks(int nx, int ny) {
    dim3 g = final_grid(nx, ny);
    return (int)(g.x * g.y);
}
int final_rows(int nx, int ny) { return (int)final_grid(nx, ny).y; }
#endif

template <class T>
void launch_final(const Consts<T> &C, const FinalPtrs<T> &F, cudaStream_t st) {
    const dim3 tg = final_grid(C.L.nx, C.L.ny), blk(FX, FY);
    const int ntiles = (int)(tg.x * tg.y);
    const bool fast = flux_fast_rcp_ok(C.h_eps);
    auto kern = C.exact_final
                    ? (F.spbt ? (fast ? k_final<T, true, true, true> : k_final<T, true, false, true>)
                              : (fast ? k_final<T, false, true, true> : k_final<T, false, false, true>))
                    : (F.spbt ? (fast ? k_final<T, true, true, false> : k_final<T, true, false, false>)
                              : (fast ? k_final<T, false, true, false> : k_final<T, false, false, false>));
    static int resident = 0;  // CTAs of k_final resident on the device (all four share one shape)
    if (!resident) {
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, FT, 0);
        resident = sms * (per > 0 ? per : 1);
    }
    const int grid = ntiles < resident ? ntiles : resident;
    launch_k(kern, dim3(grid), blk, 0, st, C, F, (int)tg.x, ntiles);
}

template <class T>
void launch_extrema(const Consts<T> &C, const T *w, const T *p, const T *q, const T *be,
                    Partial *part, cudaStream_t st) {
    k_extrema<T><<<final_grid(C.L.nx, C.L.ny), dim3(FX, FY), 0, st>>>(C, w, p, q, be, part);
}

template <class T>
void launch_gather(const T *w, const T *p, const T *q, const long long *goff, int ng, T *gval,
                   cudaStream_t st) {
    if (ng > 0) k_gather<T><<<(ng + 127) / 128, 128, 0, st>>>(w, p, q, goff, ng, gval);
}

template <class T>
void launch_fold_max(const Consts<T> &C, const T *w, T *maxw, cudaStream_t st) {
    k_fold_max<T><<<dim3((C.L.nx + 255) / 256, C.L.ny), 256, 0, st>>>(C, w, maxw);
}

#if BSQ_INST_F64
template void launch_gather<double>(const double *, const double *, const double *,
                                    const long long *, int, double *, cudaStream_t);
#endif
#if BSQ_INST_F32
template void launch_gather<float>(const float *, const float *, const float *,
                                   const long long *, int, float *, cudaStream_t);
#endif
#if BSQ_INST_F64
template void launch_fold_max<double>(const Consts<double> &, const double *, double *,
                                      cudaStream_t);
#endif
#if BSQ_INST_F32
template void launch_fold_max<float>(const Consts<float> &, const float *, float *, cudaStream_t);
#endif
#if BSQ_INST_F64
template void launch_final<double>(const Consts<double> &, const FinalPtrs<double> &,
                                   cudaStream_t);
#endif
#if BSQ_INST_F64
template void launch_extrema<double>(const Consts<double> &, const double *, const double *,
                                     const double *, const double *, Partial *, cudaStream_t);
#endif
#if BSQ_INST_F32
template void launch_final<float>(const Consts<float> &, const FinalPtrs<float> &, cudaStream_t);
#endif
#if BSQ_INST_F32
template void launch_extrema<float>(const Consts<float> &, const float *, const float *,
                                    const float *, const float *, Partial *, cudaStream_t);
#endif

}  // namespace bsq
