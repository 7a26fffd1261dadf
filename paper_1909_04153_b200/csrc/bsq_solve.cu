// bsq_solve.cu -- implicit momentum recovery: batched tridiagonal line solves
// for P (x rows) and Q (y columns), TMA-pipelined.
//
// Reference: implicit.solve_momentum (implicit.py:173-205) with thomas_batch
// (_kernels.py:360-381).  The LU factors of the static operator are
// precomputed on the host with thomas_batch's own arithmetic
// (den_i = b_i - a_i cw_{i-1}, cw_i = c_i / den_i), so the per-step forward
// sweep dw_i = (r_i - a_i dw_{i-1}) / den_i and back substitution
// x_i = dw_i - cw_i x_{i+1} reproduce thomas_batch bit for bit; the division
// by the static pivot is div_static (correctly rounded, Markstein).
//
// A CTA owns 32 lines (x: 32 consecutive rows; y: 32 consecutive columns)
// and has two warps:
//   producer (warp 1, one elected lane) streams 2-D tiles of 32 lines x EK
//     elements with bulk tensor copies (TMA) into an NS-deep smem ring,
//     gated by full/empty mbarriers -- up to NS-1 tiles per array in flight
//     without holding a single register;
//   consumer (warp 0): lane l runs line l's recurrence out of the ring, folds
//     the boundary ghosts into the first/last element, writes results into a
//     double-buffered out tile and TMA-stores it.
// x tiles use the 128-byte swizzle so the consumer's column walk through a
// row-major tile is (nearly) bank-conflict free; y tiles are naturally
// [element][line].  Out-of-range lines/elements are zero-filled on load and
// clipped on store by the TMA unit.  The forward sweep's dw is stored into
// the output array and read back by the backward sweep, which overwrites it.
#include <cstdint>
#include <cstdlib>
#include <cstdio>

#include "bsq_device.cuh"
#include "bsq_launch.h"
#include "bsq_tma.cuh"

namespace bsq {

#ifdef BSQ_SOLVE_PARK
#define SOLVE_WAIT mbar_wait_park
#else
#define SOLVE_WAIT mbar_wait
#endif

constexpr int NLINE = 32;  // lines per CTA
#ifndef BSQ_SOLVE_NS_ONCHIP
#define BSQ_SOLVE_NS_ONCHIP 3  // stages of SUB chunks (72 KB ring: 2 CTAs per SM)
#endif
#ifndef BSQ_SOLVE_SUB
#define BSQ_SOLVE_SUB 2  // chunks per ring stage (one barrier round trip per SUB chunks)
#endif

// Ring geometry.  A forward stage holds FT tiles {r, a, den[, rden]}; the
// backward pass reuses the same bytes as NS2 stages of 2 tiles {dw, cw}.
template <class T, bool ONCHIP>
struct TileGeom {
    static constexpr int EK = 128 / sizeof(T);              // elements per chunk (one 128-B row)
    static constexpr int TILE = NLINE * EK;                  // elements per tile
    static constexpr int TILE_B = TILE * sizeof(T);          // 4096 bytes
    static constexpr int FT = ONCHIP ? 3 : 4;                // tiles per forward stage
    static constexpr int NS = ONCHIP ? BSQ_SOLVE_NS_ONCHIP : 6;  // forward ring depth
    static constexpr int NS2 = NS * FT / 2;                  // backward ring depth
    static constexpr int SUB = BSQ_SOLVE_SUB;                // chunks per stage
    static constexpr int SUBT = SUB * TILE;                  // one operand's slice of a stage
    static constexpr int RING_B = NS * FT * SUB * TILE_B;
    static constexpr int SMEM_B = 1024 + RING_B + 2 * TILE_B + 8 * (2 * NS + 2 * NS2);
};

// An opaque use of all EK fp32 values: instructions that read them cannot
// move above the point where every one of them is computed.
__device__ __forceinline__ void rcp_fence(float (&v)[32]) {
#pragma unroll
    for (int k = 0; k < 32; k += 8)
        asm volatile("" : "+f"(v[k]), "+f"(v[k + 1]), "+f"(v[k + 2]), "+f"(v[k + 3]),
                     "+f"(v[k + 4]), "+f"(v[k + 5]), "+f"(v[k + 6]), "+f"(v[k + 7]));
}

// element offset of (line ln, chunk element k) inside a tile
template <class T, bool XDIR>
__device__ __forceinline__ int toff(int ln, int k) {
    if (XDIR) {  // box {EK, 32}: row = line, 128-B swizzle of 16-B units by (row & 7)
        constexpr int PER16 = 16 / sizeof(T);
        const int unit = (k / PER16) ^ (ln & 7);
        return ln * (128 / (int)sizeof(T)) + unit * PER16 + (k % PER16);
    }
    return k * NLINE + ln;  // box {32, EK}: row = element
}

// mode (y lines only; x lines always run complete): SOLVE_FULL, SOLVE_X_YFWD
// (forward sweep only: dw stays in the output array, the strip's last dw goes
// to dw_out) or SOLVE_YBWD (back substitution only).  For a y-strip with an
// internal south side the first element continues the recurrence from dw_in
// instead of folding a ghost; with an internal north side the last element
// is not folded and the back substitution starts from x_in.
// RDEN_ONCHIP: RN(1/den) is recomputed in the consumer (3 streamed operands
// instead of 4; 0.347 -> 0.310 ms per solve at 4096^2) whenever every pivot's
// exponent is within +-1000 (PIV_RDEN_INRANGE, checked at factor time)
template <class T, bool XDIR, bool POS, bool RDEN_ONCHIP, bool EXD>
__device__ __forceinline__ void solve_lines_tma(const Consts<T> &C, const SolveMaps &M, const SolvePtrs<T> &S,
                                int line0, unsigned char *smem, int mode) {
    using G = TileGeom<T, RDEN_ONCHIP>;
    constexpr int EK = G::EK, TILE = G::TILE, NS = G::NS, NS2 = G::NS2, FT = G::FT;
    const Layout L = C.L;
    const int n = XDIR ? L.nx : L.ny;
    const int nlines = XDIR ? L.ny : L.nx;
    const int nc = (n + EK - 1) / EK;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool sint = !XDIR && S.south_int, nint = !XDIR && S.north_int;
    if (XDIR) mode = SOLVE_FULL;

    T *ring = reinterpret_cast<T *>(smem);                    // NS x {r, a, den[, rden]}
    T *outb = reinterpret_cast<T *>(smem + G::RING_B);        // 2 out tiles
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + G::RING_B + 2 * G::TILE_B);
    uint64_t *empty = full + NS;
    uint64_t *full2 = empty + NS;
    uint64_t *empty2 = full2 + NS2;

    const CUtensorMap *m_rhs = XDIR ? &M.x_rhs : &M.y_rhs;
    const CUtensorMap *m_a = XDIR ? &M.x_a : &M.y_a;
    const CUtensorMap *m_den = XDIR ? &M.x_den : &M.y_den;
    const CUtensorMap *m_rden = XDIR ? &M.x_rden : &M.y_rden;
    const CUtensorMap *m_cw = XDIR ? &M.x_cw : &M.y_cw;
    const CUtensorMap *m_out = XDIR ? &M.x_out : &M.y_out;
    auto coords = [&](int c, int &c0, int &c1) {
        if (XDIR) { c0 = c * EK; c1 = line0; } else { c0 = line0; c1 = c * EK; }
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < NS2; s++) { mbar_init(&full2[s], 1); mbar_init(&empty2[s], 1); }
        fence_mbar_init();
    }
    __syncthreads();

    // ---- forward sweep --------------------------------------------------------
#ifdef BSQ_SOLVE_CLOCKS
    const long long t_start = clock64();
#endif
    constexpr int SUB = G::SUB, SUBT = G::SUBT;
    const int nsc = (nc + SUB - 1) / SUB;  // ring stages (super-chunks) per sweep
    if (mode == SOLVE_YBWD) {
        // back substitution only
    } else if (warp == 1) {
        if (lane == 0) {
            for (int u = 0; u < nsc; u++) {
                const int s = u % NS;
                if (u >= NS) SOLVE_WAIT(&empty[s], ((u / NS) - 1) & 1);
                mbar_expect_tx(&full[s], (RDEN_ONCHIP ? 3 : 4) * SUB * G::TILE_B);
#pragma unroll
                for (int j = 0; j < SUB; j++) {
                    int c0, c1;
                    coords(u * SUB + j, c0, c1);
                    T *st = ring + s * FT * SUBT + j * TILE;
                    if (!RDEN_ONCHIP) tma_load_2d(st + 3 * SUBT, m_rden, c0, c1, &full[s]);
                    tma_load_2d(st, m_rhs, c0, c1, &full[s]);
                    tma_load_2d(st + SUBT, m_a, c0, c1, &full[s]);
                    tma_load_2d(st + 2 * SUBT, m_den, c0, c1, &full[s]);
                }
            }
        }
    } else {
        const int line = line0 + lane;
        const bool lv = line < nlines;
        // ghost values folded into the first/last element (implicit.py:178-179,
        // :190-191).  The first element computes dw0 = (r0 - a0 * g0) / den0:
        // with an internal south side g0 is the south rank's last dw, which
        // makes it the ordinary recurrence step of the global column.
        const T g0 = !lv ? T(0)
                     : XDIR ? S.gp[L.at(GL + line, GL - 1)]
                     : sint ? S.dw_in[line]
                            : S.gq[L.at(GL - 1, GL + line)];
        const T g1 = (!lv || nint) ? T(0) : XDIR ? S.gp[L.at(GL + line, n + GL)] : S.gq[L.at(n + GL, GL + line)];
        const T cl = (!lv || nint) ? T(0) : XDIR ? S.cx_last[line] : S.cy_last[line];
        // dw_i = (r_i - a_i dw_{i-1}) / den_i with nr = -RN(1/den): streamed
        // from HBM, or (RDEN_ONCHIP) recomputed here off the recurrence's
        // critical path with the branch-free reciprocal (every pivot's exponent
        // is within +-1000, checked at factor time)
        // EXD (Simulator(exact_subnormal=True) or an operator the host cannot
        // vouch for): the IEEE division, exact for numerators under 2^-960 too,
        // where the Markstein step can miss by an ulp (bsq_device.cuh)
        auto step = [&](T num, T den, T nr) -> T {
            if (EXD) return num / den;
            return POS ? div_static_pos(num, den, nr) : div_static(num, den, -nr);
        };
        auto nrden = [&](const T *st, int t) -> T {
            return RDEN_ONCHIP ? -rcp_rn_inrange(st[2 * SUBT + t]) : st[3 * SUBT + t];
        };
        T dw = T(0);
        for (int c = 0; c < nc; c++) {
            const int u = c / SUB, j = c % SUB, s = u % NS;
            T *st = ring + s * FT * SUBT + j * TILE;
            T *ob = outb + (c & 1) * TILE;
            if (lane == 0) bulk_wait_read<1>();  // the store from this out tile (c-2) has read it
            __syncwarp();
            if (j == 0) SOLVE_WAIT(&full[s], (u / NS) & 1);
            const int kmax = min(EK, n - c * EK);
            // the whole chunk goes to registers first: the ring and the out tile
            // share one smem base, so interleaved loads could not be hoisted past
            // the stores and every element would pay an LDS round trip on the chain
            if (c > 0 && c < nc - 1) {  // interior chunk: pure recurrence
                T rv[EK], av[EK], dv[EK], nv[EK];
#pragma unroll
                for (int k = 0; k < EK; k++) {
                    const int t = toff<T, XDIR>(lane, k);
                    rv[k] = st[t];
                    av[k] = st[SUBT + t];
                    dv[k] = st[2 * SUBT + t];
                    nv[k] = RDEN_ONCHIP ? T(0) : st[3 * SUBT + t];
                }
                if (RDEN_ONCHIP) {
#pragma unroll
                    for (int k = 0; k < EK; k++) nv[k] = -rcp_rn_inrange(dv[k]);
                    // fp32: the chunk's reciprocals complete before its
                    // recurrence starts (interleaved element by element, each
                    // step waited on the next element's MUFU + Newton chain);
                    // fp64 measured no difference either way
                    if constexpr (sizeof(T) == 4) rcp_fence(nv);
                }
#pragma unroll
                for (int k = 0; k < EK; k++) {
                    dw = step(rv[k] - av[k] * dw, dv[k], nv[k]);
                    rv[k] = dw;
                }
#pragma unroll
                for (int k = 0; k < EK; k++) ob[toff<T, XDIR>(lane, k)] = rv[k];
            } else {  // first / last chunk of the line (2 of n/EK): fold the ghosts
                for (int k = 0; k < kmax; k++) {
                    const int t = toff<T, XDIR>(lane, k);
                    const int e = c * EK + k;
                    T r = st[t];
                    const T a = st[SUBT + t];
                    if (e == 0) {  // folded, no recurrence term (thomas_batch dw[0])
                        dw = step(r - a * g0, st[2 * SUBT + t], nrden(st, t));
                    } else {
                        if (e == n - 1) r = r - cl * g1;  // far ghost
                        dw = step(r - a * dw, st[2 * SUBT + t], nrden(st, t));
                    }
                    ob[t] = dw;
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                if (j == SUB - 1 || c == nc - 1) mbar_arrive(&empty[s]);
                int c0, c1;
                coords(c, c0, c1);
                tma_store_2d(m_out, c0, c1, ob);
                bulk_commit();
            }
        }
        if (nint && lv) S.dw_out[line] = dw;  // the north rank continues from here
        if (lane == 0) {
            bulk_wait_all();  // dw globally written before the backward loads read it
            fence_async_global();
        }
    }
    __syncthreads();

    // ---- back substitution (chunks in reverse) -----------------------------------
    if (mode == SOLVE_X_YFWD) {
        // forward sweep only
    } else if (warp == 1) {
        if (lane == 0) {
            for (int v = 0; v < nsc; v++) {  // super-chunks from the line's end
                const int u = nsc - 1 - v, s = v % NS2;
                if (v >= NS2) SOLVE_WAIT(&empty2[s], ((v / NS2) - 1) & 1);
                mbar_expect_tx(&full2[s], 2 * SUB * G::TILE_B);
#pragma unroll
                for (int j = 0; j < SUB; j++) {
                    int c0, c1;
                    coords(u * SUB + j, c0, c1);
                    T *st = ring + s * 2 * SUBT + j * TILE;
                    tma_load_2d(st, m_out, c0, c1, &full2[s]);
                    tma_load_2d(st + SUBT, m_cw, c0, c1, &full2[s]);
                }
            }
        }
    } else {
        const int line = line0 + lane;
        const bool lv = line < nlines;
        // x of the row above this strip (north rank), or none for a physical side
        const T xn = (nint && lv) ? S.x_in[line] : T(0);
        T xv = T(0);
        for (int s_ = 0; s_ < nc; s_++) {
            const int c = nc - 1 - s_, u = c / SUB, j = c % SUB, v = nsc - 1 - u, s = v % NS2;
            T *st = ring + s * 2 * SUBT + j * TILE;
            T *ob = outb + (s_ & 1) * TILE;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            if (c == min(u * SUB + SUB - 1, nc - 1)) SOLVE_WAIT(&full2[s], (v / NS2) & 1);
            const int kmax = min(EK, n - c * EK);
            if (s_ > 0 && kmax == EK) {  // interior chunk
                T dv[EK], cv[EK];
#pragma unroll
                for (int k = 0; k < EK; k++) {
                    const int t = toff<T, XDIR>(lane, k);
                    dv[k] = st[t];
                    cv[k] = st[SUBT + t];
                }
#pragma unroll
                for (int k = EK - 1; k >= 0; k--) {
                    xv = dv[k] - cv[k] * xv;
                    dv[k] = xv;
                }
#pragma unroll
                for (int k = 0; k < EK; k++) ob[toff<T, XDIR>(lane, k)] = dv[k];
            } else {  // the line's last chunk: out[n-1] = dw[n-1] (or continues from x_in)
                for (int k = kmax - 1; k >= 0; k--) {
                    const int t = toff<T, XDIR>(lane, k);
                    if (s_ == 0 && k == kmax - 1)
                        xv = nint ? st[t] - st[SUBT + t] * xn : st[t];
                    else
                        xv = st[t] - st[SUBT + t] * xv;
                    ob[t] = xv;
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                if (j == 0) mbar_arrive(&empty2[s]);
                int c0, c1;
                coords(c, c0, c1);
                tma_store_2d(m_out, c0, c1, ob);
                bulk_commit();
            }
        }
        if (sint && lv) S.x_out[line] = xv;  // the south rank continues from here
        if (lane == 0) bulk_wait_all();
#ifdef BSQ_SOLVE_CLOCKS
        if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
            printf("solve cta %d n %d total %lld cycles\n", (int)blockIdx.x, n, clock64() - t_start);
#endif
    }
}

// Few long x lines (C1: 5 lines of 1024, C2: 64 of 2048): the TMA ring above
// is paced by its data path there (without the recurrence it alone takes 80 %
// of C1's solve), so these lines run one warp per line instead.  The lanes
// load 32 consecutive elements of the line at a time (coalesced, two chunks
// ahead), compute the chunk's pivot reciprocals side by side, and stage the
// operands in shared memory; every lane then runs the same recurrence from
// broadcast reads (no divergence), lane k keeping element k.  dw stays in
// shared memory for the whole line (no round trip through HBM), and the back
// substitution writes the result once.  Same operations and order as
// thomas_batch with the folded ghosts (_kernels.py:360-381, implicit.py:178-179).
constexpr int XW_LINES = 2;  // x lines (warps) per CTA on this path
#ifndef BSQ_XW_MAX_LINES
#define BSQ_XW_MAX_LINES 256  // at most this many x lines take the path (one wave)
#endif
constexpr int XW_MAX_LINES = BSQ_XW_MAX_LINES;
template <class T>
__host__ __device__ constexpr int xw_smem_elems(int n) { return n + 5 * 32; }

template <class T, bool POS, bool ONCHIP, bool EXD>
__device__ __forceinline__ void solve_xline_warp(const Consts<T> &C, const SolveMaps &M,
                                                 const SolvePtrs<T> &S, int line, T *sm) {
    const Layout L = C.L;
    const int n = L.nx, lane = threadIdx.x & 31;
    if (line >= L.ny) return;
    const long row = L.at(GL + line, GL);
    const T *R = reinterpret_cast<const T *>(M.xp_rhs) + row;
    const T *A = reinterpret_cast<const T *>(M.xp_a) + row;
    const T *D = reinterpret_cast<const T *>(M.xp_den) + row;
    const T *RD = reinterpret_cast<const T *>(M.xp_rden) + row;
    const T *CW = reinterpret_cast<const T *>(M.xp_cw) + row;
    T *OUT = reinterpret_cast<T *>(M.xp_out) + row;
    T *dws = sm, *sr = sm + n, *sa = sr + 32, *sd = sa + 32, *sn = sd + 32, *sc = sn + 32;
    const T g0 = S.gp[L.at(GL + line, GL - 1)];
    const T g1 = S.gp[L.at(GL + line, n + GL)];
    const T cl = S.cx_last[line];
    auto step = [&](T num, T den, T nr) -> T {
        if (EXD) return num / den;
        return POS ? div_static_pos(num, den, nr) : div_static(num, den, -nr);
    };
    const int nc = (n + 31) / 32;
    // ---- forward sweep: dw_e = (r_e - a_e dw_{e-1}) / den_e, dw_{-1} = g0
    T fr[2], fa[2], fd[2], fn[2];  // operands of chunks c+1, c+2 for this lane
    auto fetch = [&](int c, int k) {
        const int e = c * 32 + lane;
        const bool in = e < n;
        fr[k] = in ? R[e] : T(0);
        fa[k] = in ? A[e] : T(0);
        fd[k] = in ? D[e] : T(1);
        fn[k] = (in && !ONCHIP) ? RD[e] : T(0);
    };
    T r0, a0, d0, n0;
    {
        fetch(0, 0);
        r0 = fr[0], a0 = fa[0], d0 = fd[0], n0 = fn[0];
        if (nc > 1) fetch(1, 0);
        if (nc > 2) fetch(2, 1);
    }
    T dw = g0;
    for (int c = 0; c < nc; c++) {
        const T nr0 = ONCHIP ? -rcp_rn_inrange(d0) : n0;
        sr[lane] = r0, sa[lane] = a0, sd[lane] = d0, sn[lane] = nr0;
        __syncwarp();
        // rotate the prefetch window and request chunk c+3
        r0 = fr[0], a0 = fa[0], d0 = fd[0], n0 = fn[0];
        fr[0] = fr[1], fa[0] = fa[1], fd[0] = fd[1], fn[0] = fn[1];
        if (c + 3 < nc) fetch(c + 3, 1);
        const int e0 = c * 32, kmax = min(32, n - e0);
        T mine = T(0);
        if (e0 > 0 && kmax == 32 && e0 + 32 < n) {  // interior chunk
#pragma unroll
            for (int k = 0; k < 32; k++) {
                dw = step(sr[k] - sa[k] * dw, sd[k], sn[k]);
                mine = lane == k ? dw : mine;
            }
        } else {
            for (int k = 0; k < kmax; k++) {
                const int e = e0 + k;
                T num;
                if (e == n - 1 && n > 1) num = (sr[k] - cl * g1) - sa[k] * dw;  // far ghost first
                else num = sr[k] - sa[k] * dw;                                 // e = 0: a_0 g0
                if (e == n - 1 && n == 1) num = num - cl * g1;
                dw = step(num, sd[k], sn[k]);
                mine = lane == k ? dw : mine;
            }
        }
        if (lane < kmax) dws[e0 + lane] = mine;
        __syncwarp();
    }
    // ---- back substitution: x_{n-1} = dw_{n-1}, x_e = dw_e - cw_e x_{e+1}
    T fc[2];
    auto fetchc = [&](int c, int k) {
        const int e = c * 32 + lane;
        fc[k] = e < n ? CW[e] : T(0);
    };
    T c0v;
    {
        fetchc(nc - 1, 0);
        c0v = fc[0];
        if (nc > 1) fetchc(nc - 2, 0);
        if (nc > 2) fetchc(nc - 3, 1);
    }
    T xv = T(0);
    for (int c = nc - 1; c >= 0; c--) {
        sc[lane] = c0v;
        __syncwarp();
        c0v = fc[0];
        fc[0] = fc[1];
        if (c - 3 >= 0) fetchc(c - 3, 1);
        const int e0 = c * 32, kmax = min(32, n - e0);
        T mine = T(0);
        if (kmax == 32 && e0 + 32 < n) {
#pragma unroll
            for (int k = 31; k >= 0; k--) {
                xv = dws[e0 + k] - sc[k] * xv;
                mine = lane == k ? xv : mine;
            }
        } else {
            for (int k = kmax - 1; k >= 0; k--) {
                const int e = e0 + k;
                xv = e == n - 1 ? dws[e] : dws[e] - sc[k] * xv;
                mine = lane == k ? xv : mine;
            }
        }
        if (lane < kmax) OUT[e0 + lane] = mine;
        __syncwarp();
    }
}

// Blocks [0, nbx) take x lines (rows -> P); blocks [nbx, ...) y lines (columns -> Q).
// xwarp: the x-line blocks run solve_xline_warp, XW_LINES lines each.
template <class T, bool POS, bool ONCHIP, bool EXD>
__global__ void __launch_bounds__(64) k_solve_tma(Consts<T> C, const __grid_constant__ SolveMaps M,
                                                  SolvePtrs<T> S, int nbx, int mode, int xwarp) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-B alignment of the ring.  fp32: pointer arithmetic on the shared
    // array keeps the address space (LDS/STS with 32-bit addresses; with the
    // reciprocal batch below, fp32 solve 0.1685 -> 0.149 ms).  fp64 keeps the
    // generic form: its schedule with LDS/STS measured slower (0.307 -> 0.320).
    unsigned char *smem;
    if constexpr (sizeof(T) == 4)
        smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    else
        smem = reinterpret_cast<unsigned char *>(
            (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    pdl_trigger();
    pdl_wait();
    if ((int)blockIdx.x < nbx && xwarp) {
        // straight from the shared array (no alignment round trip): LDS/STS
        const int w = threadIdx.x >> 5;
        T *sm = reinterpret_cast<T *>(smem_raw) + w * xw_smem_elems<T>(C.L.nx);
        solve_xline_warp<T, POS, ONCHIP, EXD>(C, M, S, blockIdx.x * XW_LINES + w, sm);
    } else if ((int)blockIdx.x < nbx)
        solve_lines_tma<T, true, POS, ONCHIP, EXD>(C, M, S, blockIdx.x * NLINE, smem, mode);
    else
        solve_lines_tma<T, false, POS, ONCHIP, EXD>(C, M, S, (blockIdx.x - nbx) * NLINE, smem, mode);
}

// pos_pivots: every Thomas pivot of both operators is > 0 (host-checked), which
// enables the select-free quotient on the recurrence's critical path.
// mode SOLVE_YBWD launches only the y-line CTAs.
template <class T>
void launch_solve(const Consts<T> &C, const SolveMaps &M, const SolvePtrs<T> &S, int pivots,
                  cudaStream_t st, int mode) {
    // few long x lines: the warp-per-line path (one wave of CTAs, the whole
    // line's dw in shared memory)
    const int smem_on = TileGeom<T, true>::SMEM_B, smem_off = TileGeom<T, false>::SMEM_B;
    const size_t xw_smem = 1024 + sizeof(T) * XW_LINES * (size_t)xw_smem_elems<T>(C.L.nx);
    static const int xw_env = [] {
        const char *e = std::getenv("BSQ_SOLVE_XWARP");  // A/B: 0 off, 1 forced
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    const bool xwarp = mode != SOLVE_YBWD && xw_smem <= (size_t)smem_on &&
                       (xw_env == 1 || (xw_env < 0 && C.L.ny <= XW_MAX_LINES));
    const int nbx = xwarp ? (C.L.ny + XW_LINES - 1) / XW_LINES : (C.L.ny + NLINE - 1) / NLINE;
    const int nby = (C.L.nx + NLINE - 1) / NLINE;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_solve_tma<T, true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_on);
        cudaFuncSetAttribute(k_solve_tma<T, false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_on);
        cudaFuncSetAttribute(k_solve_tma<T, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_off);
        cudaFuncSetAttribute(k_solve_tma<T, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_off);
        cudaFuncSetAttribute(k_solve_tma<T, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_off);
        attr_set = true;
    }
    const int bx = mode == SOLVE_YBWD ? 0 : nbx;  // x-line CTAs in this launch
    const bool pos = pivots & PIV_POSITIVE;
#ifdef BSQ_SOLVE_RDEN_HBM
    const bool onchip = false;
#else
    const bool onchip = pivots & PIV_RDEN_INRANGE;
#endif
    dim3 g(bx + nby), b(64);
    if (S.exact)
        launch_k(k_solve_tma<T, false, false, true>, g, b, smem_off, st, C, M, S, bx, mode, (int)xwarp);
    else if (pos && onchip)
        launch_k(k_solve_tma<T, true, true, false>, g, b, smem_on, st, C, M, S, bx, mode, (int)xwarp);
    else if (pos)
        launch_k(k_solve_tma<T, true, false, false>, g, b, smem_off, st, C, M, S, bx, mode, (int)xwarp);
    else if (onchip)
        launch_k(k_solve_tma<T, false, true, false>, g, b, smem_on, st, C, M, S, bx, mode, (int)xwarp);
    else
        launch_k(k_solve_tma<T, false, false, false>, g, b, smem_off, st, C, M, S, bx, mode, (int)xwarp);
}

#if BSQ_INST_F64
int solve_chunk_elems(int elem_bytes) { return 128 / elem_bytes; }
#endif

#if BSQ_INST_F64
template void launch_solve<double>(const Consts<double> &, const SolveMaps &,
                                   const SolvePtrs<double> &, int, cudaStream_t, int);
#endif
#if BSQ_INST_F32
template void launch_solve<float>(const Consts<float> &, const SolveMaps &,
                                  const SolvePtrs<float> &, int, cudaStream_t, int);
#endif

}  // namespace bsq
