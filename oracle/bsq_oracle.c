/*
 * bsq_oracle.c -- CPU restatement of the reference adaptive-AB3 Boussinesq
 * step.  TEST INFRASTRUCTURE ONLY: this file is the parity checker and the
 * CPU baseline.  It is never linked into, imported by, or called from the
 * product path (paper_1909_04153_b200/), which fails loudly without its CUDA
 * library.
 *
 * Every routine restates the reference algorithm in plain IEEE binary64 with
 * the reference's operation order (build with -ffp-contract=off, no
 * -ffast-math) so results are bitwise identical to the numba kernels, which
 * emit no FMA.  Citations are into /root/reference/pkg/src/
 * boussim/.
 *
 * Array conventions (grid.py:1-20): padded fields are (ny+4) x (nx+4)
 * row-major [j][i]; bed_face_x is (ny+4) x (nx+3), bed_face_y (ny+3) x (nx+4);
 * interior arrays are ny x nx; x fluxes ny x (nx+1), y fluxes (ny+1) x nx.
 *
 * Parallelism: OpenMP over rows / lines.  Every output is still computed by
 * exactly one thread in the reference order, so the thread count never
 * changes a bit of the result (max reductions are order free; the clamped
 * volume is summed per row then over rows in row order).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GL 2

/* ------------------------------------------------------------------ */
/* kernels: _kernels.py                                                */

/* _kernels.py:20-26 */
static inline double minmod3(double a1, double a2, double a3)
{
    /* numba's min/max keep the accumulator unless the new value is
     * strictly smaller/larger (numba cpython/builtins.py do_minmax) */
    if (a1 > 0.0 && a2 > 0.0 && a3 > 0.0) {
        double m = a3 < a2 ? a3 : a2;
        return m < a1 ? m : a1;
    }
    if (a1 < 0.0 && a2 < 0.0 && a3 < 0.0) {
        double m = a3 > a2 ? a3 : a2;
        return m > a1 ? m : a1;
    }
    return 0.0;
}

/* faces along one direction for a single cell; stride selects x (1) or y
 * (row pitch).  Mirrors faces_x / faces_y (_kernels.py:29-103). */
static inline void cell_faces(const double *w, const double *p, const double *q,
                              long c, long st, double bhi, double blo, double theta,
                              double *whi, double *wlo, double *phi, double *plo,
                              double *qhi, double *qlo)
{
    double wc = w[c];
    double s = minmod3(theta * (wc - w[c - st]), 0.5 * (w[c + st] - w[c - st]),
                       theta * (w[c + st] - wc));
    double we = wc + 0.5 * s;
    double ww = wc - 0.5 * s;
    if (we < bhi) {
        we = bhi;
        ww = 2.0 * wc - bhi;
    } else if (ww < blo) {
        ww = blo;
        we = 2.0 * wc - blo;
    }
    *whi = we;
    *wlo = ww;
    double pc = p[c];
    s = minmod3(theta * (pc - p[c - st]), 0.5 * (p[c + st] - p[c - st]),
                theta * (p[c + st] - pc));
    *phi = pc + 0.5 * s;
    *plo = pc - 0.5 * s;
    double qc = q[c];
    s = minmod3(theta * (qc - q[c - st]), 0.5 * (q[c + st] - q[c - st]),
                theta * (q[c + st] - qc));
    *qhi = qc + 0.5 * s;
    *qlo = qc - 0.5 * s;
}

/* _kernels.py:29-68 */
void orc_faces_x(int nyt, int nxt, const double *w, const double *p, const double *q,
                 const double *bfx, double theta, double *wE, double *wW, double *pE,
                 double *pW, double *qE, double *qW)
{
    int bst = nxt - 1;
#pragma omp parallel for schedule(static)
    for (int j = 1; j < nyt - 1; j++)
        for (int i = 1; i < nxt - 1; i++) {
            long c = (long)j * nxt + i;
            cell_faces(w, p, q, c, 1, bfx[(long)j * bst + i], bfx[(long)j * bst + i - 1], theta,
                       &wE[c], &wW[c], &pE[c], &pW[c], &qE[c], &qW[c]);
        }
}

/* _kernels.py:71-103 */
void orc_faces_y(int nyt, int nxt, const double *w, const double *p, const double *q,
                 const double *bfy, double theta, double *wN, double *wS, double *pN,
                 double *pS, double *qN, double *qS)
{
#pragma omp parallel for schedule(static)
    for (int j = 1; j < nyt - 1; j++)
        for (int i = 1; i < nxt - 1; i++) {
            long c = (long)j * nxt + i;
            cell_faces(w, p, q, c, nxt, bfy[(long)j * nxt + i], bfy[(long)(j - 1) * nxt + i],
                       theta, &wN[c], &wS[c], &pN[c], &pS[c], &qN[c], &qS[c]);
        }
}

/* _kernels.py:106-159 */
void orc_flux_x(int ny, int nx, const double *wE, const double *wW, const double *pE,
                const double *pW, const double *qE, const double *qW, const double *bfx,
                double g, double h_eps, double *fx1, double *fx2, double *fx3)
{
    int nxt = nx + 4, bst = nx + 3;
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj < ny; jj++) {
        int j = GL + jj;
        for (int ii = 0; ii <= nx; ii++) {
            int i = GL - 1 + ii;
            long L = (long)j * nxt + i, R = L + 1, o = (long)jj * (nx + 1) + ii;
            double bf = bfx[(long)j * bst + i];
            double hl = wE[L] - bf;
            if (hl < 0.0) hl = 0.0;
            double hr = wW[R] - bf;
            if (hr < 0.0) hr = 0.0;
            double pl, ql, pr, qr;
            if (hl > 0.0) { pl = pE[L]; ql = qE[L]; } else { pl = 0.0; ql = 0.0; }
            if (hr > 0.0) { pr = pW[R]; qr = qW[R]; } else { pr = 0.0; qr = 0.0; }
            double dl = hl > h_eps ? hl : h_eps;
            double dr = hr > h_eps ? hr : h_eps;
            double ul = pl / dl;
            double ur = pr / dr;
            double cl = sqrt(g * hl);
            double cr = sqrt(g * hr);
            double ap = ul + cl;
            if (ur + cr > ap) ap = ur + cr;
            if (0.0 > ap) ap = 0.0;
            double am = ul - cl;
            if (ur - cr < am) am = ur - cr;
            if (0.0 < am) am = 0.0;
            if (ap == 0.0 && am == 0.0) {
                fx1[o] = 0.0; fx2[o] = 0.0; fx3[o] = 0.0;
                continue;
            }
            double inv = 1.0 / (ap - am);
            double diff = ap * am * inv;
            double f2l = pl * ul + 0.5 * g * hl * hl;
            double f2r = pr * ur + 0.5 * g * hr * hr;
            double f3l = pl * ql / dl;
            double f3r = pr * qr / dr;
            double wl = wE[L], wr = wW[R];
            fx1[o] = (ap * pl - am * pr) * inv + diff * (wr - wl);
            fx2[o] = (ap * f2l - am * f2r) * inv + diff * (pr - pl);
            fx3[o] = (ap * f3l - am * f3r) * inv + diff * (qr - ql);
        }
    }
}

/* _kernels.py:162-212 */
void orc_flux_y(int ny, int nx, const double *wN, const double *wS, const double *pN,
                const double *pS, const double *qN, const double *qS, const double *bfy,
                double g, double h_eps, double *fy1, double *fy2, double *fy3)
{
    int nxt = nx + 4;
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj <= ny; jj++) {
        int j = GL - 1 + jj;
        for (int ii = 0; ii < nx; ii++) {
            int i = GL + ii;
            long L = (long)j * nxt + i, R = L + nxt, o = (long)jj * nx + ii;
            double bf = bfy[(long)j * nxt + i];
            double hl = wN[L] - bf;
            if (hl < 0.0) hl = 0.0;
            double hr = wS[R] - bf;
            if (hr < 0.0) hr = 0.0;
            double pl, ql, pr, qr;
            if (hl > 0.0) { pl = pN[L]; ql = qN[L]; } else { pl = 0.0; ql = 0.0; }
            if (hr > 0.0) { pr = pS[R]; qr = qS[R]; } else { pr = 0.0; qr = 0.0; }
            double dl = hl > h_eps ? hl : h_eps;
            double dr = hr > h_eps ? hr : h_eps;
            double vl = ql / dl;
            double vr = qr / dr;
            double cl = sqrt(g * hl);
            double cr = sqrt(g * hr);
            double ap = vl + cl;
            if (vr + cr > ap) ap = vr + cr;
            if (0.0 > ap) ap = 0.0;
            double am = vl - cl;
            if (vr - cr < am) am = vr - cr;
            if (0.0 < am) am = 0.0;
            if (ap == 0.0 && am == 0.0) {
                fy1[o] = 0.0; fy2[o] = 0.0; fy3[o] = 0.0;
                continue;
            }
            double inv = 1.0 / (ap - am);
            double diff = ap * am * inv;
            double f2l = ql * pl / dl;
            double f2r = qr * pr / dr;
            double f3l = ql * vl + 0.5 * g * hl * hl;
            double f3r = qr * vr + 0.5 * g * hr * hr;
            double wl = wN[L], wr = wS[R];
            fy1[o] = (ap * ql - am * qr) * inv + diff * (wr - wl);
            fy2[o] = (ap * f2l - am * f2r) * inv + diff * (pr - pl);
            fy3[o] = (ap * f3l - am * f3r) * inv + diff * (qr - ql);
        }
    }
}

/* _kernels.py:215-251 */
void orc_fv_rates(int ny, int nx, const double *fx1, const double *fx2, const double *fx3,
                  const double *fy1, const double *fy2, const double *fy3, const double *w,
                  const double *p, const double *q, const double *bed, const double *bfx,
                  const double *bfy, double g, double c_f, double h_eps, double dx, double dy,
                  double *rw, double *rp, double *rq)
{
    int nxt = nx + 4, bst = nx + 3;
    double inv_dx = 1.0 / dx, inv_dy = 1.0 / dy;
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj < ny; jj++) {
        int j = GL + jj;
        for (int ii = 0; ii < nx; ii++) {
            int i = GL + ii;
            long c = (long)j * nxt + i, o = (long)jj * nx + ii;
            long ox = (long)jj * (nx + 1) + ii, oy = (long)jj * nx + ii;
            rw[o] = -(fx1[ox + 1] - fx1[ox]) * inv_dx - (fy1[oy + nx] - fy1[oy]) * inv_dy;
            double be = bfx[(long)j * bst + i], bw = bfx[(long)j * bst + i - 1];
            double bn = bfy[(long)j * nxt + i], bs = bfy[(long)(j - 1) * nxt + i];
            double wc = w[c];
            double src_x = -g * (wc - 0.5 * (be + bw)) * (be - bw) * inv_dx;
            double src_y = -g * (wc - 0.5 * (bn + bs)) * (bn - bs) * inv_dy;
            double h = wc - bed[c];
            if (h < 0.0) h = 0.0;
            double hstar = h > h_eps ? h : h_eps;
            double fric = 0.0;
            if (c_f > 0.0) fric = c_f * sqrt(p[c] * p[c] + q[c] * q[c]) / (hstar * hstar);
            rp[o] = -(fx2[ox + 1] - fx2[ox]) * inv_dx - (fy2[oy + nx] - fy2[oy]) * inv_dy + src_x -
                    fric * p[c];
            rq[o] = -(fx3[ox + 1] - fx3[ox]) * inv_dx - (fy3[oy + nx] - fy3[oy]) * inv_dy + src_y -
                    fric * q[c];
        }
    }
}

/* _kernels.py:254-288 */
void orc_dispersive_rates(int ny, int nx, const double *eta, const double *depth,
                          const double *ddx, const double *ddy, double g, double b_disp,
                          double dx, double dy, double *rp, double *rq)
{
    int nxt = nx + 4;
    double inv_dx = 1.0 / dx, inv_dy = 1.0 / dy;
    double inv_dx2 = inv_dx * inv_dx, inv_dy2 = inv_dy * inv_dy;
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj < ny; jj++) {
        int j = GL + jj;
        for (int ii = 0; ii < nx; ii++) {
            int i = GL + ii;
            long c = (long)j * nxt + i, o = (long)jj * nx + ii;
            double d = depth[c];
            if (d <= 0.0) continue;
            const double *e = eta;
            long N = c + nxt, S = c - nxt;
            double e_xx = (e[c + 1] - 2.0 * e[c] + e[c - 1]) * inv_dx2;
            double e_yy = (e[N] - 2.0 * e[c] + e[S]) * inv_dy2;
            double e_xy = (e[N + 1] - e[N - 1] - e[S + 1] + e[S - 1]) * 0.25 * inv_dx * inv_dy;
            double e_xxx = (e[c + 2] - 2.0 * e[c + 1] + 2.0 * e[c - 1] - e[c - 2]) * 0.5 * inv_dx *
                           inv_dx2;
            double e_yyy = (e[N + nxt] - 2.0 * e[N] + 2.0 * e[S] - e[S - nxt]) * 0.5 * inv_dy *
                           inv_dy2;
            double e_xyy = ((e[N + 1] - 2.0 * e[c + 1] + e[S + 1]) -
                            (e[N - 1] - 2.0 * e[c - 1] + e[S - 1])) * 0.5 * inv_dx * inv_dy2;
            double e_xxy = ((e[N + 1] - 2.0 * e[N] + e[N - 1]) -
                            (e[S + 1] - 2.0 * e[S] + e[S - 1])) * 0.5 * inv_dy * inv_dx2;
            double gd2 = g * d * d;
            double gd3 = gd2 * d;
            rp[o] += b_disp * gd3 * (e_xxx + e_xyy) +
                     b_disp * gd2 * (ddx[c] * (2.0 * e_xx + e_yy) + ddy[c] * e_xy);
            rq[o] += b_disp * gd3 * (e_yyy + e_xxy) +
                     b_disp * gd2 * (ddy[c] * (2.0 * e_yy + e_xx) + ddx[c] * e_xy);
        }
    }
}

/* _kernels.py:291-321 */
void orc_cross_rates(int ny, int nx, const double *p, const double *q, const double *depth,
                     const double *ddx, const double *ddy, double bp13, double dx, double dy,
                     double *sp, double *sq)
{
    int nxt = nx + 4;
    double inv_dx = 1.0 / dx, inv_dy = 1.0 / dy;
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj < ny; jj++) {
        int j = GL + jj;
        for (int ii = 0; ii < nx; ii++) {
            int i = GL + ii;
            long c = (long)j * nxt + i, o = (long)jj * nx + ii;
            long N = c + nxt, S = c - nxt;
            double d = depth[c];
            if (d <= 0.0) {
                sp[o] = 0.0;
                sq[o] = 0.0;
                continue;
            }
            double q_x = (q[c + 1] - q[c - 1]) * 0.5 * inv_dx;
            double q_y = (q[N] - q[S]) * 0.5 * inv_dy;
            double q_xy = (q[N + 1] - q[N - 1] - q[S + 1] + q[S - 1]) * 0.25 * inv_dx * inv_dy;
            double p_x = (p[c + 1] - p[c - 1]) * 0.5 * inv_dx;
            double p_y = (p[N] - p[S]) * 0.5 * inv_dy;
            double p_xy = (p[N + 1] - p[N - 1] - p[S + 1] + p[S - 1]) * 0.25 * inv_dx * inv_dy;
            double sixth = d / 6.0;
            double d2 = bp13 * d * d;
            sp[o] = sixth * (ddx[c] * q_y + ddy[c] * q_x) + d2 * q_xy;
            sq[o] = sixth * (ddx[c] * p_y + ddy[c] * p_x) + d2 * p_xy;
        }
    }
}

/* _kernels.py:324-353.  out = {max_rate, max_speed, max_depth}.  Per-row
 * maxima combined in row order; max is order free so this equals the
 * reference's serial scan bit for bit. */
void orc_speed_extrema(int ny, int nx, const double *w, const double *p, const double *q,
                       const double *bed, double g, double h_eps, double dx, double dy,
                       double *out)
{
    int nxt = nx + 4;
    double inv_dx = 1.0 / dx, inv_dy = 1.0 / dy;
    double *rows = (double *)malloc(sizeof(double) * 3 * (size_t)ny);
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj < ny; jj++) {
        int j = GL + jj;
        double mr = 0.0, ms = 0.0, md = 0.0;
        for (int ii = 0; ii < nx; ii++) {
            long c = (long)j * nxt + GL + ii;
            double h = w[c] - bed[c];
            if (h < 0.0) h = 0.0;
            if (h > md) md = h;
            double hstar = h > h_eps ? h : h_eps;
            double cc = sqrt(g * h);
            double su = fabs(p[c]) / hstar + cc;
            double sv = fabs(q[c]) / hstar + cc;
            if (su > ms) ms = su;
            if (sv > ms) ms = sv;
            double a = su * inv_dx, b = sv * inv_dy;
            double rate = b > a ? b : a;
            if (rate > mr) mr = rate;
        }
        rows[3 * jj] = mr;
        rows[3 * jj + 1] = ms;
        rows[3 * jj + 2] = md;
    }
    double mr = 0.0, ms = 0.0, md = 0.0;
    for (int jj = 0; jj < ny; jj++) {
        if (rows[3 * jj] > mr) mr = rows[3 * jj];
        if (rows[3 * jj + 1] > ms) ms = rows[3 * jj + 1];
        if (rows[3 * jj + 2] > md) md = rows[3 * jj + 2];
    }
    free(rows);
    out[0] = mr;
    out[1] = ms;
    out[2] = md;
}

/* _kernels.py:360-381.  Returns 0, or -1 on an exactly zero pivot. */
static int thomas_one(int n, const double *dl, const double *dd, const double *du,
                      const double *rhs, double *out, double *cw, double *dw)
{
    double den = dd[0];
    if (den == 0.0) return -1;
    cw[0] = du[0] / den;
    dw[0] = rhs[0] / den;
    for (int i = 1; i < n; i++) {
        den = dd[i] - dl[i] * cw[i - 1];
        if (den == 0.0) return -1;
        cw[i] = du[i] / den;
        dw[i] = (rhs[i] - dl[i] * dw[i - 1]) / den;
    }
    out[n - 1] = dw[n - 1];
    for (int i = n - 2; i >= 0; i--) out[i] = dw[i] - cw[i] * out[i + 1];
    return 0;
}

int orc_thomas_batch(int m, int n, const double *dl, const double *dd, const double *du,
                     const double *rhs, double *out)
{
    int bad = 0;
#pragma omp parallel
    {
        double *cw = (double *)malloc(sizeof(double) * (size_t)n);
        double *dw = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(static)
        for (int k = 0; k < m; k++) {
            long o = (long)k * n;
            if (thomas_one(n, dl + o, dd + o, du + o, rhs + o, out + o, cw, dw)) {
#pragma omp atomic write
                bad = 1;
            }
        }
        free(cw);
        free(dw);
    }
    return bad ? -1 : 0;
}

/* _kernels.py:384-451 */
static int cr_one(int n, int n2, const double *dl, const double *dd, const double *du,
                  const double *rhs, double *out, double *a, double *b, double *c, double *r,
                  double *x)
{
    for (int i = 0; i < n; i++) { a[i] = dl[i]; b[i] = dd[i]; c[i] = du[i]; r[i] = rhs[i]; }
    for (int i = n; i < n2; i++) { a[i] = 0.0; b[i] = 1.0; c[i] = 0.0; r[i] = 0.0; }
    int stride = 1;
    while (stride < n2 / 2) {
        for (int idx = 2 * stride - 1; idx < n2; idx += 2 * stride) {
            int il = idx - stride;
            if (b[il] == 0.0) return -1;
            double alpha = -a[idx] / b[il];
            a[idx] = alpha * a[il];
            b[idx] += alpha * c[il];
            r[idx] += alpha * r[il];
            int ir = idx + stride;
            if (ir < n2) {
                if (b[ir] == 0.0) return -1;
                double beta = -c[idx] / b[ir];
                c[idx] = beta * c[ir];
                b[idx] += beta * a[ir];
                r[idx] += beta * r[ir];
            } else {
                c[idx] = 0.0;
            }
        }
        stride *= 2;
    }
    int i1 = n2 / 2 - 1, i2 = n2 - 1;
    double det = b[i1] * b[i2] - c[i1] * a[i2];
    if (det == 0.0) return -2;
    x[i1] = (r[i1] * b[i2] - c[i1] * r[i2]) / det;
    x[i2] = (b[i1] * r[i2] - a[i2] * r[i1]) / det;
    stride = n2 / 4;
    while (stride >= 1) {
        for (int idx = stride - 1; idx < n2; idx += 2 * stride) {
            if (b[idx] == 0.0) return -3;
            double lower = idx - stride >= 0 ? x[idx - stride] : 0.0;
            x[idx] = (r[idx] - a[idx] * lower - c[idx] * x[idx + stride]) / b[idx];
        }
        stride /= 2;
    }
    for (int i = 0; i < n; i++) out[i] = x[i];
    return 0;
}

int orc_cr_batch(int m, int n, const double *dl, const double *dd, const double *du,
                 const double *rhs, double *out)
{
    int n2 = 1;
    while (n2 < n) n2 *= 2;
    if (n2 < 2) n2 = 2;
    /* the reference raises at the first failing line: keep the lowest k */
    int bad_k = m, bad_rc = 0;
#pragma omp parallel
    {
        double *buf = (double *)malloc(sizeof(double) * 5 * (size_t)n2);
#pragma omp for schedule(static)
        for (int k = 0; k < m; k++) {
            long o = (long)k * n;
            int rc = cr_one(n, n2, dl + o, dd + o, du + o, rhs + o, out + o, buf, buf + n2,
                            buf + 2 * n2, buf + 3 * n2, buf + 4 * n2);
            if (rc) {
#pragma omp critical(orc_cr_bad)
                if (k < bad_k) {
                    bad_k = k;
                    bad_rc = rc;
                }
            }
        }
        free(buf);
    }
    return bad_rc;
}

/* ------------------------------------------------------------------ */
/* full step: stepper.py:225-325 with its numpy glue                   */

enum { SIDE_N = 0, SIDE_S = 1, SIDE_E = 2, SIDE_W = 3 };
enum { KIND_WALL = 0, KIND_MAKER = 1, KIND_SPONGE = 2 };

typedef struct {
    int nx, ny;
    double dx, dy, dx2, dy2; /* dx2 = dx**2 as Python computes it */
    double g, b_disp, bp13, c_f, theta, h_eps, h_dry, ws;
    int side_kind[4]; /* N, S, E, W */
    int solver;       /* 0 thomas, 1 cr */
    int cross_correction;
} orc_config;

typedef struct {
    double t, dt;
    int euler;
    int pad_;
    double wc, wp, wp2; /* ab3_weights (multistep.py:118-136) */
    double sc, sp, sp2; /* increment_weights (multistep.py:200-228) */
    double eta_t[4], flux_t[4];     /* maker_surface_flux at t, per side */
    double eta_n[4], flux_n[4];     /* at t + dt */
    const double *sponge_fac[4];    /* per side, band cells in index order */
    int sponge_lo[4], sponge_len[4];
} orc_params;

typedef struct {
    double max_rate, max_speed, max_depth, max_dev, clamped;
    int64_t stage_bad[5]; /* first row-major interior index or -1: e,f,g,fstar,gstar */
    int64_t state_bad[3]; /* w, P, Q of the new state */
} orc_result;

typedef struct {
    orc_config cfg;
    long npad;
    double *bed_eff, *depth, *ddx, *ddy, *bfx, *bfy, *rest;
    double *ax, *bx, *cx, *ay_t, *by_t, *cy_t;
    double *w, *p, *q;          /* current state */
    double *nw, *np_, *nq;      /* pending new state */
    double *hist[4][5];         /* ring slots */
    int head;                   /* slot holding the newest committed level */
    int nlev;
    int pend_slot;
    double *faces[12], *fx[3], *fy[3], *eta;
    double *ustar, *vstar, *base_u, *base_v, *us, *vs, *p1, *q1, *fsp, *gsp, *tmp_t, *out_t;
} orc_sim;

static double *dalloc(long n) { return (double *)calloc((size_t)n, sizeof(double)); }

/* implicit.py:84-90 */
static void coefficients(double d, double slope, double delta2, double six_delta, double bp13,
                         double *a, double *b, double *c)
{
    double curv = bp13 * d * d / delta2;
    double drift = d * slope / six_delta;
    *a = drift - curv;
    *b = 1.0 + 2.0 * curv;
    *c = -drift - curv;
}

orc_sim *orc_create(const orc_config *cfg, const double *bed_eff, const double *depth,
                    const double *ddx, const double *ddy, const double *bfx,
                    const double *bfy)
{
    orc_sim *s = (orc_sim *)calloc(1, sizeof(orc_sim));
    s->cfg = *cfg;
    int nx = cfg->nx, ny = cfg->ny, nxt = nx + 4, nyt = ny + 4;
    long np = (long)nxt * nyt, ni = (long)nx * ny;
    s->npad = np;
    s->bed_eff = dalloc(np); memcpy(s->bed_eff, bed_eff, sizeof(double) * np);
    s->depth = dalloc(np); memcpy(s->depth, depth, sizeof(double) * np);
    s->ddx = dalloc(np); memcpy(s->ddx, ddx, sizeof(double) * np);
    s->ddy = dalloc(np); memcpy(s->ddy, ddy, sizeof(double) * np);
    s->bfx = dalloc((long)nyt * (nxt - 1)); memcpy(s->bfx, bfx, sizeof(double) * nyt * (nxt - 1));
    s->bfy = dalloc((long)(nyt - 1) * nxt); memcpy(s->bfy, bfy, sizeof(double) * (nyt - 1) * nxt);
    s->rest = dalloc(np);
    for (long k = 0; k < np; k++) s->rest[k] = cfg->ws > bed_eff[k] ? cfg->ws : bed_eff[k];
    /* implicit.py:93-119: x rows, y stored transposed (column-major lines) */
    s->ax = dalloc(ni); s->bx = dalloc(ni); s->cx = dalloc(ni);
    s->ay_t = dalloc(ni); s->by_t = dalloc(ni); s->cy_t = dalloc(ni);
    double six_dx = 6.0 * cfg->dx, six_dy = 6.0 * cfg->dy;
    for (int jj = 0; jj < ny; jj++)
        for (int ii = 0; ii < nx; ii++) {
            long c = (long)(jj + GL) * nxt + ii + GL, o = (long)jj * nx + ii,
                 t = (long)ii * ny + jj;
            coefficients(depth[c], ddx[c], cfg->dx2, six_dx, cfg->bp13, &s->ax[o], &s->bx[o],
                         &s->cx[o]);
            coefficients(depth[c], ddy[c], cfg->dy2, six_dy, cfg->bp13, &s->ay_t[t],
                         &s->by_t[t], &s->cy_t[t]);
        }
    s->w = dalloc(np); s->p = dalloc(np); s->q = dalloc(np);
    s->nw = dalloc(np); s->np_ = dalloc(np); s->nq = dalloc(np);
    for (int k = 0; k < 4; k++)
        for (int f = 0; f < 5; f++) s->hist[k][f] = dalloc(ni);
    s->head = 0;
    s->nlev = 0;
    for (int k = 0; k < 12; k++) s->faces[k] = dalloc(np);
    for (int k = 0; k < 3; k++) {
        s->fx[k] = dalloc((long)ny * (nx + 1));
        s->fy[k] = dalloc((long)(ny + 1) * nx);
    }
    s->eta = dalloc(np);
    s->ustar = dalloc(ni); s->vstar = dalloc(ni); s->base_u = dalloc(ni); s->base_v = dalloc(ni);
    s->us = dalloc(ni); s->vs = dalloc(ni); s->p1 = dalloc(ni); s->q1 = dalloc(ni);
    s->fsp = dalloc(ni); s->gsp = dalloc(ni); s->tmp_t = dalloc(ni); s->out_t = dalloc(ni);
    return s;
}

void orc_destroy(orc_sim *s)
{
    if (!s) return;
    double *all[] = {s->bed_eff, s->depth, s->ddx, s->ddy, s->bfx, s->bfy, s->rest, s->ax, s->bx,
                     s->cx, s->ay_t, s->by_t, s->cy_t, s->w, s->p, s->q, s->nw, s->np_, s->nq,
                     s->eta, s->ustar, s->vstar, s->base_u, s->base_v, s->us, s->vs, s->p1,
                     s->q1, s->fsp, s->gsp, s->tmp_t, s->out_t};
    for (size_t k = 0; k < sizeof(all) / sizeof(all[0]); k++) free(all[k]);
    for (int k = 0; k < 4; k++)
        for (int f = 0; f < 5; f++) free(s->hist[k][f]);
    for (int k = 0; k < 12; k++) free(s->faces[k]);
    for (int k = 0; k < 3; k++) { free(s->fx[k]); free(s->fy[k]); }
    free(s);
}

void orc_set_state(orc_sim *s, const double *w, const double *p, const double *q)
{
    memcpy(s->w, w, sizeof(double) * s->npad);
    memcpy(s->p, p, sizeof(double) * s->npad);
    memcpy(s->q, q, sizeof(double) * s->npad);
}

void orc_get_state(const orc_sim *s, int pending, double *w, double *p, double *q)
{
    memcpy(w, pending ? s->nw : s->w, sizeof(double) * s->npad);
    memcpy(p, pending ? s->np_ : s->p, sizeof(double) * s->npad);
    memcpy(q, pending ? s->nq : s->q, sizeof(double) * s->npad);
}

/* newest-first history level k (0 newest) field f (e,f,g,fstar,gstar) */
void orc_get_history(const orc_sim *s, int k, int f, double *out)
{
    int slot = (s->head - k + 4) % 4;
    memcpy(out, s->hist[slot][f], sizeof(double) * s->cfg.nx * s->cfg.ny);
}

/* boundary.py:206-232 */
static void wall(const orc_sim *s, double *w, double *p, double *q, int side)
{
    int nxt = s->cfg.nx + 4, nyt = s->cfg.ny + 4;
    if (side == SIDE_W || side == SIDE_E) {
        double *arr[3] = {w, q, p};
        double sg[3] = {1.0, 1.0, -1.0};
        for (int k = 0; k < 3; k++)
            for (int j = 0; j < nyt; j++) {
                double *r = arr[k] + (long)j * nxt;
                if (side == SIDE_W) {
                    r[GL - 1] = sg[k] * r[GL];
                    r[GL - 2] = sg[k] * r[GL + 1];
                } else {
                    r[nxt - GL] = sg[k] * r[nxt - GL - 1];
                    r[nxt - GL + 1] = sg[k] * r[nxt - GL - 2];
                }
            }
    } else {
        double *arr[3] = {w, p, q};
        double sg[3] = {1.0, 1.0, -1.0};
        for (int k = 0; k < 3; k++) {
            double *a = arr[k];
            for (int i = 0; i < nxt; i++) {
                if (side == SIDE_S) {
                    a[(long)(GL - 1) * nxt + i] = sg[k] * a[(long)GL * nxt + i];
                    a[(long)(GL - 2) * nxt + i] = sg[k] * a[(long)(GL + 1) * nxt + i];
                } else {
                    a[(long)(nyt - GL) * nxt + i] = sg[k] * a[(long)(nyt - GL - 1) * nxt + i];
                    a[(long)(nyt - GL + 1) * nxt + i] = sg[k] * a[(long)(nyt - GL - 2) * nxt + i];
                }
            }
        }
    }
}

/* boundary.py:235-261 */
static void maker(const orc_sim *s, double *w, double *p, double *q, int side, double eta,
                  double flux)
{
    int nxt = s->cfg.nx + 4, nyt = s->cfg.ny + 4;
    double wv = s->cfg.ws + eta;
    for (int j = 0; j < nyt; j++)
        for (int i = 0; i < nxt; i++) {
            long c = (long)j * nxt + i;
            int in = 0;
            double pv = 0.0, qv = 0.0;
            if (side == SIDE_W && i < GL) { in = 1; pv = flux; }
            if (side == SIDE_E && i >= nxt - GL) { in = 1; pv = -flux; }
            if (side == SIDE_S && j < GL) { in = 1; qv = flux; }
            if (side == SIDE_N && j >= nyt - GL) { in = 1; qv = -flux; }
            if (in) { w[c] = wv; p[c] = pv; q[c] = qv; }
        }
}

/* Boundaries.apply_ghosts, boundary.py:316-323: order N, S, E, W */
static void ghosts(const orc_sim *s, double *w, double *p, double *q, const double *eta,
                   const double *flux)
{
    for (int side = 0; side < 4; side++) {
        if (s->cfg.side_kind[side] == KIND_MAKER)
            maker(s, w, p, q, side, eta[side], flux[side]);
        else
            wall(s, w, p, q, side);
    }
}

static int64_t first_nonfinite(const double *a, int ny, int nx, long pitch, long off)
{
    for (int jj = 0; jj < ny; jj++)
        for (int ii = 0; ii < nx; ii++)
            if (!isfinite(a[off + (long)jj * pitch + ii])) return (int64_t)jj * nx + ii;
    return -1;
}

/* implicit.py:173-194 with the chosen batched solver */
static int solve_momentum(orc_sim *s, const double *us, const double *vs, const double *pg_w,
                          const double *pg_e, const double *qg_s, const double *qg_n,
                          double *p_out, double *q_out)
{
    int nx = s->cfg.nx, ny = s->cfg.ny;
    long ni = (long)nx * ny;
    int (*solver)(int, int, const double *, const double *, const double *, const double *,
                  double *) = s->cfg.solver == 1 ? orc_cr_batch : orc_thomas_batch;
    /* x: folded = rhs copy; [:,0] -= ax[:,0]*gw; [:,-1] -= cx[:,-1]*ge */
    memcpy(s->tmp_t, us, sizeof(double) * ni);
    for (int jj = 0; jj < ny; jj++) {
        s->tmp_t[(long)jj * nx] -= s->ax[(long)jj * nx] * pg_w[jj];
        s->tmp_t[(long)jj * nx + nx - 1] -= s->cx[(long)jj * nx + nx - 1] * pg_e[jj];
    }
    int rc = solver(ny, nx, s->ax, s->bx, s->cx, s->tmp_t, p_out);
    if (rc) return rc;
    /* y: transposed */
    for (int jj = 0; jj < ny; jj++)
        for (int ii = 0; ii < nx; ii++) s->tmp_t[(long)ii * ny + jj] = vs[(long)jj * nx + ii];
    for (int ii = 0; ii < nx; ii++) {
        s->tmp_t[(long)ii * ny] -= s->ay_t[(long)ii * ny] * qg_s[ii];
        s->tmp_t[(long)ii * ny + ny - 1] -= s->cy_t[(long)ii * ny + ny - 1] * qg_n[ii];
    }
    rc = solver(nx, ny, s->ay_t, s->by_t, s->cy_t, s->tmp_t, s->out_t);
    if (rc) return rc;
    for (int jj = 0; jj < ny; jj++)
        for (int ii = 0; ii < nx; ii++) q_out[(long)jj * nx + ii] = s->out_t[(long)ii * ny + jj];
    return 0;
}

/*
 * One step into the pending buffers (stepper.py:225-305 minus the host-side
 * controller).  Returns 0 on success, 1 if a stage value is non-finite (the
 * reference raises before pushing history: nothing is pending), or the
 * solver's error code: -1 a zero pivot (Thomas) / zero pivot in reduction
 * (CR), -2 a zero CR core determinant, -3 a zero pivot in CR back
 * substitution.  The caller commits with orc_commit.
 */
int orc_step(orc_sim *s, const orc_params *pr, orc_result *res)
{
    const orc_config *cf = &s->cfg;
    int nx = cf->nx, ny = cf->ny, nxt = nx + 4, nyt = ny + 4;
    long ni = (long)nx * ny, np = s->npad;
    (void)nyt;
    memset(res, 0, sizeof(*res));
    for (int k = 0; k < 5; k++) res->stage_bad[k] = -1;
    for (int k = 0; k < 3; k++) res->state_bad[k] = -1;

    /* 1. ghosts at t (stepper.py:233) */
    ghosts(s, s->w, s->p, s->q, pr->eta_t, pr->flux_t);

    /* 2. stages (dispersion.py:67-99) into the next ring slot */
    int slot = (s->head + 1) % 4;
    double *E = s->hist[slot][0], *F = s->hist[slot][1], *G = s->hist[slot][2],
           *FS = s->hist[slot][3], *GS = s->hist[slot][4];
    double **fc = s->faces;
    orc_faces_x(ny + 4, nxt, s->w, s->p, s->q, s->bfx, cf->theta, fc[0], fc[1], fc[2], fc[3],
                fc[4], fc[5]);
    orc_faces_y(ny + 4, nxt, s->w, s->p, s->q, s->bfy, cf->theta, fc[6], fc[7], fc[8], fc[9],
                fc[10], fc[11]);
    orc_flux_x(ny, nx, fc[0], fc[1], fc[2], fc[3], fc[4], fc[5], s->bfx, cf->g, cf->h_eps,
               s->fx[0], s->fx[1], s->fx[2]);
    orc_flux_y(ny, nx, fc[6], fc[7], fc[8], fc[9], fc[10], fc[11], s->bfy, cf->g, cf->h_eps,
               s->fy[0], s->fy[1], s->fy[2]);
    orc_fv_rates(ny, nx, s->fx[0], s->fx[1], s->fx[2], s->fy[0], s->fy[1], s->fy[2], s->w, s->p,
                 s->q, s->bed_eff, s->bfx, s->bfy, cf->g, cf->c_f, cf->h_eps, cf->dx, cf->dy, E,
                 F, G);
    for (long k = 0; k < np; k++) s->eta[k] = (s->w[k] - s->bed_eff[k]) - s->depth[k];
    orc_dispersive_rates(ny, nx, s->eta, s->depth, s->ddx, s->ddy, cf->g, cf->b_disp, cf->dx,
                         cf->dy, F, G);
    orc_cross_rates(ny, nx, s->p, s->q, s->depth, s->ddx, s->ddy, cf->bp13, cf->dx, cf->dy, FS,
                    GS);
    int bad = 0;
    for (int f = 0; f < 5; f++) {
        res->stage_bad[f] = first_nonfinite(s->hist[slot][f], ny, nx, nx, 0);
        if (res->stage_bad[f] >= 0) bad = 1;
    }
    if (bad) return 1;
    s->pend_slot = slot;

    /* 3. U*, V* (dispersion.py:120-149) */
    double two_dx = 2.0 * cf->dx, two_dy = 2.0 * cf->dy;
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj < ny; jj++)
        for (int ii = 0; ii < nx; ii++) {
            long c = (long)(jj + GL) * nxt + ii + GL, o = (long)jj * nx + ii;
            double d = s->depth[c];
            double pc = s->p[c], pw = s->p[c - 1], pe = s->p[c + 1];
            double p_x = (pe - pw) / two_dx;
            double p_xx = (pe - 2.0 * pc + pw) / cf->dx2;
            s->ustar[o] = pc - (d * s->ddx[c] / 3.0) * p_x - cf->bp13 * d * d * p_xx;
            double qc = s->q[c], qs = s->q[c - nxt], qn = s->q[c + nxt];
            double q_y = (qn - qs) / two_dy;
            double q_yy = (qn - 2.0 * qc + qs) / cf->dy2;
            s->vstar[o] = qc - (d * s->ddy[c] / 3.0) * q_y - cf->bp13 * d * d * q_yy;
        }

    /* 4. predictors (stepper.py:239-250; multistep.py:139-153) */
    int s1 = slot, s2 = (slot + 3) % 4, s3 = (slot + 2) % 4;
    memcpy(s->nw, s->w, sizeof(double) * np);
    memcpy(s->np_, s->p, sizeof(double) * np);
    memcpy(s->nq, s->q, sizeof(double) * np);
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj < ny; jj++)
        for (int ii = 0; ii < nx; ii++) {
            long c = (long)(jj + GL) * nxt + ii + GL, o = (long)jj * nx + ii;
            if (pr->euler) {
                s->nw[c] = s->w[c] + pr->dt * s->hist[s1][0][o];
                s->base_u[o] = s->ustar[o] + pr->dt * s->hist[s1][1][o];
                s->base_v[o] = s->vstar[o] + pr->dt * s->hist[s1][2][o];
                s->us[o] = s->base_u[o];
                s->vs[o] = s->base_v[o];
            } else {
                s->nw[c] = s->w[c] + (pr->wc * s->hist[s1][0][o] + pr->wp * s->hist[s2][0][o] +
                                      pr->wp2 * s->hist[s3][0][o]);
                s->base_u[o] = s->ustar[o] + (pr->wc * s->hist[s1][1][o] +
                                              pr->wp * s->hist[s2][1][o] +
                                              pr->wp2 * s->hist[s3][1][o]);
                s->base_v[o] = s->vstar[o] + (pr->wc * s->hist[s1][2][o] +
                                              pr->wp * s->hist[s2][2][o] +
                                              pr->wp2 * s->hist[s3][2][o]);
                s->us[o] = s->base_u[o] + (pr->sc * s->hist[s1][3][o] +
                                           pr->sp * s->hist[s2][3][o] +
                                           pr->sp2 * s->hist[s3][3][o]);
                s->vs[o] = s->base_v[o] + (pr->sc * s->hist[s1][4][o] +
                                           pr->sp * s->hist[s2][4][o] +
                                           pr->sp2 * s->hist[s3][4][o]);
            }
        }

    /* 5. ghosts of the new state at t+dt (stepper.py:252-254) */
    ghosts(s, s->nw, s->np_, s->nq, pr->eta_n, pr->flux_n);
    double *pgw = (double *)malloc(sizeof(double) * ny), *pge = (double *)malloc(sizeof(double) * ny);
    double *qgs = (double *)malloc(sizeof(double) * nx), *qgn = (double *)malloc(sizeof(double) * nx);
    for (int jj = 0; jj < ny; jj++) {
        pgw[jj] = s->np_[(long)(jj + GL) * nxt + GL - 1];
        pge[jj] = s->np_[(long)(jj + GL) * nxt + nx + GL];
    }
    for (int ii = 0; ii < nx; ii++) {
        qgs[ii] = s->nq[(long)(GL - 1) * nxt + ii + GL];
        qgn[ii] = s->nq[(long)(ny + GL) * nxt + ii + GL];
    }

    /* 6. first solve (stepper.py:255-261) */
    int rc = solve_momentum(s, s->us, s->vs, pgw, pge, qgs, qgn, s->p1, s->q1);
    /* 7. cross correction (stepper.py:262-280) */
    if (rc == 0 && cf->cross_correction) {
        for (int jj = 0; jj < ny; jj++)
            for (int ii = 0; ii < nx; ii++) {
                long c = (long)(jj + GL) * nxt + ii + GL, o = (long)jj * nx + ii;
                s->np_[c] = s->p1[o];
                s->nq[c] = s->q1[o];
            }
        orc_cross_rates(ny, nx, s->np_, s->nq, s->depth, s->ddx, s->ddy, cf->bp13, cf->dx,
                        cf->dy, s->fsp, s->gsp);
        for (long o = 0; o < ni; o++) {
            s->us[o] = s->base_u[o] + (s->fsp[o] - FS[o]);
            s->vs[o] = s->base_v[o] + (s->gsp[o] - GS[o]);
        }
        rc = solve_momentum(s, s->us, s->vs, pgw, pge, qgs, qgn, s->p1, s->q1);
    }
    free(pgw); free(pge); free(qgs); free(qgn);
    if (rc) return rc; /* -1 zero pivot / reduction, -2 core determinant, -3 back substitution */

    /* 8. clamp, set momenta, film cutoff (stepper.py:281-292) */
    double *rowsum = (double *)malloc(sizeof(double) * ny);
#pragma omp parallel for schedule(static)
    for (int jj = 0; jj < ny; jj++) {
        double acc = 0.0;
        for (int ii = 0; ii < nx; ii++) {
            long c = (long)(jj + GL) * nxt + ii + GL, o = (long)jj * nx + ii;
            double be = s->bed_eff[c];
            double def = be - s->nw[c];
            if (def > 0.0 || def != def) acc += def; /* np.maximum(def, 0) */
            double wv = s->nw[c];
            s->nw[c] = (wv >= be || wv != wv) ? wv : be; /* np.maximum propagates NaN */
            s->np_[c] = s->p1[o];
            s->nq[c] = s->q1[o];
            if (cf->h_dry > 0.0 && (s->nw[c] - be) < cf->h_dry) {
                s->np_[c] = 0.0;
                s->nq[c] = 0.0;
            }
        }
        rowsum[jj] = acc;
    }
    double clamped = 0.0;
    for (int jj = 0; jj < ny; jj++) clamped += rowsum[jj];
    free(rowsum);
    res->clamped = clamped;

    /* 9. sponge bands, order N, S, E, W (boundary.py:264-300, :325-330) */
    for (int side = 0; side < 4; side++) {
        if (cf->side_kind[side] != KIND_SPONGE || pr->sponge_len[side] <= 0) continue;
        const double *fac = pr->sponge_fac[side];
        int lo = pr->sponge_lo[side], len = pr->sponge_len[side];
        for (int jj = 0; jj < ny; jj++)
            for (int ii = 0; ii < nx; ii++) {
                int k;
                if (side == SIDE_E || side == SIDE_W) k = ii - lo; else k = jj - lo;
                if (k < 0 || k >= len) continue;
                long c = (long)(jj + GL) * nxt + ii + GL;
                double f = fac[k];
                double rest = s->rest[c];
                s->nw[c] = rest + (s->nw[c] - rest) * f;
                s->np_[c] *= f;
                s->nq[c] *= f;
            }
    }

    /* 10. blow-up deviation, non-finite scan, extrema (stepper.py:295-305) */
    double dev = 0.0;
    int devnan = 0;
    for (int jj = 0; jj < ny; jj++)
        for (int ii = 0; ii < nx; ii++) {
            long c = (long)(jj + GL) * nxt + ii + GL;
            double d = fabs(s->nw[c] - s->rest[c]);
            if (d != d) devnan = 1;
            else if (d > dev) dev = d;
        }
    res->max_dev = devnan ? NAN : dev;
    res->state_bad[0] = first_nonfinite(s->nw, ny, nx, nxt, (long)GL * nxt + GL);
    res->state_bad[1] = first_nonfinite(s->np_, ny, nx, nxt, (long)GL * nxt + GL);
    res->state_bad[2] = first_nonfinite(s->nq, ny, nx, nxt, (long)GL * nxt + GL);
    double ext[3];
    orc_speed_extrema(ny, nx, s->nw, s->np_, s->nq, s->bed_eff, cf->g, cf->h_eps, cf->dx, cf->dy,
                      ext);
    res->max_rate = ext[0];
    res->max_speed = ext[1];
    res->max_depth = ext[2];
    return 0;
}

/* accept the pending step: state <- new state, history ring advances */
void orc_commit(orc_sim *s)
{
    double *t;
    t = s->w; s->w = s->nw; s->nw = t;
    t = s->p; s->p = s->np_; s->np_ = t;
    t = s->q; s->q = s->nq; s->nq = t;
    s->head = s->pend_slot;
    if (s->nlev < 3) s->nlev++;
}

/* speed_extrema of the current state (used at construction, stepper.py:210) */
void orc_state_extrema(const orc_sim *s, double *out)
{
    orc_speed_extrema(s->cfg.ny, s->cfg.nx, s->w, s->p, s->q, s->bed_eff, s->cfg.g, s->cfg.h_eps,
                      s->cfg.dx, s->cfg.dy, out);
}

void orc_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
