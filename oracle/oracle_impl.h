/* TEST INFRASTRUCTURE — included twice by oracle.c (REAL = double, float).
 *
 * Scalar restatement of one reference translation, one request at a time,
 * bit-mirroring the arithmetic the reference performs when GCC builds it with
 * `-mfma -ffp-contract=fast` (oracle/Makefile, pairing B of SURVEY §7.1):
 *   contractions   acc = fma(A, x, acc), k ascending from acc = +0
 *                  (kernels.cpp:38-46, 122-131, 172-195)
 *   rotations      re' = s*fma(a, c, -(b*sm)),  im' = s*fma(a, sm, b*c)
 *                  (kernels.cpp:198-221)
 *   angle tables   c' = fma(c, c1, -(s*s1)),    s' = fma(s, c1, c*s1)
 *                  (pipeline.cpp:62-79)
 * Structural zeros of the chequerboard are skipped exactly as the packed
 * stream skips them (operators.cpp:68-89, kernels.cpp:38-46).
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SUFFIX)

/* geometry.cpp:11-30 */
static int FN(angles)(const REAL* r, REAL* rn, REAL* ca, REAL* sa, REAL* cb,
                      REAL* sb) {
    const REAL h = HYPOT(r[0], r[1]);
    const REAL n = HYPOT(h, r[2]);
    if (n < REAL_MIN) return ORC_DOMAIN_ERROR;
    *rn = n;
    if (h == (REAL)0) {
        *ca = (REAL)1;
        *sa = (REAL)0;
    } else {
        *ca = r[1] / h;
        *sa = r[0] / h;
    }
    *cb = r[2] / n;
    *sb = -h / n;
    return 0;
}

/* y[i] = sum_{k asc, (i+k)%2 == parity} a(i,k) * x[k]; a(i,k) = A[i*rows+k]
 * or A[k*rows+i] when transposed (operators.cpp:160-163, kernels.cpp:102-114) */
static void FN(swap_apply)(const double* A, int rows, int parity, int transposed,
                           const REAL* x, REAL* y) {
    for (int i = 0; i < rows; ++i) {
        REAL acc = (REAL)0;
        for (int k = 0; k < rows; ++k) {
            if (((i + k) & 1) != parity) continue;
            const REAL a = (REAL)(transposed ? A[k * rows + i] : A[i * rows + k]);
            acc = FMA(a, x[k], acc);
        }
        y[i] = acc;
    }
}

/* kernels.cpp:198-221, scale == NULL variant when has_scale == 0 */
static void FN(rotate)(REAL* re, REAL* im, int rows, int has_scale, REAL scale,
                       const REAL* c, const REAL* s) {
    for (int m = 0; m < rows; ++m) {
        const REAL a = re[m], b = im[m];
        const REAL nr = FMA(a, c[m], -(b * s[m]));
        const REAL ni = FMA(a, s[m], b * c[m]);
        re[m] = has_scale ? scale * nr : nr;
        im[m] = has_scale ? scale * ni : ni;
    }
}

/* pipeline.cpp:118-136 plus the halving/doubling of :155-157 / :247-249 */
static void FN(swap_pass)(const struct orc_tables* t, int n, int local_side,
                          const REAL* cb, const REAL* sb, REAL* re, REAL* im,
                          REAL* tre, REAL* tim) {
    const int rows = n + 1;
    const double* F = t->f[n];
    const double* G = t->g[n];
    const int fp = n & 1, gp = (n + 1) & 1;
    if (local_side) re[0] *= (REAL)0.5;
    FN(swap_apply)(F, rows, fp, local_side, re, tre);
    FN(swap_apply)(G, rows, gp, local_side, im, tim);
    FN(rotate)(tre, tim, rows, 0, (REAL)1, cb, sb);
    FN(swap_apply)(F, rows, fp, local_side, tre, re);
    FN(swap_apply)(G, rows, gp, local_side, tim, im);
    if (local_side) re[0] *= (REAL)2;
}

/* One request. kind: 0 m2l, 1 m2m, 2 l2l (pipeline.cpp:33-49). */
static int FN(translate_one)(const struct orc_tables* t, int kind, int p_in,
                             int p_out, const REAL* src, const REAL* shift,
                             REAL* dst) {
    enum { PM = ORC_MAX_ORDER };
    REAL rn, c1a, s1a, c1b, s1b;
    const int st = FN(angles)(shift, &rn, &c1a, &s1a, &c1b, &s1b);
    if (st) return st;
    const int p_rot = p_in > p_out ? p_in : p_out;

    /* pipeline.cpp:52-91 */
    REAL ca[PM], sa[PM], nsa[PM], cb[PM], sb[PM], nsb[PM], pw[PM + 1], ipw[PM + 1];
    {
        REAL c = 1, s = 0, d = 1, e = 0;
        for (int m = 0; m < p_rot; ++m) {
            ca[m] = c; sa[m] = s; nsa[m] = -s;
            cb[m] = d; sb[m] = e; nsb[m] = -e;
            const REAL nc = FMA(c, c1a, -(s * s1a));
            const REAL ns = FMA(s, c1a, c * s1a);
            c = nc; s = ns;
            const REAL nd = FMA(d, c1b, -(e * s1b));
            const REAL ne = FMA(e, c1b, d * s1b);
            d = nd; e = ne;
        }
        REAL p = 1, q = 1;
        const REAL inv = (REAL)1 / rn;
        for (int n = 0; n <= p_rot; ++n) {
            pw[n] = p; ipw[n] = q;
            p *= rn; q *= inv;
        }
    }

    const int src_local = kind == 2;
    const int dst_local = kind != 1;
    const int cols = p_in < p_out ? p_in : p_out;

    /* translation columns: tin[m][k] = row (m+k) coefficient m */
    static _Thread_local REAL tin_re[PM][PM], tin_im[PM][PM];
    static _Thread_local REAL tout_re[PM][PM], tout_im[PM][PM];
    REAL re[PM], im[PM], tre[PM], tim[PM];

    /* forward pass, pipeline.cpp:142-169 */
    for (int n = 0; n < p_in; ++n) {
        for (int m = 0; m <= n; ++m) {
            re[m] = src[n * (n + 1) + 2 * m];
            im[m] = src[n * (n + 1) + 2 * m + 1];
        }
        FN(rotate)(re, im, n + 1, 1, src_local ? pw[n] : ipw[n + 1], ca, sa);
        FN(swap_pass)(t, n, src_local, cb, sb, re, im, tre, tim);
        for (int m = 0; m <= n; ++m) {
            tin_re[m][n - m] = re[m];
            tin_im[m][n - m] = im[m];
        }
    }

    /* z-axis step */
    for (int m = 0; m < cols; ++m) {
        const int kin = p_in - m, kout = p_out - m;
        for (int i = 0; i < kout; ++i) {
            REAL ar = 0, ai = 0;
            if (kind == 0) { /* pipeline.cpp:171-186, kernels.cpp:118-167 */
                const REAL* f = FN(t->fac) + 2 * m + i;
                for (int k = 0; k < kin; ++k) {
                    ar = FMA(f[k], tin_re[m][k], ar);
                    ai = FMA(f[k], tin_im[m][k], ai);
                }
            } else if (kind == 1) { /* lower, w[d] = (-1)^d / d!, kernels.cpp:169-182 */
                const int klim = i < kin - 1 ? i : kin - 1;
                for (int k = 0; k <= klim; ++k) {
                    const int d = i - k;
                    const REAL w = (d & 1) ? -FN(t->inv)[d] : FN(t->inv)[d];
                    ar = FMA(w, tin_re[m][k], ar);
                    ai = FMA(w, tin_im[m][k], ai);
                }
            } else { /* upper, w[d] = 1 / d!, kernels.cpp:184-196 */
                for (int k = i; k < kin; ++k) {
                    const REAL w = FN(t->inv)[k - i];
                    ar = FMA(w, tin_re[m][k], ar);
                    ai = FMA(w, tin_im[m][k], ai);
                }
            }
            tout_re[m][i] = ar;
            tout_im[m][i] = ai;
        }
    }

    /* backward pass, pipeline.cpp:216-267 */
    for (int n = 0; n < p_out; ++n) {
        const int mmax = n < cols - 1 ? n : cols - 1;
        for (int m = 0; m <= n; ++m) { re[m] = 0; im[m] = 0; }
        for (int m = 0; m <= mmax; ++m) {
            const int neg = kind == 0 && ((n + m) & 1);
            re[m] = neg ? -tout_re[m][n - m] : tout_re[m][n - m];
            im[m] = neg ? -tout_im[m][n - m] : tout_im[m][n - m];
        }
        FN(swap_pass)(t, n, dst_local, cb, nsb, re, im, tre, tim);
        FN(rotate)(re, im, n + 1, 1, dst_local ? ipw[n] : pw[n + 1], ca, nsa);
        for (int m = 0; m <= n; ++m) {
            dst[n * (n + 1) + 2 * m] = re[m];
            dst[n * (n + 1) + 2 * m + 1] = im[m];
        }
    }
    return 0;
}

/* run_batch validation, pipeline.cpp:280-298: everything is checked before
 * any output is written. */
static int FN(validate)(long n, const int* p_in, const int* p_out, int p_in_u,
                        int p_out_u, const REAL* shifts, int* pmax_out) {
    int pmax = 0;
    for (long i = 0; i < n; ++i) {
        const int pi = p_in ? p_in[i] : p_in_u;
        const int po = p_out ? p_out[i] : p_out_u;
        if (pi < 1 || po < 1) return ORC_INVALID_ARGUMENT;
        const int need = pi > po ? pi : po;
        if (need > FN(orc_max_order)()) return ORC_INVALID_ARGUMENT;
        if (need > pmax) pmax = need;
        /* norm(): std::hypot(x, y, z), solid.hpp:21-23 */
        const REAL* r = shifts + 3 * i;
        const REAL ax = FABS(r[0]), ay = FABS(r[1]), az = FABS(r[2]);
        REAL mx = ax > ay ? ax : ay;
        if (az > mx) mx = az;
        if (mx < REAL_MIN) {
            /* all components subnormal or zero: |r| may still reach REAL_MIN */
            if (HYPOT(HYPOT(r[0], r[1]), r[2]) < REAL_MIN) return ORC_DOMAIN_ERROR;
        }
    }
    *pmax_out = pmax;
    return 0;
}

int FN(orc_translate)(int kind, long n, int p_in, int p_out, const REAL* in,
                      const REAL* shifts, REAL* out) {
    if (n <= 0) return 0;
    if (!in || !shifts || !out || kind < 0 || kind > 2) return ORC_INVALID_ARGUMENT;
    int pmax;
    const int st = FN(validate)(n, 0, 0, p_in, p_out, shifts, &pmax);
    if (st) return st;
    const struct orc_tables* t = orc_tables_get(pmax);
    if (!t) return ORC_INVALID_ARGUMENT;
    const long si = (long)p_in * (p_in + 1), so = (long)p_out * (p_out + 1);
    for (long i = 0; i < n; ++i) {
        const int s = FN(translate_one)(t, kind, p_in, p_out, in + i * si,
                                        shifts + 3 * i, out + i * so);
        if (s) return s;
    }
    return 0;
}

int FN(orc_translate_mixed)(int kind, long n, const int* p_in, const int* p_out,
                            const REAL* in, const long* in_off,
                            const REAL* shifts, REAL* out, const long* out_off) {
    if (n <= 0) return 0;
    if (!in || !shifts || !out || !p_in || !p_out || !in_off || !out_off ||
        kind < 0 || kind > 2)
        return ORC_INVALID_ARGUMENT;
    int pmax;
    const int st = FN(validate)(n, p_in, p_out, 0, 0, shifts, &pmax);
    if (st) return st;
    const struct orc_tables* t = orc_tables_get(pmax);
    if (!t) return ORC_INVALID_ARGUMENT;
    for (long i = 0; i < n; ++i) {
        const int s = FN(translate_one)(t, kind, p_in[i], p_out[i], in + in_off[i],
                                        shifts + 3 * i, out + out_off[i]);
        if (s) return s;
    }
    return 0;
}

int FN(orc_angles)(const REAL* r, REAL* out5) {
    return FN(angles)(r, out5, out5 + 1, out5 + 2, out5 + 3, out5 + 4);
}

#undef FN
#undef CAT
#undef CAT_
