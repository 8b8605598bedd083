/*
 * material_oracle.c -- CPU restatement of the reference's automatic
 * implicit-Euler material-law path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker for the CUDA material kernel
 * (paper_2006_04391_b200/csrc/material.cu).  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / reference arm
 * may load it.  The product path never links or calls it.
 *
 * It restates, operation by operation, the reference package gsmkit
 * (/root/reference/pkg/src/gsmkit) for
 *   StrategyConfig(strategy="automatic", integrator="implicit-euler"):
 *   - ad.py:46-131      Dual1 forward vector mode (payload arithmetic below)
 *   - ad.py:247-517     reverse expression nodes with recomputation: v()
 *                       re-evaluates a subtree, back(bv) pushes adjoints,
 *                       RLeaf accumulates, RConst drops (no tape)
 *   - gsm.py:62-79      dev_components / mises_components (guarded sqrt)
 *   - gsm.py:100-117    LinearElastic.omega
 *   - gsm.py:210-256    MichelSuquet.omega / psi / clamp_state
 *   - gsm.py:431-461    stress_generic / gen_stress_generic / flow_generic
 *   - gsm.py:494-518    rhs_and_jacobians (tangent-over-adjoint, W = 6 + m)
 *   - gsm.py:520-560    stress_and_tangent / elastic_tangent
 *   - odeint.py:241-304 MaterialStepProblem (ramp, rhs_and_jac, rhs_dual)
 *   - odeint.py:357-426 _newton_implicit_euler / implicit_euler_step
 *   - linalg.py:75-143  lu_factor / lu_solve_factored (partial pivoting)
 *   - evaluator.py:124-203 _evaluate_chunk (m == 0, dt == 0, clamp, sigma)
 * The expression trees are built in the same shape Python's operator
 * overloading builds them, so the floating-point operation sequence matches
 * the reference's (pinned against the npz fixtures in tests/golden made by the reference).
 *
 * Payloads are either plain doubles (has == 0) or Dual1 values with a
 * tangent of width g_W (has == 1), mirroring the mixed float / Dual1
 * arithmetic of the Python classes.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXW 13
#define MAXN 320

typedef struct {
    int has;
    double v;
    double d[MAXW];
} P;

static __thread int g_W = 0; /* tangent width of the sweep in progress */

static P pf(double v) { P r; r.has = 0; r.v = v; return r; }

/* ---------------------------------------------------------------- Dual1 ops
 * ad.py:64-127; float-op-Dual cases go through the reflected methods. */
static P p_add(P x, P y) {
    P r;
    if (x.has && y.has) {
        r.has = 1; r.v = x.v + y.v;
        for (int k = 0; k < g_W; ++k) r.d[k] = x.d[k] + y.d[k];
    } else if (x.has) {
        r = x; r.v = x.v + y.v;
    } else if (y.has) {
        r = y; r.v = y.v + x.v;
    } else {
        r = pf(x.v + y.v);
    }
    return r;
}

static P p_sub(P x, P y) {
    P r;
    if (x.has && y.has) {
        r.has = 1; r.v = x.v - y.v;
        for (int k = 0; k < g_W; ++k) r.d[k] = x.d[k] - y.d[k];
    } else if (x.has) {
        r = x; r.v = x.v - y.v;
    } else if (y.has) { /* Dual1.__rsub__ */
        r.has = 1; r.v = x.v - y.v;
        for (int k = 0; k < g_W; ++k) r.d[k] = -y.d[k];
    } else {
        r = pf(x.v - y.v);
    }
    return r;
}

static P p_mul(P x, P y) {
    P r;
    if (x.has && y.has) {
        r.has = 1; r.v = x.v * y.v;
        for (int k = 0; k < g_W; ++k) r.d[k] = x.d[k] * y.v + x.v * y.d[k];
    } else if (x.has) {
        r.has = 1; r.v = x.v * y.v;
        for (int k = 0; k < g_W; ++k) r.d[k] = x.d[k] * y.v;
    } else if (y.has) { /* __rmul__ = __mul__(self=y, o=x) */
        r.has = 1; r.v = y.v * x.v;
        for (int k = 0; k < g_W; ++k) r.d[k] = y.d[k] * x.v;
    } else {
        r = pf(x.v * y.v);
    }
    return r;
}

static P p_div(P x, P y) {
    P r;
    if (x.has && y.has) {
        double inv = 1.0 / y.v;
        r.has = 1; r.v = x.v * inv;
        for (int k = 0; k < g_W; ++k) r.d[k] = (x.d[k] - x.v * inv * y.d[k]) * inv;
    } else if (x.has) {
        r.has = 1; r.v = x.v / y.v;
        for (int k = 0; k < g_W; ++k) r.d[k] = x.d[k] / y.v;
    } else if (y.has) { /* __rtruediv__ */
        double inv = 1.0 / y.v;
        r.has = 1; r.v = x.v * inv;
        for (int k = 0; k < g_W; ++k) r.d[k] = -x.v * inv * inv * y.d[k];
    } else {
        r = pf(x.v / y.v);
    }
    return r;
}

static P p_neg(P x) {
    P r = x;
    r.v = -x.v;
    if (x.has) for (int k = 0; k < g_W; ++k) r.d[k] = -x.d[k];
    return r;
}

static P p_pow(P x, double c) {
    P r;
    r.has = x.has; r.v = pow(x.v, c);
    if (x.has) {
        double f = c * pow(x.v, c - 1.0);
        for (int k = 0; k < g_W; ++k) r.d[k] = f * x.d[k];
    }
    return r;
}

static P p_sqrt(P x) {
    P r;
    double s = sqrt(x.v);
    r.has = x.has; r.v = s;
    if (x.has) {
        double g = 0.5 / s;
        for (int k = 0; k < g_W; ++k) r.d[k] = g * x.d[k];
    }
    return r;
}

static P p_exp(P x) {
    P r;
    double e = exp(x.v);
    r.has = x.has; r.v = e;
    if (x.has) for (int k = 0; k < g_W; ++k) r.d[k] = e * x.d[k];
    return r;
}

static P p_log(P x) {
    P r;
    r.has = x.has; r.v = log(x.v);
    if (x.has) for (int k = 0; k < g_W; ++k) r.d[k] = x.d[k] / x.v;
    return r;
}

static double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : (v == 0.0 ? 0.0 : v)); }

static P p_abs(P x) {
    double s = sgn(x.v);
    P r;
    r.has = x.has; r.v = x.v * s;
    if (x.has) for (int k = 0; k < g_W; ++k) r.d[k] = x.d[k] * s;
    return r;
}

static P p_pos(P x) {
    if (x.has) { /* Dual1.pos, ad.py:113-115 */
        double gate = x.v > 0.0 ? 1.0 : 0.0;
        P r; r.has = 1; r.v = x.v * gate;
        for (int k = 0; k < g_W; ++k) r.d[k] = x.d[k] * gate;
        return r;
    }
    /* np.maximum(x, 0.0) propagates NaN */
    return pf(isnan(x.v) ? x.v : (x.v > 0.0 ? x.v : 0.0));
}

/* ---------------------------------------------------------------- reverse tree
 * ad.py:247-517.  Nodes live in a per-sweep pool; shared subexpressions
 * are shared node indices (Python shares the objects), and back()
 * visits them once per path like the reference. */
enum { N_LEAF, N_CONST, N_ADD, N_SUB, N_MUL, N_DIV, N_NEG, N_POW, N_SQRT, N_EXP, N_LOG, N_POS, N_ABS };

typedef struct {
    int op, a, b;
    double c;
    P val;   /* leaf / const payload */
    P adj;   /* leaf adjoint */
    int adj_set;
} Node;

typedef struct {
    Node n[MAXN];
    int count;
} Tree;

static int t_new(Tree *t, int op, int a, int b, double c) {
    Node *x = &t->n[t->count];
    x->op = op; x->a = a; x->b = b; x->c = c; x->adj_set = 0;
    return t->count++;
}
static int t_leaf(Tree *t, P v) { int i = t_new(t, N_LEAF, -1, -1, 0.0); t->n[i].val = v; return i; }
static int t_const(Tree *t, P v) { int i = t_new(t, N_CONST, -1, -1, 0.0); t->n[i].val = v; return i; }
static int t_cst(Tree *t, double v) { return t_const(t, pf(v)); }
static int t_add(Tree *t, int a, int b) { return t_new(t, N_ADD, a, b, 0.0); }
static int t_sub(Tree *t, int a, int b) { return t_new(t, N_SUB, a, b, 0.0); }
static int t_mul(Tree *t, int a, int b) { return t_new(t, N_MUL, a, b, 0.0); }
static int t_pow(Tree *t, int a, double c) { return t_new(t, N_POW, a, -1, c); }
static int t_sqrt(Tree *t, int a) { return t_new(t, N_SQRT, a, -1, 0.0); }
static int t_pos(Tree *t, int a) { return t_new(t, N_POS, a, -1, 0.0); }

static P t_v(const Tree *t, int i) {
    const Node *x = &t->n[i];
    switch (x->op) {
    case N_LEAF:
    case N_CONST: return x->val;
    case N_ADD: return p_add(t_v(t, x->a), t_v(t, x->b));
    case N_SUB: return p_sub(t_v(t, x->a), t_v(t, x->b));
    case N_MUL: return p_mul(t_v(t, x->a), t_v(t, x->b));
    case N_DIV: return p_div(t_v(t, x->a), t_v(t, x->b));
    case N_NEG: return p_neg(t_v(t, x->a));
    case N_POW: return p_pow(t_v(t, x->a), x->c);
    case N_SQRT: return p_sqrt(t_v(t, x->a));
    case N_EXP: return p_exp(t_v(t, x->a));
    case N_LOG: return p_log(t_v(t, x->a));
    case N_POS: return p_pos(t_v(t, x->a));
    case N_ABS: return p_abs(t_v(t, x->a));
    }
    return pf(NAN);
}

static void t_back(Tree *t, int i, P bv) {
    Node *x = &t->n[i];
    switch (x->op) {
    case N_LEAF: /* RLeaf.back, ad.py:339-340 */
        if (x->adj_set) x->adj = p_add(x->adj, bv);
        else { x->adj = bv; x->adj_set = 1; }
        return;
    case N_CONST: return;
    case N_ADD: t_back(t, x->a, bv); t_back(t, x->b, bv); return;
    case N_SUB: t_back(t, x->a, bv); t_back(t, x->b, p_neg(bv)); return;
    case N_MUL:
        t_back(t, x->a, p_mul(bv, t_v(t, x->b)));
        t_back(t, x->b, p_mul(bv, t_v(t, x->a)));
        return;
    case N_DIV: {
        P bval = t_v(t, x->b);
        t_back(t, x->a, p_div(bv, bval));
        t_back(t, x->b, p_div(p_mul(p_neg(bv), t_v(t, x->a)), p_mul(bval, bval)));
        return;
    }
    case N_NEG: t_back(t, x->a, p_neg(bv)); return;
    case N_POW: {
        P av = t_v(t, x->a);
        t_back(t, x->a, p_mul(bv, p_mul(pf(x->c), p_pow(av, x->c - 1.0))));
        return;
    }
    case N_SQRT: t_back(t, x->a, p_mul(bv, p_div(pf(0.5), p_sqrt(t_v(t, x->a))))); return;
    case N_EXP: t_back(t, x->a, p_mul(bv, p_exp(t_v(t, x->a)))); return;
    case N_LOG: t_back(t, x->a, p_div(bv, t_v(t, x->a))); return;
    case N_POS: {
        double gate = t_v(t, x->a).v > 0.0 ? 1.0 : 0.0;
        t_back(t, x->a, p_mul(bv, pf(gate)));
        return;
    }
    case N_ABS: t_back(t, x->a, p_mul(bv, pf(sgn(t_v(t, x->a).v)))); return;
    }
}

/* RLeaf.adjoint, ad.py:342-343 */
static P t_adjoint(const Tree *t, int i) {
    const Node *x = &t->n[i];
    if (x->adj_set) return x->adj;
    return p_mul(x->val, pf(0.0));
}

/* ---------------------------------------------------------------- laws */
typedef struct {
    int kind; /* 0 linear elastic, 1 Michel-Suquet */
    double E, nu, sigma_Y, H, eps0_dot, sigma_d, n;
    double lam, mu;
} Law;

/* linalg.py:49-53 */
static void lame(double E, double nu, double *lam, double *mu) {
    *lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    *mu = E / (2.0 * (1.0 + nu));
}

static int law_m(const Law *L) { return L->kind == 1 ? 7 : 0; }

/* sum of squares x0*x0 + x1*x1 + x2*x2 as Python builds it */
static int sq3(Tree *t, int x0, int x1, int x2) {
    return t_add(t, t_add(t, t_mul(t, x0, x0), t_mul(t, x1, x1)), t_mul(t, x2, x2));
}

/* LinearElastic.omega gsm.py:112-117 and MichelSuquet.omega gsm.py:234-244 */
static int build_omega(Tree *t, const Law *L, const int *eps, const int *a) {
    int ee[6];
    if (L->kind == 1) {
        for (int i = 0; i < 6; ++i) ee[i] = t_sub(t, eps[i], a[i]);
    } else {
        for (int i = 0; i < 6; ++i) ee[i] = eps[i];
    }
    int tr = t_add(t, t_add(t, ee[0], ee[1]), ee[2]);
    int w = t_mul(t, t_mul(t, t_cst(t, 0.5 * L->lam), tr), tr);
    w = t_add(t, w, t_mul(t, t_cst(t, L->mu), sq3(t, ee[0], ee[1], ee[2])));
    w = t_add(t, w, t_mul(t, t_cst(t, 0.5 * L->mu), sq3(t, ee[3], ee[4], ee[5])));
    if (L->kind == 1) {
        w = t_add(t, w, t_mul(t, t_cst(t, L->H / 3.0), sq3(t, a[0], a[1], a[2])));
        w = t_add(t, w, t_mul(t, t_cst(t, L->H / 6.0), sq3(t, a[3], a[4], a[5])));
        w = t_add(t, w, t_mul(t, t_cst(t, L->sigma_Y), a[6]));
    }
    return w;
}

/* MichelSuquet.psi gsm.py:246-250 with mises_components gsm.py:62-79 */
static int build_psi(Tree *t, const Law *L, const int *A) {
    int s012 = t_add(t, t_add(t, A[0], A[1]), A[2]);
    int p = t_mul(t, s012, t_cst(t, 1.0 / 3.0));
    int d[6];
    for (int i = 0; i < 3; ++i) d[i] = t_sub(t, A[i], p);
    for (int i = 3; i < 6; ++i) d[i] = A[i];
    int x = sq3(t, d[0], d[1], d[2]);
    int y2 = t_mul(t, t_cst(t, 2.0), sq3(t, d[3], d[4], d[5]));
    int q = t_mul(t, t_cst(t, 1.5), t_add(t, x, y2));
    double mask = t_v(t, q).v > 0.0 ? 1.0 : 0.0;
    int norm = t_mul(t, t_sqrt(t, t_add(t, q, t_cst(t, 1.0 - mask))), t_cst(t, mask));
    int y = t_add(t, norm, A[6]);
    int ys = t_mul(t, y, t_cst(t, 1.0 / L->sigma_d));
    int pw = t_pow(t, t_pos(t, ys), L->n + 1.0);
    double K = L->sigma_d * L->eps0_dot / (L->n + 1.0);
    return t_mul(t, t_cst(t, K), pw);
}

/* LawOps.stress_generic gsm.py:431-439: eps leaves, a consts */
static void stress_generic(const Law *L, const P *eps, const P *a, P *sig) {
    Tree t; t.count = 0;
    int e[6], ai[7];
    for (int i = 0; i < 6; ++i) e[i] = t_leaf(&t, eps[i]);
    for (int k = 0; k < law_m(L); ++k) ai[k] = t_const(&t, a[k]);
    int root = build_omega(&t, L, e, ai);
    t_back(&t, root, pf(1.0));
    for (int i = 0; i < 6; ++i) sig[i] = t_adjoint(&t, e[i]);
}

/* LawOps.gen_stress_generic gsm.py:441-449: eps consts, a leaves, A = -adj */
static void gen_stress_generic(const Law *L, const P *eps, const P *a, P *A) {
    Tree t; t.count = 0;
    int e[6], ai[7];
    for (int i = 0; i < 6; ++i) e[i] = t_const(&t, eps[i]);
    for (int k = 0; k < 7; ++k) ai[k] = t_leaf(&t, a[k]);
    int root = build_omega(&t, L, e, ai);
    t_back(&t, root, pf(1.0));
    for (int k = 0; k < 7; ++k) A[k] = p_neg(t_adjoint(&t, ai[k]));
}

/* LawOps.flow_generic gsm.py:451-458 */
static void flow_generic(const Law *L, const P *A, P *f) {
    Tree t; t.count = 0;
    int ai[7];
    for (int k = 0; k < 7; ++k) ai[k] = t_leaf(&t, A[k]);
    int root = build_psi(&t, L, ai);
    t_back(&t, root, pf(1.0));
    for (int k = 0; k < 7; ++k) f[k] = t_adjoint(&t, ai[k]);
}

static void rhs_generic(const Law *L, const P *eps, const P *a, P *f) {
    P A[7];
    gen_stress_generic(L, eps, a, A);
    flow_generic(L, A, f);
}

static P seeded(double v, int dir) {
    P r; r.has = 1; r.v = v;
    for (int k = 0; k < g_W; ++k) r.d[k] = 0.0;
    r.d[dir] = 1.0;
    return r;
}

/* LawOps.rhs_and_jacobians gsm.py:494-518 (automatic): W = 13 */
static void rhs_and_jacobians(const Law *L, const double *eps, const double *a,
                              double *f, double *J /*7x7*/, double *dfde /*7x6*/) {
    g_W = 13;
    P pe[6], pa[7], pfv[7];
    for (int i = 0; i < 6; ++i) pe[i] = seeded(eps[i], i);
    for (int k = 0; k < 7; ++k) pa[k] = seeded(a[k], 6 + k);
    rhs_generic(L, pe, pa, pfv);
    for (int i = 0; i < 7; ++i) {
        f[i] = pfv[i].v;
        for (int k = 0; k < 7; ++k) J[i * 7 + k] = pfv[i].has ? pfv[i].d[6 + k] : 0.0;
        if (dfde) for (int k = 0; k < 6; ++k) dfde[i * 6 + k] = pfv[i].has ? pfv[i].d[k] : 0.0;
    }
}

/* stress_of odeint.py:339-341 (plain payloads) */
static void stress_plain(const Law *L, const double *eps, const double *a, double *sig) {
    g_W = 0;
    P pe[6], pa[7], ps[6];
    for (int i = 0; i < 6; ++i) pe[i] = pf(eps[i]);
    for (int k = 0; k < law_m(L); ++k) pa[k] = pf(a[k]);
    stress_generic(L, pe, pa, ps);
    for (int i = 0; i < 6; ++i) sig[i] = ps[i].v;
}

/* rhs_dual odeint.py:298-304 with ydot = 0: eps seeded with ramp r */
static void rhs_dual(const Law *L, const double *eps, double r, const double *a, double *dfp /*7x6*/) {
    g_W = 6;
    P pe[6], pa[7], pfv[7];
    for (int i = 0; i < 6; ++i) {
        pe[i].has = 1; pe[i].v = eps[i];
        for (int k = 0; k < 6; ++k) pe[i].d[k] = 0.0;
        pe[i].d[i] = r;
    }
    for (int k = 0; k < 7; ++k) {
        pa[k].has = 1; pa[k].v = a[k];
        for (int j = 0; j < 6; ++j) pa[k].d[j] = 0.0;
    }
    rhs_generic(L, pe, pa, pfv);
    for (int i = 0; i < 7; ++i)
        for (int k = 0; k < 6; ++k) dfp[i * 6 + k] = pfv[i].has ? pfv[i].d[k] : 0.0;
}

/* LawOps.stress_and_tangent gsm.py:520-551 */
static void stress_and_tangent(const Law *L, const double *eps, const double *a,
                               const double *da /* m x 6 */, double *sig, double *C) {
    g_W = 6;
    int m = law_m(L);
    Tree t; t.count = 0;
    int e[6], ai[7];
    for (int i = 0; i < 6; ++i) e[i] = t_leaf(&t, seeded(eps[i], i));
    for (int k = 0; k < m; ++k) {
        P q; q.has = 1; q.v = a[k];
        for (int j = 0; j < 6; ++j) q.d[j] = da[k * 6 + j];
        ai[k] = t_const(&t, q);
    }
    int root = build_omega(&t, L, e, ai);
    t_back(&t, root, pf(1.0));
    for (int i = 0; i < 6; ++i) {
        P adj = t_adjoint(&t, e[i]);
        sig[i] = adj.v;
        for (int j = 0; j < 6; ++j) C[i * 6 + j] = adj.has ? adj.d[j] : 0.0;
    }
}

/* ---------------------------------------------------------------- LU (n = 7) */
/* linalg.py:75-109; returns ok flag */
static int lu_factor7(double *lu, int *piv, int n) {
    double scale = 0.0;
    int scale_nan = 0;
    for (int i = 0; i < n * n; ++i) {
        double v = fabs(lu[i]);
        if (isnan(v)) scale_nan = 1;
        if (v > scale) scale = v;
    }
    if (scale_nan) scale = NAN;
    int ok = scale > 0.0;
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(lu[k * n + k]);
        if (!isnan(best)) {
            for (int i = k + 1; i < n; ++i) {
                double v = fabs(lu[i * n + k]);
                if (isnan(v)) { p = i; break; }
                if (v > best) { best = v; p = i; }
            }
        }
        piv[k] = p;
        if (p != k) {
            for (int j = 0; j < n; ++j) {
                double tmp = lu[k * n + j]; lu[k * n + j] = lu[p * n + j]; lu[p * n + j] = tmp;
            }
        }
        double pivot = lu[k * n + k];
        ok = ok && (fabs(pivot) >= 1e-14 * scale);
        if (k < n - 1) {
            double safe = pivot == 0.0 ? 1.0 : pivot;
            for (int i = k + 1; i < n; ++i) lu[i * n + k] /= safe;
            for (int i = k + 1; i < n; ++i)
                for (int j = k + 1; j < n; ++j) lu[i * n + j] -= lu[i * n + k] * lu[k * n + j];
        }
    }
    return ok;
}

/* numpy's einsum("bj,bjr->br") contraction (linalg.py:133,137) accumulates
 * in two interleaved lanes (even / odd j) that are added at the end; the
 * same order is used here so the oracle reproduces the reference bitwise. */
static double dot2(const double *l, const double *x, int stride, int len) {
    double s0 = 0.0, s1 = 0.0;
    for (int j = 0; j < len; ++j) {
        if (j & 1) s1 += l[j] * x[j * stride];
        else s0 += l[j] * x[j * stride];
    }
    return s0 + s1;
}

/* linalg.py:112-143, nrhs columns stored row-major x[row*nrhs + r] */
static void lu_solve7(const double *lu, const int *piv, double *x, int n, int nrhs) {
    for (int k = 0; k < n; ++k) {
        int p = piv[k];
        if (p != k)
            for (int r = 0; r < nrhs; ++r) {
                double tmp = x[k * nrhs + r]; x[k * nrhs + r] = x[p * nrhs + r]; x[p * nrhs + r] = tmp;
            }
    }
    for (int k = 1; k < n; ++k)
        for (int r = 0; r < nrhs; ++r) {
            x[k * nrhs + r] -= dot2(lu + k * n, x + r, nrhs, k);
        }
    for (int k = n - 1; k >= 0; --k)
        for (int r = 0; r < nrhs; ++r) {
            if (k < n - 1) {
                x[k * nrhs + r] -= dot2(lu + k * n + k + 1, x + (k + 1) * nrhs + r, nrhs, n - k - 1);
            }
            x[k * nrhs + r] /= lu[k * n + k];
        }
}

static double rms(const double *x, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * x[i];
    return sqrt(s / n);
}

/* ---------------------------------------------------------------- one voxel */
enum { ST_NEWTON = 1, ST_SINGULAR = 2, ST_NONFINITE = 4 };

typedef struct {
    int newton_mode; /* 0 internal, 1 stress */
    double newton_tol;
    int max_newton;
} Cfg;

/* odeint.py:357-401 for a single voxel; returns ok, writes a and count */
static int newton_ie(const Law *L, const Cfg *cfg, const double *eps_t1, double h,
                     const double *a0, double *a, int *iters) {
    int m = 7;
    double res_prev = INFINITY;
    int growth = 0;
    double sig_prev[6];
    memcpy(a, a0, sizeof(double) * m);
    if (cfg->newton_mode == 1) stress_plain(L, eps_t1, a, sig_prev);
    int it = 0;
    for (int pass = 0; pass < cfg->max_newton; ++pass) {
        ++it;
        double f[7], J[49], F[7], M[49], dlt[7], an[7];
        int piv[7];
        rhs_and_jacobians(L, eps_t1, a, f, J, NULL);
        int finite = 1;
        for (int i = 0; i < m; ++i) {
            F[i] = a[i] - a0[i] - h * f[i];
            if (!isfinite(F[i])) finite = 0;
        }
        for (int i = 0; i < m; ++i)
            for (int k = 0; k < m; ++k) M[i * m + k] = (i == k ? 1.0 : 0.0) - h * J[i * m + k];
        int fac_ok = lu_factor7(M, piv, m);
        int bad = !fac_ok || !finite;
        for (int i = 0; i < m; ++i) dlt[i] = bad ? 0.0 : F[i];
        lu_solve7(M, piv, dlt, m, 1);
        for (int i = 0; i < m; ++i) an[i] = a[i] - dlt[i];
        double sc[7];
        for (int i = 0; i < m; ++i) sc[i] = F[i] / (1.0 + fabs(a[i]));
        double res = rms(sc, m);
        growth = res > res_prev ? growth + 1 : 0;
        res_prev = res;
        int conv;
        if (cfg->newton_mode == 1) {
            double sn[6], ds[6];
            stress_plain(L, eps_t1, an, sn);
            for (int i = 0; i < 6; ++i) ds[i] = sn[i] - sig_prev[i];
            double dsig = rms(ds, 6), ref = rms(sn, 6);
            conv = dsig <= cfg->newton_tol * (ref > 1e-300 ? ref : 1e-300);
            memcpy(sig_prev, sn, sizeof(sn));
        } else {
            for (int i = 0; i < m; ++i) sc[i] = dlt[i] / (1.0 + fabs(an[i]));
            conv = rms(sc, m) <= cfg->newton_tol;
        }
        memcpy(a, an, sizeof(double) * m);
        int failed = bad || growth >= 5;
        if (failed) { *iters = it; return 0; }
        if (conv) { *iters = it; return 1; }
    }
    *iters = it;
    return 0; /* iteration cap, odeint.py:400 */
}

/* _evaluate_chunk evaluator.py:124-203, implicit Euler, single voxel */
static int eval_voxel(const Law *L, const Cfg *cfg, const double *eps_n, const double *a_n,
                      const double *eps_np1, double dt, int want_tangent,
                      double *sig, double *a_out, double *C, int *iters) {
    int m = law_m(L);
    *iters = 0;
    if (m == 0) {
        double da[1] = {0.0};
        if (want_tangent) stress_and_tangent(L, eps_np1, a_n, da, sig, C);
        else stress_plain(L, eps_np1, a_n, sig);
        return 0;
    }
    if (dt == 0.0) { /* frozen: a = a_n, no clamp */
        memcpy(a_out, a_n, sizeof(double) * m);
        stress_plain(L, eps_np1, a_n, sig);
        if (want_tangent) {
            double da[42] = {0}, s2[6];
            stress_and_tangent(L, eps_np1, a_n, da, s2, C);
        }
        return 0;
    }
    int status = 0;
    /* MaterialStepProblem odeint.py:241-264: t1 = 0 + h, r = min(t1/dt, 1) */
    double h = dt, t1 = 0.0 + h;
    double r = t1 / dt;
    if (!(r <= 1.0) && !isnan(r)) r = 1.0;
    double deps[6], e1[6];
    for (int i = 0; i < 6; ++i) {
        deps[i] = eps_np1[i] - eps_n[i];
        e1[i] = eps_n[i] + r * deps[i];
    }
    double a[7];
    int ok = newton_ie(L, cfg, e1, h, a_n, a, iters);
    if (!ok) status |= ST_NEWTON;
    double da[42];
    if (want_tangent) {
        /* implicit_euler_step tangent post-process odeint.py:417-426 */
        double dfp[42], f[7], J[49], M[49];
        int piv[7];
        rhs_dual(L, e1, r, a, dfp);
        rhs_and_jacobians(L, e1, a, f, J, NULL);
        for (int i = 0; i < 7; ++i)
            for (int k = 0; k < 7; ++k) M[i * 7 + k] = (i == k ? 1.0 : 0.0) - h * J[i * 7 + k];
        for (int i = 0; i < 42; ++i) da[i] = 0.0 + h * dfp[i];
        if (!lu_factor7(M, piv, 7)) status |= ST_SINGULAR;
        lu_solve7(M, piv, da, 7, 6);
    }
    /* clamp_state gsm.py:252-256 */
    if (a[6] < 0.0) a[6] = 0.0;
    memcpy(a_out, a, sizeof(a));
    if (want_tangent) stress_and_tangent(L, eps_np1, a, da, sig, C);
    else stress_plain(L, eps_np1, a, sig);
    return status;
}

/* ---------------------------------------------------------------- C entry points */
static void make_law(Law *L, int kind, const double *prm) {
    L->kind = kind;
    L->E = prm[0]; L->nu = prm[1];
    L->sigma_Y = prm[2]; L->H = prm[3]; L->eps0_dot = prm[4]; L->sigma_d = prm[5]; L->n = prm[6];
    lame(L->E, L->nu, &L->lam, &L->mu);
}

/*
 * Batch evaluation, AoS like evaluate_arrays (evaluator.py:206-248):
 *   eps_n, eps_np1 (B,6); a_n, a_out (B,m); sig (B,6); C (B,6,6) or NULL.
 * prm = {E, nu, sigma_Y, H, eps0_dot, sigma_d, n}.  Returns the OR of the
 * per-voxel status bits; iters/status per voxel.  nthreads > 1 splits the
 * batch into contiguous spans over pthreads (results are per-voxel).
 */
typedef struct {
    const Law *L; const Cfg *cfg; int m;
    int64_t lo, hi;
    const double *eps_n, *a_n, *eps_np1, *dt;
    int want_tangent;
    double *sig, *a_out, *C;
    int32_t *iters; uint8_t *status;
    int any;
} Job;

static void *run_job(void *arg) {
    Job *j = (Job *)arg;
    int m = j->m;
    for (int64_t b = j->lo; b < j->hi; ++b) {
        int it = 0;
        double Cv[36];
        int st = eval_voxel(j->L, j->cfg, j->eps_n + 6 * b, m ? j->a_n + m * b : NULL, j->eps_np1 + 6 * b,
                            j->dt[b], j->want_tangent, j->sig + 6 * b, m ? j->a_out + m * b : NULL, Cv, &it);
        if (j->want_tangent && j->C) memcpy(j->C + 36 * b, Cv, sizeof(Cv));
        if (j->iters) j->iters[b] = it;
        if (j->status) j->status[b] = (uint8_t)st;
        j->any |= st;
    }
    return NULL;
}

int oracle_eval_batch(int kind, const double *prm, int newton_mode, double newton_tol,
                      int64_t B, const double *eps_n, const double *a_n, const double *eps_np1,
                      const double *dt, int want_tangent, double *sig, double *a_out, double *C,
                      int32_t *iters, uint8_t *status, int nthreads) {
    Law L;
    make_law(&L, kind, prm);
    Cfg cfg = {newton_mode, newton_tol, 50};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > B) nthreads = B > 0 ? (int)B : 1;
    Job jobs[256];
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) {
        Job j = {&L, &cfg, law_m(&L), B * t / nthreads, B * (t + 1) / nthreads,
                 eps_n, a_n, eps_np1, dt, want_tangent, sig, a_out, C, iters, status, 0};
        jobs[t] = j;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, run_job, &jobs[t]);
    run_job(&jobs[0]);
    int any = jobs[0].any;
    for (int t = 1; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        any |= jobs[t].any;
    }
    return any;
}

/* gsm.py:574-602 module-level constitutive operations at one point */
void oracle_constitutive(int kind, const double *prm, const double *eps, const double *a,
                         double *sig, double *A, double *f, double *J, double *dfde) {
    Law L;
    make_law(&L, kind, prm);
    stress_plain(&L, eps, a, sig);
    if (law_m(&L) == 0) return;
    g_W = 0;
    P pe[6], pa[7], pA[7];
    for (int i = 0; i < 6; ++i) pe[i] = pf(eps[i]);
    for (int k = 0; k < 7; ++k) pa[k] = pf(a[k]);
    gen_stress_generic(&L, pe, pa, pA);
    for (int k = 0; k < 7; ++k) A[k] = pA[k].v;
    rhs_and_jacobians(&L, eps, a, f, J, dfde);
}

/* Generic AD entry for unit tests: gradient of omega or psi by one reverse
 * sweep (grad_reverse, ad.py:555-568) at plain payloads. which: 0 omega
 * w.r.t. (eps, a), 1 psi w.r.t. A. */
void oracle_grad(int kind, const double *prm, int which, const double *x, double *g) {
    Law L;
    make_law(&L, kind, prm);
    g_W = 0;
    Tree t; t.count = 0;
    if (which == 0) {
        int e[6], ai[7];
        for (int i = 0; i < 6; ++i) e[i] = t_leaf(&t, pf(x[i]));
        for (int k = 0; k < 7; ++k) ai[k] = t_leaf(&t, pf(x[6 + k]));
        int root = build_omega(&t, &L, e, ai);
        t_back(&t, root, pf(1.0));
        for (int i = 0; i < 6; ++i) g[i] = t_adjoint(&t, e[i]).v;
        for (int k = 0; k < 7; ++k) g[6 + k] = t_adjoint(&t, ai[k]).v;
    } else {
        int ai[7];
        for (int k = 0; k < 7; ++k) ai[k] = t_leaf(&t, pf(x[k]));
        int root = build_psi(&t, &L, ai);
        t_back(&t, root, pf(1.0));
        for (int k = 0; k < 7; ++k) g[k] = t_adjoint(&t, ai[k]).v;
    }
}
