/*
 * oracle/netsimplex.c -- exact solver for the transportation LP, Eq. (1)
 * (lines 41-46):  min <C,X>  s.t.  X e_n = a,  X^T e_m = b,  X >= 0.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path (paper_2502_03749_b200/)
 * may link or call this file; it is the independent ground truth used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 *
 * Method: primal network simplex on the complete bipartite graph (the textbook
 * algorithm: spanning-tree bases, big-M artificial root, strongly feasible
 * trees for anti-cycling, block pivot search).  Own implementation:
 *   - tree = parent pointers + depth + doubly-linked child lists;
 *   - the flow of a basic arc is stored at the tree node it hangs from
 *     (non-basic arcs of an uncapacitated problem carry zero flow);
 *   - after a pivot the detached subtree is re-rooted along its stem and its
 *     depths / potentials are refreshed by an explicit DFS.
 * Output: an optimal vertex (<= m+n-1 positive entries), its cost, and the
 * node potentials as LP duals (u_i + v_j <= C_ij), so the caller can check a
 * zero duality gap.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    long long m, n, N, root, mn;
    const double *C;
    double art;
    int8_t *nonbasic;   /* per real arc: 1 = at lower bound (flow 0), 0 = basic */
    int *parent, *first_child, *next_sib, *prev_sib, *depth;
    long long *pred;    /* arc id of the tree arc joining v to parent[v]     */
    int8_t *up;         /* 1 if pred arc is oriented v -> parent[v]           */
    double *flow;       /* flow on pred arc of v                              */
    double *pi;         /* node potentials, reduced cost c + pi[s] - pi[t]    */
    int *stack;
} ns_t;

static inline long long arc_src(const ns_t *S, long long e) {
    if (e < S->mn) return e / S->n;
    long long v = e - S->mn;
    return v < S->m ? v : S->root;
}
static inline long long arc_tgt(const ns_t *S, long long e) {
    if (e < S->mn) return S->m + e % S->n;
    long long v = e - S->mn;
    return v < S->m ? S->root : v;
}
static inline double arc_cost(const ns_t *S, long long e) {
    return e < S->mn ? S->C[e] : S->art;
}

static void child_detach(ns_t *S, int v) {
    int p = S->parent[v];
    if (p < 0) return;
    if (S->prev_sib[v] >= 0) S->next_sib[S->prev_sib[v]] = S->next_sib[v];
    else S->first_child[p] = S->next_sib[v];
    if (S->next_sib[v] >= 0) S->prev_sib[S->next_sib[v]] = S->prev_sib[v];
    S->next_sib[v] = S->prev_sib[v] = -1;
}
static void child_attach(ns_t *S, int v, int p) {
    S->parent[v] = p;
    S->prev_sib[v] = -1;
    S->next_sib[v] = S->first_child[p];
    if (S->first_child[p] >= 0) S->prev_sib[S->first_child[p]] = v;
    S->first_child[p] = v;
}

/* refresh depth and shift potentials by sigma over the subtree rooted at r */
static void subtree_refresh(ns_t *S, int r, double sigma) {
    int top = 0;
    S->stack[top++] = r;
    while (top) {
        int v = S->stack[--top];
        S->depth[v] = S->depth[S->parent[v]] + 1;
        S->pi[v] += sigma;
        for (int c = S->first_child[v]; c >= 0; c = S->next_sib[c]) S->stack[top++] = c;
    }
}

/*
 * Solve.  Returns 0 on success, 1 if the pivot budget ran out, 2 on bad input.
 * X (m*n, row-major) receives the optimal plan (zero-filled first).
 * u (m), v (n) receive LP duals; stats[0]=pivots, stats[1]=max artificial flow,
 * stats[2]=min reduced cost over all arcs (>= -tol at optimality).
 */
int ns_solve(long long m, long long n, const double *C, const double *a, const double *b,
             double *X, double *u, double *v, double *obj, double *stats,
             long long max_pivots) {
    if (m <= 0 || n <= 0) return 2;
    ns_t S;
    memset(&S, 0, sizeof S);
    S.m = m; S.n = n; S.N = m + n + 1; S.root = m + n; S.mn = m * n; S.C = C;
    long long N = S.N;
    double cmax = 0.0;
    for (long long e = 0; e < S.mn; ++e) if (fabs(C[e]) > cmax) cmax = fabs(C[e]);
    S.art = (cmax + 1.0) * (double)N;
    S.nonbasic = (int8_t *)malloc((size_t)S.mn);
    S.parent = (int *)malloc(sizeof(int) * N);
    S.first_child = (int *)malloc(sizeof(int) * N);
    S.next_sib = (int *)malloc(sizeof(int) * N);
    S.prev_sib = (int *)malloc(sizeof(int) * N);
    S.depth = (int *)malloc(sizeof(int) * N);
    S.stack = (int *)malloc(sizeof(int) * N);
    S.pred = (long long *)malloc(sizeof(long long) * N);
    S.up = (int8_t *)malloc((size_t)N);
    S.flow = (double *)malloc(sizeof(double) * N);
    S.pi = (double *)malloc(sizeof(double) * N);
    if (!S.nonbasic || !S.parent || !S.first_child || !S.next_sib || !S.prev_sib ||
        !S.depth || !S.stack || !S.pred || !S.up || !S.flow || !S.pi) return 2;
    memset(S.nonbasic, 1, (size_t)S.mn);

    /* initial strongly feasible tree: every node hangs from the root by its
     * artificial arc; supply nodes point up (v->root), demand nodes down.   */
    for (long long k = 0; k < N; ++k) {
        S.first_child[k] = S.next_sib[k] = S.prev_sib[k] = -1;
    }
    S.parent[S.root] = -1; S.depth[S.root] = 0; S.pi[S.root] = 0.0;
    S.pred[S.root] = -1; S.up[S.root] = 0; S.flow[S.root] = 0.0;
    for (long long k = 0; k < m + n; ++k) {
        child_attach(&S, (int)k, (int)S.root);
        S.depth[k] = 1;
        S.pred[k] = S.mn + k;
        if (k < m) { S.up[k] = 1; S.flow[k] = a[k]; S.pi[k] = 0.0; }
        else { S.up[k] = 0; S.flow[k] = b[k - m]; S.pi[k] = S.art; }
    }

    const double eps = 1e-11 * (1.0 + cmax);
    long long block = (long long)sqrt((double)S.mn);
    if (block < 64) block = 64;
    if (block > S.mn) block = S.mn;
    long long next = 0, pivots = 0;
    int status = 0;

    for (;;) {
        /* ---- block pivot search for an entering arc (most negative rc) ---- */
        long long in = -1, scanned = 0, cnt = 0;
        double best = -eps;
        long long e = next;
        while (scanned < S.mn) {
            long long i = e / n, j = e % n;
            if (S.nonbasic[e]) {
                double rc = C[e] + S.pi[i] - S.pi[m + j];
                if (rc < best) { best = rc; in = e; }
            }
            ++scanned; ++cnt;
            if (++e == S.mn) e = 0;
            if (cnt == block) { if (in >= 0) break; cnt = 0; }
        }
        if (in < 0) break;               /* optimal */
        next = e;
        if (pivots++ >= max_pivots) { status = 1; break; }

        /* ---- cycle: apex (join) of src(in) and tgt(in) ---- */
        long long s = arc_src(&S, in), t = arc_tgt(&S, in);
        long long x = s, y = t;
        while (x != y) {
            if (S.depth[x] >= S.depth[y]) x = S.parent[x]; else y = S.parent[y];
        }
        long long join = x;

        /* ---- leaving arc, strongly-feasible tie rule ----
         * flow travels join -> ... -> s -> t -> ... -> join.  On the s side an
         * arc blocks if it points up (its flow decreases); on the t side if it
         * points down.  Ties: the last blocking arc met from the apex wins. */
        double delta = INFINITY;
        long long u_out = -1;
        int side = 0;
        for (long long w = s; w != join; w = S.parent[w]) {
            if (S.up[w] && S.flow[w] < delta) { delta = S.flow[w]; u_out = w; side = 1; }
        }
        for (long long w = t; w != join; w = S.parent[w]) {
            if (!S.up[w] && S.flow[w] <= delta) { delta = S.flow[w]; u_out = w; side = 2; }
        }
        if (u_out < 0) { status = 2; break; }  /* unbounded: impossible here */

        /* ---- push delta around the cycle ---- */
        if (delta > 0.0) {
            for (long long w = s; w != join; w = S.parent[w]) S.flow[w] += S.up[w] ? -delta : delta;
            for (long long w = t; w != join; w = S.parent[w]) S.flow[w] += S.up[w] ? delta : -delta;
        }
        long long u_in = side == 1 ? s : t;
        long long v_in = side == 1 ? t : s;

        /* ---- basis exchange ---- */
        long long leaving = S.pred[u_out];
        if (leaving < S.mn) S.nonbasic[leaving] = 1;
        S.nonbasic[in] = 0;

        /* re-root the detached subtree at u_in: reverse the stem u_in..u_out */
        child_detach(&S, (int)u_out);
        long long w = u_in;
        long long carry_pred = in;
        int8_t carry_up = (u_in == s) ? 1 : 0;
        double carry_flow = delta;
        long long newpar = v_in;
        for (;;) {
            long long oldpar = S.parent[w];
            long long opred = S.pred[w];
            int8_t oup = S.up[w];
            double oflow = S.flow[w];
            if (w != u_out) child_detach(&S, (int)w);
            child_attach(&S, (int)w, (int)newpar);
            S.pred[w] = carry_pred; S.up[w] = carry_up; S.flow[w] = carry_flow;
            if (w == u_out) break;
            carry_pred = opred; carry_up = (int8_t)!oup; carry_flow = oflow;
            newpar = w;
            w = oldpar;
        }
        /* potentials: make rc(in) = 0 by shifting the moved subtree */
        double cin = arc_cost(&S, in);
        double sigma = (u_in == s) ? (S.pi[v_in] - cin - S.pi[u_in])
                                   : (S.pi[v_in] + cin - S.pi[u_in]);
        subtree_refresh(&S, (int)u_in, sigma);
    }

    /* ---- extract plan, duals, certificate ---- */
    memset(X, 0, sizeof(double) * (size_t)S.mn);
    double maxart = 0.0, total = 0.0;
    for (long long k = 0; k < m + n; ++k) {
        long long e = S.pred[k];
        if (e < 0) continue;
        if (e >= S.mn) { if (S.flow[k] > maxart) maxart = S.flow[k]; continue; }
        X[e] = S.flow[k];
    }
    for (long long e = 0; e < S.mn; ++e) total += C[e] * X[e];
    for (long long i = 0; i < m; ++i) u[i] = -S.pi[i];
    for (long long j = 0; j < n; ++j) v[j] = S.pi[m + j];
    double minrc = INFINITY;
    for (long long i = 0; i < m; ++i)
        for (long long j = 0; j < n; ++j) {
            double rc = C[i * n + j] - u[i] - v[j];
            if (rc < minrc) minrc = rc;
        }
    *obj = total;
    stats[0] = (double)pivots;
    stats[1] = maxart;
    stats[2] = minrc;

    free(S.nonbasic); free(S.parent); free(S.first_child); free(S.next_sib);
    free(S.prev_sib); free(S.depth); free(S.stack); free(S.pred); free(S.up);
    free(S.flow); free(S.pi);
    return status;
}
