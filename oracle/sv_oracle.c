/*
 * sv_oracle.c -- the CPU ORACLE for the state-vector gate-application path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2106_13995_b200/) never links, imports or executes anything here, and this
 * file shares no code, header, table or helper with it.
 *
 * What it computes: psi_out = U_G ... U_1 psi_in, where U_j is gate j's
 * matrix embedded on its qubits in controlled form and the identity elsewhere, under the
 * little-endian convention (qubit q = bit q of the basis index).
 *   - PAPER.md:38 (Background): the state of an n-qubit circuit is a 2^n complex vector
 *     and each moment is a 2^n x 2^n matrix; Schroedinger simulation stores all amplitudes.
 *   - PAPER.md:55 (Methods, assumption a): a simulator is matrix-vector multiplication.
 *   - SPEC S:167-176: gate-local semantics by bit-mask iteration over groups.
 * Algorithm, step by step as SURVEY 8(c) lists it:
 *   1. parse the IR text with this file's own parser and gate table;
 *   2. psi holds 2^n complex doubles (fp64, reading R4);
 *   3. for each gate in file order: Q = controls ++ targets, m = |Q|;
 *      M (2^m x 2^m) = identity except the block where all control bits are 1, which is U;
 *      for g = 0 .. 2^(n-m)-1: base = g with zero bits inserted at sorted(Q);
 *      v[r] = psi[base | sum_j bit_j(r) 2^Q[j]];  w[r] = sum_{c ascending} M[r][c] v[c]
 *      with the complex product written out as (ac - bd, ad + bc); scatter w back;
 *      OpenMP static schedule over g is allowed because groups are disjoint, so
 *      the result is bit-identical for any thread count;
 *   4. readout: norm = sqrt(pairwise tree sum of |a|^2 in index order);
 *      marginal probabilities by fixed-order sums in index order.
 * Build: gcc -O2 -ffp-contract=off -fopenmp (reading R18: no FMA contraction, no fast-math).
 * Parity pins: tests/test_oracle.py (brute-force 2^n x 2^n products, closed forms, QFT,
 * multiplier truth tables, classical reversible map).  Pinned: every function below.
 */
#include <ctype.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { double re, im; } cplx;

#define OR_MAXQ 10   /* max |controls ++ targets| per gate */

static void set_err(char* err, int errlen, const char* fmt, int line, const char* what) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, fmt, line, what);
}

/* ------------------------------------------------------------------ gate table (App. A) */
/* Each named gate -> (number of controls, target count, U row-major on the targets). */
static int named_gate(const char* name, int* nc, int* k, cplx* U) {
    const double h = M_SQRT1_2;
    memset(U, 0, sizeof(cplx) * 16);
#define SET(i, a, b) do { U[i].re = (a); U[i].im = (b); } while (0)
    if (!strcmp(name, "X"))  { *nc = 0; *k = 1; SET(1, 1, 0); SET(2, 1, 0); return 1; }
    if (!strcmp(name, "Y"))  { *nc = 0; *k = 1; SET(1, 0, -1); SET(2, 0, 1); return 1; }
    if (!strcmp(name, "Z"))  { *nc = 0; *k = 1; SET(0, 1, 0); SET(3, -1, 0); return 1; }
    if (!strcmp(name, "H"))  { *nc = 0; *k = 1; SET(0, h, 0); SET(1, h, 0); SET(2, h, 0); SET(3, -h, 0); return 1; }
    if (!strcmp(name, "S"))  { *nc = 0; *k = 1; SET(0, 1, 0); SET(3, 0, 1); return 1; }
    if (!strcmp(name, "Sdg")) { *nc = 0; *k = 1; SET(0, 1, 0); SET(3, 0, -1); return 1; }
    if (!strcmp(name, "T"))  { *nc = 0; *k = 1; SET(0, 1, 0); SET(3, h, h); return 1; }
    if (!strcmp(name, "Tdg")) { *nc = 0; *k = 1; SET(0, 1, 0); SET(3, h, -h); return 1; }
    /* SqrtX = 1/2 [[1+i, 1-i], [1-i, 1+i]]  (R3) */
    if (!strcmp(name, "SqrtX"))  { *nc = 0; *k = 1; SET(0, .5, .5); SET(1, .5, -.5); SET(2, .5, -.5); SET(3, .5, .5); return 1; }
    if (!strcmp(name, "SqrtXdg")) { *nc = 0; *k = 1; SET(0, .5, -.5); SET(1, .5, .5); SET(2, .5, .5); SET(3, .5, -.5); return 1; }
    /* SqrtY = 1/2 [[1+i, -1-i], [1+i, 1+i]]  (R3) */
    if (!strcmp(name, "SqrtY"))  { *nc = 0; *k = 1; SET(0, .5, .5); SET(1, -.5, -.5); SET(2, .5, .5); SET(3, .5, .5); return 1; }
    if (!strcmp(name, "SqrtYdg")) { *nc = 0; *k = 1; SET(0, .5, -.5); SET(1, .5, -.5); SET(2, -.5, .5); SET(3, .5, -.5); return 1; }
    if (!strcmp(name, "CZ"))   { *nc = 1; *k = 1; SET(0, 1, 0); SET(3, -1, 0); return 1; }
    if (!strcmp(name, "CNOT")) { *nc = 1; *k = 1; SET(1, 1, 0); SET(2, 1, 0); return 1; }
    if (!strcmp(name, "Toffoli")) { *nc = 2; *k = 1; SET(1, 1, 0); SET(2, 1, 0); return 1; }
    if (!strcmp(name, "SWAP")) { *nc = 0; *k = 2; SET(0, 1, 0); SET(6, 1, 0); SET(9, 1, 0); SET(15, 1, 0); return 1; }
#undef SET
    return 0;
}

/* ------------------------------------------------------------------ parsed circuit */
typedef struct {
    int nc, k;             /* controls, targets */
    int q[OR_MAXQ];        /* controls ++ targets */
    cplx* U;               /* 2^k x 2^k row-major, row/col bit j <-> target j */
    int line;
} ogate;

typedef struct {
    int n;
    int ngates, cap;
    ogate* g;
} ocircuit;

static void free_circuit(ocircuit* c) {
    for (int i = 0; i < c->ngates; ++i) free(c->g[i].U);
    free(c->g);
    c->g = NULL; c->ngates = c->cap = 0;
}

static const char* skip_ws(const char* p, const char* e) {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    return p;
}

/* parse "a,b,c" integers up to terminator set; returns count or -1 */
static int parse_ints(const char** pp, const char* e, int* out, int maxn) {
    const char* p = *pp;
    int cnt = 0;
    for (;;) {
        p = skip_ws(p, e);
        if (p >= e || !isdigit((unsigned char)*p)) return -1;
        long v = 0;
        while (p < e && isdigit((unsigned char)*p)) { v = v * 10 + (*p - '0'); if (v > 100000) return -1; ++p; }
        if (cnt >= maxn) return -1;
        out[cnt++] = (int)v;
        p = skip_ws(p, e);
        if (p < e && *p == ',') { ++p; continue; }
        break;
    }
    *pp = p;
    return cnt;
}

static int parse_gate(const char* p, const char* e, int n, int line, ogate* g, char* err, int errlen) {
    char name[32];
    int len = 0;
    p = skip_ws(p, e);
    while (p < e && (isalnum((unsigned char)*p) || *p == '_') && len < 31) name[len++] = *p++;
    name[len] = 0;
    if (!len) { set_err(err, errlen, "line %d: expected gate name%s", line, ""); return -1; }
    memset(g, 0, sizeof(*g));
    g->line = line;
    if (!strcmp(name, "U") || !strcmp(name, "CU")) {
        int ctrl[OR_MAXQ], tg[OR_MAXQ], nc = 0, k;
        if (name[0] == 'C') {
            nc = parse_ints(&p, e, ctrl, OR_MAXQ);
            if (nc < 1 || p >= e || *p != '|') { set_err(err, errlen, "line %d: bad CU control list%s", line, ""); return -1; }
            ++p;
        }
        k = parse_ints(&p, e, tg, OR_MAXQ);
        if (k < 1 || k > 6 || nc + k > OR_MAXQ) { set_err(err, errlen, "line %d: bad %s target list", line, name); return -1; }
        p = skip_ws(p, e);
        if (p >= e || *p != ':') { set_err(err, errlen, "line %d: %s needs ': matrix'", line, name); return -1; }
        ++p;
        int d = 1 << k;
        g->U = (cplx*)malloc(sizeof(cplx) * (size_t)d * d);
        for (int i = 0; i < 2 * d * d; ++i) {
            p = skip_ws(p, e);
            char* endp;
            double v = strtod(p, &endp);
            if (endp == p || endp > e) { free(g->U); g->U = NULL; set_err(err, errlen, "line %d: bad number in %s matrix", line, name); return -1; }
            if (i & 1) g->U[i >> 1].im = v; else g->U[i >> 1].re = v;
            p = skip_ws(endp, e);
            if (i + 1 < 2 * d * d) {
                if (p >= e || *p != ',') { free(g->U); g->U = NULL; set_err(err, errlen, "line %d: %s matrix too short", line, name); return -1; }
                ++p;
            }
        }
        p = skip_ws(p, e);
        if (p != e) { free(g->U); g->U = NULL; set_err(err, errlen, "line %d: trailing text after %s matrix", line, name); return -1; }
        g->nc = nc; g->k = k;
        for (int i = 0; i < nc; ++i) g->q[i] = ctrl[i];
        for (int i = 0; i < k; ++i) g->q[nc + i] = tg[i];
    } else {
        int nc, k, qs[OR_MAXQ];
        cplx U[16];
        if (!named_gate(name, &nc, &k, U)) { set_err(err, errlen, "line %d: unknown gate '%s'", line, name); return -1; }
        int cnt = parse_ints(&p, e, qs, OR_MAXQ);
        if (cnt != nc + k) { set_err(err, errlen, "line %d: wrong qubit count for %s", line, name); return -1; }
        p = skip_ws(p, e);
        if (p != e) { set_err(err, errlen, "line %d: trailing text after %s", line, name); return -1; }
        g->nc = nc; g->k = k;
        for (int i = 0; i < cnt; ++i) g->q[i] = qs[i];
        int d = 1 << k;
        g->U = (cplx*)malloc(sizeof(cplx) * (size_t)d * d);
        memcpy(g->U, U, sizeof(cplx) * (size_t)d * d);
    }
    int m = g->nc + g->k;
    for (int i = 0; i < m; ++i) {
        if (g->q[i] < 0 || g->q[i] >= n) { free(g->U); g->U = NULL; set_err(err, errlen, "line %d: qubit out of range in %s", line, name); return -1; }
        for (int j = 0; j < i; ++j)
            if (g->q[i] == g->q[j]) { free(g->U); g->U = NULL; set_err(err, errlen, "line %d: duplicate qubit in %s", line, name); return -1; }
    }
    return 0;
}

static int parse_circuit(const char* text, ocircuit* c, char* err, int errlen) {
    memset(c, 0, sizeof(*c));
    c->n = -1;
    const char* p = text;
    int line = 0;
    while (*p) {
        const char* e = strchr(p, '\n');
        if (!e) e = p + strlen(p);
        ++line;
        const char* s = skip_ws(p, e);
        const char* t = e;
        while (t > s && (t[-1] == ' ' || t[-1] == '\t' || t[-1] == '\r')) --t;
        if (s < t && *s != '#') {
            if (!strncmp(s, "qubits:", 7)) {
                c->n = atoi(s + 7);
                if (c->n < 1 || c->n > 62) { set_err(err, errlen, "line %d: bad qubit count%s", line, ""); free_circuit(c); return -1; }
            } else if (!strncmp(s, "family:", 7) || !strncmp(s, "meta.", 5)) {
                /* metadata: ignored by the simulation */
            } else {
                if (c->n < 0) { set_err(err, errlen, "line %d: gate before 'qubits:' header%s", line, ""); free_circuit(c); return -1; }
                const char* gs = s;
                while (gs < t) {
                    const char* ge = gs;
                    while (ge < t && *ge != ';') ++ge;
                    const char* ge2 = ge;
                    while (ge2 > gs && (ge2[-1] == ' ' || ge2[-1] == '\t')) --ge2;
                    if (c->ngates == c->cap) {
                        c->cap = c->cap ? 2 * c->cap : 64;
                        c->g = (ogate*)realloc(c->g, sizeof(ogate) * (size_t)c->cap);
                    }
                    if (parse_gate(gs, ge2, c->n, line, &c->g[c->ngates], err, errlen)) { free_circuit(c); return -1; }
                    c->ngates++;
                    gs = ge < t ? ge + 1 : t;
                }
            }
        }
        p = *e ? e + 1 : e;
    }
    if (c->n < 0) { set_err(err, errlen, "line %d: missing 'qubits:' header%s", line, ""); return -1; }
    return 0;
}

/* ------------------------------------------------------------------ apply (step 3) */
static int apply_full(int n, cplx* psi, const cplx* U, int k, const int* Q, int nc, int nthreads) {
    int m = nc + k;
    if (m > n || m > OR_MAXQ) return -1;
    int D = 1 << m;
    /* controlled-form matrix M: identity except the all-controls-one block, which is U */
    cplx* M = (cplx*)calloc((size_t)D * D, sizeof(cplx));
    int cm = (1 << nc) - 1;
    for (int r = 0; r < D; ++r) {
        if ((r & cm) != cm) { M[(size_t)r * D + r].re = 1.0; continue; }
        for (int c = 0; c < D; ++c)
            if ((c & cm) == cm) M[(size_t)r * D + c] = U[(size_t)(r >> nc) * (1 << k) + (c >> nc)];
    }
    int sorted[OR_MAXQ];
    for (int i = 0; i < m; ++i) sorted[i] = Q[i];
    for (int i = 1; i < m; ++i)
        for (int j = i; j > 0 && sorted[j - 1] > sorted[j]; --j) { int t = sorted[j]; sorted[j] = sorted[j - 1]; sorted[j - 1] = t; }
    uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)D);
    for (int r = 0; r < D; ++r) {
        uint64_t o = 0;
        for (int j = 0; j < m; ++j) if ((r >> j) & 1) o |= (uint64_t)1 << Q[j];
        off[r] = o;
    }
    int64_t groups = (int64_t)1 << (n - m);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        cplx* v = (cplx*)malloc(sizeof(cplx) * (size_t)D);
        cplx* w = (cplx*)malloc(sizeof(cplx) * (size_t)D);
#pragma omp for schedule(static)
        for (int64_t g = 0; g < groups; ++g) {
            /* insert zero bits at sorted(Q), lowest position first */
            uint64_t base = (uint64_t)g;
            for (int j = 0; j < m; ++j) {
                uint64_t low = base & (((uint64_t)1 << sorted[j]) - 1);
                base = ((base >> sorted[j]) << (sorted[j] + 1)) | low;
            }
            for (int r = 0; r < D; ++r) v[r] = psi[base | off[r]];
            for (int r = 0; r < D; ++r) {
                double ar = 0.0, ai = 0.0;
                const cplx* row = M + (size_t)r * D;
                for (int c = 0; c < D; ++c) {
                    double pr = row[c].re * v[c].re - row[c].im * v[c].im;
                    double pi = row[c].re * v[c].im + row[c].im * v[c].re;
                    ar += pr;
                    ai += pi;
                }
                w[r].re = ar; w[r].im = ai;
            }
            for (int r = 0; r < D; ++r) psi[base | off[r]] = w[r];
        }
        free(v); free(w);
    }
    free(off); free(M);
    return 0;
}

/* ------------------------------------------------------------------ exported API */
int or_apply_gate(int n, double* psi, const double* U, int k, const int* targets,
                  const int* controls, int nc, int nthreads) {
    int Q[OR_MAXQ];
    if (k < 1 || nc < 0 || nc + k > OR_MAXQ || nc + k > n) return -1;
    for (int i = 0; i < nc; ++i) Q[i] = controls[i];
    for (int i = 0; i < k; ++i) Q[nc + i] = targets[i];
    for (int i = 0; i < nc + k; ++i) {
        if (Q[i] < 0 || Q[i] >= n) return -2;
        for (int j = 0; j < i; ++j) if (Q[i] == Q[j]) return -2;
    }
    return apply_full(n, (cplx*)psi, (const cplx*)U, k, Q, nc, nthreads);
}

int or_circuit_info(const char* text, int* n, int* ngates, char* err, int errlen) {
    ocircuit c;
    if (parse_circuit(text, &c, err, errlen)) return -1;
    *n = c.n; *ngates = c.ngates;
    free_circuit(&c);
    return 0;
}

/* apply gates [first, first+count) of the circuit (count < 0: all) to psi in place */
int or_run(const char* text, double* psi, int n_expected, int first, int count, int nthreads,
           char* err, int errlen) {
    ocircuit c;
    if (parse_circuit(text, &c, err, errlen)) return -1;
    if (c.n != n_expected) { set_err(err, errlen, "line %d: circuit width does not match state%s", 0, ""); free_circuit(&c); return -1; }
    int last = count < 0 ? c.ngates : first + count;
    if (last > c.ngates) last = c.ngates;
    for (int i = first; i < last; ++i) {
        if (apply_full(c.n, (cplx*)psi, c.g[i].U, c.g[i].k, c.g[i].q, c.g[i].nc, nthreads)) {
            set_err(err, errlen, "line %d: gate too wide for the oracle%s", c.g[i].line, "");
            free_circuit(&c);
            return -1;
        }
    }
    free_circuit(&c);
    return 0;
}

void or_init_zero(int n, double* psi) {
    memset(psi, 0, sizeof(double) * 2 * ((size_t)1 << n));
    psi[0] = 1.0;
}

/* 2^(-n/2): ldexp(1,-n/2) for even n, ldexp(fl(1/sqrt2), -(n-1)/2) for odd n (App. A) */
void or_init_uniform(int n, double* psi) {
    double a = (n % 2 == 0) ? ldexp(1.0, -n / 2) : ldexp(M_SQRT1_2, -(n - 1) / 2);
    size_t N = (size_t)1 << n;
    for (size_t i = 0; i < N; ++i) { psi[2 * i] = a; psi[2 * i + 1] = 0.0; }
}

/* 2^n amplitudes x bytes_per_amp, saturating at UINT64_MAX (R20) */
uint64_t or_memory_estimate(int n, int bytes_per_amp) {
    if (n < 0 || bytes_per_amp <= 0) return 0;
    int sh = 0;
    while ((1 << sh) < bytes_per_amp) ++sh;
    if ((1 << sh) != bytes_per_amp) {
        if (n >= 60) return UINT64_MAX;
        unsigned __int128 v = ((unsigned __int128)1 << n) * (unsigned)bytes_per_amp;
        return v > UINT64_MAX ? UINT64_MAX : (uint64_t)v;
    }
    if (n + sh >= 64) return UINT64_MAX;
    return (uint64_t)1 << (n + sh);
}

static double pairwise(const double* psi, uint64_t lo, uint64_t hi) {
    if (hi - lo == 1) return psi[2 * lo] * psi[2 * lo] + psi[2 * lo + 1] * psi[2 * lo + 1];
    uint64_t mid = lo + (hi - lo) / 2;
    return pairwise(psi, lo, mid) + pairwise(psi, mid, hi);
}

/* sqrt of the pairwise (tree) sum of |a_i|^2 in index order */
double or_norm(int n, const double* psi) {
    return sqrt(pairwise(psi, 0, (uint64_t)1 << n));
}

/* marginal P(qubits[j] = bit j of k), summed in index order */
int or_probabilities(int n, const double* psi, const int* qubits, int nq, double* out) {
    if (nq < 0 || nq > n) return -1;
    for (int j = 0; j < nq; ++j) if (qubits[j] < 0 || qubits[j] >= n) return -2;
    memset(out, 0, sizeof(double) * ((size_t)1 << nq));
    uint64_t N = (uint64_t)1 << n;
    for (uint64_t i = 0; i < N; ++i) {
        uint64_t k = 0;
        for (int j = 0; j < nq; ++j) k |= ((i >> qubits[j]) & 1) << j;
        out[k] += psi[2 * i] * psi[2 * i] + psi[2 * i + 1] * psi[2 * i + 1];
    }
    return 0;
}

/* Classical reversible map of a permutation circuit (X/CNOT/Toffoli/SWAP and 0/1 U, CU):
 * out[i] = f(in[i]) evaluated bit by bit, one gate at a time (S:217 conditional swaps).
 * Returns -1 with an error message if a gate is not a 0/1 permutation. */
int or_classical_map(const char* text, const uint64_t* in, uint64_t* out, uint64_t count,
                     char* err, int errlen) {
    ocircuit c;
    if (parse_circuit(text, &c, err, errlen)) return -1;
    /* for each gate: perm[col] = row with U[row][col] == 1 */
    int** perm = (int**)calloc((size_t)c.ngates, sizeof(int*));
    for (int i = 0; i < c.ngates; ++i) {
        int d = 1 << c.g[i].k;
        perm[i] = (int*)malloc(sizeof(int) * (size_t)d);
        for (int col = 0; col < d; ++col) {
            int found = -1;
            for (int row = 0; row < d; ++row) {
                cplx u = c.g[i].U[row * d + col];
                if (u.re == 1.0 && u.im == 0.0) { if (found >= 0) found = -2; else found = row; }
                else if (u.re != 0.0 || u.im != 0.0) found = -2;
            }
            if (found < 0) {
                set_err(err, errlen, "line %d: gate is not a classical permutation%s", c.g[i].line, "");
                for (int j = 0; j <= i; ++j) free(perm[j]);
                free(perm); free_circuit(&c);
                return -1;
            }
            perm[i][col] = found;
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)count; ++t) {
        uint64_t x = in[t];
        for (int i = 0; i < c.ngates; ++i) {
            const ogate* g = &c.g[i];
            int ok = 1;
            for (int j = 0; j < g->nc; ++j) ok &= (int)((x >> g->q[j]) & 1);
            if (!ok) continue;
            int col = 0;
            for (int j = 0; j < g->k; ++j) col |= (int)((x >> g->q[g->nc + j]) & 1) << j;
            int row = perm[i][col];
            for (int j = 0; j < g->k; ++j) {
                uint64_t b = (uint64_t)1 << g->q[g->nc + j];
                x = ((row >> j) & 1) ? (x | b) : (x & ~b);
            }
        }
        out[t] = x;
    }
    for (int i = 0; i < c.ngates; ++i) free(perm[i]);
    free(perm);
    free_circuit(&c);
    return 0;
}

/* Classical reversible map over a whole index range, bit-sliced (SURVEY 8(c) comparison
 * step 5: "64 indices per uint64 word per gate (Toffoli = AND + XOR on bit planes)").  For
 * 64 consecutive inputs x = first + 64 w + j, plane[b] holds bit b of the 64 inputs (bit j
 * of the plane = input j).  Each gate acts on the planes as its classical definition: a
 * controlled X flips its target where every control is 1 (plane[t] ^= AND of the control
 * planes); a controlled SWAP exchanges its two targets where every control is 1 and they
 * differ.  out[64 w + j] = f(first + 64 w + j).  Only X-type and SWAP-type gates (with any
 * controls) are accepted; first and count must be multiples of 64.  Pinned against the
 * per-index or_classical_map and the multiplier's a*b (tests/test_oracle.py). */
int or_classical_map_range(const char* text, uint64_t first, uint64_t count, uint64_t* out, char* err, int errlen) {
    if ((first | count) & 63) {
        set_err(err, errlen, "line %d: first and count must be multiples of 64%s", 0, "");
        return -1;
    }
    ocircuit c;
    if (parse_circuit(text, &c, err, errlen)) return -1;
    if (c.n > 63) {
        set_err(err, errlen, "line %d: at most 63 qubits%s", 0, "");
        free_circuit(&c);
        return -1;
    }
    /* kind[i]: 1 = X on q[nc], 2 = SWAP of q[nc], q[nc+1] */
    int* kind = (int*)calloc((size_t)c.ngates + 1, sizeof(int));
    for (int i = 0; i < c.ngates; ++i) {
        const ogate* g = &c.g[i];
        const cplx* U = g->U;
        int isx = g->k == 1;
        if (isx) {
            static const double X[8] = {0, 0, 1, 0, 1, 0, 0, 0};
            for (int e = 0; e < 4; ++e) isx &= U[e].re == X[2 * e] && U[e].im == X[2 * e + 1];
        }
        int issw = g->k == 2;
        if (issw)
            for (int r = 0; r < 4; ++r)
                for (int cc = 0; cc < 4; ++cc) {
                    const int sw = ((cc & 1) << 1) | (cc >> 1);
                    const double want = (r == sw) ? 1.0 : 0.0;
                    issw &= U[r * 4 + cc].re == want && U[r * 4 + cc].im == 0.0;
                }
        kind[i] = isx ? 1 : issw ? 2 : 0;
        if (!kind[i]) {
            set_err(err, errlen, "line %d: not an X- or SWAP-type gate%s", g->line, "");
            free(kind);
            free_circuit(&c);
            return -1;
        }
    }
    static const uint64_t low[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                                    0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
    const int n = c.n;
    const int64_t words = (int64_t)(count / 64);
#pragma omp parallel for schedule(static)
    for (int64_t w = 0; w < words; ++w) {
        const uint64_t base = first + 64 * (uint64_t)w;
        uint64_t plane[64];
        for (int b = 0; b < n; ++b) plane[b] = b < 6 ? low[b] : (((base >> b) & 1) ? ~0ull : 0ull);
        for (int i = 0; i < c.ngates; ++i) {
            const ogate* g = &c.g[i];
            uint64_t on = ~0ull;
            for (int j = 0; j < g->nc; ++j) on &= plane[g->q[j]];
            if (kind[i] == 1) {
                plane[g->q[g->nc]] ^= on;
            } else {
                const int a = g->q[g->nc], b = g->q[g->nc + 1];
                const uint64_t d = on & (plane[a] ^ plane[b]);
                plane[a] ^= d;
                plane[b] ^= d;
            }
        }
        for (int j = 0; j < 64; ++j) {
            uint64_t x = 0;
            for (int b = 0; b < n; ++b) x |= ((plane[b] >> j) & 1ull) << b;
            out[64 * w + j] = x;
        }
    }
    free(kind);
    free_circuit(&c);
    return 0;
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
