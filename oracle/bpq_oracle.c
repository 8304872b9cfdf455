/*
 * bpq_oracle.c -- CPU restatement of the reference bilayer-PQ search path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port" arm of bench.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_1404_1831_b200) never links or calls it.
 *
 * Every function restates one reference function, cited file:line against
 * /root/reference/pkg/src/bilayerpq/ (abbreviated bpq/).  Arithmetic is IEEE
 * float32 in the reference's operation order; the build uses
 * -ffp-contract=off so no multiply-add is fused (numba does not fuse either,
 * which the survey verified bit-for-bit).
 *
 * Pinned against the reference itself: tests/golden/make_golden.py runs the
 * reference package and stores its outputs; tests/test_oracle_golden.py
 * checks this file against them.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* traverse_cells: bpq/kernels/numba_backend.py:11-146                       */
/* Multi-sequence min-heap keyed (key f64, oi, oj) with the popped bitmap.  */
/* Returns the number of visited non-empty cells written to the outputs,    */
/* which must hold cap = max(1, min(budget, total, t*t)) entries (:14-19).  */
/* ------------------------------------------------------------------------ */
static int heap_less(double ka, int32_t ia, int32_t ja, double kb, int32_t ib, int32_t jb) {
    if (ka < kb) return 1;
    if (ka == kb) return (ia < ib) || (ia == ib && ja < jb);
    return 0;
}

int64_t orc_traverse_cells(const double *sr1, const double *sr2, const int32_t *order1,
                           const int32_t *order2, const int64_t *offsets, int64_t t,
                           int64_t budget, int32_t *vis_i, int32_t *vis_j, int64_t *starts,
                           int64_t *ends) {
    uint8_t *popped = (uint8_t *)calloc((size_t)(t * t), 1); /* :25 */
    int64_t hcap = 2 * t + 4;                                  /* :28 */
    double *hkey = (double *)malloc(sizeof(double) * hcap);
    int32_t *hoi = (int32_t *)malloc(sizeof(int32_t) * hcap);
    int32_t *hoj = (int32_t *)malloc(sizeof(int32_t) * hcap);
    int32_t *ha = (int32_t *)malloc(sizeof(int32_t) * hcap);
    int32_t *hb = (int32_t *)malloc(sizeof(int32_t) * hcap);
    int64_t hn = 1, nvis = 0, collected = 0;
    hkey[0] = sr1[0] + sr2[0]; /* :36-42 */
    hoi[0] = order1[0];
    hoj[0] = order2[0];
    ha[0] = 0;
    hb[0] = 0;
    while (hn > 0) { /* :46 */
        int32_t oi = hoi[0], oj = hoj[0], a = ha[0], b = hb[0];
        hn -= 1; /* pop root, sift the last element down (:53-89) */
        if (hn > 0) {
            double ck = hkey[hn];
            int32_t coi = hoi[hn], coj = hoj[hn], ca = ha[hn], cb = hb[hn];
            int64_t pos = 0;
            for (;;) {
                int64_t child = 2 * pos + 1;
                if (child >= hn) break;
                int64_t right = child + 1;
                if (right < hn && heap_less(hkey[right], hoi[right], hoj[right], hkey[child],
                                            hoi[child], hoj[child]))
                    child = right;
                if (heap_less(hkey[child], hoi[child], hoj[child], ck, coi, coj)) {
                    hkey[pos] = hkey[child];
                    hoi[pos] = hoi[child];
                    hoj[pos] = hoj[child];
                    ha[pos] = ha[child];
                    hb[pos] = hb[child];
                    pos = child;
                } else {
                    break;
                }
            }
            hkey[pos] = ck;
            hoi[pos] = coi;
            hoj[pos] = coj;
            ha[pos] = ca;
            hb[pos] = cb;
        }
        popped[(int64_t)a * t + b] = 1; /* :91 */
        int64_t lin = (int64_t)oi * t + oj;
        int64_t s = offsets[lin], e = offsets[lin + 1];
        if (e > s) { /* :95-102 */
            vis_i[nvis] = oi;
            vis_j[nvis] = oj;
            starts[nvis] = s;
            ends[nvis] = e;
            nvis++;
            collected += e - s;
        }
        for (int push = 0; push < 2; push++) { /* :104-141 */
            int32_t na, nb;
            int ok;
            if (push == 0) {
                na = a + 1;
                nb = b;
                ok = na < t && (b == 0 || popped[(int64_t)na * t + (b - 1)]);
            } else {
                na = a;
                nb = b + 1;
                ok = nb < t && (a == 0 || popped[(int64_t)(a - 1) * t + nb]);
            }
            if (!ok) continue;
            double nkey = sr1[na] + sr2[nb];
            int32_t noi = order1[na], noj = order2[nb];
            int64_t pos = hn++;
            while (pos > 0) {
                int64_t parent = (pos - 1) / 2;
                if (heap_less(nkey, noi, noj, hkey[parent], hoi[parent], hoj[parent])) {
                    hkey[pos] = hkey[parent];
                    hoi[pos] = hoi[parent];
                    hoj[pos] = hoj[parent];
                    ha[pos] = ha[parent];
                    hb[pos] = hb[parent];
                    pos = parent;
                } else {
                    break;
                }
            }
            hkey[pos] = nkey;
            hoi[pos] = noi;
            hoj[pos] = noj;
            ha[pos] = na;
            hb[pos] = nb;
        }
        if (collected >= budget) break; /* :143-144 */
    }
    free(popped);
    free(hkey);
    free(hoi);
    free(hoj);
    free(ha);
    free(hb);
    return nvis;
}

/* ------------------------------------------------------------------------ */
/* scan_global: bpq/kernels/numba_backend.py:149-180 (sequential f32).      */
/* e1/e2 are the (t, dh) query displacement tables (multi_index.py:342-347) */
/* ------------------------------------------------------------------------ */
void orc_scan_global(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                     const int64_t *ends, int64_t nvis, const uint32_t *ids,
                     const uint8_t *codes, const float *e1, const float *e2, const float *books,
                     int64_t m, int64_t k, int64_t ds, uint32_t *out_ids, float *out_d) {
    int64_t m2 = m / 2, dh = m2 * ds, pos = 0;
    for (int64_t v = 0; v < nvis; v++) {
        const float *r1 = e1 + (int64_t)vis_i[v] * dh;
        const float *r2 = e2 + (int64_t)vis_j[v] * dh;
        for (int64_t e = starts[v]; e < ends[v]; e++) {
            float acc = 0.0f;
            for (int64_t p = 0; p < m2; p++) {
                const float *bk = books + (p * k + codes[e * m + p]) * ds;
                for (int64_t u = 0; u < ds; u++) {
                    float d = r1[p * ds + u] - bk[u];
                    acc += d * d;
                }
            }
            for (int64_t p = m2; p < m; p++) {
                const float *bk = books + (p * k + codes[e * m + p]) * ds;
                for (int64_t u = 0; u < ds; u++) {
                    float d = r2[(p - m2) * ds + u] - bk[u];
                    acc += d * d;
                }
            }
            out_ids[pos] = ids[e];
            out_d[pos] = acc;
            pos++;
        }
    }
}

/* scan_local: bpq/kernels/numba_backend.py:183-213; books1/2 (t, m2, k, ds) */
void orc_scan_local(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                    const int64_t *ends, int64_t nvis, const uint32_t *ids, const uint8_t *codes,
                    const float *e1, const float *e2, const float *books1, const float *books2,
                    int64_t m2, int64_t k, int64_t ds, uint32_t *out_ids, float *out_d) {
    int64_t m = 2 * m2, dh = m2 * ds, pos = 0;
    for (int64_t v = 0; v < nvis; v++) {
        int64_t i = vis_i[v], j = vis_j[v];
        const float *r1 = e1 + i * dh;
        const float *r2 = e2 + j * dh;
        for (int64_t e = starts[v]; e < ends[v]; e++) {
            float acc = 0.0f;
            for (int64_t p = 0; p < m2; p++) {
                const float *bk = books1 + ((i * m2 + p) * k + codes[e * m + p]) * ds;
                for (int64_t u = 0; u < ds; u++) {
                    float d = r1[p * ds + u] - bk[u];
                    acc += d * d;
                }
            }
            for (int64_t p = 0; p < m2; p++) {
                const float *bk = books2 + ((j * m2 + p) * k + codes[e * m + m2 + p]) * ds;
                for (int64_t u = 0; u < ds; u++) {
                    float d = r2[p * ds + u] - bk[u];
                    acc += d * d;
                }
            }
            out_ids[pos] = ids[e];
            out_d[pos] = acc;
            pos++;
        }
    }
}

/* scan_tables: bpq/kernels/numba_backend.py:216-246 (FBPQ, clamp < 0). */
void orc_scan_tables(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                     const int64_t *ends, int64_t nvis, const uint32_t *ids,
                     const uint8_t *codes, float q_norm, const float *qd1, const float *qd2,
                     const float *cn1, const float *cn2, const float *fold, const float *cross1,
                     const float *cross2, int64_t m, int64_t k, uint32_t *out_ids, float *out_d) {
    int64_t m2 = m / 2, pos = 0;
    const float two = 2.0f;
    for (int64_t v = 0; v < nvis; v++) {
        int64_t i = vis_i[v], j = vis_j[v];
        float cell_base = q_norm - two * (qd1[i] + qd2[j]) + cn1[i] + cn2[j]; /* :232 */
        for (int64_t e = starts[v]; e < ends[v]; e++) {
            float acc = cell_base;
            for (int64_t p = 0; p < m2; p++) {
                int64_t c = codes[e * m + p];
                acc += fold[p * k + c] + two * cross1[(i * m2 + p) * k + c];
            }
            for (int64_t p = m2; p < m; p++) {
                int64_t c = codes[e * m + p];
                acc += fold[p * k + c] + two * cross2[(j * m2 + (p - m2)) * k + c];
            }
            if (acc < 0.0f) acc = 0.0f;
            out_ids[pos] = ids[e];
            out_d[pos] = acc;
            pos++;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* select_top: bpq/multi_index.py:326-339 -- top-r by (dist asc, id asc).   */
/* argpartition + threshold + lexsort equals a full (dist, id) sort cut at  */
/* r; float comparison treats -0.0 == +0.0 as numpy's lexsort does.         */
/* ------------------------------------------------------------------------ */
typedef struct {
    float d;
    uint32_t id;
} orc_cand;

static int cand_cmp(const void *pa, const void *pb) {
    const orc_cand *a = (const orc_cand *)pa, *b = (const orc_cand *)pb;
    if (a->d < b->d) return -1;
    if (a->d > b->d) return 1;
    if (a->id < b->id) return -1;
    if (a->id > b->id) return 1;
    return 0;
}

int64_t orc_select_top(const uint32_t *ids, const float *d, int64_t n, int64_t r,
                       uint32_t *out_ids, float *out_d) {
    if (n == 0) return 0;
    orc_cand *c = (orc_cand *)malloc(sizeof(orc_cand) * n);
    for (int64_t x = 0; x < n; x++) {
        c[x].d = d[x];
        c[x].id = ids[x];
    }
    qsort(c, (size_t)n, sizeof(orc_cand), cand_cmp);
    int64_t cnt = r < n ? r : n;
    for (int64_t x = 0; x < cnt; x++) {
        out_ids[x] = c[x].id;
        out_d[x] = c[x].d;
    }
    free(c);
    return cnt;
}

/* ------------------------------------------------------------------------ */
/* Whole-query search in C, used only as the multi-threaded CPU baseline.   */
/* coarse_scan (multi_index.py:270-293) with plain sequential f32 dots in   */
/* place of OpenBLAS sgemv; stable argsort (multi_index.py:319-322);        */
/* traverse; the engine's scan; select_top.                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    float r;
    int32_t idx;
} orc_rkey;

static int rkey_cmp(const void *pa, const void *pb) {
    const orc_rkey *a = (const orc_rkey *)pa, *b = (const orc_rkey *)pb;
    if (a->r < b->r) return -1;
    if (a->r > b->r) return 1;
    return (a->idx > b->idx) - (a->idx < b->idx); /* stable: original index */
}

typedef struct {
    int engine; /* 0 baseline, 1 fbpq, 2 hbpq */
    int64_t t, dh, m, k, n;
    const float *c1, *c2, *cn1, *cn2;
    const int64_t *offsets;
    const uint32_t *ids;
    const uint8_t *codes;
    const float *books;                  /* baseline / fbpq prepare: (m, k, ds) */
    const float *fine_norms;             /* fbpq (m, k) */
    const float *cross1, *cross2;        /* fbpq (t, m2, k) */
    const float *bank1, *bank2;          /* hbpq (t, m2, k, ds) */
    const float *queries;
    int64_t l, r;
    float *out_d;
    uint32_t *out_ids;
    int32_t *out_count;
    int64_t *out_cands;
    int64_t q0, q1;
} orc_job;

static float dotf(const float *a, const float *b, int64_t n) {
    float s = 0.0f;
    for (int64_t x = 0; x < n; x++) s += a[x] * b[x];
    return s;
}

static void *orc_worker(void *arg) {
    orc_job *J = (orc_job *)arg;
    int64_t t = J->t, dh = J->dh, m = J->m, k = J->k, m2 = J->m / 2, ds = 2 * dh / J->m;
    int64_t total = J->offsets[t * t];
    int64_t cap = J->l < total ? J->l : total;
    if (cap > t * t) cap = t * t;
    if (cap < 1) cap = 1;
    float *dots1 = malloc(sizeof(float) * t), *dots2 = malloc(sizeof(float) * t);
    orc_rkey *rk = malloc(sizeof(orc_rkey) * t);
    double *sr1 = malloc(sizeof(double) * t), *sr2 = malloc(sizeof(double) * t);
    int32_t *o1 = malloc(sizeof(int32_t) * t), *o2 = malloc(sizeof(int32_t) * t);
    int32_t *vi = malloc(sizeof(int32_t) * cap), *vj = malloc(sizeof(int32_t) * cap);
    int64_t *vs = malloc(sizeof(int64_t) * cap), *ve = malloc(sizeof(int64_t) * cap);
    float *e1 = NULL, *e2 = NULL, *fold = NULL;
    if (J->engine != 1) {
        e1 = malloc(sizeof(float) * t * dh);
        e2 = malloc(sizeof(float) * t * dh);
    } else {
        fold = malloc(sizeof(float) * m * k);
    }
    int64_t cand_cap = 0;
    uint32_t *cid = NULL;
    float *cd = NULL;
    for (int64_t q = J->q0; q < J->q1; q++) {
        const float *qv = J->queries + q * 2 * dh;
        float q1n = dotf(qv, qv, dh), q2n = dotf(qv + dh, qv + dh, dh);
        for (int64_t x = 0; x < t; x++) {
            dots1[x] = dotf(J->c1 + x * dh, qv, dh);
            dots2[x] = dotf(J->c2 + x * dh, qv + dh, dh);
        }
        for (int h = 0; h < 2; h++) {
            const float *dots = h ? dots2 : dots1;
            const float *cn = h ? J->cn2 : J->cn1;
            float qn = h ? q2n : q1n;
            for (int64_t x = 0; x < t; x++) {
                float rv = (cn[x] - 2.0f * dots[x]) + qn;
                rk[x].r = rv < 0.0f ? 0.0f : rv;
                rk[x].idx = (int32_t)x;
            }
            qsort(rk, (size_t)t, sizeof(orc_rkey), rkey_cmp);
            double *sr = h ? sr2 : sr1;
            int32_t *o = h ? o2 : o1;
            for (int64_t x = 0; x < t; x++) {
                sr[x] = (double)rk[x].r;
                o[x] = rk[x].idx;
            }
        }
        int64_t nvis = 0;
        if (total > 0)
            nvis = orc_traverse_cells(sr1, sr2, o1, o2, J->offsets, t, J->l, vi, vj, vs, ve);
        int64_t nc = 0;
        for (int64_t v = 0; v < nvis; v++) nc += ve[v] - vs[v];
        if (nc > cand_cap) {
            cand_cap = nc * 2;
            cid = realloc(cid, sizeof(uint32_t) * cand_cap);
            cd = realloc(cd, sizeof(float) * cand_cap);
        }
        if (J->engine == 1) {
            for (int64_t p = 0; p < m; p++)
                for (int64_t c = 0; c < k; c++)
                    fold[p * k + c] =
                        J->fine_norms[p * k + c] -
                        2.0f * dotf(J->books + (p * k + c) * ds, qv + p * ds, ds);
            float qn = dotf(qv, qv, 2 * dh);
            orc_scan_tables(vi, vj, vs, ve, nvis, J->ids, J->codes, qn, dots1, dots2, J->cn1,
                            J->cn2, fold, J->cross1, J->cross2, m, k, cid, cd);
        } else {
            for (int64_t x = 0; x < t; x++)
                for (int64_t u = 0; u < dh; u++) {
                    e1[x * dh + u] = qv[u] - J->c1[x * dh + u];
                    e2[x * dh + u] = qv[dh + u] - J->c2[x * dh + u];
                }
            if (J->engine == 0)
                orc_scan_global(vi, vj, vs, ve, nvis, J->ids, J->codes, e1, e2, J->books, m, k,
                                ds, cid, cd);
            else
                orc_scan_local(vi, vj, vs, ve, nvis, J->ids, J->codes, e1, e2, J->bank1,
                               J->bank2, m2, k, ds, cid, cd);
        }
        int64_t cnt = orc_select_top(cid, cd, nc, J->r, J->out_ids + q * J->r, J->out_d + q * J->r);
        for (int64_t x = cnt; x < J->r; x++) {
            J->out_ids[q * J->r + x] = 0xFFFFFFFFu;
            J->out_d[q * J->r + x] = INFINITY;
        }
        J->out_count[q] = (int32_t)cnt;
        if (J->out_cands) J->out_cands[q] = nc;
    }
    free(dots1); free(dots2); free(rk); free(sr1); free(sr2); free(o1); free(o2);
    free(vi); free(vj); free(vs); free(ve); free(e1); free(e2); free(fold); free(cid); free(cd);
    return NULL;
}

/* Batched search over nq queries with nthreads POSIX threads (queries split */
/* contiguously).  Outputs are padded to r per query with (inf, 0xFFFFFFFF). */
int orc_search_batch(int engine, int64_t t, int64_t dh, int64_t m, int64_t k, const float *c1,
                     const float *c2, const float *cn1, const float *cn2,
                     const int64_t *offsets, const uint32_t *ids, const uint8_t *codes,
                     const float *books, const float *fine_norms, const float *cross1,
                     const float *cross2, const float *bank1, const float *bank2,
                     const float *queries, int64_t nq, int64_t l, int64_t r, float *out_d,
                     uint32_t *out_ids, int32_t *out_count, int64_t *out_cands, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > nq) nthreads = (int)(nq > 0 ? nq : 1);
    pthread_t *th = malloc(sizeof(pthread_t) * nthreads);
    orc_job *jobs = malloc(sizeof(orc_job) * nthreads);
    for (int x = 0; x < nthreads; x++) {
        orc_job *J = &jobs[x];
        J->engine = engine; J->t = t; J->dh = dh; J->m = m; J->k = k;
        J->c1 = c1; J->c2 = c2; J->cn1 = cn1; J->cn2 = cn2; J->offsets = offsets;
        J->ids = ids; J->codes = codes; J->books = books; J->fine_norms = fine_norms;
        J->cross1 = cross1; J->cross2 = cross2; J->bank1 = bank1; J->bank2 = bank2;
        J->queries = queries; J->l = l; J->r = r; J->out_d = out_d; J->out_ids = out_ids;
        J->out_count = out_count; J->out_cands = out_cands;
        J->q0 = nq * x / nthreads;
        J->q1 = nq * (x + 1) / nthreads;
        pthread_create(&th[x], NULL, orc_worker, J);
    }
    for (int x = 0; x < nthreads; x++) pthread_join(th[x], NULL);
    free(th);
    free(jobs);
    return 0;
}
