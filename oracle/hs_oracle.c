/*
 * CPU ORACLE (C restatement) -- test infrastructure only, never the product.
 *
 * Same recurrence as oracle/hs_oracle.py::fitness_one, which restates the
 * reference decoder /root/reference/pkg/src/hetsched/heuristics.py:43-148
 * (try_place :92-106, ready_time :67-78, non-insertion _slot :80-84,
 * commit :108-120) with comm_time core.py:148-155. Tables come from
 * oracle/hs_oracle.py::build_tables (NOT from the product's plan compiler),
 * so the two implementations stay independent. Parity is pinned by
 * tests/test_oracle_golden.py against fixtures produced by the reference.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library. Built by oracle/Makefile with -ffp-contract=off so that no
 * multiply-add is fused (the reference computes in plain IEEE binary64).
 *
 * Status codes: 0 ok, 1 batch size, 2 memory, 3 link, 4 missing latency,
 * 5 gene out of range.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int V, K;
    const int32_t *pred_off;  /* [V+1] */
    const int32_t *pred_pos;  /* [E] predecessor positions */
    const double *dur;        /* [V*K] */
    const uint8_t *dur_ok;    /* [V*K] */
    const double *extra;      /* [V] */
    const double *cap;        /* [K] */
    const uint8_t *okL;       /* [K] */
    const double *comm;       /* [V*K*K] comm[p][u][v] */
    const uint8_t *link;      /* [K*K] */
} hso_tables;

static inline double pymax(double a, double b) { return b > a ? b : a; }

/* One candidate. Returns status; *ms gets the makespan (inf if status). */
static int eval_one(const hso_tables *t, const uint8_t *g, double *ms_out,
                    double *starts, double *avail, double *mem, double *end)
{
    const int V = t->V, K = t->K;
    for (int i = 0; i < V; ++i)
        if (g[i] >= K) { *ms_out = INFINITY; return 5; }
    for (int k = 0; k < K; ++k) { avail[k] = 0.0; mem[k] = 0.0; }
    double ms = 0.0;
    for (int i = 0; i < V; ++i) {
        const int d = g[i];
        if (!t->okL[d]) { *ms_out = INFINITY; return 1; }
        if (mem[d] + t->extra[i] > t->cap[d]) { *ms_out = INFINITY; return 2; }
        double r = 0.0;
        for (int e = t->pred_off[i]; e < t->pred_off[i + 1]; ++e) {
            const int p = t->pred_pos[e];
            const int gp = g[p];
            if (!t->link[gp * K + d]) { *ms_out = INFINITY; return 3; }
            const double c = (gp == d) ? 0.0 : t->comm[((size_t)p * K + gp) * K + d];
            r = pymax(r, end[p] + c);
        }
        if (!t->dur_ok[(size_t)i * K + d]) { *ms_out = INFINITY; return 4; }
        const double s = pymax(r, avail[d]);
        const double e = s + t->dur[(size_t)i * K + d];
        if (starts) starts[i] = s;
        end[i] = e;
        avail[d] = e;
        mem[d] += t->extra[i];
        ms = pymax(ms, e);
    }
    *ms_out = ms;
    return 0;
}

typedef struct {
    const hso_tables *t;
    const uint8_t *genes;
    int64_t ld, lo, hi;
    double *out;
    uint8_t *status;
} job_t;

static void *run_job(void *arg)
{
    job_t *j = (job_t *)arg;
    const int V = j->t->V, K = j->t->K;
    double *buf = (double *)malloc(sizeof(double) * (size_t)(2 * K + V + 1));
    double *avail = buf, *mem = buf + K, *end = buf + 2 * K;
    for (int64_t c = j->lo; c < j->hi; ++c) {
        double ms;
        int st = eval_one(j->t, j->genes + c * j->ld, &ms, NULL, avail, mem, end);
        j->out[c] = ms;
        if (j->status) j->status[c] = (uint8_t)st;
    }
    free(buf);
    return NULL;
}

/* Batch fitness over n genomes (row stride ld bytes) on nthreads threads. */
int hso_fitness(const hso_tables *t, const uint8_t *genes, int64_t n,
                int64_t ld, double *out, uint8_t *status, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > n) nthreads = (int)(n > 0 ? n : 1);
    pthread_t th[256];
    job_t jobs[256];
    for (int k = 0; k < nthreads; ++k) {
        jobs[k].t = t; jobs[k].genes = genes; jobs[k].ld = ld;
        jobs[k].lo = n * k / nthreads; jobs[k].hi = n * (k + 1) / nthreads;
        jobs[k].out = out; jobs[k].status = status;
    }
    if (nthreads == 1) { run_job(&jobs[0]); return 0; }
    for (int k = 0; k < nthreads; ++k)
        pthread_create(&th[k], NULL, run_job, &jobs[k]);
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    return 0;
}

/* decode() trace of one genome: per-position start times. */
int hso_trace(const hso_tables *t, const uint8_t *genes, double *starts,
              double *ms)
{
    const int V = t->V, K = t->K;
    double *buf = (double *)malloc(sizeof(double) * (size_t)(2 * K + V + 1));
    int st = eval_one(t, genes, ms, starts, buf, buf + K, buf + 2 * K);
    free(buf);
    return st;
}
