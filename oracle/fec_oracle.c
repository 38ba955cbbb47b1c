/*
 * FEC ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of what the FEC hot path computes.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, table or constant generator with
 * the CUDA path (paper_2208_07678_b200/csrc); neither side includes the other.
 *
 * What it computes (the plain definition; DESIGN.md §2 "Readings"):
 *
 *   d  = fp32(d_th);  t2 = fl32(d*d)                                  (reading A3)
 *   pred(i,j): dx = fl(x_j - x_i), dy = fl(y_j - y_i), dz = fl(z_j - z_i)
 *              d2 = fl(fl(fl(dx*dx) + fl(dy*dy)) + fl(dz*dz));  d2 <= t2
 *        -- PAPER.md L187-194 (§2.2, Eq. 1, the Euclidean proximity criterion), with the
 *           inclusive boundary and fixed fp32 operation order of readings A1/A2.
 *   G = ({0..n-1}, {{i,j}: i != j and pred(i,j)})
 *   C(i) = connected component of i in G         -- the clusters Algorithm 1 is meant to
 *          output (Alg. 1 I/O L132-145; EC semantics L215, L227).
 *   labels[i] = min C(i)  if  min_size <= |C(i)| <= max_size,  else -1   (readings A7/A8/A10)
 *
 * How: bucket the points in a uniform grid of edge c_o = 1.01*d (double), then flood-fill
 * (breadth first) from every unvisited point in increasing index order.  A visited point
 * is swap-removed from its bucket so it is never tested again.  Because components are
 * started in increasing index order, the seed i is the minimum index of its component.
 *
 * Why the grid is exact: a pred-true pair has |x_j - x_i| <= d*(1 + 2^-21) on every axis
 * (fp32 rounding of the differences/squares/sums), which is < c_o, so the two points lie
 * in the same or adjacent cells on each axis; scanning the 27 surrounding cells therefore
 * tests every pred-true pair.
 *
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC   (x86-64 SSE2, so every
 * float operation is a single IEEE binary32 round-to-nearest-even; no FMA, no x87).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#define ORACLE_OK 0
#define ORACLE_ERR_INVALID_ARGUMENT (-1)
#define ORACLE_ERR_NONFINITE (-2)
#define ORACLE_ERR_RANGE (-3)
#define ORACLE_ERR_NOMEM (-4)

/* ---- the predicate (Eq. 1, readings A1-A3) ------------------------------------------ */

float oracle_t2(float d) {
    float t2 = d * d;
    return t2;
}

int oracle_pred(const float* a, const float* b, float t2) {
    float dx = b[0] - a[0];
    float dy = b[1] - a[1];
    float dz = b[2] - a[2];
    float sx = dx * dx;
    float sy = dy * dy;
    float sz = dz * dz;
    float s = sx + sy;
    s = s + sz;
    return s <= t2;
}

/* d2 exactly as the predicate computes it (exported for the rounding pins). */
float oracle_d2(const float* a, const float* b) {
    float dx = b[0] - a[0];
    float dy = b[1] - a[1];
    float dz = b[2] - a[2];
    float sx = dx * dx;
    float sy = dy * dy;
    float sz = dz * dz;
    float s = sx + sy;
    s = s + sz;
    return s;
}

/* Argument checks (readings A12, A13, A7). */
static int check_args(const float* p, int64_t n, float d, int64_t mn, int64_t mx) {
    if (n < 0 || n > INT32_MAX) return ORACLE_ERR_INVALID_ARGUMENT;
    if (!(d > 0.0f) || !isfinite(d)) return ORACLE_ERR_INVALID_ARGUMENT;
    float t2 = oracle_t2(d);
    if (!isfinite(t2) || t2 < FLT_MIN) return ORACLE_ERR_INVALID_ARGUMENT;
    if (mn < 0 || mx < 1 || mn > mx) return ORACLE_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < 3 * n; ++i)
        if (!isfinite(p[i])) return ORACLE_ERR_NONFINITE;
    return ORACLE_OK;
}

/* ---- grid buckets -------------------------------------------------------------------- */

typedef struct {
    int64_t n;
    const float* p;
    float t2;
    int64_t* cx;          /* cell coordinate of each point, 3 per point */
    int64_t ncell;
    int64_t* cstart;      /* first slot of cell k in items */
    int64_t* calive;      /* one past the last alive slot of cell k */
    int64_t* ccoord;      /* 3 per cell */
    int32_t* items;       /* point ids grouped by cell */
    int64_t* slot;        /* slot of each point in items */
    int64_t* pcell;       /* cell id of each point */
    int64_t hcap;         /* hash: cell coordinate -> cell id */
    int64_t* htab;
} grid_t;

static const int64_t* g_sort_cx;
static int cmp_pts(const void* A, const void* B) {
    int32_t a = *(const int32_t*)A, b = *(const int32_t*)B;
    for (int k = 0; k < 3; ++k) {
        int64_t u = g_sort_cx[3 * (int64_t)a + k], v = g_sort_cx[3 * (int64_t)b + k];
        if (u != v) return u < v ? -1 : 1;
    }
    return a < b ? -1 : (a > b);
}

static uint64_t hash3(int64_t x, int64_t y, int64_t z) {
    uint64_t h = (uint64_t)x * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)y * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
    h ^= (uint64_t)z * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
    return h ^ (h >> 29);
}

static int64_t grid_find(const grid_t* g, int64_t x, int64_t y, int64_t z) {
    uint64_t m = (uint64_t)g->hcap - 1;
    for (uint64_t h = hash3(x, y, z) & m;; h = (h + 1) & m) {
        int64_t c = g->htab[h];
        if (c < 0) return -1;
        const int64_t* q = g->ccoord + 3 * c;
        if (q[0] == x && q[1] == y && q[2] == z) return c;
    }
}

static void grid_free(grid_t* g) {
    free(g->cx); free(g->cstart); free(g->calive); free(g->ccoord); free(g->items);
    free(g->slot); free(g->pcell); free(g->htab);
    memset(g, 0, sizeof(*g));
}

static int grid_build(grid_t* g, const float* p, int64_t n, float d) {
    memset(g, 0, sizeof(*g));
    g->n = n; g->p = p; g->t2 = oracle_t2(d);
    if (n == 0) return ORACLE_OK;
    double lo[3];
    for (int k = 0; k < 3; ++k) lo[k] = p[k];
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k)
            if ((double)p[3 * i + k] < lo[k]) lo[k] = p[3 * i + k];
    double c = 1.01 * (double)d;
    g->cx = malloc(sizeof(int64_t) * 3 * n);
    g->items = malloc(sizeof(int32_t) * n);
    g->slot = malloc(sizeof(int64_t) * n);
    g->pcell = malloc(sizeof(int64_t) * n);
    if (!g->cx || !g->items || !g->slot || !g->pcell) { grid_free(g); return ORACLE_ERR_NOMEM; }
    for (int64_t i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) {
            double q = floor(((double)p[3 * i + k] - lo[k]) / c);
            if (!(q < 4.0e18)) { grid_free(g); return ORACLE_ERR_RANGE; }
            g->cx[3 * i + k] = (int64_t)q;
        }
        g->items[i] = (int32_t)i;
    }
    g_sort_cx = g->cx;
    qsort(g->items, (size_t)n, sizeof(int32_t), cmp_pts);
    /* cells = runs of equal coordinates */
    int64_t nc = 0;
    for (int64_t s = 0; s < n; ++s) {
        if (s == 0 || memcmp(g->cx + 3 * (int64_t)g->items[s], g->cx + 3 * (int64_t)g->items[s - 1],
                             3 * sizeof(int64_t)) != 0)
            ++nc;
    }
    g->ncell = nc;
    g->cstart = malloc(sizeof(int64_t) * (nc + 1));
    g->calive = malloc(sizeof(int64_t) * nc);
    g->ccoord = malloc(sizeof(int64_t) * 3 * nc);
    g->hcap = 1;
    while (g->hcap < 2 * nc) g->hcap <<= 1;
    g->htab = malloc(sizeof(int64_t) * g->hcap);
    if (!g->cstart || !g->calive || !g->ccoord || !g->htab) { grid_free(g); return ORACLE_ERR_NOMEM; }
    for (int64_t h = 0; h < g->hcap; ++h) g->htab[h] = -1;
    int64_t k = -1;
    for (int64_t s = 0; s < n; ++s) {
        int32_t i = g->items[s];
        if (s == 0 || memcmp(g->cx + 3 * (int64_t)i, g->cx + 3 * (int64_t)g->items[s - 1],
                             3 * sizeof(int64_t)) != 0) {
            ++k;
            g->cstart[k] = s;
            memcpy(g->ccoord + 3 * k, g->cx + 3 * (int64_t)i, 3 * sizeof(int64_t));
            uint64_t m = (uint64_t)g->hcap - 1;
            uint64_t h = hash3(g->ccoord[3 * k], g->ccoord[3 * k + 1], g->ccoord[3 * k + 2]) & m;
            while (g->htab[h] >= 0) h = (h + 1) & m;
            g->htab[h] = k;
        }
        g->slot[i] = s;
        g->pcell[i] = k;
    }
    g->cstart[nc] = n;
    for (int64_t c2 = 0; c2 < nc; ++c2) g->calive[c2] = g->cstart[c2 + 1];
    return ORACLE_OK;
}

/* swap-remove point v (in cell c) from the alive part of its bucket; optionally log it */
static void grid_remove(grid_t* g, int32_t v) {
    int64_t c = g->pcell[v];
    int64_t s = g->slot[v];
    int64_t last = g->calive[c] - 1;
    int32_t w = g->items[last];
    g->items[last] = v; g->slot[v] = last;
    g->items[s] = w; g->slot[w] = s;
    g->calive[c] = last;
}

/* Breadth-first flood fill from `seed` (already removed).  Appends members to queue[*tail].
 * Returns the number of predicate evaluations (for instrumentation). */
static int64_t flood(grid_t* g, int32_t* queue, int64_t head, int64_t* tail) {
    int64_t tests = 0;
    while (head < *tail) {
        int32_t u = queue[head++];
        const float* pu = g->p + 3 * (int64_t)u;
        const int64_t* cu = g->cx + 3 * (int64_t)u;
        for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dz = -1; dz <= 1; ++dz) {
                    int64_t c = grid_find(g, cu[0] + dx, cu[1] + dy, cu[2] + dz);
                    if (c < 0) continue;
                    int64_t s = g->cstart[c];
                    while (s < g->calive[c]) {
                        int32_t v = g->items[s];
                        ++tests;
                        if (oracle_pred(pu, g->p + 3 * (int64_t)v, g->t2)) {
                            grid_remove(g, v);     /* slot s now holds another alive point */
                            queue[(*tail)++] = v;
                        } else {
                            ++s;
                        }
                    }
                }
    }
    return tests;
}

/* Full clustering: labels[i] = min C(i) if min_size <= |C(i)| <= max_size else -1. */
int oracle_fec(const float* p, int64_t n, float d, int64_t min_size, int64_t max_size,
               int32_t* labels, int64_t* stats /* nullable: [components, pred tests] */) {
    int rc = check_args(p, n, d, min_size, max_size);
    if (rc) return rc;
    if (stats) { stats[0] = 0; stats[1] = 0; }
    if (n == 0) return ORACLE_OK;
    grid_t g;
    rc = grid_build(&g, p, n, d);
    if (rc) return rc;
    int32_t* queue = malloc(sizeof(int32_t) * n);
    if (!queue) { grid_free(&g); return ORACLE_ERR_NOMEM; }
    char* visited = calloc((size_t)n, 1);
    if (!visited) { free(queue); grid_free(&g); return ORACLE_ERR_NOMEM; }
    int64_t ncomp = 0, tests = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (visited[i]) continue;
        int64_t head = 0, tail = 0;
        grid_remove(&g, (int32_t)i);
        queue[tail++] = (int32_t)i;
        tests += flood(&g, queue, head, &tail);
        int64_t size = tail;
        int32_t lab = (size >= min_size && size <= max_size) ? (int32_t)i : -1;
        for (int64_t k = 0; k < tail; ++k) {
            visited[queue[k]] = 1;
            labels[queue[k]] = lab;
        }
        ++ncomp;
    }
    if (stats) { stats[0] = ncomp; stats[1] = tests; }
    free(visited); free(queue); grid_free(&g);
    return ORACLE_OK;
}

/* ---- one-component queries (for sampled parity at full size) ------------------------
 * oracle_index_build() buckets the cloud once; oracle_component() flood-fills from one
 * seed and then restores the buckets, returning min C(seed) and |C(seed)|. */

typedef struct { grid_t g; int32_t* queue; } oracle_index_t;

void* oracle_index_build(const float* p, int64_t n, float d, int32_t* rc_out) {
    int rc = check_args(p, n, d, 1, 1);
    if (rc) { *rc_out = rc; return NULL; }
    oracle_index_t* ix = calloc(1, sizeof(oracle_index_t));
    if (!ix) { *rc_out = ORACLE_ERR_NOMEM; return NULL; }
    rc = grid_build(&ix->g, p, n, d);
    if (rc) { free(ix); *rc_out = rc; return NULL; }
    ix->queue = malloc(sizeof(int32_t) * (n > 0 ? n : 1));
    if (!ix->queue) { grid_free(&ix->g); free(ix); *rc_out = ORACLE_ERR_NOMEM; return NULL; }
    *rc_out = ORACLE_OK;
    return ix;
}

void oracle_index_free(void* h) {
    oracle_index_t* ix = h;
    if (!ix) return;
    grid_free(&ix->g);
    free(ix->queue);
    free(ix);
}

int oracle_component(void* h, int64_t seed, int64_t* min_out, int64_t* size_out) {
    oracle_index_t* ix = h;
    grid_t* g = &ix->g;
    if (seed < 0 || seed >= g->n) return ORACLE_ERR_INVALID_ARGUMENT;
    int64_t tail = 0;
    grid_remove(g, (int32_t)seed);
    ix->queue[tail++] = (int32_t)seed;
    flood(g, ix->queue, 0, &tail);
    int64_t mn = seed;
    for (int64_t k = 0; k < tail; ++k)
        if (ix->queue[k] < mn) mn = ix->queue[k];
    /* restore: every removal decremented calive of the member's cell; a member's slot is
     * inside its cell's range, so re-opening the ranges restores the bucket *sets*. */
    for (int64_t k = 0; k < tail; ++k) g->calive[g->pcell[ix->queue[k]]] += 1;
    *min_out = mn;
    *size_out = tail;
    return ORACLE_OK;
}
