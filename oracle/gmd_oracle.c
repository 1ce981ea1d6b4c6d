/* ORACLE TEST INFRASTRUCTURE -- not part of the product (see gmd_oracle.h).
 *
 * Plain-C fp64 restatement of the reference graphmd hot path.  Every
 * floating-point decision is written with the same operand order as the
 * reference so that graphs, partitions and line graphs are bit-identical
 * (compiled with -ffp-contract=off; the x86-64 baseline has no FMA anyway).
 * Each function cites the reference file:line it restates.
 */
#define _GNU_SOURCE
#include "gmd_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define PI_D 3.14159265358979323846

static __thread char g_err[512];

static int fail(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return 1;
}

const char* orc_last_error(void) { return g_err; }

static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s);
    if (!p) {
        fprintf(stderr, "oracle: out of memory\n");
        abort();
    }
    return p;
}

/* growable int64 vector */
typedef struct {
    int64_t* v;
    int64_t n, cap;
} vec64;

static void v_push(vec64* a, int64_t x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 8;
        a->v = (int64_t*)realloc(a->v, (size_t)a->cap * sizeof(int64_t));
    }
    a->v[a->n++] = x;
}
static void v_free(vec64* a) {
    free(a->v);
    a->v = NULL;
    a->n = a->cap = 0;
}

/* ------------------------------------------------------------------------ */
/* small fp64 vector algebra, operand order as system.hpp:26-40             */
/* ------------------------------------------------------------------------ */
typedef struct {
    double c[3];
} v3;

static v3 mk(double x, double y, double z) {
    v3 r = {{x, y, z}};
    return r;
}
static v3 vadd(v3 a, v3 b) { return mk(a.c[0] + b.c[0], a.c[1] + b.c[1], a.c[2] + b.c[2]); }
static v3 vsub(v3 a, v3 b) { return mk(a.c[0] - b.c[0], a.c[1] - b.c[1], a.c[2] - b.c[2]); }
static v3 vscale(v3 a, double s) { return mk(a.c[0] * s, a.c[1] * s, a.c[2] * s); }
static v3 vdiv(v3 a, double s) { return mk(a.c[0] / s, a.c[1] / s, a.c[2] / s); }
static double vdot(v3 a, v3 b) { return a.c[0] * b.c[0] + a.c[1] * b.c[1] + a.c[2] * b.c[2]; }
static v3 vcross(v3 a, v3 b) {
    return mk(a.c[1] * b.c[2] - a.c[2] * b.c[1], a.c[2] * b.c[0] - a.c[0] * b.c[2],
              a.c[0] * b.c[1] - a.c[1] * b.c[0]);
}
static double vnorm(v3 a) { return sqrt(vdot(a, a)); }

typedef struct {
    v3 r[3];
} m3;

static double mdet(const m3* m) { return vdot(m->r[0], vcross(m->r[1], m->r[2])); }

/* v * M with M's rows: rows[0]*v.x + rows[1]*v.y + rows[2]*v.z (system.hpp:59-61) */
static v3 rowvec(const m3* m, v3 v) {
    return vadd(vadd(vscale(m->r[0], v.c[0]), vscale(m->r[1], v.c[1])),
                vscale(m->r[2], v.c[2]));
}

/* Mat3::inverse (system.cpp:55-70) */
static int minverse(const m3* m, m3* inv) {
    double d = mdet(m);
    if (fabs(d) < 1e-10) return fail("lattice is singular (|det| < 1e-10)");
    v3 bc = vdiv(vcross(m->r[1], m->r[2]), d);
    v3 ca = vdiv(vcross(m->r[2], m->r[0]), d);
    v3 ab = vdiv(vcross(m->r[0], m->r[1]), d);
    for (int k = 0; k < 3; ++k) inv->r[k] = mk(bc.c[k], ca.c[k], ab.c[k]);
    return 0;
}

/* AtomicSystem::perpendicular_width (system.cpp:87-93) */
static double perp_width(const m3* L, int axis) {
    double area = vnorm(vcross(L->r[(axis + 1) % 3], L->r[(axis + 2) % 3]));
    return fabs(mdet(L)) / area;
}

/* ------------------------------------------------------------------------ */
/* RNG: mt19937_64 + inline Box-Muller (system.hpp:121-149)                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t mt[312];
    int idx;
    int have_spare;
    double spare;
} rng_t;

static void rng_seed(rng_t* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
    g->have_spare = 0;
    g->spare = 0.0;
}

static uint64_t rng_next(rng_t* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

static double rng_uniform(rng_t* g) { return (double)(rng_next(g) >> 11) * 0x1.0p-53; }

static double rng_normal(rng_t* g) {
    if (g->have_spare) {
        g->have_spare = 0;
        return g->spare;
    }
    double u1 = 0.0;
    while (u1 == 0.0) u1 = rng_uniform(g);
    double u2 = rng_uniform(g);
    double rad = sqrt(-2.0 * log(u1));
    double ang = 2.0 * PI_D * u2;
    g->spare = rad * sin(ang);
    g->have_spare = 1;
    return rad * cos(ang);
}

void orc_rng_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out) {
    rng_t g;
    rng_seed(&g, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * rng_uniform(&g);
}

void orc_rng_normal(uint64_t seed, int64_t count, double* out) {
    rng_t g;
    rng_seed(&g, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = rng_normal(&g);
}

/* make_supercell (system.cpp:188-214) then random_perturb (:231-240) */
void orc_supercell(int64_t n, const double* pos, const int32_t* z, const double* lat,
                   int rx, int ry, int rz, double amp, uint64_t seed, double* out_pos,
                   int32_t* out_z, double* out_lat) {
    m3 L;
    for (int k = 0; k < 3; ++k) L.r[k] = mk(lat[3 * k], lat[3 * k + 1], lat[3 * k + 2]);
    int reps[3] = {rx, ry, rz};
    for (int k = 0; k < 3; ++k) {
        v3 row = vscale(L.r[k], (double)reps[k]);
        for (int c = 0; c < 3; ++c) out_lat[3 * k + c] = row.c[c];
    }
    int64_t o = 0;
    for (int a = 0; a < rx; ++a)
        for (int b = 0; b < ry; ++b)
            for (int c = 0; c < rz; ++c) {
                v3 sh = vadd(vadd(vscale(L.r[0], a), vscale(L.r[1], b)), vscale(L.r[2], c));
                for (int64_t i = 0; i < n; ++i, ++o) {
                    v3 p = vadd(mk(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), sh);
                    for (int k = 0; k < 3; ++k) out_pos[3 * o + k] = p.c[k];
                    out_z[o] = z[i];
                }
            }
    if (amp > 0.0) {
        rng_t g;
        rng_seed(&g, seed);
        for (int64_t i = 0; i < o; ++i)
            for (int k = 0; k < 3; ++k)
                out_pos[3 * i + k] += -amp + (amp - -amp) * rng_uniform(&g);
    }
}

/* ------------------------------------------------------------------------ */
/* params (potential.cpp:119-148)                                           */
/* ------------------------------------------------------------------------ */
int64_t orc_params_size(int F, int K, int L) {
    return 119LL * F + (int64_t)L * F * F + (int64_t)L * F + 2LL * F * K + 2LL * F * F + F;
}

void orc_params_init(uint64_t seed, int F, int K, int L, double r_atom, double r3,
                     double* blob) {
    (void)r_atom;
    (void)r3;
    rng_t g;
    rng_seed(&g, seed ^ 0x9e3779b97f4a7c15ULL);
    struct {
        int64_t n;
        double scale;
    } seg[8] = {
        {119LL * F, 0.5},
        {(int64_t)L * F * F, 1.0 / sqrt((double)F)},
        {(int64_t)L * F, 0.1},
        {(int64_t)F * K, 1.0 / sqrt((double)K)},
        {(int64_t)F * K, 0.5 / sqrt((double)K)},
        {(int64_t)F * F, 1.0 / sqrt((double)F)},
        {(int64_t)F * F, 0.5 / sqrt((double)F)},
        {(int64_t)F, 0.5},
    };
    double* q = blob;
    for (int s = 0; s < 8; ++s)
        for (int64_t i = 0; i < seg[s].n; ++i) *q++ = seg[s].scale * rng_normal(&g);
}

/* ------------------------------------------------------------------------ */
/* system: ensure_periodic (system.cpp:242-270)                             */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t n;
    v3* pos;
    int32_t* z;
    m3 L;
} sys_t;

static int sys_make(sys_t* s, int64_t n, const double* pos, const int32_t* z,
                    const double* lat, const uint8_t* pbc, double cutoff) {
    s->n = n;
    s->pos = (v3*)xcalloc((size_t)n, sizeof(v3));
    s->z = (int32_t*)xcalloc((size_t)n, sizeof(int32_t));
    for (int64_t i = 0; i < n; ++i) {
        s->pos[i] = mk(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
        s->z[i] = z ? z[i] : 1;
    }
    for (int k = 0; k < 3; ++k) s->L.r[k] = mk(lat[3 * k], lat[3 * k + 1], lat[3 * k + 2]);
    int all = 1;
    for (int k = 0; k < 3; ++k)
        if (pbc && !pbc[k]) all = 0;
    if (!all) {
        if (cutoff <= 0.0) return fail("cutoff must be positive");
        for (int k = 0; k < 3; ++k) {
            if (pbc[k]) continue;
            v3 dir = s->L.r[k];
            double len = vnorm(dir);
            if (len == 0.0)
                dir = mk(k == 0, k == 1, k == 2);
            else
                dir = vdiv(dir, len);
            double lo = 1.7976931348623157e308, hi = -1.7976931348623157e308;
            for (int64_t i = 0; i < n; ++i) {
                double t = vdot(s->pos[i], dir);
                lo = t < lo ? t : lo;
                hi = t > hi ? t : hi;
            }
            if (n == 0) lo = hi = 0.0;
            double extent = hi - lo + 2.0 * cutoff;
            s->L.r[k] = vscale(dir, extent);
            for (int64_t i = 0; i < n; ++i) s->pos[i] = vadd(s->pos[i], vscale(dir, cutoff - lo));
        }
    }
    if (fabs(mdet(&s->L)) < 1e-10) return fail("periodic system requires an invertible lattice");
    return 0;
}

static void sys_free(sys_t* s) {
    free(s->pos);
    free(s->z);
    s->pos = NULL;
    s->z = NULL;
}

/* ------------------------------------------------------------------------ */
/* neighbour list (neighborlist.cpp:33-239)                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t src;
    int32_t off[3];
    double d;
    v3 v;
} raw_edge;

typedef struct {
    raw_edge* e;
    int64_t n, cap;
} edge_list;

static void el_push(edge_list* l, raw_edge x) {
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 16;
        l->e = (raw_edge*)realloc(l->e, (size_t)l->cap * sizeof(raw_edge));
    }
    l->e[l->n++] = x;
}

static int raw_cmp(const void* pa, const void* pb) {
    const raw_edge* a = (const raw_edge*)pa;
    const raw_edge* b = (const raw_edge*)pb;
    if (a->src != b->src) return a->src < b->src ? -1 : 1;
    for (int k = 0; k < 3; ++k)
        if (a->off[k] != b->off[k]) return a->off[k] < b->off[k] ? -1 : 1;
    return 0;
}

typedef struct {
    int64_t n, ne;
    int64_t *src, *dst;
    int32_t* off;
    double *dist, *vec;
    double cutoff;
    int64_t* row; /* n+1 CSR by dst */
} graph_t;

static void graph_free(graph_t* g) {
    free(g->src);
    free(g->dst);
    free(g->off);
    free(g->dist);
    free(g->vec);
    free(g->row);
    memset(g, 0, sizeof *g);
}

/* per-dst sort then dst-major concat (neighborlist.cpp:60-85) */
static void assemble(graph_t* g, int64_t n, double cutoff, edge_list* per) {
    int64_t tot = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (per[i].n > 1) qsort(per[i].e, (size_t)per[i].n, sizeof(raw_edge), raw_cmp);
        tot += per[i].n;
    }
    g->n = n;
    g->ne = tot;
    g->cutoff = cutoff;
    g->src = (int64_t*)xcalloc((size_t)tot, 8);
    g->dst = (int64_t*)xcalloc((size_t)tot, 8);
    g->off = (int32_t*)xcalloc((size_t)tot * 3, 4);
    g->dist = (double*)xcalloc((size_t)tot, 8);
    g->vec = (double*)xcalloc((size_t)tot * 3, 8);
    g->row = (int64_t*)xcalloc((size_t)n + 1, 8);
    int64_t e = 0;
    for (int64_t i = 0; i < n; ++i) {
        g->row[i] = e;
        for (int64_t k = 0; k < per[i].n; ++k, ++e) {
            raw_edge* r = &per[i].e[k];
            g->src[e] = r->src;
            g->dst[e] = i;
            memcpy(&g->off[3 * e], r->off, 12);
            g->dist[e] = r->d;
            memcpy(&g->vec[3 * e], r->v.c, 24);
        }
        free(per[i].e);
    }
    g->row[n] = e;
    free(per);
}

/* wrap_for_search (neighborlist.cpp:33-58) */
static int wrap_atoms(const sys_t* s, int32_t* cell, v3* frac, v3* wrapped) {
    m3 inv;
    if (minverse(&s->L, &inv)) return 1;
    for (int64_t i = 0; i < s->n; ++i) {
        v3 f = rowvec(&inv, s->pos[i]);
        for (int k = 0; k < 3; ++k) {
            double fl = floor(f.c[k]);
            cell[3 * i + k] = (int32_t)fl;
            double w = f.c[k] - fl;
            if (w >= 1.0) {
                w = 0.0;
                cell[3 * i + k] += 1;
            }
            frac[i].c[k] = w;
        }
    }
    for (int64_t i = 0; i < s->n; ++i) wrapped[i] = rowvec(&s->L, frac[i]);
    return 0;
}

/* exact inclusion test through raw positions (neighborlist.cpp:178-191) */
static void try_edge(const sys_t* s, int64_t i, int64_t j, const int32_t off[3],
                     double cutoff2, edge_list* out) {
    v3 raw = vadd(vadd(vscale(s->L.r[0], (double)off[0]), vscale(s->L.r[1], (double)off[1])),
                  vscale(s->L.r[2], (double)off[2]));
    v3 vr = vadd(vsub(s->pos[j], s->pos[i]), raw);
    double d2 = vdot(vr, vr);
    if (d2 > cutoff2 || d2 == 0.0) return;
    raw_edge r;
    r.src = j;
    memcpy(r.off, off, 12);
    r.d = sqrt(d2);
    r.v = vr;
    el_push(out, r);
}

static int build_nl(const sys_t* s, double cutoff, int brute, graph_t* g) {
    if (cutoff <= 0.0) return fail("cutoff must be positive");
    if (s->n == 0) return fail("cannot build neighbor list for empty system");
    if (brute && s->n > 5000) return fail("brute force guard: N > 5000");
    const int64_t n = s->n;
    int32_t* cell = (int32_t*)xcalloc((size_t)n * 3, 4);
    v3* frac = (v3*)xcalloc((size_t)n, sizeof(v3));
    v3* wr = (v3*)xcalloc((size_t)n, sizeof(v3));
    if (wrap_atoms(s, cell, frac, wr)) {
        free(cell);
        free(frac);
        free(wr);
        return 1;
    }
    const double cutoff2 = cutoff * cutoff;
    edge_list* per = (edge_list*)xcalloc((size_t)n, sizeof(edge_list));

    if (brute) { /* neighborlist.cpp:199-239 */
        int span[3];
        for (int k = 0; k < 3; ++k) span[k] = (int)ceil(cutoff / perp_width(&s->L, k)) + 1;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j)
                for (int a = -span[0]; a <= span[0]; ++a)
                    for (int b = -span[1]; b <= span[1]; ++b)
                        for (int c = -span[2]; c <= span[2]; ++c) {
                            int32_t off[3] = {a - cell[3 * j] + cell[3 * i],
                                              b - cell[3 * j + 1] + cell[3 * i + 1],
                                              c - cell[3 * j + 2] + cell[3 * i + 2]};
                            try_edge(s, i, j, off, cutoff2, &per[i]);
                        }
    } else { /* cell list, neighborlist.cpp:119-194 */
        int bins[3], sten[3];
        for (int k = 0; k < 3; ++k) {
            double w = perp_width(&s->L, k);
            int b = (int)floor(w / cutoff);
            bins[k] = b > 1 ? b : 1;
            double bw = w / bins[k];
            sten[k] = (int)floor(cutoff / bw) + 1;
        }
        int64_t nb = (int64_t)bins[0] * bins[1] * bins[2];
        int64_t* bin_of = (int64_t*)xcalloc((size_t)n, 8);
        int64_t* start = (int64_t*)xcalloc((size_t)nb + 1, 8);
        int64_t* members = (int64_t*)xcalloc((size_t)n, 8);
        int32_t* bi3 = (int32_t*)xcalloc((size_t)n * 3, 4);
        for (int64_t i = 0; i < n; ++i) {
            for (int k = 0; k < 3; ++k) {
                int b = (int)(frac[i].c[k] * bins[k]);
                bi3[3 * i + k] = b < bins[k] - 1 ? b : bins[k] - 1;
            }
            bin_of[i] = ((int64_t)bi3[3 * i] * bins[1] + bi3[3 * i + 1]) * bins[2] + bi3[3 * i + 2];
            start[bin_of[i] + 1]++;
        }
        for (int64_t b = 0; b < nb; ++b) start[b + 1] += start[b];
        int64_t* fill = (int64_t*)xcalloc((size_t)nb, 8);
        for (int64_t i = 0; i < n; ++i) members[start[bin_of[i]] + fill[bin_of[i]]++] = i;
        free(fill);
        for (int64_t i = 0; i < n; ++i) {
            const v3 ri = wr[i];
            for (int dx = -sten[0]; dx <= sten[0]; ++dx)
                for (int dy = -sten[1]; dy <= sten[1]; ++dy)
                    for (int dz = -sten[2]; dz <= sten[2]; ++dz) {
                        int cc[3] = {bi3[3 * i] + dx, bi3[3 * i + 1] + dy, bi3[3 * i + 2] + dz};
                        int q[3], cw[3];
                        for (int k = 0; k < 3; ++k) {
                            q[k] = cc[k] >= 0 ? cc[k] / bins[k] : -((-cc[k] + bins[k] - 1) / bins[k]);
                            cw[k] = cc[k] - q[k] * bins[k];
                        }
                        v3 shift = vadd(vadd(vscale(s->L.r[0], (double)q[0]),
                                             vscale(s->L.r[1], (double)q[1])),
                                        vscale(s->L.r[2], (double)q[2]));
                        int64_t b = ((int64_t)cw[0] * bins[1] + cw[1]) * bins[2] + cw[2];
                        for (int64_t m = start[b]; m < start[b + 1]; ++m) {
                            int64_t j = members[m];
                            v3 v = vsub(vadd(wr[j], shift), ri);
                            if (vdot(v, v) > cutoff2 * 1.000001) continue;
                            int32_t off[3];
                            for (int k = 0; k < 3; ++k) off[k] = q[k] - cell[3 * j + k] + cell[3 * i + k];
                            try_edge(s, i, j, off, cutoff2, &per[i]);
                        }
                    }
        }
        free(bin_of);
        free(start);
        free(members);
        free(bi3);
    }
    free(cell);
    free(frac);
    free(wr);
    assemble(g, n, cutoff, per);
    return 0;
}

void* orc_neighbor_list(int64_t n, const double* pos, const int32_t* z, const double* lat,
                        const uint8_t* pbc, double rc, int brute) {
    if (rc <= 0.0) {
        fail("cutoff must be positive");
        return NULL;
    }
    sys_t s;
    if (sys_make(&s, n, pos, z, lat, pbc, rc)) {
        sys_free(&s);
        return NULL;
    }
    graph_t* g = (graph_t*)xcalloc(1, sizeof(graph_t));
    int rcode = build_nl(&s, rc, brute, g);
    sys_free(&s);
    if (rcode) {
        free(g);
        return NULL;
    }
    return g;
}

int64_t orc_graph_num_edges(void* g) { return ((graph_t*)g)->ne; }

static void graph_copy_out(const graph_t* g, int64_t* src, int64_t* dst, int32_t* off,
                           double* dist, double* vec) {
    if (src) memcpy(src, g->src, (size_t)g->ne * 8);
    if (dst) memcpy(dst, g->dst, (size_t)g->ne * 8);
    if (off) memcpy(off, g->off, (size_t)g->ne * 12);
    if (dist) memcpy(dist, g->dist, (size_t)g->ne * 8);
    if (vec) memcpy(vec, g->vec, (size_t)g->ne * 24);
}

void orc_graph_get(void* g, int64_t* src, int64_t* dst, int32_t* off, double* dist,
                   double* vec) {
    graph_copy_out((graph_t*)g, src, dst, off, dist, vec);
}

void orc_graph_destroy(void* g) {
    if (!g) return;
    graph_free((graph_t*)g);
    free(g);
}

/* ------------------------------------------------------------------------ */
/* partitions (partitioner.cpp:15-218)                                      */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t* nodes; /* node_array */
    int64_t size;
    int64_t* markers; /* 2 + 2p */
    int64_t* dups;    /* pairs */
    int64_t ndups;
    int64_t* g2l; /* dense map over the id space, -1 if absent (canonical) */
} layout_t;

typedef struct {
    layout_t lay;
    vec64 owned, lsrc, ldst, border;
} apart_t;

typedef struct {
    layout_t lay;
    vec64 line; /* pairs (local e, local e') */
} bpart_t;

typedef struct {
    sys_t s;
    graph_t g;
    int p, axis;
    double* bnd;
    int32_t* owner;
    apart_t* ap;
    int has_lg;
    int64_t nb;
    int64_t* edge_of_bond;
    int32_t* bond_owner;
    bpart_t* bp;
} dist_t;

static double wrapped_frac(double f) {
    double w = f - floor(f);
    if (w >= 1.0) w = 0.0;
    return w;
}

static int cmp_d(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* which_partition (partitioner.cpp:93-100): right-hand slab on ties */
static int which_part(const double* bnd, int p, double f) {
    if (f >= 1.0) return p - 1;
    int k = 1;
    while (k <= p - 1 && !(f < bnd[k])) ++k;
    return k - 1;
}

/* build_span_layout (partitioner.cpp:153-180) over an id space of size nid,
 * lists[b] for b in [pure, to_0..to_{p-1}, from_0..from_{p-1}] */
static void make_layout(layout_t* L, vec64* lists, int p, int64_t nid) {
    int64_t tot = 0;
    for (int b = 0; b < 1 + 2 * p; ++b) tot += lists[b].n;
    L->size = tot;
    L->nodes = (int64_t*)xcalloc((size_t)tot, 8);
    L->markers = (int64_t*)xcalloc((size_t)(2 + 2 * p), 8);
    L->g2l = (int64_t*)xcalloc((size_t)nid, 8);
    for (int64_t v = 0; v < nid; ++v) L->g2l[v] = -1;
    vec64 dups = {0};
    int64_t row = 0;
    for (int b = 0; b < 1 + 2 * p; ++b) {
        for (int64_t k = 0; k < lists[b].n; ++k, ++row) {
            int64_t gid = lists[b].v[k];
            L->nodes[row] = gid;
            if (L->g2l[gid] < 0)
                L->g2l[gid] = row;
            else {
                v_push(&dups, L->g2l[gid]);
                v_push(&dups, row);
            }
        }
        L->markers[b + 1] = row;
    }
    L->dups = dups.v;
    L->ndups = dups.n / 2;
}

static void free_layout(layout_t* L) {
    free(L->nodes);
    free(L->markers);
    free(L->dups);
    free(L->g2l);
}

/* PURE/TO/FROM lists from requirement masks (partitioner.cpp:136-150) for
 * partition i, in ascending id order */
static void bucket_lists(vec64* lists, int i, int p, int64_t nid, const int32_t* own,
                         const uint64_t* req) {
    for (int64_t v = 0; v < nid; ++v) {
        if (own[v] == i) {
            if (req[v] == 0)
                v_push(&lists[0], v);
            else
                for (int j = 0; j < p; ++j)
                    if (req[v] >> j & 1ULL) v_push(&lists[1 + j], v);
        } else if (req[v] >> i & 1ULL) {
            v_push(&lists[1 + p + own[v]], v);
        }
    }
}

static int is_rev(const graph_t* g, int64_t e, int64_t f) {
    return g->dst[f] == g->src[e] && g->src[f] == g->dst[e] && g->off[3 * f] == -g->off[3 * e] &&
           g->off[3 * f + 1] == -g->off[3 * e + 1] && g->off[3 * f + 2] == -g->off[3 * e + 2];
}

static int cmp_pair_key(const void* a, const void* b) {
    const int64_t* x = (const int64_t*)a;
    const int64_t* y = (const int64_t*)b;
    for (int k = 0; k < 2; ++k)
        if (x[k] != y[k]) return x[k] < y[k] ? -1 : 1;
    return 0;
}

void orc_destroy(void* hv);

void* orc_create(int64_t n, const double* pos, const int32_t* z, const double* lat,
                 const uint8_t* pbc, double rc, double r3, double tau, int p,
                 int allow_narrow) {
    if (p < 1) {
        fail("partition count must be >= 1");
        return NULL;
    }
    dist_t* d = (dist_t*)xcalloc(1, sizeof(dist_t));
    d->p = p;
    /* create_distributed: ensure_periodic then build_neighbor_list (engine.cpp:50-53) */
    if (sys_make(&d->s, n, pos, z, lat, pbc, rc)) goto bad;
    if (build_nl(&d->s, rc, 0, &d->g)) goto bad;

    /* choose_partition_rule (partitioner.cpp:46-91) */
    if (p > 64) {
        fail("partition count limited to 64");
        goto bad;
    }
    if ((int64_t)p > n) {
        fail("more partitions than atoms");
        goto bad;
    }
    {
        double best = -1.0;
        for (int k = 0; k < 3; ++k) {
            double len = vnorm(d->s.L.r[k]);
            if (len > best) {
                best = len;
                d->axis = k;
            }
        }
    }
    d->bnd = (double*)xcalloc((size_t)p + 1, 8);
    d->bnd[0] = 0.0;
    d->bnd[p] = 1.0;
    double* fr = (double*)xcalloc((size_t)n, 8);
    {
        m3 inv;
        if (minverse(&d->s.L, &inv)) {
            free(fr);
            goto bad;
        }
        for (int64_t i = 0; i < n; ++i) fr[i] = wrapped_frac(rowvec(&inv, d->s.pos[i]).c[d->axis]);
    }
    if (p > 1) {
        double* sorted = (double*)xcalloc((size_t)n, 8);
        memcpy(sorted, fr, (size_t)n * 8);
        qsort(sorted, (size_t)n, 8, cmp_d);
        for (int k = 1; k < p; ++k) {
            int64_t c = n * k / p;
            d->bnd[k] = (c >= 1 && c < n) ? 0.5 * (sorted[c - 1] + sorted[c]) : (double)k / p;
        }
        free(sorted);
        for (int k = 1; k <= p; ++k)
            if (d->bnd[k] <= d->bnd[k - 1]) {
                free(fr);
                fail("cannot place distinct partition boundaries; coordinates along the axis are degenerate");
                goto bad;
            }
    }
    /* check_slab_widths (partitioner.cpp:21-33) */
    if (p > 1 && !allow_narrow) {
        double perp = perp_width(&d->s.L, d->axis);
        for (int i = 0; i < p; ++i) {
            double w = (d->bnd[i + 1] - d->bnd[i]) * perp;
            if (w < rc) {
                free(fr);
                fail("partition-width error: slab %d is %f A wide, below the cutoff %f A", i, w, rc);
                goto bad;
            }
        }
    }
    d->owner = (int32_t*)xcalloc((size_t)n, 4);
    for (int64_t i = 0; i < n; ++i) d->owner[i] = which_part(d->bnd, p, fr[i]);
    free(fr);

    /* requirement masks (partitioner.cpp:124-134), layouts, edge ownership */
    {
        const graph_t* g = &d->g;
        uint64_t* req = (uint64_t*)xcalloc((size_t)n, 8);
        for (int64_t e = 0; e < g->ne; ++e) {
            int ps = d->owner[g->src[e]], pd = d->owner[g->dst[e]];
            if (ps != pd) req[g->src[e]] |= 1ULL << pd;
        }
        d->ap = (apart_t*)xcalloc((size_t)p, sizeof(apart_t));
        for (int i = 0; i < p; ++i) {
            vec64* lists = (vec64*)xcalloc((size_t)(1 + 2 * p), sizeof(vec64));
            bucket_lists(lists, i, p, n, d->owner, req);
            make_layout(&d->ap[i].lay, lists, p, n);
            for (int b = 0; b < 1 + 2 * p; ++b) v_free(&lists[b]);
            free(lists);
        }
        free(req);
        for (int64_t e = 0; e < g->ne; ++e) {
            int pi = d->owner[g->dst[e]];
            apart_t* a = &d->ap[pi];
            int64_t ls = a->lay.g2l[g->src[e]], ld = a->lay.g2l[g->dst[e]];
            if (ls < 0 || ld < 0) {
                fail("internal: edge endpoint missing from partition layout");
                goto bad;
            }
            if (d->owner[g->src[e]] != pi) v_push(&a->border, a->owned.n);
            v_push(&a->owned, e);
            v_push(&a->lsrc, ls);
            v_push(&a->ldst, ld);
        }
    }

    /* three-body line graph (linegraph.cpp:10-171), restated from its
     * definition: bond = edge with !(d > r + tau); bond owner = owner(dst);
     * line edge (e, e') iff dst(e) = src(e') and e' is not the reverse of e,
     * drawn by owner(e') and ordered by (e', e). */
    if (r3 > 0.0) {
        const graph_t* g = &d->g;
        if (r3 > g->cutoff) {
            fail("three-body range cannot exceed the atom graph cutoff");
            goto bad;
        }
        if (tau < 0.0) {
            fail("tolerance tau must be >= 0");
            goto bad;
        }
        d->has_lg = 1;
        double bound = r3 + tau;
        int64_t* bond_of_edge = (int64_t*)xcalloc((size_t)g->ne, 8);
        vec64 eob = {0};
        for (int64_t e = 0; e < g->ne; ++e) {
            bond_of_edge[e] = -1;
            if (g->dist[e] > bound) continue;
            bond_of_edge[e] = eob.n;
            v_push(&eob, e);
        }
        d->nb = eob.n;
        d->edge_of_bond = eob.v;
        d->bond_owner = (int32_t*)xcalloc((size_t)d->nb, 4);
        for (int64_t b = 0; b < d->nb; ++b) d->bond_owner[b] = d->owner[g->dst[d->edge_of_bond[b]]];
        /* bonds into each atom, ascending bond id (BondSet::by_dst) */
        int64_t* bstart = (int64_t*)xcalloc((size_t)n + 1, 8);
        for (int64_t b = 0; b < d->nb; ++b) bstart[g->dst[d->edge_of_bond[b]] + 1]++;
        for (int64_t v = 0; v < n; ++v) bstart[v + 1] += bstart[v];
        int64_t* bin = (int64_t*)xcalloc((size_t)d->nb, 8);
        {
            int64_t* fillc = (int64_t*)xcalloc((size_t)n, 8);
            for (int64_t b = 0; b < d->nb; ++b) {
                int64_t v = g->dst[d->edge_of_bond[b]];
                bin[bstart[v] + fillc[v]++] = b;
            }
            free(fillc);
        }
        /* bond requirement masks (linegraph.cpp:95-105) */
        uint64_t* breq = (uint64_t*)xcalloc((size_t)d->nb, 8);
        for (int64_t ep = 0; ep < d->nb; ++ep) {
            int64_t eep = d->edge_of_bond[ep];
            int own = d->bond_owner[ep];
            int64_t s = g->src[eep];
            for (int64_t k = bstart[s]; k < bstart[s + 1]; ++k) {
                int64_t e = bin[k];
                if (is_rev(g, d->edge_of_bond[e], eep)) continue;
                if (d->bond_owner[e] != own) breq[e] |= 1ULL << own;
            }
        }
        d->bp = (bpart_t*)xcalloc((size_t)p, sizeof(bpart_t));
        for (int i = 0; i < p; ++i) {
            vec64* lists = (vec64*)xcalloc((size_t)(1 + 2 * p), sizeof(vec64));
            bucket_lists(lists, i, p, d->nb, d->bond_owner, breq);
            make_layout(&d->bp[i].lay, lists, p, d->nb);
            for (int b = 0; b < 1 + 2 * p; ++b) v_free(&lists[b]);
            free(lists);
        }
        free(breq);
        /* line edges in (e', e) order: e' ascending, then bonds into src(e')
         * ascending */
        for (int64_t ep = 0; ep < d->nb; ++ep) {
            int own = d->bond_owner[ep];
            bpart_t* bp = &d->bp[own];
            int64_t eep = d->edge_of_bond[ep];
            int64_t s = g->src[eep];
            for (int64_t k = bstart[s]; k < bstart[s + 1]; ++k) {
                int64_t e = bin[k];
                if (is_rev(g, d->edge_of_bond[e], eep)) continue;
                int64_t le = bp->lay.g2l[e], lep = bp->lay.g2l[ep];
                if (le < 0 || lep < 0) {
                    free(bstart);
                    free(bin);
                    free(bond_of_edge);
                    fail("dangling bond reference in line graph");
                    goto bad;
                }
                v_push(&bp->line, le);
                v_push(&bp->line, lep);
            }
        }
        free(bstart);
        free(bin);
        free(bond_of_edge);
    }
    return d;
bad:
    orc_destroy(d);
    return NULL;
}

void orc_destroy(void* hv) {
    dist_t* d = (dist_t*)hv;
    if (!d) return;
    if (d->ap)
        for (int i = 0; i < d->p; ++i) {
            free_layout(&d->ap[i].lay);
            v_free(&d->ap[i].owned);
            v_free(&d->ap[i].lsrc);
            v_free(&d->ap[i].ldst);
            v_free(&d->ap[i].border);
        }
    if (d->bp)
        for (int i = 0; i < d->p; ++i) {
            free_layout(&d->bp[i].lay);
            v_free(&d->bp[i].line);
        }
    free(d->ap);
    free(d->bp);
    free(d->bnd);
    free(d->owner);
    free(d->edge_of_bond);
    free(d->bond_owner);
    graph_free(&d->g);
    sys_free(&d->s);
    free(d);
}

int64_t orc_num_nodes(void* h) { return ((dist_t*)h)->s.n; }
int64_t orc_num_edges(void* h) { return ((dist_t*)h)->g.ne; }
void orc_graph(void* h, int64_t* src, int64_t* dst, int32_t* off, double* dist, double* vec) {
    graph_copy_out(&((dist_t*)h)->g, src, dst, off, dist, vec);
}
void orc_system(void* h, double* pos, double* lat) {
    dist_t* d = (dist_t*)h;
    for (int64_t i = 0; i < d->s.n; ++i) memcpy(&pos[3 * i], d->s.pos[i].c, 24);
    for (int k = 0; k < 3; ++k) memcpy(&lat[3 * k], d->s.L.r[k].c, 24);
}
int orc_rule(void* h, double* boundaries) {
    dist_t* d = (dist_t*)h;
    memcpy(boundaries, d->bnd, (size_t)(d->p + 1) * 8);
    return d->axis;
}
void orc_owner(void* h, int32_t* owner) {
    dist_t* d = (dist_t*)h;
    memcpy(owner, d->owner, (size_t)d->s.n * 4);
}
static layout_t* lay_of(void* h, int part, int bonds) {
    dist_t* d = (dist_t*)h;
    return bonds ? &d->bp[part].lay : &d->ap[part].lay;
}
int64_t orc_layout_size(void* h, int part, int bonds) { return lay_of(h, part, bonds)->size; }
void orc_layout(void* h, int part, int bonds, int64_t* node_array, int64_t* markers) {
    layout_t* L = lay_of(h, part, bonds);
    memcpy(node_array, L->nodes, (size_t)L->size * 8);
    memcpy(markers, L->markers, (size_t)(2 + 2 * ((dist_t*)h)->p) * 8);
}
int64_t orc_num_dups(void* h, int part, int bonds) { return lay_of(h, part, bonds)->ndups; }
void orc_dups(void* h, int part, int bonds, int64_t* pairs) {
    layout_t* L = lay_of(h, part, bonds);
    memcpy(pairs, L->dups, (size_t)L->ndups * 16);
}
int64_t orc_num_owned_edges(void* h, int part) { return ((dist_t*)h)->ap[part].owned.n; }
void orc_owned_edges(void* h, int part, int64_t* owned, int64_t* lsrc, int64_t* ldst) {
    apart_t* a = &((dist_t*)h)->ap[part];
    memcpy(owned, a->owned.v, (size_t)a->owned.n * 8);
    memcpy(lsrc, a->lsrc.v, (size_t)a->lsrc.n * 8);
    memcpy(ldst, a->ldst.v, (size_t)a->ldst.n * 8);
}
int64_t orc_num_border(void* h, int part) { return ((dist_t*)h)->ap[part].border.n; }
void orc_border(void* h, int part, int64_t* out) {
    apart_t* a = &((dist_t*)h)->ap[part];
    memcpy(out, a->border.v, (size_t)a->border.n * 8);
}
int orc_has_line_graph(void* h) { return ((dist_t*)h)->has_lg; }
int64_t orc_num_bonds(void* h) { return ((dist_t*)h)->nb; }
void orc_bonds(void* h, int64_t* edge_of_bond, int32_t* bond_owner) {
    dist_t* d = (dist_t*)h;
    memcpy(edge_of_bond, d->edge_of_bond, (size_t)d->nb * 8);
    memcpy(bond_owner, d->bond_owner, (size_t)d->nb * 4);
}
int64_t orc_num_line_edges(void* h, int part) { return ((dist_t*)h)->bp[part].line.n / 2; }
void orc_line_edges(void* h, int part, int64_t* pairs) {
    bpart_t* b = &((dist_t*)h)->bp[part];
    memcpy(pairs, b->line.v, (size_t)b->line.n * 8);
}

/* ------------------------------------------------------------------------ */
/* global line graphs (linegraph.cpp:183-219)                               */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t* v;
    int64_t n;
} pairs_t;

void* orc_line_graph(int64_t n, const double* pos, const int32_t* z, const double* lat,
                     const uint8_t* pbc, double rc, double r, double tau, int brute) {
    graph_t* g = (graph_t*)orc_neighbor_list(n, pos, z, lat, pbc, rc, 0);
    if (!g) return NULL;
    if (r > g->cutoff) {
        orc_graph_destroy(g);
        fail("three-body range cannot exceed the atom graph cutoff");
        return NULL;
    }
    if (tau < 0.0) {
        orc_graph_destroy(g);
        fail("tolerance tau must be >= 0");
        return NULL;
    }
    if (brute && g->n > 2000) {
        orc_graph_destroy(g);
        fail("brute force guard: N > 2000");
        return NULL;
    }
    double bound = r + tau;
    vec64 out = {0};
    if (brute) {
        /* every atom u: bonds into u x bonds out of u, by exhaustive scan */
        for (int64_t u = 0; u < g->n; ++u)
            for (int64_t e = 0; e < g->ne; ++e) {
                if (g->dst[e] != u || g->dist[e] > bound) continue;
                for (int64_t f = 0; f < g->ne; ++f) {
                    if (g->src[f] != u || g->dist[f] > bound || is_rev(g, e, f)) continue;
                    v_push(&out, e);
                    v_push(&out, f);
                }
            }
    } else {
        /* every bond e: bonds leaving dst(e), through a by-source index */
        int64_t* st = (int64_t*)xcalloc((size_t)g->n + 1, 8);
        for (int64_t f = 0; f < g->ne; ++f)
            if (!(g->dist[f] > bound)) st[g->src[f] + 1]++;
        for (int64_t v = 0; v < g->n; ++v) st[v + 1] += st[v];
        int64_t* by = (int64_t*)xcalloc((size_t)st[g->n], 8);
        int64_t* fc = (int64_t*)xcalloc((size_t)g->n, 8);
        for (int64_t f = 0; f < g->ne; ++f)
            if (!(g->dist[f] > bound)) by[st[g->src[f]] + fc[g->src[f]]++] = f;
        for (int64_t e = 0; e < g->ne; ++e) {
            if (g->dist[e] > bound) continue;
            int64_t u = g->dst[e];
            for (int64_t k = st[u]; k < st[u + 1]; ++k) {
                if (is_rev(g, e, by[k])) continue;
                v_push(&out, e);
                v_push(&out, by[k]);
            }
        }
        free(st);
        free(by);
        free(fc);
    }
    qsort(out.v, (size_t)(out.n / 2), 16, cmp_pair_key);
    orc_graph_destroy(g);
    pairs_t* ph = (pairs_t*)xcalloc(1, sizeof(pairs_t));
    ph->v = out.v;
    ph->n = out.n / 2;
    return ph;
}
int64_t orc_pairs_size(void* ph) { return ((pairs_t*)ph)->n; }
void orc_pairs_get(void* ph, int64_t* out) { memcpy(out, ((pairs_t*)ph)->v, (size_t)((pairs_t*)ph)->n * 16); }
void orc_pairs_destroy(void* ph) {
    if (!ph) return;
    free(((pairs_t*)ph)->v);
    free(ph);
}

/* ------------------------------------------------------------------------ */
/* model: forward_serial (potential.cpp:19-78, 269-530)                     */
/* ------------------------------------------------------------------------ */
static double fcut(double d, double rc) { return d >= rc ? 0.0 : 0.5 * (cos(PI_D * d / rc) + 1.0); }
static double fcut_d(double d, double rc) { return d >= rc ? 0.0 : -0.5 * PI_D / rc * sin(PI_D * d / rc); }

/* s = P u(d), ds = P u'(d) (potential.cpp:30-50) */
static void radial(const double* P, int F, int K, double rc, double d, double* s, double* ds) {
    double w = fcut(d, rc), dw = fcut_d(d, rc), sigma = rc / K;
    for (int f = 0; f < F; ++f) {
        s[f] = 0.0;
        if (ds) ds[f] = 0.0;
    }
    for (int k = 0; k < K; ++k) {
        double mu = K > 1 ? rc * k / (K - 1) : 0.0;
        double x = (d - mu) / sigma;
        double phi = exp(-x * x);
        double u = w * phi;
        double du = dw * phi + w * (-2.0 * x / sigma) * phi;
        for (int f = 0; f < F; ++f) {
            s[f] += P[f * K + k] * u;
            if (ds) ds[f] += P[f * K + k] * du;
        }
    }
}

static void mv(const double* W, int F, const double* x, double* y) {
    for (int i = 0; i < F; ++i) {
        double a = 0.0;
        for (int j = 0; j < F; ++j) a += W[i * F + j] * x[j];
        y[i] = a;
    }
}
static void mvt(const double* W, int F, const double* x, double* y) {
    for (int j = 0; j < F; ++j) y[j] = 0.0;
    for (int i = 0; i < F; ++i)
        for (int j = 0; j < F; ++j) y[j] += W[i * F + j] * x[i];
}

int orc_forward_serial(int64_t n, const double* pos, const int32_t* z, const double* lat,
                       const uint8_t* pbc, int F, int K, int L, double r_atom, double r3,
                       const double* blob, double* energy, double* per_atom, double* forces,
                       double* stress) {
    if (L < 1) return fail("layer count must be >= 1");
    if (r3 > 0.0 && r3 > r_atom) return fail("three-body cutoff cannot exceed the atom cutoff");
    const double* emb = blob;
    const double* lw = emb + 119 * F;
    const double* lb = lw + (size_t)L * F * F;
    const double* P = lb + (size_t)L * F;
    const double* P3 = P + F * K;
    const double* W3 = P3 + F * K;
    const double* W4 = W3 + F * F;
    const double* ro = W4 + F * F;
    const int tb = r3 > 0.0;

    sys_t s;
    if (sys_make(&s, n, pos, z, lat, pbc, r_atom)) {
        sys_free(&s);
        return 1;
    }
    graph_t g;
    if (build_nl(&s, r_atom, 0, &g)) {
        sys_free(&s);
        return 1;
    }
    const int64_t ne = g.ne;
    double* se = (double*)xcalloc((size_t)ne * F, 8);
    for (int64_t e = 0; e < ne; ++e) radial(P, F, K, r_atom, g.dist[e], se + e * F, NULL);

    /* bonds and serial line pairs grouped by e' (potential.cpp:86-105) */
    int64_t nb = 0, np = 0;
    int64_t *eob = NULL, *pe = NULL, *pep = NULL;
    if (tb) {
        vec64 vb = {0};
        for (int64_t e = 0; e < ne; ++e)
            if (!(g.dist[e] > r3)) v_push(&vb, e);
        eob = vb.v;
        nb = vb.n;
        int64_t* bs = (int64_t*)xcalloc((size_t)n + 1, 8);
        for (int64_t b = 0; b < nb; ++b) bs[g.dst[eob[b]] + 1]++;
        for (int64_t v = 0; v < n; ++v) bs[v + 1] += bs[v];
        int64_t* bl = (int64_t*)xcalloc((size_t)nb, 8);
        int64_t* fc = (int64_t*)xcalloc((size_t)n, 8);
        for (int64_t b = 0; b < nb; ++b) {
            int64_t v = g.dst[eob[b]];
            bl[bs[v] + fc[v]++] = b;
        }
        free(fc);
        vec64 a = {0}, c = {0};
        for (int64_t ep = 0; ep < nb; ++ep) {
            int64_t sv = g.src[eob[ep]];
            for (int64_t k = bs[sv]; k < bs[sv + 1]; ++k) {
                if (is_rev(&g, eob[bl[k]], eob[ep])) continue;
                v_push(&a, bl[k]);
                v_push(&c, ep);
            }
        }
        pe = a.v;
        pep = c.v;
        np = a.n;
        free(bs);
        free(bl);
    }

    const size_t NF = (size_t)n * F, BF = (size_t)nb * F;
    double* h = (double*)xcalloc(NF, 8);
    double* hin = (double*)xcalloc(NF * L, 8);
    double* zl = (double*)xcalloc(NF * L, 8);
    double* m = (double*)xcalloc(NF, 8);
    double* sc = (double*)xcalloc((size_t)F, 8);
    double* dsv = (double*)xcalloc((size_t)F, 8);
    double *t0 = NULL, *z3 = NULL, *tp = NULL, *z4 = NULL, *q = NULL;
    if (tb) {
        t0 = (double*)xcalloc(BF, 8);
        z3 = (double*)xcalloc(BF, 8);
        tp = (double*)xcalloc(BF, 8);
        z4 = (double*)xcalloc(NF, 8);
        q = (double*)xcalloc(NF, 8);
    }
    for (int64_t i = 0; i < n; ++i) memcpy(h + i * F, emb + (size_t)s.z[i] * F, (size_t)F * 8);

    int rcode = 0;
    for (int l = 0; l < L; ++l) {
        if (tb && l == L - 1) { /* three-body stage (potential.cpp:317-362) */
            for (int64_t b = 0; b < nb; ++b) radial(P3, F, K, r3, g.dist[eob[b]], t0 + b * F, NULL);
            double* m3 = (double*)xcalloc(BF, 8);
            for (int64_t k = 0; k < np; ++k) {
                int64_t ee = eob[pe[k]], eep = eob[pep[k]];
                v3 va = mk(g.vec[3 * ee], g.vec[3 * ee + 1], g.vec[3 * ee + 2]);
                v3 vb = mk(g.vec[3 * eep], g.vec[3 * eep + 1], g.vec[3 * eep + 2]);
                double c = -vdot(va, vb) / (g.dist[ee] * g.dist[eep]);
                for (int f = 0; f < F; ++f) m3[pep[k] * F + f] += c * t0[pe[k] * F + f];
            }
            for (int64_t b = 0; b < nb; ++b) {
                mv(W3, F, m3 + b * F, sc);
                double fw = fcut(g.dist[eob[b]], r3);
                for (int f = 0; f < F; ++f) {
                    z3[b * F + f] = sc[f];
                    tp[b * F + f] = t0[b * F + f] + fw * tanh(sc[f]);
                }
            }
            free(m3);
            for (int64_t b = 0; b < nb; ++b) {
                int64_t u = g.dst[eob[b]];
                for (int f = 0; f < F; ++f) q[u * F + f] += tp[b * F + f];
            }
            for (int64_t i = 0; i < n; ++i) {
                mv(W4, F, q + i * F, sc);
                for (int f = 0; f < F; ++f) {
                    z4[i * F + f] = sc[f];
                    h[i * F + f] += tanh(sc[f]);
                }
            }
        }
        /* conv (potential.cpp:364-384) */
        double* hl = hin + (size_t)l * NF;
        memcpy(hl, h, NF * 8);
        memset(m, 0, NF * 8);
        for (int64_t e = 0; e < ne; ++e) {
            const double* hs = hl + g.src[e] * F;
            double* mi = m + g.dst[e] * F;
            for (int f = 0; f < F; ++f) mi[f] += hs[f] * se[e * F + f];
        }
        const double* W = lw + (size_t)l * F * F;
        const double* bias = lb + (size_t)l * F;
        double* zz = zl + (size_t)l * NF;
        for (int64_t i = 0; i < n; ++i) {
            mv(W, F, m + i * F, sc);
            for (int f = 0; f < F; ++f) {
                zz[i * F + f] = sc[f] + bias[f];
                h[i * F + f] += tanh(zz[i * F + f]);
            }
        }
        for (size_t k = 0; k < NF; ++k)
            if (!isfinite(h[k])) {
                rcode = fail("non-finite feature at layer %d, atom %lld", l, (long long)(k / F));
                goto done;
            }
    }

    {
        double E = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double ei = 0.0;
            for (int f = 0; f < F; ++f) ei += ro[f] * h[i * F + f];
            if (per_atom) per_atom[i] = ei;
            E += ei;
        }
        if (energy) *energy = E;
    }

    /* backward (potential.cpp:400-529) */
    {
        double* hb = (double*)xcalloc(NF, 8);
        double* mb = (double*)xcalloc(NF, 8);
        double* gp = (double*)xcalloc((size_t)n * 3, 8);
        double vir[9] = {0};
        for (int64_t i = 0; i < n; ++i) memcpy(hb + i * F, ro, (size_t)F * 8);
#define ADD_GRAD(edge, gx, gy, gz)                                              \
    do {                                                                        \
        int64_t _e = (edge);                                                    \
        double _g[3] = {gx, gy, gz};                                            \
        for (int _a = 0; _a < 3; ++_a) {                                        \
            gp[g.src[_e] * 3 + _a] += _g[_a];                                   \
            gp[g.dst[_e] * 3 + _a] -= _g[_a];                                   \
        }                                                                       \
        for (int _a = 0; _a < 3; ++_a)                                          \
            for (int _b = 0; _b < 3; ++_b) vir[3 * _a + _b] += _g[_a] * g.vec[3 * _e + _b]; \
    } while (0)
        for (int l = L - 1; l >= 0; --l) {
            const double* W = lw + (size_t)l * F * F;
            const double* zz = zl + (size_t)l * NF;
            const double* hl = hin + (size_t)l * NF;
            for (int64_t i = 0; i < n; ++i) {
                for (int f = 0; f < F; ++f) {
                    double th = tanh(zz[i * F + f]);
                    sc[f] = hb[i * F + f] * (1.0 - th * th);
                }
                mvt(W, F, sc, mb + i * F);
            }
            for (int64_t e = 0; e < ne; ++e) {
                const double* mbv = mb + g.dst[e] * F;
                const double* hs = hl + g.src[e] * F;
                double* hbs = hb + g.src[e] * F;
                radial(P, F, K, r_atom, g.dist[e], sc, dsv);
                double db = 0.0;
                for (int f = 0; f < F; ++f) {
                    hbs[f] += mbv[f] * se[e * F + f];
                    db += mbv[f] * hs[f] * dsv[f];
                }
                double r = db / g.dist[e];
                ADD_GRAD(e, g.vec[3 * e] * r, g.vec[3 * e + 1] * r, g.vec[3 * e + 2] * r);
            }
            if (tb && l == L - 1) { /* potential.cpp:447-519 */
                double* tbar = (double*)xcalloc(BF, 8);
                double* vbar = (double*)xcalloc((size_t)nb * 3, 8);
                double* m3b = (double*)xcalloc(BF, 8);
                double* tpb = (double*)xcalloc(BF, 8);
                for (int64_t i = 0; i < n; ++i) {
                    for (int f = 0; f < F; ++f) {
                        double th = tanh(z4[i * F + f]);
                        sc[f] = hb[i * F + f] * (1.0 - th * th);
                    }
                    mvt(W4, F, sc, mb + i * F);
                }
                for (int64_t b = 0; b < nb; ++b) memcpy(tpb + b * F, mb + g.dst[eob[b]] * F, (size_t)F * 8);
                for (int64_t b = 0; b < nb; ++b) {
                    int64_t ed = eob[b];
                    double d = g.dist[ed], fw = fcut(d, r3), dfw = fcut_d(d, r3), db = 0.0;
                    for (int f = 0; f < F; ++f) {
                        double th = tanh(z3[b * F + f]);
                        tbar[b * F + f] += tpb[b * F + f];
                        db += tpb[b * F + f] * th * dfw;
                        sc[f] = tpb[b * F + f] * fw * (1.0 - th * th);
                    }
                    mvt(W3, F, sc, m3b + b * F);
                    for (int a = 0; a < 3; ++a) vbar[3 * b + a] += g.vec[3 * ed + a] * (db / d);
                }
                for (int64_t k = 0; k < np; ++k) {
                    int64_t e = pe[k], ep = pep[k];
                    int64_t ee = eob[e], eep = eob[ep];
                    double de = g.dist[ee], dep = g.dist[eep];
                    v3 va = mk(g.vec[3 * ee], g.vec[3 * ee + 1], g.vec[3 * ee + 2]);
                    v3 vb = mk(g.vec[3 * eep], g.vec[3 * eep + 1], g.vec[3 * eep + 2]);
                    double c = -vdot(va, vb) / (de * dep);
                    double cb = 0.0;
                    for (int f = 0; f < F; ++f) {
                        tbar[e * F + f] += c * m3b[ep * F + f];
                        cb += m3b[ep * F + f] * t0[e * F + f];
                    }
                    /* cos_gradients (potential.cpp:72-78) */
                    v3 ah = vdiv(va, de), bh = vdiv(vb, dep);
                    v3 dca = vdiv(vscale(vadd(bh, vscale(ah, c)), -1.0), de);
                    v3 dcb = vdiv(vscale(vadd(ah, vscale(bh, c)), -1.0), dep);
                    for (int a = 0; a < 3; ++a) {
                        vbar[3 * e + a] += dca.c[a] * cb;
                        vbar[3 * ep + a] += dcb.c[a] * cb;
                    }
                }
                for (int64_t b = 0; b < nb; ++b) {
                    int64_t ed = eob[b];
                    radial(P3, F, K, r3, g.dist[ed], sc, dsv);
                    double db = 0.0;
                    for (int f = 0; f < F; ++f) db += tbar[b * F + f] * dsv[f];
                    for (int a = 0; a < 3; ++a) vbar[3 * b + a] += g.vec[3 * ed + a] * (db / g.dist[ed]);
                }
                for (int64_t b = 0; b < nb; ++b)
                    ADD_GRAD(eob[b], vbar[3 * b], vbar[3 * b + 1], vbar[3 * b + 2]);
                free(tbar);
                free(vbar);
                free(m3b);
                free(tpb);
            }
        }
#undef ADD_GRAD
        if (forces)
            for (int64_t i = 0; i < n * 3; ++i) forces[i] = -gp[i];
        double vol = fabs(mdet(&s.L));
        if (stress)
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) stress[3 * a + b] = 0.5 * (vir[3 * a + b] + vir[3 * b + a]) / vol;
        free(hb);
        free(mb);
        free(gp);
    }
done:
    free(se);
    free(h);
    free(hin);
    free(zl);
    free(m);
    free(sc);
    free(dsv);
    free(t0);
    free(z3);
    free(tp);
    free(z4);
    free(q);
    free(eob);
    free(pe);
    free(pep);
    graph_free(&g);
    sys_free(&s);
    return rcode;
}

/* ------------------------------------------------------------------------ */
/* MD (md.cpp:11-160): Maxwell-Boltzmann init, velocity Verlet with a        */
/* forward_serial evaluation per step (the reference uses                    */
/* forward_distributed, equal to serial within 1e-10).                        */
/* ------------------------------------------------------------------------ */
static const double ORC_MASSES[55] = {
    0.0,    1.008,  4.0026, 6.94,   9.0122, 10.81,  12.011, 14.007, 15.999, 18.998, 20.180,
    22.990, 24.305, 26.982, 28.085, 30.974, 32.06,  35.45,  39.948, 39.098, 40.078, 44.956,
    47.867, 50.942, 51.996, 54.938, 55.845, 58.933, 58.693, 63.546, 65.38,  69.723, 72.630,
    74.922, 78.971, 79.904, 83.798, 85.468, 87.62,  88.906, 91.224, 92.906, 95.95,  97.0,
    101.07, 102.91, 106.42, 107.87, 112.41, 114.82, 118.71, 121.76, 127.60, 126.90, 131.29};
#define ORC_KACCEL 9.648533212e-3
#define ORC_KKIN 103.642697
#define ORC_KB 8.617333262e-5

double orc_atomic_mass(int z) { /* system.cpp:289-293 */
    return z < 55 ? ORC_MASSES[z] : 2.5 * z;
}

static void md_record(int64_t n, const double* m, const double* v, const double* f, double pot,
                      double* rec) {
    double e = 0.0, fm = 0.0;
    for (int64_t i = 0; i < n; ++i) { /* MDState::kinetic_energy (md.cpp:11-16) */
        const v3 vi = mk(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
        e += 0.5 * m[i] * vdot(vi, vi);
        const double fn = vnorm(mk(f[3 * i], f[3 * i + 1], f[3 * i + 2]));
        fm = fn > fm ? fn : fm;
    }
    rec[0] = pot;
    rec[1] = e * ORC_KKIN;
    rec[2] = rec[0] + rec[1];
    rec[3] = fm;
}

int orc_md_run(int64_t n, const double* pos0, const int32_t* z, const double* lat,
               const uint8_t* pbc, int F, int K, int L, double r_atom, double r3,
               const double* blob, double dt, int64_t steps, double temperature, uint64_t seed,
               double* pos, double* vel, double* forces, double* rec) {
    if (dt < 0.0) return fail("time step must be >= 0");
    double* m = (double*)xcalloc((size_t)n, 8);
    for (int64_t i = 0; i < n; ++i) m[i] = orc_atomic_mass(z[i]);
    for (int64_t i = 0; i < 3 * n; ++i) {
        pos[i] = pos0[i];
        vel[i] = 0.0;
    }
    if (temperature > 0.0 && n > 0) { /* maxwell_boltzmann_velocities (md.cpp:20-52) */
        rng_t g;
        rng_seed(&g, seed ^ 0xd1b54a32d192ed03ull);
        for (int64_t i = 0; i < n; ++i) {
            const double sigma = sqrt(ORC_KB * temperature / (m[i] * ORC_KKIN));
            for (int k = 0; k < 3; ++k) vel[3 * i + k] = sigma * rng_normal(&g);
        }
        v3 ptot = mk(0, 0, 0);
        double mtot = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            ptot = vadd(ptot, vscale(mk(vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]), m[i]));
            mtot += m[i];
        }
        const v3 vcm = vdiv(ptot, mtot);
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) vel[3 * i + k] -= vcm.c[k];
    }
    m3 Lm, inv;
    for (int k = 0; k < 3; ++k) Lm.r[k] = mk(lat[3 * k], lat[3 * k + 1], lat[3 * k + 2]);
    if (minverse(&Lm, &inv)) {
        free(m);
        return 1;
    }
    double pot = 0.0;
    if (orc_forward_serial(n, pos, z, lat, pbc, F, K, L, r_atom, r3, blob, &pot, NULL, forces,
                           NULL)) {
        free(m);
        return 1;
    }
    md_record(n, m, vel, forces, pot, rec);
    for (int64_t step = 1; step <= steps; ++step) { /* velocity_verlet_step (md.cpp:85-110) */
        for (int64_t i = 0; i < n; ++i) {
            const double s = ORC_KACCEL / m[i];
            for (int k = 0; k < 3; ++k) {
                vel[3 * i + k] += (forces[3 * i + k] * s) * (0.5 * dt);
                pos[3 * i + k] += vel[3 * i + k] * dt;
            }
        }
        for (int64_t i = 0; i < n; ++i) { /* wrap_positions (system.cpp:216-229) */
            v3 fr = rowvec(&inv, mk(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]));
            for (int k = 0; k < 3; ++k) {
                fr.c[k] -= floor(fr.c[k]);
                if (fr.c[k] >= 1.0) fr.c[k] = 0.0;
            }
            const v3 r = rowvec(&Lm, fr);
            for (int k = 0; k < 3; ++k) pos[3 * i + k] = r.c[k];
        }
        if (orc_forward_serial(n, pos, z, lat, pbc, F, K, L, r_atom, r3, blob, &pot, NULL,
                               forces, NULL)) {
            free(m);
            return 1;
        }
        for (int64_t i = 0; i < 3 * n; ++i)
            if (!isfinite(forces[i])) {
                free(m);
                return fail("non-finite force on atom %lld at step %lld", (long long)(i / 3),
                            (long long)step);
            }
        for (int64_t i = 0; i < n; ++i) {
            const double s = ORC_KACCEL / m[i];
            for (int k = 0; k < 3; ++k) vel[3 * i + k] += (forces[3 * i + k] * s) * (0.5 * dt);
        }
        md_record(n, m, vel, forces, pot, rec + 4 * step);
    }
    free(m);
    return 0;
}
