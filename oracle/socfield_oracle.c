/*
 * socfield_oracle.c — CPU ORACLE (test infrastructure; see socfield_oracle.h).
 *
 * Plain-C restatement of the reference's per-tick pipeline.  "ref:" comments give the file
 * and line range under /root/reference/proj that each function follows.  The arithmetic is
 * kept in the reference's evaluation order (doubles, no contraction: build with
 * -ffp-contract=off) because decisions and images are compared bit for bit.
 *
 * Parity status: PINNED against the reference's golden digests and against oracle/_ref
 * (tests/test_oracle_golden.py, tests/test_oracle_vs_ref.py).
 */
#include "socfield_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#ifndef M_SQRT1_2
#define M_SQRT1_2 0.70710678118654752440
#endif

/* ---------------------------------------------------------------------------------------
 * tables
 * ------------------------------------------------------------------------------------- */

typedef struct plan_entry {
    int32_t dx, dy; /* centre position relative to the target su */
    double mag;
} plan_entry;

typedef struct write_plan {
    plan_entry* e[SO_SECTS];
    int n[SO_SECTS];
    int fanout;
} write_plan;

typedef struct gather_entry {
    int32_t dx, dy;
    double mag;
    uint8_t mask;
} gather_entry;

struct so_sim {
    so_config cfg;
    int32_t W, H;
    int64_t C, P;
    int64_t tick;
    /* SimState (ref: engine.hpp:91-98) */
    int32_t* occ;
    float* stat;
    float* dyn[SO_KINDS];
    int32_t *cx, *cy, *fw, *fh, *period, *phase, *goal;
    int32_t* orient[SO_KINDS]; /* FieldSpec::orientation per pedestrian per kind */
    /* Engine temporaries (ref: engine.hpp:222-227) */
    int32_t* enroll_ids;
    double* enroll_scores;
    int32_t* winners;
    int32_t *moved_from, *moved_to;
    uint8_t* from_mask[SO_KINDS];
    uint8_t* to_mask[SO_KINDS];
    int32_t* dec_dir;
    double* dec_score;
    /* plans: directional kinds hold 8, the recurrent kind 1 (ref: engine.cpp:179-191) */
    write_plan plans[SO_KINDS][SO_SECTS];
    int n_plans[SO_KINDS];
    gather_entry* gather[SO_KINDS][SO_SECTS];
    int n_gather[SO_KINDS][SO_SECTS];
    char err[256];
    int err_phase;
};

static int kind_of_dyn(int k) { /* ref: engine.cpp:22-29 to_field_kind */
    return k == 0 ? SO_DIR_ATTRACTIVE : k == 1 ? SO_DIR_REPULSIVE : SO_RECURRENT_REPULSIVE;
}
static int is_attractive(int kind) { return kind == SO_OMNI_ATTRACTIVE || kind == SO_DIR_ATTRACTIVE; }
static int is_directional(int kind) { return kind == SO_DIR_ATTRACTIVE || kind == SO_DIR_REPULSIVE; }

static int mod_floor(int a, int m) { /* ref: grid.cpp:8-11 */
    int r = a % m;
    return r < 0 ? r + m : r;
}

/* ref: grid.cpp:15-21 wrap.  Returns 0 when the pair falls off a closed grid. */
static int wrap_xy(const so_sim* s, int x, int y, int* ox, int* oy) {
    if (!s->cfg.closed) {
        *ox = mod_floor(x, s->W);
        *oy = mod_floor(y, s->H);
        return 1;
    }
    if (x < 0 || x >= s->W || y < 0 || y >= s->H) return 0;
    *ox = x;
    *oy = y;
    return 1;
}

static size_t flat(const so_sim* s, int x, int y) { return (size_t)y * (size_t)s->W + (size_t)x; }

/* ref: fields.cpp:54-60 sect_index */
int so_sect_index(double x, double y) {
    if (x == 0.0 && y == 0.0) return -1;
    const double deg = atan2(y, x) * 180.0 / M_PI;
    int sct = (int)floor((deg + 22.5) / 45.0);
    return ((sct % SO_SECTS) + SO_SECTS) % SO_SECTS;
}

/* ref: fields.cpp:62-65 sect_distance */
int so_sect_distance(int a, int b) {
    int d = ((a - b) % SO_SECTS + SO_SECTS) % SO_SECTS;
    return d < SO_SECTS - d ? d : SO_SECTS - d;
}

/* ref: fields.cpp:67-72 sect_step */
void so_sect_step(int sect, int* dx, int* dy) {
    static const int sx[8] = {1, 1, 0, -1, -1, -1, 0, 1};
    static const int sy[8] = {0, 1, 1, 1, 0, -1, -1, -1};
    *dx = sx[sect];
    *dy = sy[sect];
}

/* ref: fields.cpp:74-86 strength_at_offset */
void so_strength_at_offset(int kind, const so_field* f, int orientation, int dx, int dy, double* sx,
                           double* sy) {
    *sx = 0.0;
    *sy = 0.0;
    if (dx == 0 && dy == 0) return;
    const int hw = (f->width - 1) / 2, hh = (f->height - 1) / 2;
    if (abs(dx) > hw || abs(dy) > hh) return;
    if (is_directional(kind)) {
        const int target_sect = so_sect_index((double)dx, (double)dy);
        if (so_sect_distance(target_sect, orientation) > 1) return;
    }
    const double r = hypot((double)dx, (double)dy);
    const double magnitude = f->gain * exp(f->decay * r);
    if (magnitude == 0.0) return;
    const double sign = is_attractive(kind) ? -1.0 : 1.0;
    *sx = sign * magnitude * dx / r;
    *sy = sign * magnitude * dy / r;
}

static int plan_entry_less(const void* a, const void* b) { /* ref: fields.hpp:55-57 Offset < */
    const plan_entry* x = (const plan_entry*)a;
    const plan_entry* y = (const plan_entry*)b;
    if (x->dx != y->dx) return x->dx < y->dx ? -1 : 1;
    if (x->dy != y->dy) return x->dy < y->dy ? -1 : 1;
    return 0;
}

/* ref: fields.cpp:93-121 support + build_write_plan */
static void build_write_plan(write_plan* plan, int kind, const so_field* f, int orientation) {
    const int hw = (f->width - 1) / 2, hh = (f->height - 1) / 2;
    const int cap = f->width * f->height;
    for (int sct = 0; sct < SO_SECTS; ++sct) {
        plan->e[sct] = (plan_entry*)malloc(sizeof(plan_entry) * (size_t)cap);
        plan->n[sct] = 0;
    }
    for (int dy = -hh; dy <= hh; ++dy) {     /* support(): row-major over offsets */
        for (int dx = -hw; dx <= hw; ++dx) {
            double sx, sy;
            so_strength_at_offset(kind, f, orientation, dx, dy, &sx, &sy);
            if (!(sx != 0.0 || sy != 0.0)) continue;
            const int sct = so_sect_index(sx, sy);
            plan_entry* e = &plan->e[sct][plan->n[sct]++];
            e->dx = -dx; /* a field centred at target - o writes (target, sect) */
            e->dy = -dy;
            e->mag = hypot(sx, sy); /* Vec2::norm, fields.cpp:40 */
        }
    }
    plan->fanout = 0;
    for (int sct = 0; sct < SO_SECTS; ++sct) {
        qsort(plan->e[sct], (size_t)plan->n[sct], sizeof(plan_entry), plan_entry_less);
        if (plan->n[sct] > plan->fanout) plan->fanout = plan->n[sct];
    }
}

/* ref: engine.cpp:201-221 build_gather_tables.  std::map<Offset,...>::try_emplace keeps the
 * first magnitude seen for an offset and ORs the orientation bits; iteration is in Offset
 * order.  Restated as: concatenate, stable-merge equal offsets, sort. */
static void build_gather_tables(so_sim* s) {
    for (int k = 0; k < SO_KINDS; ++k) {
        const int directional = is_directional(kind_of_dyn(k));
        for (int sct = 0; sct < SO_SECTS; ++sct) {
            int total = 0;
            for (int o = 0; o < s->n_plans[k]; ++o) total += s->plans[k][o].n[sct];
            gather_entry* list = (gather_entry*)malloc(sizeof(gather_entry) * (size_t)(total > 0 ? total : 1));
            int n = 0;
            for (int o = 0; o < s->n_plans[k]; ++o) {
                const write_plan* p = &s->plans[k][o];
                for (int i = 0; i < p->n[sct]; ++i) {
                    const plan_entry* e = &p->e[sct][i];
                    const uint8_t bit = directional ? (uint8_t)(1u << o) : (uint8_t)0xFF;
                    int found = -1;
                    for (int j = 0; j < n; ++j) {
                        if (list[j].dx == e->dx && list[j].dy == e->dy) {
                            found = j;
                            break;
                        }
                    }
                    if (found >= 0) {
                        list[found].mask |= (uint8_t)(1u << o);
                    } else {
                        list[n].dx = e->dx;
                        list[n].dy = e->dy;
                        list[n].mag = e->mag;
                        list[n].mask = bit;
                        ++n;
                    }
                }
            }
            /* insertion sort by (dx, dy): offsets are unique after the merge */
            for (int i = 1; i < n; ++i) {
                gather_entry key = list[i];
                int j = i - 1;
                while (j >= 0 && (list[j].dx > key.dx || (list[j].dx == key.dx && list[j].dy > key.dy))) {
                    list[j + 1] = list[j];
                    --j;
                }
                list[j + 1] = key;
            }
            s->gather[k][sct] = list;
            s->n_gather[k][sct] = n;
        }
    }
}

/* ---------------------------------------------------------------------------------------
 * rasterization (ref: fields.cpp:152-168, engine.cpp:158-168)
 * ------------------------------------------------------------------------------------- */

static void rasterize_into(const so_sim* s, float* img, int kind, const so_field* f, int orientation,
                           int cx, int cy) {
    const int hw = (f->width - 1) / 2, hh = (f->height - 1) / 2;
    for (int dy = -hh; dy <= hh; ++dy) {
        for (int dx = -hw; dx <= hw; ++dx) {
            double sx, sy;
            so_strength_at_offset(kind, f, orientation, dx, dy, &sx, &sy);
            if (!(sx != 0.0 || sy != 0.0)) continue; /* not in support() */
            int tx, ty;
            if (!wrap_xy(s, cx + dx, cy + dy, &tx, &ty)) continue; /* clipped under Closed */
            img[flat(s, tx, ty) * SO_SECTS + (size_t)so_sect_index(sx, sy)] += (float)hypot(sx, sy);
        }
    }
}

void so_rebuild_images(const so_sim* s, float* out) {
    const size_t n = (size_t)s->C * SO_SECTS;
    memset(out, 0, sizeof(float) * n * SO_KINDS);
    for (int64_t i = 0; i < s->P; ++i) { /* id order, kinds inner: engine.cpp:162-166 */
        for (int k = 0; k < SO_KINDS; ++k) {
            rasterize_into(s, out + (size_t)k * n, kind_of_dyn(k), &s->cfg.templates[k], s->orient[k][i],
                           s->cx[i], s->cy[i]);
        }
    }
}

int so_set_static_fields(so_sim* s, int64_t n, const so_anchor* anchors) {
    memset(s->stat, 0, sizeof(float) * (size_t)s->C * SO_SECTS);
    for (int64_t i = 0; i < n; ++i) {
        so_field f = {anchors[i].width, anchors[i].height, anchors[i].gain, anchors[i].decay};
        rasterize_into(s, s->stat, anchors[i].kind, &f, 0, anchors[i].x, anchors[i].y);
    }
    return 0;
}

/* ---------------------------------------------------------------------------------------
 * construction
 * ------------------------------------------------------------------------------------- */

static int valid_chunk_width(int k) { return k == 2 || k == 4 || k == 8 || k == 16; } /* accumulator.cpp:5-7 */

static void* zalloc(size_t n, size_t sz) { return calloc(n > 0 ? n : 1, sz); }

static so_sim* alloc_sim(const so_config* cfg, int64_t n, char* err, size_t errlen) {
    if (!valid_chunk_width(cfg->chunk_k)) { /* ref: engine.cpp:173 */
        snprintf(err, errlen, "chunk_k: must be 2, 4, 8, or 16");
        return NULL;
    }
    if (cfg->density_radius < 0) {
        snprintf(err, errlen, "density_radius: must be >= 0");
        return NULL;
    }
    if (cfg->width < 1 || cfg->height < 1) {
        snprintf(err, errlen, "grid: must be at least 1x1");
        return NULL;
    }
    so_sim* s = (so_sim*)zalloc(1, sizeof(so_sim));
    s->cfg = *cfg;
    s->W = cfg->width;
    s->H = cfg->height;
    s->C = (int64_t)s->W * s->H;
    s->P = n;
    const size_t C = (size_t)s->C, P = (size_t)n;
    s->occ = (int32_t*)malloc(sizeof(int32_t) * C);
    for (size_t i = 0; i < C; ++i) s->occ[i] = SO_NO_PED;
    s->stat = (float*)zalloc(C * SO_SECTS, sizeof(float));
    for (int k = 0; k < SO_KINDS; ++k) {
        s->dyn[k] = (float*)zalloc(C * SO_SECTS, sizeof(float));
        s->orient[k] = (int32_t*)zalloc(P, sizeof(int32_t));
        s->from_mask[k] = (uint8_t*)zalloc(C, 1);
        s->to_mask[k] = (uint8_t*)zalloc(C, 1);
    }
    s->cx = (int32_t*)zalloc(P, sizeof(int32_t));
    s->cy = (int32_t*)zalloc(P, sizeof(int32_t));
    s->fw = (int32_t*)zalloc(P, sizeof(int32_t));
    s->fh = (int32_t*)zalloc(P, sizeof(int32_t));
    s->period = (int32_t*)zalloc(P, sizeof(int32_t));
    s->phase = (int32_t*)zalloc(P, sizeof(int32_t));
    s->goal = (int32_t*)zalloc(P, sizeof(int32_t));
    s->enroll_ids = (int32_t*)malloc(sizeof(int32_t) * C * SO_SECTS);
    s->enroll_scores = (double*)zalloc(C * SO_SECTS, sizeof(double));
    s->winners = (int32_t*)malloc(sizeof(int32_t) * C);
    s->moved_from = (int32_t*)malloc(sizeof(int32_t) * C);
    s->moved_to = (int32_t*)malloc(sizeof(int32_t) * C);
    for (size_t i = 0; i < C * SO_SECTS; ++i) s->enroll_ids[i] = SO_NO_PED;
    for (size_t i = 0; i < C; ++i) s->winners[i] = s->moved_from[i] = s->moved_to[i] = SO_NO_PED;
    s->dec_dir = (int32_t*)malloc(sizeof(int32_t) * (P > 0 ? P : 1));
    s->dec_score = (double*)zalloc(P, sizeof(double));
    for (size_t i = 0; i < P; ++i) s->dec_dir[i] = SO_STILL;
    /* ref: engine.cpp:179-192 */
    for (int k = 0; k < SO_KINDS; ++k) {
        const int kind = kind_of_dyn(k);
        s->n_plans[k] = is_directional(kind) ? SO_SECTS : 1;
        for (int o = 0; o < s->n_plans[k]; ++o) build_write_plan(&s->plans[k][o], kind, &cfg->templates[k], o);
    }
    build_gather_tables(s);
    return s;
}

/* ref: grid.cpp:36-50 footprint_cells + scenario.cpp:336-338 occupy */
static int stamp_footprint(so_sim* s, int cx, int cy, int fw, int fh, int32_t id) {
    int clipped = 0;
    for (int oy = -(fh - 1) / 2; oy <= (fh - 1) / 2; ++oy) {
        for (int ox = -(fw - 1) / 2; ox <= (fw - 1) / 2; ++ox) {
            int x, y;
            if (wrap_xy(s, cx + ox, cy + oy, &x, &y)) s->occ[flat(s, x, y)] = id;
            else clipped = 1;
        }
    }
    return clipped;
}

so_sim* so_create(const so_config* cfg, int64_t n, const int32_t* cx, const int32_t* cy,
                  const int32_t* fw, const int32_t* fh, const int32_t* period, const int32_t* phase,
                  const int32_t* goal, char* err, size_t errlen) {
    so_sim* s = alloc_sim(cfg, n, err, errlen);
    if (!s) return NULL;
    for (int64_t i = 0; i < n; ++i) { /* test fixture make_ped/make_state, test_engine.cpp:22-50 */
        s->cx[i] = cx[i];
        s->cy[i] = cy[i];
        s->fw[i] = fw[i];
        s->fh[i] = fh[i];
        s->period[i] = period[i];
        s->phase[i] = phase[i];
        s->goal[i] = goal[i];
        s->orient[0][i] = goal[i];
        s->orient[1][i] = goal[i];
        s->orient[2][i] = 0;
        stamp_footprint(s, cx[i], cy[i], fw[i], fh[i], (int32_t)i);
    }
    float* fresh = (float*)malloc(sizeof(float) * (size_t)s->C * SO_SECTS * SO_KINDS);
    so_rebuild_images(s, fresh);
    for (int k = 0; k < SO_KINDS; ++k)
        memcpy(s->dyn[k], fresh + (size_t)k * (size_t)s->C * SO_SECTS, sizeof(float) * (size_t)s->C * SO_SECTS);
    free(fresh);
    return s;
}

static void* dup_mem(const void* p, size_t bytes) {
    void* q = malloc(bytes > 0 ? bytes : 1);
    memcpy(q, p, bytes);
    return q;
}

so_sim* so_clone(const so_sim* a) {
    char err[64];
    so_sim* s = alloc_sim(&a->cfg, a->P, err, sizeof err);
    const size_t C = (size_t)a->C, P = (size_t)a->P;
    s->tick = a->tick;
    memcpy(s->occ, a->occ, sizeof(int32_t) * C);
    memcpy(s->stat, a->stat, sizeof(float) * C * SO_SECTS);
    for (int k = 0; k < SO_KINDS; ++k) {
        memcpy(s->dyn[k], a->dyn[k], sizeof(float) * C * SO_SECTS);
        memcpy(s->orient[k], a->orient[k], sizeof(int32_t) * P);
    }
    int32_t** dst[] = {&s->cx, &s->cy, &s->fw, &s->fh, &s->period, &s->phase, &s->goal};
    int32_t* const src[] = {a->cx, a->cy, a->fw, a->fh, a->period, a->phase, a->goal};
    for (int i = 0; i < 7; ++i) {
        free(*dst[i]);
        *dst[i] = (int32_t*)dup_mem(src[i], sizeof(int32_t) * P);
    }
    return s;
}

void so_free(so_sim* s) {
    if (!s) return;
    free(s->occ);
    free(s->stat);
    for (int k = 0; k < SO_KINDS; ++k) {
        free(s->dyn[k]);
        free(s->orient[k]);
        free(s->from_mask[k]);
        free(s->to_mask[k]);
        for (int o = 0; o < s->n_plans[k]; ++o)
            for (int sct = 0; sct < SO_SECTS; ++sct) free(s->plans[k][o].e[sct]);
        for (int sct = 0; sct < SO_SECTS; ++sct) free(s->gather[k][sct]);
    }
    free(s->cx); free(s->cy); free(s->fw); free(s->fh); free(s->period); free(s->phase); free(s->goal);
    free(s->enroll_ids); free(s->enroll_scores); free(s->winners); free(s->moved_from); free(s->moved_to);
    free(s->dec_dir); free(s->dec_score);
    free(s);
}

/* ---------------------------------------------------------------------------------------
 * seeding (ref: scenario.cpp:309-429).  The reference draws from std::mt19937_64 through
 * libstdc++'s std::uniform_int_distribution<int> and std::shuffle; neither is specified by
 * the C++ standard, so their published libstdc++ 13 algorithms are restated here
 * (bits/uniform_int_dist.h: Lemire's nearly-divisionless method on a 128-bit product;
 * bits/stl_algo.h: pairwise-swap shuffle) and pinned by the golden digests.
 * ------------------------------------------------------------------------------------- */

typedef struct mt64 {
    uint64_t x[312];
    int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->x[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->x[i] = 6364136223846793005ull * (g->x[i - 1] ^ (g->x[i - 1] >> 62)) + (uint64_t)i;
    g->i = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->i >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
        for (int k = 0; k < 312; ++k) {
            const uint64_t y = (g->x[k] & upper) | (g->x[(k + 1) % 312] & lower);
            g->x[k] = g->x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ull : 0);
        }
        g->i = 0;
    }
    uint64_t z = g->x[g->i++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

/* uniform integer in [0, range) for range >= 1 (libstdc++ _S_nd<unsigned __int128>) */
static uint64_t lemire_below(mt64* g, uint64_t range) {
    unsigned __int128 product = (unsigned __int128)mt64_next(g) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
        const uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            product = (unsigned __int128)mt64_next(g) * range;
            low = (uint64_t)product;
        }
    }
    return (uint64_t)(product >> 64);
}

static int uniform_int(mt64* g, int lo, int hi) { /* std::uniform_int_distribution<int>(lo,hi)(g) */
    const uint64_t urange = (uint64_t)hi - (uint64_t)lo;
    return (int)(lemire_below(g, urange + 1) + (uint64_t)lo);
}

void so_rng_check(uint64_t seed, int lo, int hi, int n, int32_t* out) {
    mt64 g;
    mt64_seed(&g, seed);
    for (int i = 0; i < n; ++i) out[i] = uniform_int(&g, lo, hi);
}

static void shuffle_pairs(int32_t* xs, int32_t* ys, size_t n, mt64* g) { /* std::shuffle, stl_algo.h:3741-3800 */
    if (n == 0) return;
#define SWAP_AT(a, b) do { int32_t t = xs[a]; xs[a] = xs[b]; xs[b] = t; t = ys[a]; ys[a] = ys[b]; ys[b] = t; } while (0)
    const uint64_t urngrange = UINT64_MAX, urange = (uint64_t)n;
    if (urngrange / urange >= urange) {
        size_t i = 1;
        if ((urange % 2) == 0) {
            const size_t j = (size_t)lemire_below(g, 2);
            SWAP_AT(i, j);
            ++i;
        }
        while (i != n) {
            const uint64_t swap_range = (uint64_t)i + 1;
            const uint64_t b1 = swap_range + 1;
            const uint64_t x = lemire_below(g, swap_range * b1);
            const size_t p0 = (size_t)(x / b1), p1 = (size_t)(x % b1);
            SWAP_AT(i, p0);
            ++i;
            SWAP_AT(i, p1);
            ++i;
        }
        return;
    }
    for (size_t i = 1; i < n; ++i) {
        const size_t j = (size_t)lemire_below(g, (uint64_t)i + 1);
        SWAP_AT(i, j);
    }
#undef SWAP_AT
}

int64_t so_planned_population(const so_config* cfg, const so_seed_spec* spec) { /* ref: scenario.cpp:309-313 */
    const double cells = (double)((int64_t)cfg->width * cfg->height);
    return (int64_t)floor(spec->density * cells / (double)(spec->ped_width * spec->ped_height));
}

/* ref: scenario.cpp:320-334 center_feasible + area_free */
static int center_ok(const so_sim* s, int x, int y, int fw, int fh) {
    const int hw = (fw - 1) / 2, hh = (fh - 1) / 2;
    if (s->cfg.closed && !(x >= hw && x + hw < s->W && y >= hh && y + hh < s->H)) return 0;
    for (int oy = -hh; oy <= hh; ++oy) {
        for (int ox = -hw; ox <= hw; ++ox) {
            int px, py;
            if (!wrap_xy(s, x + ox, y + oy, &px, &py)) return 0;
            if (s->occ[flat(s, px, py)] != SO_NO_PED) return 0;
        }
    }
    return 1;
}

so_sim* so_seed(const so_config* cfg, const so_seed_spec* spec, char* err, size_t errlen) {
    const int64_t count = so_planned_population(cfg, spec);
    so_sim* s = alloc_sim(cfg, count, err, errlen);
    if (!s) return NULL;
    const int fw = spec->ped_width, fh = spec->ped_height;
    mt64 rng;
    mt64_seed(&rng, spec->seed);

    /* place_centers, ref: scenario.cpp:342-388 */
    int64_t placed = 0, budget = 64 * count;
    int exhausted = 0;
    while (placed < count && !exhausted) {
        for (;;) {
            if (budget-- <= 0) {
                exhausted = 1;
                break;
            }
            const int x = uniform_int(&rng, 0, s->W - 1);
            const int y = uniform_int(&rng, 0, s->H - 1);
            if (!center_ok(s, x, y, fw, fh)) continue; /* infeasible or overlapping */
            stamp_footprint(s, x, y, fw, fh, (int32_t)placed);
            s->cx[placed] = x;
            s->cy[placed] = y;
            ++placed;
            break;
        }
    }
    if (exhausted) { /* sublattice fallback */
        const int hw = (fw - 1) / 2, hh = (fh - 1) / 2;
        size_t nslots = 0, cap = 0;
        for (int y = hh; y + hh < s->H; y += fh)
            for (int x = hw; x + hw < s->W; x += fw) ++cap;
        int32_t* sx = (int32_t*)zalloc(cap, sizeof(int32_t));
        int32_t* sy = (int32_t*)zalloc(cap, sizeof(int32_t));
        for (int y = hh; y + hh < s->H; y += fh)
            for (int x = hw; x + hw < s->W; x += fw) {
                sx[nslots] = x;
                sy[nslots] = y;
                ++nslots;
            }
        if ((int64_t)nslots < count) {
            snprintf(err, errlen, "cannot place %lld pedestrians: density too high for the footprint",
                     (long long)count);
            free(sx);
            free(sy);
            so_free(s);
            return NULL;
        }
        shuffle_pairs(sx, sy, nslots, &rng);
        memcpy(s->cx, sx, sizeof(int32_t) * (size_t)count);
        memcpy(s->cy, sy, sizeof(int32_t) * (size_t)count);
        free(sx);
        free(sy);
    }

    /* seed_population, ref: scenario.cpp:392-429: the occupancy grid is rebuilt from the
     * final centres (the rejection-sampling scratch grid is discarded) */
    for (int64_t i = 0; i < s->C; ++i) s->occ[i] = SO_NO_PED;
    for (int64_t i = 0; i < count; ++i) {
        s->fw[i] = fw;
        s->fh[i] = fh;
        s->period[i] = spec->walk_period_min == spec->walk_period_max
                           ? spec->walk_period_min
                           : uniform_int(&rng, spec->walk_period_min, spec->walk_period_max);
        s->phase[i] = (int)i % s->period[i];
        s->goal[i] = spec->goal_sects[(size_t)i % (size_t)spec->n_goal_sects];
        s->orient[0][i] = s->goal[i];
        s->orient[1][i] = s->goal[i];
        s->orient[2][i] = 0;
        stamp_footprint(s, s->cx[i], s->cy[i], fw, fh, (int32_t)i);
    }
    float* fresh = (float*)malloc(sizeof(float) * (size_t)s->C * SO_SECTS * SO_KINDS);
    so_rebuild_images(s, fresh);
    for (int k = 0; k < SO_KINDS; ++k)
        memcpy(s->dyn[k], fresh + (size_t)k * (size_t)s->C * SO_SECTS, sizeof(float) * (size_t)s->C * SO_SECTS);
    free(fresh);
    return s;
}

/* ---------------------------------------------------------------------------------------
 * the tick (ref: engine.cpp:242-550)
 * ------------------------------------------------------------------------------------- */

/* ref: engine.cpp:31-50 sort8_desc — fixed 19-comparator network, ties to the lower sect */
void so_sort8_desc(const double scores[8], int32_t p[8]) {
    static const int net[19][2] = {{0, 1}, {2, 3}, {0, 2}, {1, 3}, {1, 2}, {4, 5}, {6, 7}, {4, 6}, {5, 7}, {5, 6},
                                   {0, 4}, {1, 5}, {1, 4}, {2, 6}, {3, 7}, {3, 6}, {2, 4}, {3, 5}, {3, 4}};
    for (int i = 0; i < 8; ++i) p[i] = i;
    for (int c = 0; c < 19; ++c) {
        const int a = net[c][0], b = net[c][1];
        const int pa = p[a], pb = p[b];
        const int swap = (scores[pa] < scores[pb]) || (scores[pa] == scores[pb] && pa > pb);
        p[a] = swap ? pb : pa;
        p[b] = swap ? pa : pb;
    }
}

/* ref: accumulator.hpp:54-83 */
double so_one_step_sum(const double* terms, int64_t n) {
    double sum = 0.0;
    for (int64_t i = 0; i < n; ++i) sum += terms[i];
    return sum;
}

double so_multi_step_sum(const double* terms, int64_t n, int k) {
    double partials[16] = {0};
    const int64_t m = (n + k - 1) / k;
    for (int64_t i = 0; i < m; ++i)
        for (int j = 0; j < k; ++j) {
            const int64_t idx = i * k + j;
            partials[idx & (k - 1)] += idx < n ? terms[idx] : 0.0;
        }
    double sum = 0.0;
    for (int j = 0; j < k; ++j) sum += partials[j];
    return sum;
}

/* ref: grid.cpp:58-72 local_density */
double so_local_density(const so_sim* s, int cx, int cy, int radius) {
    int64_t occupied = 0, window = 0;
    for (int oy = -radius; oy <= radius; ++oy) {
        for (int ox = -radius; ox <= radius; ++ox) {
            int x, y;
            if (!wrap_xy(s, cx + ox, cy + oy, &x, &y)) continue;
            ++window;
            occupied += s->occ[flat(s, x, y)] != SO_NO_PED;
        }
    }
    if (window == 0) return 0.0;
    return (double)occupied / (double)window;
}

/* ref: engine.cpp:256-287 move_cells_empty / move_new_cells.  Visits the cells a step in
 * `direction` would newly cover.  Returns 0 if one falls off a closed grid; with
 * need_empty, also 0 if one is occupied.  Cells are appended to out_flat when non-NULL. */
static int new_cells(const so_sim* s, int64_t i, int direction, int need_empty, size_t* out_flat, int* n_out) {
    int ux, uy;
    so_sect_step(direction, &ux, &uy);
    const int rw = (s->fw[i] - 1) / 2, rh = (s->fh[i] - 1) / 2;
    int n = 0;
    for (int oy = -rh; oy <= rh; ++oy) {
        for (int ox = -rw; ox <= rw; ++ox) {
            if (abs(ox + ux) <= rw && abs(oy + uy) <= rh) continue; /* still covered by the old footprint */
            int x, y;
            if (!wrap_xy(s, s->cx[i] + ux + ox, s->cy[i] + uy + oy, &x, &y)) return 0;
            if (need_empty && s->occ[flat(s, x, y)] != SO_NO_PED) return 0;
            if (out_flat) out_flat[n] = flat(s, x, y);
            ++n;
        }
    }
    if (n_out) *n_out = n;
    return 1;
}

/* ref: engine.cpp:289-324 decide_core (+ :242-254 regulate, goal_bias) */
static void decide_core(const so_sim* s, int64_t i, int32_t* direction, double* score) {
    *direction = SO_STILL;
    *score = 0.0;
    if (s->tick % s->period[i] != s->phase[i]) return;
    double g = 1.0;
    if (s->cfg.regulation != 0) {
        const double rho = so_local_density(s, s->cx[i], s->cy[i], s->cfg.density_radius);
        g = 1.0 - rho;
        if (g < 0.1) g = 0.1; /* std::max(0.1, 1.0 - rho) */
    }
    static const double kCos[5] = {1.0, M_SQRT1_2, 0.0, 0.0, 0.0};
    const double w[SO_KINDS] = {s->cfg.weight_dir_attractive, s->cfg.weight_dir_repulsive, s->cfg.weight_recurrent};
    const size_t base = flat(s, s->cx[i], s->cy[i]) * SO_SECTS;
    double scores[8];
    for (int sct = 0; sct < SO_SECTS; ++sct) {
        double raw = s->cfg.weight_static * s->stat[base + (size_t)sct];
        for (int k = 0; k < SO_KINDS; ++k) raw += w[k] * s->dyn[k][base + (size_t)sct];
        scores[sct] = g * raw + s->cfg.goal_bias * kCos[so_sect_distance(sct, s->goal[i])];
    }
    int32_t order[8];
    so_sort8_desc(scores, order);
    for (int r = 0; r < 8; ++r) {
        const int sct = order[r];
        if (scores[sct] <= 0.0) break;
        if (!new_cells(s, i, sct, 1, NULL, NULL)) continue;
        *direction = sct;
        *score = scores[sct];
        return;
    }
}

int so_decide(so_sim* s, int64_t ped, int32_t* direction, double* score) {
    decide_core(s, ped, direction, score);
    return 0;
}

static int fail(so_sim* s, int phase, const char* msg) {
    snprintf(s->err, sizeof s->err, "tick %lld phase k-%d: %s", (long long)s->tick, phase, msg);
    s->err_phase = phase;
    return 1;
}

/* ref: engine.cpp:335-339 k1_init_range */
static void k1_init(so_sim* s) {
    const size_t C = (size_t)s->C;
    for (size_t i = 0; i < C * SO_SECTS; ++i) {
        s->enroll_ids[i] = SO_NO_PED;
        s->enroll_scores[i] = 0.0;
    }
    for (size_t i = 0; i < C; ++i) s->winners[i] = s->moved_from[i] = s->moved_to[i] = SO_NO_PED;
    for (int k = 0; k < SO_KINDS; ++k) {
        memset(s->from_mask[k], 0, C);
        memset(s->to_mask[k], 0, C);
    }
}

/* ref: engine.cpp:341-363 k2_decide_range */
static int k2_decide(so_sim* s) {
    size_t* cells = (size_t*)malloc(sizeof(size_t) * 4096);
    size_t cap = 4096;
    for (int64_t i = 0; i < s->P; ++i) {
        decide_core(s, i, &s->dec_dir[i], &s->dec_score[i]);
        if (s->dec_dir[i] == SO_STILL) continue;
        const size_t need = (size_t)(s->fw[i] * s->fh[i]);
        if (need > cap) {
            cap = need;
            cells = (size_t*)realloc(cells, sizeof(size_t) * cap);
        }
        int n = 0;
        new_cells(s, i, s->dec_dir[i], 0, cells, &n);
        for (int c = 0; c < n; ++c) {
            const size_t slot = cells[c] * SO_SECTS + (size_t)s->dec_dir[i];
            if (s->enroll_ids[slot] != SO_NO_PED) {
                free(cells);
                return fail(s, 2, "enrollment slot conflict");
            }
            s->enroll_ids[slot] = (int32_t)i;
            s->enroll_scores[slot] = s->dec_score[i];
        }
    }
    free(cells);
    return 0;
}

/* ref: engine.cpp:365-386 k3_vote_range */
static void k3_vote(so_sim* s) {
    const int fault = s->cfg.fault_invert_vote_tiebreak;
    for (size_t su = 0; su < (size_t)s->C; ++su) {
        int32_t best_id = SO_NO_PED;
        double best_score = 0.0;
        for (int slot = 0; slot < SO_SECTS; ++slot) {
            const int32_t id = s->enroll_ids[su * SO_SECTS + (size_t)slot];
            if (id == SO_NO_PED) continue;
            const double score = s->enroll_scores[su * SO_SECTS + (size_t)slot];
            int better = best_id == SO_NO_PED || score > best_score;
            if (!better && score == best_score) better = fault ? id > best_id : id < best_id;
            if (better) {
                best_id = id;
                best_score = score;
            }
        }
        s->winners[su] = best_id;
    }
}

/* ref: engine.cpp:388-426 k4_move_range */
static int64_t k4_move(so_sim* s) {
    int64_t moved = 0;
    size_t* cells = (size_t*)malloc(sizeof(size_t) * 4096);
    size_t cap = 4096;
    for (int64_t i = 0; i < s->P; ++i) {
        const int d = s->dec_dir[i];
        if (d == SO_STILL) continue;
        const size_t need = (size_t)(s->fw[i] * s->fh[i]);
        if (need > cap) {
            cap = need;
            cells = (size_t*)realloc(cells, sizeof(size_t) * cap);
        }
        int n = 0;
        if (!new_cells(s, i, d, 0, cells, &n)) n = 0;
        int won = n > 0;
        for (int c = 0; c < n; ++c) won = won && s->winners[cells[c]] == (int32_t)i;
        if (!won) continue;
        int ux, uy;
        so_sect_step(d, &ux, &uy);
        const int ox0 = s->cx[i], oy0 = s->cy[i];
        int nx, ny;
        wrap_xy(s, ox0 + ux, oy0 + uy, &nx, &ny);
        const int rw = (s->fw[i] - 1) / 2, rh = (s->fh[i] - 1) / 2;
        for (int oy = -rh; oy <= rh; ++oy) { /* release cells the new footprint no longer covers */
            for (int ox = -rw; ox <= rw; ++ox) {
                if (abs(ox - ux) <= rw && abs(oy - uy) <= rh) continue;
                int x, y;
                wrap_xy(s, ox0 + ox, oy0 + oy, &x, &y);
                s->occ[flat(s, x, y)] = SO_NO_PED;
            }
        }
        for (int c = 0; c < n; ++c) s->occ[cells[c]] = (int32_t)i;
        s->cx[i] = nx;
        s->cy[i] = ny;
        const size_t from = flat(s, ox0, oy0), to = flat(s, nx, ny);
        s->moved_from[from] = (int32_t)i;
        s->moved_to[to] = (int32_t)i;
        for (int k = 0; k < SO_KINDS; ++k) {
            const uint8_t mask = is_directional(kind_of_dyn(k)) ? (uint8_t)(1u << s->orient[k][i]) : (uint8_t)0xFF;
            s->from_mask[k][from] = mask;
            s->to_mask[k][to] = mask;
        }
        ++moved;
    }
    free(cells);
    return moved;
}

/* ref: engine.cpp:428-472 k5_writeback_range with accumulator.hpp:36-46 StepCache */
static void k5_range(so_sim* s, size_t su_begin, size_t su_end) {
    const int K = s->cfg.chunk_k;
    for (size_t su = su_begin; su < su_end; ++su) {
        const int tx = (int)(su % (size_t)s->W), ty = (int)(su / (size_t)s->W);
        for (int kind = 0; kind < SO_KINDS; ++kind) {
            const uint8_t* from_mask = s->from_mask[kind];
            const uint8_t* to_mask = s->to_mask[kind];
            for (int sct = 0; sct < SO_SECTS; ++sct) {
                const int n = s->n_gather[kind][sct];
                if (n == 0) continue;
                const gather_entry* list = s->gather[kind][sct];
                double partials[16] = {0};
                size_t idx = 0;
                for (int j = 0; j < n; ++j) {
                    int cx = tx + list[j].dx, cy = ty + list[j].dy;
                    if (!s->cfg.closed) {
                        while (cx < 0) cx += s->W;
                        while (cx >= s->W) cx -= s->W;
                        while (cy < 0) cy += s->H;
                        while (cy >= s->H) cy -= s->H;
                    } else if (cx < 0 || cx >= s->W || cy < 0 || cy >= s->H) {
                        idx += 2;
                        continue;
                    }
                    const size_t c = (size_t)cy * (size_t)s->W + (size_t)cx;
                    const double left = (list[j].mask & from_mask[c]) != 0 ? 1.0 : 0.0;
                    partials[idx & (size_t)(K - 1)] += -list[j].mag * left;
                    ++idx;
                    const double arrived = (list[j].mask & to_mask[c]) != 0 ? 1.0 : 0.0;
                    partials[idx & (size_t)(K - 1)] += list[j].mag * arrived;
                    ++idx;
                }
                double total = 0.0;
                for (int j = 0; j < K; ++j) total += partials[j];
                s->dyn[kind][su * SO_SECTS + (size_t)sct] += (float)total;
            }
        }
    }
}

/* The reference runs k-5 as a parallel_for over su with a static contiguous partition
 * (engine.cpp:524-528, thread_pool.cpp:52-54): every su is written by exactly one worker and reads
 * only the movement log, so the result does not depend on the worker count.  so_set_threads > 1 does
 * the same here (large parity cases); the default is the plain loop. */
static int g_threads = 1;
void so_set_threads(int n) { g_threads = n < 1 ? 1 : (n > 64 ? 64 : n); }

typedef struct {
    so_sim* s;
    size_t begin, end;
} k5_job;

static void* k5_worker(void* arg) {
    k5_job* j = (k5_job*)arg;
    k5_range(j->s, j->begin, j->end);
    return NULL;
}

static void k5_writeback(so_sim* s) {
    const size_t n = (size_t)s->C;
    const int workers = g_threads;
    if (workers <= 1 || n < 4096) {
        k5_range(s, 0, n);
        return;
    }
    pthread_t tid[64];
    k5_job job[64];
    int started = 0;
    for (int w = 0; w < workers; ++w) { /* [n*w/workers, n*(w+1)/workers), thread_pool.cpp:52-54 */
        job[w].s = s;
        job[w].begin = n * (size_t)w / (size_t)workers;
        job[w].end = n * (size_t)(w + 1) / (size_t)workers;
        if (pthread_create(&tid[w], NULL, k5_worker, &job[w]) != 0) break;
        ++started;
    }
    for (int w = started; w < workers; ++w) k5_range(s, job[w].begin, job[w].end);
    for (int w = 0; w < started; ++w) pthread_join(tid[w], NULL);
}

/* ref: engine.cpp:538-550 maybe_rebuild + fields.cpp:144-150 max_abs_difference */
static int maybe_rebuild(so_sim* s) {
    if (s->cfg.rebuild_interval <= 0 || s->tick % s->cfg.rebuild_interval != 0) return 0;
    const size_t n = (size_t)s->C * SO_SECTS;
    float* fresh = (float*)malloc(sizeof(float) * n * SO_KINDS);
    so_rebuild_images(s, fresh);
    for (int k = 0; k < SO_KINDS; ++k) {
        float worst = 0.0f;
        for (size_t i = 0; i < n; ++i) {
            const float d = fabsf(s->dyn[k][i] - fresh[(size_t)k * n + i]);
            if (worst < d) worst = d; /* std::max(worst, d) */
        }
        if (worst > s->cfg.rebuild_tolerance) {
            free(fresh);
            return fail(s, 5, "image drifted");
        }
    }
    for (int k = 0; k < SO_KINDS; ++k) memcpy(s->dyn[k], fresh + (size_t)k * n, sizeof(float) * n);
    free(fresh);
    return 0;
}

/* ref: engine.cpp:478-536 Engine::tick */
int so_tick(so_sim* s, int until_phase, int64_t* moved_out) {
    int64_t moved = 0;
    k1_init(s);
    if (until_phase == 1) goto done;
    if (k2_decide(s)) return 1;
    if (until_phase == 2) goto done;
    k3_vote(s);
    if (until_phase == 3) goto done;
    moved = k4_move(s);
    if (until_phase == 4) goto done;
    if (moved > 0) k5_writeback(s);
    if (until_phase == 5) goto done;
    s->tick += 1;
    if (maybe_rebuild(s)) return 1;
done:
    if (moved_out) *moved_out = moved;
    return 0;
}

/* ref: engine.cpp:556-563 Engine::run */
int so_run(so_sim* s, int64_t ticks, int64_t* moved) {
    if (so_verify(s)) return 1;
    for (int64_t t = 0; t < ticks; ++t) {
        int64_t m = 0;
        if (so_tick(s, 0, &m)) return 1;
        if (moved) moved[t] = m;
    }
    return 0;
}

/* ref: engine.cpp:569-618 verify_state (the structural checks that can fail for flat arrays) */
int so_verify(so_sim* s) {
    const size_t C = (size_t)s->C;
    int32_t* expected = (int32_t*)malloc(sizeof(int32_t) * C);
    for (size_t i = 0; i < C; ++i) expected[i] = SO_NO_PED;
    for (int64_t i = 0; i < s->P; ++i) {
        int x, y;
        if (!wrap_xy(s, s->cx[i], s->cy[i], &x, &y) || x != s->cx[i] || y != s->cy[i]) {
            free(expected);
            return fail(s, 0, "pedestrian center not normalized");
        }
        if (s->period[i] < 1 || s->phase[i] < 0 || s->phase[i] >= s->period[i]) {
            free(expected);
            return fail(s, 0, "walk gate out of range");
        }
        if (s->goal[i] < 0 || s->goal[i] >= SO_SECTS) {
            free(expected);
            return fail(s, 0, "goal sect out of range");
        }
        const int rw = (s->fw[i] - 1) / 2, rh = (s->fh[i] - 1) / 2;
        for (int oy = -rh; oy <= rh; ++oy) {
            for (int ox = -rw; ox <= rw; ++ox) {
                if (!wrap_xy(s, s->cx[i] + ox, s->cy[i] + oy, &x, &y)) {
                    free(expected);
                    return fail(s, 0, "footprint crosses a closed edge");
                }
                if (expected[flat(s, x, y)] != SO_NO_PED) {
                    free(expected);
                    return fail(s, 0, "pedestrians overlap");
                }
                expected[flat(s, x, y)] = (int32_t)i;
            }
        }
    }
    const int same = memcmp(expected, s->occ, sizeof(int32_t) * C) == 0;
    free(expected);
    if (!same) return fail(s, 0, "occupancy does not match the pedestrians");
    return 0;
}

/* ref: tests/acceptance/acceptance_main.cpp:39-58 fnv1a + state_digest */
static uint64_t fnv1a(const void* data, size_t bytes, uint64_t h) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

uint64_t so_digest(const so_sim* s) {
    uint64_t h = 14695981039346656037ull;
    h = fnv1a(s->occ, sizeof(int32_t) * (size_t)s->C, h);
    for (int k = 0; k < SO_KINDS; ++k) h = fnv1a(s->dyn[k], sizeof(float) * (size_t)s->C * SO_SECTS, h);
    for (int64_t i = 0; i < s->P; ++i) {
        const int32_t xy[2] = {s->cx[i], s->cy[i]};
        h = fnv1a(xy, sizeof xy, h);
    }
    return h;
}

/* ---------------------------------------------------------------------------------------
 * accessors
 * ------------------------------------------------------------------------------------- */
const char* so_last_error(const so_sim* s) { return s->err; }
int so_error_phase(const so_sim* s) { return s->err_phase; }
int64_t so_population(const so_sim* s) { return s->P; }
int64_t so_tick_count(const so_sim* s) { return s->tick; }
void so_set_tick(so_sim* s, int64_t t) { s->tick = t; }
int32_t* so_occupancy(so_sim* s) { return s->occ; }
float* so_image(so_sim* s, int which) { return which < 0 ? s->stat : s->dyn[which]; }
int32_t* so_centers_x(so_sim* s) { return s->cx; }
int32_t* so_centers_y(so_sim* s) { return s->cy; }
const int32_t* so_ped_attr(const so_sim* s, int which) {
    switch (which) {
        case 0: return s->period;
        case 1: return s->phase;
        case 2: return s->goal;
        case 3: return s->fw;
        default: return s->fh;
    }
}
const int32_t* so_decisions(const so_sim* s) { return s->dec_dir; }
const double* so_decision_scores(const so_sim* s) { return s->dec_score; }
const int32_t* so_enroll_ids(const so_sim* s) { return s->enroll_ids; }
const double* so_enroll_scores(const so_sim* s) { return s->enroll_scores; }
const int32_t* so_winners(const so_sim* s) { return s->winners; }
const int32_t* so_moved_from(const so_sim* s) { return s->moved_from; }
const int32_t* so_moved_to(const so_sim* s) { return s->moved_to; }
const uint8_t* so_from_mask(const so_sim* s, int kind) { return s->from_mask[kind]; }
const uint8_t* so_to_mask(const so_sim* s, int kind) { return s->to_mask[kind]; }

int so_plan_entries(const so_sim* s, int kind, int orientation, int sect, int32_t* dxdy, double* mag, int cap) {
    const write_plan* p = &s->plans[kind][s->n_plans[kind] == 1 ? 0 : orientation];
    for (int i = 0; i < p->n[sect] && i < cap; ++i) {
        if (dxdy) {
            dxdy[2 * i] = p->e[sect][i].dx;
            dxdy[2 * i + 1] = p->e[sect][i].dy;
        }
        if (mag) mag[i] = p->e[sect][i].mag;
    }
    return p->n[sect];
}

int so_gather_entries(const so_sim* s, int kind, int sect, int32_t* dxdy, double* mag, uint8_t* mask, int cap) {
    const int n = s->n_gather[kind][sect];
    for (int i = 0; i < n && i < cap; ++i) {
        if (dxdy) {
            dxdy[2 * i] = s->gather[kind][sect][i].dx;
            dxdy[2 * i + 1] = s->gather[kind][sect][i].dy;
        }
        if (mag) mag[i] = s->gather[kind][sect][i].mag;
        if (mask) mask[i] = s->gather[kind][sect][i].mask;
    }
    return n;
}
