/*
 * socfield_shim.h — flat C view of the socfield C++ API (Engine / SimState /
 * ScenarioConfig), for driving an implementation of that API from ctypes.
 *
 * TEST INFRASTRUCTURE.  The same shim source (socfield_shim.cpp) is compiled
 * twice, against two different implementations of the *same* C++ headers:
 *
 *   1. the unmodified reference sources under /root/reference/proj
 *      -> oracle/_ref/libsocfield_ref.so          (the CPU oracle, "reference")
 *   2. this repository's host mirror (include/socfield/*.hpp + CUDA C-ABI)
 *      -> paper_1803_04782_b200/lib/libsocfield_b200_shim.so   (the product)
 *
 * Because one client source builds against both, the shim doubles as the
 * drop-in proof: everything it touches (types, signatures, error behaviour)
 * must exist with the reference's names in the product.
 *
 * Conventions: every call that can fail returns 0 on success and writes a
 * message into (err, errlen) otherwise:  1 = IntegrityError, 2 = ConfigError,
 * 3 = ParseError, 4 = SeedingError, 5 = anything else.
 */
#ifndef SOCFIELD_SHIM_H
#define SOCFIELD_SHIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct shim_sim shim_sim;

typedef struct shim_engine_cfg {
    int32_t chunk_k;
    double weight_static;
    double weight_dir_attractive;
    double weight_dir_repulsive;
    double weight_recurrent;
    double goal_bias;
    int32_t regulation;       /* 0 identity, 1 linear */
    int32_t density_radius;
    int64_t rebuild_interval;
    double rebuild_tolerance;
    int32_t workers;
    int32_t fault_invert_vote_tiebreak;
} shim_engine_cfg;

typedef struct shim_field {
    int32_t width, height;
    double gain, decay;
} shim_field;

/* Static (anchored) field: kind 0 omni-attractive, 1 omni-repulsive (FieldKind order). */
typedef struct shim_anchor {
    int32_t kind;
    int32_t width, height;
    double gain, decay;
    int32_t x, y;
} shim_anchor;

/* Per-phase capture buffers for one inspected tick; any pointer may be NULL. */
typedef struct shim_capture {
    int32_t* decisions;       /* [P]     after k-2: Engine::decision_direction       */
    int32_t* enroll_ids;      /* [C*8]   after k-2: EnrollmentTable::id_at           */
    double* enroll_scores;    /* [C*8]   after k-2: EnrollmentTable::score_at        */
    int32_t* winners;         /* [C]     after k-3: Engine::vote_winners             */
    int32_t* moved_from;      /* [C]     after k-4: MovementLog::moved_from          */
    int32_t* moved_to;        /* [C]     after k-4                                   */
    uint8_t* from_mask;       /* [3*C]   after k-4: MovementLog::from_mask[kind]     */
    uint8_t* to_mask;         /* [3*C]   after k-4                                   */
    int32_t* occupancy_k4;    /* [C]     after k-4                                   */
    int32_t* centers_k4;      /* [P*2]   after k-4                                   */
    float* images_k5;         /* [3*C*8] after k-5 (before the periodic rebuild)     */
    int32_t phases_seen;      /* bit p set when the inspector ran for phase p (1..5) */
} shim_capture;

const char* shim_impl_name(void);

/* parse_scenario + seed_population + Engine(cfg.grid, cfg.engine_config(), cfg.field_templates()) */
int shim_from_scenario(const char* text, int workers, shim_sim** out, char* err, size_t errlen);

/* Hand-built population in the style of the reference's unit-test fixtures
 * (make_ped / make_state): occupancy from footprint_cells, dynamic images from
 * rasterize_dynamic, zero static image. */
int shim_from_arrays(int width, int height, int closed, const shim_engine_cfg* cfg,
                     const shim_field templates[3], int64_t n, const int32_t* cx,
                     const int32_t* cy, const int32_t* fw, const int32_t* fh,
                     const int32_t* period, const int32_t* phase, const int32_t* goal,
                     shim_sim** out, char* err, size_t errlen);

void shim_free(shim_sim* s);

/* static_image = rasterize_static(anchors, grid) */
int shim_set_static_fields(shim_sim* s, int64_t n, const shim_anchor* anchors, char* err,
                           size_t errlen);

int shim_grid(const shim_sim* s, int32_t* width, int32_t* height, int32_t* closed);
int64_t shim_population(const shim_sim* s);
int64_t shim_tick_count(const shim_sim* s);
void shim_set_tick(shim_sim* s, int64_t tick);

/* Engine::run(state, ticks, mode); moved[ticks] and wall_us[ticks] optional. mode 0 seq, 1 par */
int shim_run(shim_sim* s, int64_t ticks, int mode, int64_t* moved, int64_t* phase_us5,
             char* err, size_t errlen);
/* Engine::tick(state, mode[, inspector]) */
int shim_tick(shim_sim* s, int mode, int64_t* moved, char* err, size_t errlen);
int shim_tick_capture(shim_sim* s, int mode, shim_capture* cap, int64_t* moved, char* err,
                      size_t errlen);

int shim_verify(const shim_sim* s, char* err, size_t errlen);
/* Engine::decide for pedestrian i: direction, score, new cells (x,y pairs, up to cap). */
int shim_decide(const shim_sim* s, int64_t ped, int32_t* direction, double* score,
                int32_t* ncells, int32_t* cells_xy, int32_t cap, char* err, size_t errlen);
/* Engine::rebuild_images -> out[3*C*8] */
int shim_rebuild_images(const shim_sim* s, float* out, char* err, size_t errlen);
/* Engine::plan(kind, orientation).entries(sect): returns count; fills up to cap. */
int shim_plan_entries(const shim_sim* s, int kind, int orientation, int sect, int32_t* dxdy,
                      double* magnitude, int32_t cap);
int shim_plan_fanout(const shim_sim* s, int kind, int orientation);

/* State accessors (copies). which: -1 static image, 0..2 dynamic kinds. */
void shim_get_centers(const shim_sim* s, int32_t* xy);
void shim_get_ped_attrs(const shim_sim* s, int32_t* period, int32_t* phase, int32_t* goal,
                        int32_t* fw, int32_t* fh);
void shim_get_occupancy(const shim_sim* s, int32_t* out);
void shim_get_image(const shim_sim* s, int which, float* out);
void shim_set_centers(shim_sim* s, const int32_t* xy);
void shim_set_occupancy(shim_sim* s, const int32_t* in);
void shim_set_image(shim_sim* s, int which, const float* in);

/* FNV-1a over occupancy, the three dynamic images, the centres — the digest of
 * the reference's acceptance suite (tests/acceptance/acceptance_main.cpp:39-58). */
uint64_t shim_digest(const shim_sim* s);
/* states_identical(a, b, &diagnosis): returns 1 if identical. */
int shim_states_identical(const shim_sim* a, const shim_sim* b, char* diag, size_t diaglen);
/* Deep copy (state + a fresh engine with the same configuration). */
int shim_clone(const shim_sim* s, shim_sim** out, char* err, size_t errlen);

/* Free functions of the API, for table-level parity. */
int shim_sect_index(double x, double y);
void shim_sort8_desc(const double scores[8], int32_t order[8]);
double shim_multi_step_sum(const double* terms, int64_t n, int k);
void shim_strength_at_offset(int kind, int w, int h, double gain, double decay, int orientation,
                             int dx, int dy, double* sx, double* sy);

#ifdef __cplusplus
}
#endif
#endif
