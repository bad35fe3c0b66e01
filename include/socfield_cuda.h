/*
 * socfield_cuda.h — the C ABI of the B200 (sm_100a) engine for the per-tick hot path of the
 * discrete social-field pedestrian model.
 *
 * This is the drop-in boundary.  The reference has no FFI: its boundary is the C++ class
 * socfield::Engine acting on the value type socfield::SimState
 * (reference proj/include/socfield/engine.hpp:91-98,142-230).  The host mirror in
 * include/socfield/ keeps that class signature for signature and forwards every device
 * operation through the entry points below — plain pointers and sizes, no C++ or torch
 * types, no exceptions across the line.  Each entry point names the reference interface it
 * replaces.
 *
 * Threading: an sfc_engine is not thread-safe; every call is synchronous for the caller
 * (the reference's Engine::tick is synchronous too, engine.hpp:150-158).
 */
#ifndef SOCFIELD_CUDA_H
#define SOCFIELD_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFC_ABI_VERSION 1
#define SFC_KINDS 3 /* dir-attractive, dir-repulsive, recurrent-repulsive (engine.hpp:19) */
#define SFC_SECTS 8

/* Status codes.  The host mirror rethrows them as the reference's exception types
 * (errors.hpp): INTEGRITY -> IntegrityError(tick, phase), CONFIG -> ConfigError,
 * everything else -> std::runtime_error. */
enum {
    SFC_OK = 0,
    SFC_E_INTEGRITY = -1,
    SFC_E_CONFIG = -2,
    SFC_E_CUDA = -3,
    SFC_E_NOMEM = -4,
    SFC_E_STATE = -5, /* call sequence error, e.g. run before upload */
    SFC_E_NO_DEVICE = -6
};

typedef struct sfc_engine sfc_engine;

/* GridGeometry (grid.hpp:26-45) + EngineConfig (engine.hpp:108-121). */
typedef struct sfc_config {
    int32_t width, height;
    int32_t closed;                /* BoundaryMode::Closed */
    int32_t chunk_k;               /* K of the multi-step sum: 2, 4, 8 or 16 */
    double weight_static, weight_dir_attractive, weight_dir_repulsive, weight_recurrent;
    double goal_bias;
    int32_t regulation;            /* 0 identity, 1 linear */
    int32_t density_radius;
    int64_t rebuild_interval;      /* 0 = never */
    double rebuild_tolerance;
    int32_t fault_invert_vote_tiebreak; /* test hook, engine.hpp:120 */
    int32_t device;                /* CUDA device ordinal */
    /* Row slab owned by this engine (multi-GPU): rows [slab_row0, slab_row0 + slab_rows).
     * slab_rows = 0 means the whole grid. */
    int32_t slab_row0, slab_rows;
    int32_t slab_halo;             /* resident rows beyond each slab edge (see sfc_slab_halo_rows) */
    /* > 1: band-swapped engine (sfc_band_run): slab_rows is the band height, the window moves over the grid */
    int32_t bands;
} sfc_config;

/* Merged contributor table of one dynamic kind, replacing Engine::build_gather_tables
 * (engine.cpp:201-221).  Indexed by centre offset (dx, dy) = mover centre - target su:
 * entry (dy + height/2) * width + (dx + width/2).
 *   magnitude  strength the field incurs at the target (double, WritePlan::Entry::magnitude)
 *   info       bits 0-2  sect of the (target, sect) address the offset feeds
 *              bits 3-10 orientation mask (all ones for the non-directional kind; 0 = the
 *                        offset is outside the support)
 *              bits 11-31 j, the offset's rank in the (kind, sect) contributor list, ordered
 *                        lexicographically by (dx, dy) — fixes the StepCache slot
 *                        (accumulator.hpp:36-40)
 * The host computes these with the same libm calls as the reference (fields.cpp:74-121). */
typedef struct sfc_kind_table {
    int32_t width, height;
    const double* magnitude;
    const uint32_t* info;
} sfc_kind_table;

typedef struct sfc_tables {
    sfc_kind_table kind[SFC_KINDS];
} sfc_tables;

/* Host view of a SimState (engine.hpp:91-98): raw pointers into OccupancyGrid::raw(),
 * StrengthImage::raw() and per-pedestrian attribute arrays gathered from
 * std::vector<Pedestrian>.  Arrays marked [out] are written by sfc_download. */
typedef struct sfc_state_view {
    int64_t tick;                 /* [in/out] SimState::tick */
    int64_t n_peds;
    int32_t* occupancy;           /* [in/out] [H*W], -1 empty */
    float* static_image;          /* [in]     [H*W*8] (may be NULL on download) */
    float* dyn_images[SFC_KINDS]; /* [in/out] [H*W*8] each */
    int32_t* center_xy;           /* [in/out] [P*2] */
    const int32_t* walk_period;   /* [in] [P] */
    const int32_t* walk_phase;    /* [in] [P] */
    const int32_t* goal_sect;     /* [in] [P] */
    const int32_t* orient_attractive; /* [in] [P] FieldSpec::orientation of the dir-attractive field */
    const int32_t* orient_repulsive;  /* [in] [P] ... of the dir-repulsive field */
    const int32_t* foot_w;        /* [in] [P] odd */
    const int32_t* foot_h;        /* [in] [P] odd */
} sfc_state_view;

/* TickMetrics (engine.hpp:123-128); phase_us from CUDA events when requested. */
typedef struct sfc_tick_metrics {
    int64_t tick;
    int64_t moved;
    int64_t phase_us[5];
    int64_t wall_us;
} sfc_tick_metrics;

/* Host mirrors of the per-tick temporaries the reference exposes through
 * Engine::enrollment(), vote_winners(), movement_log(), decision_direction()
 * (engine.hpp:172-177).  Any pointer may be NULL. */
typedef struct sfc_temporaries {
    int32_t* decisions;      /* [P] */
    double* decision_scores; /* [P] */
    int32_t* enroll_ids;     /* [C*8] */
    double* enroll_scores;   /* [C*8] */
    int32_t* winners;        /* [C] */
    int32_t* moved_from;     /* [C] */
    int32_t* moved_to;       /* [C] */
    uint8_t* from_mask;      /* [3*C] */
    uint8_t* to_mask;        /* [3*C] */
} sfc_temporaries;

/* A static field anchored at a su (fields.hpp:151-154 AnchoredField).  `table` is built by
 * the host exactly like a dynamic kind's (info mask is 0xFF inside the support); anchors
 * that share a FieldSpec share a table. */
typedef struct sfc_anchor {
    int32_t x, y;
    int32_t table;       /* index into the tables array passed alongside */
    int32_t orientation; /* facing sect of a directional field, -1 for non-directional kinds */
} sfc_anchor;

int sfc_abi_version(void);
/* Number of visible CUDA devices (<= 0: none; the engine never falls back to the CPU). */
int sfc_device_count(void);

/* Engine::Engine (engine.cpp:170-199): validates the configuration, uploads the tables,
 * allocates the SU field buffers and per-tick temporaries on the device. */
int sfc_create(const sfc_config* cfg, const sfc_tables* tables, sfc_engine** out, char* err,
               size_t errlen);
void sfc_destroy(sfc_engine* e);

/* Last error text and the (tick, phase, su) detail of an integrity violation. */
const char* sfc_last_error(const sfc_engine* e);
void sfc_error_detail(const sfc_engine* e, int64_t* tick, int32_t* phase, int32_t* su_x,
                      int32_t* su_y, double* value);

/* Host -> device copy of a whole SimState; device -> host copy of what a tick mutates
 * (occupancy, dynamic images, centres, tick).  Engine::tick / Engine::run entry and exit.
 *
 * sfc_upload with the dense arrays NULL (occupancy, static_image, all three dyn_images) describes a
 * freshly seeded population: the device then derives the occupancy grid from the footprints and
 * rasterises the dynamic images itself, exactly as seed_population does (scenario.cpp:392-429),
 * with a zero static image — no whole-grid host state is needed (a 32768^2 SimState is 141 GB).
 * sfc_download skips every array that is NULL (e.g. only center_xy set: positions alone). */
int sfc_upload(sfc_engine* e, const sfc_state_view* view);
int sfc_download(sfc_engine* e, sfc_state_view* view);

/* Engine::run body (engine.cpp:556-563 minus verify_state): `ticks` iterations of
 * Engine::tick (engine.cpp:478-536) including the periodic rebuild (engine.cpp:538-550), on
 * the device-resident state.  metrics: NULL or [ticks].  with_phase_times != 0 brackets each
 * phase with CUDA events (slower). */
int sfc_run(sfc_engine* e, int64_t ticks, sfc_tick_metrics* metrics, int with_phase_times);

/* One phase of the current tick for the Engine::Inspector path (engine.hpp:150-155):
 * phase 1..5 = k-1..k-5, 6 = end of tick (tick += 1, maybe_rebuild).  *moved is TickMetrics::moved
 * (valid after phase 4). */
int sfc_phase(sfc_engine* e, int phase, int64_t* moved);
int sfc_download_temporaries(sfc_engine* e, sfc_temporaries* out);

/* Engine::decide (engine.cpp:326-333) for one pedestrian of the uploaded state. */
int sfc_decide(sfc_engine* e, int64_t ped, int32_t* direction, double* score);

/* rasterize_dynamic / Engine::rebuild_images (engine.cpp:158-168,565-567) from the uploaded
 * pedestrians: out[k] receives image k ([H*W*8] host floats).  The device images are untouched. */
int sfc_rasterize_dynamic(sfc_engine* e, float* out[SFC_KINDS]);
/* Same, but replaces the device-resident dynamic images (seed_population, scenario.cpp:427). */
int sfc_reset_dynamic_images(sfc_engine* e);
/* rasterize_static / rasterize_into (fields.cpp:152-168): adds the anchored fields, in list
 * order, into the device static image — zeroed first, or initialised from `base` ([H*W*8] host
 * floats) when that is not NULL — and copies the result to `out` ([H*W*8], may be NULL). */
int sfc_rasterize_static(sfc_engine* e, int32_t n_tables, const sfc_kind_table* tables, int64_t n_anchors,
                         const sfc_anchor* anchors, const float* base, float* out);

/* Page-lock / unlock a host array the caller hands to sfc_upload / sfc_download again and again
 * (cudaHostRegister): copies from a locked array are single DMAs at PCIe rate, the copy path detects the
 * lock by itself.  Returns 0 on success; failure only means the staged copy path is used. */
int sfc_host_pin(const void* ptr, size_t bytes);
int sfc_host_unpin(const void* ptr);

/* ---- Row slabs across GPUs (no counterpart in the reference, which is single address space;
 * SURVEY.md 8e).  An engine created with sfc_config.slab_rows < height owns rows
 * [slab_row0, slab_row0 + slab_rows) and keeps slab_halo more rows resident on each side.
 * sfc_upload takes the WHOLE-grid host state and copies the slab's part; sfc_download writes back
 * only the rows and pedestrians the slab owns.  One tick = three device steps with a halo exchange
 * after step 0 (kind 0) and after step 1 (kinds 1, 2, 3):
 *   kind 0 decisions of boundary pedestrians   kind 1 positions of boundary pedestrians
 *   kind 2 occupancy rows                      kind 3 event-map rows
 * My `edge` (0 = low-y, 1 = high-y) send buffer goes to the ring neighbour's facing (1 - edge)
 * receive buffer.  sfc_slab_buffer returns device pointers so the transport (peer copy, NCCL) is
 * the caller's choice. */
int sfc_slab_halo_rows(int field_half_h, int ped_half_h, int density_radius_if_regulated);
int sfc_slab_begin(sfc_engine* e, int64_t ticks);
int sfc_slab_step(sfc_engine* e, int step);
int sfc_slab_buffer(sfc_engine* e, int kind, int edge, int recv, void** ptr, size_t* bytes);
/* The CUDA stream (cudaStream_t) every kernel of this engine is enqueued on: a transport that orders its
 * sends / receives on it (NCCL under a torch ExternalStream, peer copies with events) keeps the tick loop
 * free of host synchronisation — the reference's phase barrier (thread_pool.hpp:13-16) becomes stream order. */
void* sfc_stream(sfc_engine* e);
/* Synchronises, reports a device-side error, returns TickMetrics::moved of ticks [first, first+ticks)
 * counted since sfc_slab_begin (this slab's movers only). */
int sfc_slab_finish(sfc_engine* e, int64_t first_tick, int64_t ticks, int64_t* moved);
/* Single-process driver: runs `ticks` ticks over n slab engines (ordered by slab_row0), exchanging
 * halos with peer copies.  metrics: NULL or [ticks] (moved summed over slabs). */
int sfc_group_run(sfc_engine** engines, int n, int64_t ticks, sfc_tick_metrics* metrics);

/* ---- Band-swapped pass: a state LARGER than device memory (the paper's divide-and-conquer against
 * global-memory depletion; reference accumulator.hpp:68-83 multi_step_sum,
 * bench.cpp:14-24 memory_plan).  The reference holds one SimState in host memory; here that host
 * state is the backing store and the SU grid streams through the device in `bands` row bands of
 * slab_rows rows (+ slab_halo rows each side), one phase at a time:
 *   pass A  k-2   per band: occupancy (with halo), static + dynamic images in -> decisions
 *   pass B  k-3   per band: occupancy in -> vote results
 *   pass C  k-4   per band: occupancy, event map in -> moved, both out (halo rows included: a mover
 *                 that crosses a band edge writes into the neighbour's rows; bands run in order, so
 *                 the neighbour loads those rows after the store)
 *   pass D  k-5   per band: event map (with field halo), dynamic images in -> images out
 *   rebuild       check pass over every band, verdict, commit pass over every band
 * Pedestrians (31 B each) stay resident for the whole run, so no pedestrian halo exchange exists.
 * The engine must have been created with sfc_config.bands > 1; `host` holds every dense array
 * (occupancy, static_image, dyn_images) and is updated in place; results are bit-identical to sfc_run
 * on the undivided grid.  sfc_band_plan returns the smallest band count whose window (134 B per
 * resident su) plus the population fits `device_bytes` (0: what cudaMemGetInfo reports free). */
int sfc_band_run(sfc_engine* e, sfc_state_view* host, int64_t ticks, sfc_tick_metrics* metrics);
int sfc_band_plan(int32_t width, int32_t height, int32_t halo, int64_t n_peds, int64_t device_bytes, int device);

/* ---- Validation without host copies.
 * sfc_digest: the acceptance digest of the resident state — FNV-1a over occupancy, the three dynamic
 * images, the centres — bit-identical to state_digest (tests/acceptance/acceptance_main.cpp:39-58),
 * computed on the device (whole-grid engines only).
 * sfc_compare: states_identical (engine.cpp:103-156) between the resident states of two whole-grid
 * engines on the same device: the first difference in the reference's order. */
typedef struct sfc_difference {
    int32_t what;      /* 0 identical, 1 tick, 2 pedestrian count, 3 centre, 4 occupancy, 5 static image, 6 + k dynamic image k */
    int64_t index;     /* pedestrian id / flat su index / flat image index (su * 8 + sect) */
    int32_t ax, ay, bx, by; /* what == 3: the two centres; what == 4: ax, bx the two occupants */
    float av, bv;      /* what >= 5: the two image values */
} sfc_difference;
int sfc_digest(sfc_engine* e, uint64_t* digest);
int sfc_compare(sfc_engine* a, sfc_engine* b, sfc_difference* out);

/* Counters for bench.py: kernels launched by this engine since creation, bytes copied. */
typedef struct sfc_counters {
    int64_t kernel_launches;
    int64_t graph_launches;
    int64_t h2d_bytes, d2h_bytes;
    int32_t k5_path;        /* k-5 formulation chosen for the uploaded state: 0 scatter / event-walk gather, 1 window, 2 list walk, 3 pairs, 4 large-field */
    int32_t k5_active_list; /* 1: k-5 visits only the tiles k-4 listed */
} sfc_counters;
void sfc_get_counters(const sfc_engine* e, sfc_counters* out);

/* CUDA-event time of the device work enqueued by the last sfc_run, in milliseconds, and the
 * share spent in the k-5 write-back kernel when phase timing was requested. */
double sfc_last_run_ms(const sfc_engine* e);

#ifdef __cplusplus
}
#endif
#endif
