// sfc_internal.cuh — device-side data model shared by the sm_100a kernels.
//
// HBM layout (one engine = one row slab of the SU grid, normally the whole grid):
//   occ   int32 [rows_local][W]            occupant id per su, -1 empty        (grid.hpp:94-116)
//   stat  float [rows_local][W][8]         static strength image               (fields.hpp:89-112)
//   dyn   float [rows_local][W][3][8]      the three dynamic images INTERLEAVED per su: one
//                                          96-byte record, so the k-5 read-modify-write and the
//                                          k-2 centre read are single contiguous runs
//   ev    uint8 [rows_local][W][2]         movement events of the current tick (replaces the
//                                          reference's 14-byte MovementLog, engine.hpp:81-89):
//                                          byte 0 = "a pedestrian left this centre", byte 1 =
//                                          "arrived"; 0x80 | orient_attr | orient_rep << 3
//   per pedestrian (SoA): centre int2, gate int2 (period, phase), attr u32, decision dir int8 +
//   score f64, vote result u8, direction of the previous tick's move int8.
// rows_local = slab_rows + 2 * halo; the whole-grid engine has halo 0.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <vector>

#include "socfield_cuda.h"

namespace sfc {

constexpr int kSects = 8;
constexpr int kKinds = 3;
constexpr int kStill = -1;
constexpr int kNoPed = -1;

struct GridDev {
    int W, H;      // global extent
    int closed;    // BoundaryMode::Closed
    int row0;      // first owned global row
    int rows;      // owned rows
    int halo;      // resident rows beyond each slab edge
};

// Euclidean modulo (grid.cpp:8-11).
__host__ __device__ __forceinline__ int emod(int a, int m) {
    if (a >= 0 && a < m) return a;
    int r = a % m;
    return r < 0 ? r + m : r;
}

// Local flat su index of unwrapped global coordinates, or -1 when the su does not exist
// (closed boundary, grid.cpp:15-21) or is not resident in this slab.
__host__ __device__ __forceinline__ long long cell_index(const GridDev& g, int x, int y) {
    if (g.closed) {
        if (x < 0 || x >= g.W || y < 0 || y >= g.H) return -1;
    } else {
        x = emod(x, g.W);
        y = emod(y, g.H);
    }
    int ly = y - g.row0;
    if (!g.closed) ly = emod(ly + g.halo, g.H) - g.halo;
    if (ly < -g.halo || ly >= g.rows + g.halo) return -1;
    return (long long)(ly + g.halo) * g.W + x;
}

__host__ __device__ __forceinline__ bool row_owned(const GridDev& g, int y) {
    int ly = y - g.row0;
    if (!g.closed) ly = emod(ly, g.H);
    return ly >= 0 && ly < g.rows;
}

// True when global row y lies at most `depth` rows beyond this slab's owned range (depth 0 = owned).
__host__ __device__ __forceinline__ bool row_within(const GridDev& g, int y, int depth) {
    int ly = y - g.row0;
    if (!g.closed) ly = emod(ly + depth, g.H) - depth;
    return ly >= -depth && ly < g.rows + depth;
}

// ---- chained launches (programmatic dependent launch) ----------------------------------------
// A tick is four small-to-medium kernels in a row, hundreds of ticks in a run: the gap between two
// kernels of a stream (drain, then launch) is a visible share of a tick.  Kernels launched with
// launch_chained may be scheduled while their predecessor drains: they do whatever needs nothing from it
// (constant tables into shared memory) and then wait for its writes (chain_wait) before touching anything a
// kernel produces.  Every kernel launched this way must call chain_wait before its first global access to
// mutable state; on a plain launch the call does nothing.  chain_release lets the successor be scheduled
// before this kernel ends; measured (profiles/README.md, chained launches), that only pays for crowds small
// enough to be latency-bound — config 1: 27.4 -> 24.4 us a tick — and costs 3 to 5 % elsewhere (early CTAs of
// k-5 crowd k-4's SMs), so only the per-pedestrian kernels of small crowds call it.  SFC_CHAIN=0 launches
// everything plainly.
constexpr long long kChainReleasePeds = 4096;
__device__ __forceinline__ void chain_release(bool on) {
    if (on) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void chain_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool chain_enabled();   // sfc_ped_kernels.cu
void chain_configure(); // reads SFC_CHAIN (sfc_create)

template <typename... Params, typename... Args>
cudaError_t launch_chained(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = chain_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Multi-GPU row slabs: what the per-pedestrian kernels need to know beyond GridDev.
struct SlabDev {
    int active;               // this engine owns a proper sub-range of rows
    int reach;                // k-3 / k-4 also run for neighbours' pedestrians this many rows beyond the edge
    long long* ev_written;    // event-map cells written this tick (cleared at the start of the next)
    long long ev_capacity;
    int band;                 // band-swapped engine: every pedestrian is resident and processed by the band that owns
                              // its centre NOW — k-4 retires its vote flag so a mover is not moved again by the next band
};

// sect_step (fields.cpp:67-72) without a table: sect 0 = +x, counter-clockwise.
__host__ __device__ __forceinline__ int step_dx(int sect) {
    return (sect == 0 || sect == 1 || sect == 7) ? 1 : ((sect >= 3 && sect <= 5) ? -1 : 0);
}
__host__ __device__ __forceinline__ int step_dy(int sect) {
    return (sect >= 1 && sect <= 3) ? 1 : ((sect >= 5) ? -1 : 0);
}

// attr word of a pedestrian
__host__ __device__ __forceinline__ uint32_t pack_attr(int goal, int o_att, int o_rep, int half_w, int half_h) {
    return (uint32_t)goal | ((uint32_t)o_att << 3) | ((uint32_t)o_rep << 6) | ((uint32_t)half_w << 9) |
           ((uint32_t)half_h << 20);
}
__host__ __device__ __forceinline__ int attr_goal(uint32_t a) { return a & 7; }
__host__ __device__ __forceinline__ int attr_orient(uint32_t a, int kind) { return (a >> (3 + 3 * kind)) & 7; }
__host__ __device__ __forceinline__ int attr_half_w(uint32_t a) { return (a >> 9) & 0x7FF; }
__host__ __device__ __forceinline__ int attr_half_h(uint32_t a) { return (a >> 20) & 0x7FF; }
constexpr int kMaxHalfExtent = 0x7FF;

// event byte: 0x80 | orient(dir-attractive) | orient(dir-repulsive) << 3
__host__ __device__ __forceinline__ uint8_t event_code(uint32_t attr) { return (uint8_t)(0x80u | ((attr >> 3) & 0x3Fu)); }

struct PedArrays {
    long long n;
    int2* center;
    int2* gate;       // (walk_period, walk_phase)
    uint32_t* attr;
    int8_t* dir;      // decision of the current tick (k-2)
    double* score;
    uint8_t* won;     // k-3 result: wins every newly covered su
    int8_t* moved_dir; // direction moved in the previous tick, -1 none (for event clearing)
    int* order;        // ids by centre, row-major, as of the last ordering pass (valid while Ctl::order_ok); may be null
};

struct DecideParams {
    double w_static, w_kind[kKinds], goal_bias;
    int regulated;      // Regulation::Linear
    int density_radius;
    int fault_invert;
};

// Device-resident control block: lets a captured CUDA graph replay tick after tick with no
// host-side parameter patching.
struct Ctl {
    long long tick;          // SimState::tick
    long long run_base;      // tick at the start of the current sfc_run
    int error_code;          // first error wins (atomicCAS)
    int error_phase;
    long long error_tick;
    int error_x, error_y;
    double error_value;
    unsigned int drift_bits[kKinds]; // max |old - fresh| per kind as float bits (rebuild)
    int dense_count;         // k-5: tiles the scatter kernel handed to the gather kernel this tick
    int ev_written_count;    // slab mode: entries of SlabDev::ev_written
    int halo_counts[4];      // slab mode: records packed per (edge, kind): [edge*2 + kind]
    int active_count;        // k-5: tiles within reach of this tick's movers (TileMarks::list), reset by k-3
    unsigned int epoch;      // k-5: this tick's tile stamp (set by k-3, read by k-4 and k-5; never 0)
    int tiny_image;          // upload: an uploaded dynamic-image value is non-zero below 2^-92 — sums could be
                             // subnormal, so k-5 may not use flush-to-zero float reductions (sfc_k5_pairs.cu)
    int order_ok;            // PedArrays::order is a permutation of this population's ids
    int negative_zero;       // upload: a dynamic-image value is -0.0f.  The reference's k-5 adds (float)total to EVERY
                             // address once anybody moved (engine.cpp:468,524), which turns -0.0f into +0.0f; k-5 here skips
                             // untouched addresses, so the first moving tick is followed by one normalising pass
};

// Optional reference-shaped temporaries for the Inspector path (engine.hpp:172-177).
struct DebugArrays {
    int32_t* enroll_ids;     // [C*8]
    double* enroll_scores;   // [C*8]
    int32_t* winners;        // [C]
    int32_t* moved_from;     // [C]
    int32_t* moved_to;       // [C]
    uint8_t* from_mask;      // [3*C]
    uint8_t* to_mask;        // [3*C]
    long long cells;
};

struct KindTableDev {
    int fw, fh, hw, hh;
    const double* mag;     // [fh*fw]
    const uint32_t* info;  // [fh*fw]
};

struct TablesDev {
    KindTableDev k[kKinds];
    int max_hw, max_hh;
    int total_entries;
};

__device__ __forceinline__ void raise_error(Ctl* ctl, int code, int phase, int x, int y, double value) {
    if (atomicCAS(&ctl->error_code, 0, code) == 0) {
        ctl->error_phase = phase;
        ctl->error_tick = ctl->tick;
        ctl->error_x = x;
        ctl->error_y = y;
        ctl->error_value = value;
    }
}

// k-5 work list.  The su grid is cut into tiles of 32 x 8 su (tile id = tile_y * tiles_x + tile_x,
// rows counted from the slab's first owned row).  k-4 stamps every tile within field reach of a
// mover's old or new centre with the tick's epoch and appends it to `list` the first time, so the
// write-back touches only tiles that can change: its cost follows the movers, not the grid.
// In slab mode the tiles whose field region reaches into the halo rows ("edge tiles") are not
// listed — the neighbours' events arrive there as plain row copies — and are always processed.
constexpr int kMarkTileW = 32, kMarkTileH = 8;
constexpr unsigned kEpochPeriod = (1u << 16) - 1u; // stamps are erased once per period (sfc_run)
constexpr unsigned kMarkCountMax = 0xFFu;
struct TileMarks {
    unsigned* epoch; // [tiles_x * tiles_y] stamp << 16 | blocks within reach << 8 | movers within reach (saturating);
                     // stamp = tick % period + 1; block bit = 4 * (row of 8 x 4 blocks) + column
    int* list;       // [tiles_x * tiles_y]
    int tiles_x, tiles_y;
    int hw, hh;      // field reach (largest half extents over the three kinds)
    int edge_lo;     // slab mode: tile rows [0, edge_lo) and [edge_hi, tiles_y) are edge tiles
    int edge_hi;     //            (whole grid: edge_lo = 0, edge_hi = tiles_y)
};
__host__ __device__ __forceinline__ int tile_edge_count(const TileMarks& m) {
    return (m.edge_lo + (m.tiles_y - m.edge_hi)) * m.tiles_x;
}

// Contributor lists for the list-walk formulation of k-5 (sfc_k5_listwalk.cu): the offsets of the
// support grouped by the sect they feed (kind 0's sect; sect_of maps a group to kind k's sect),
// each group in list order (rank 0, 1, 2, ...), shared by the three kinds.
struct WalkLists {
    const uint32_t* meta;  // [n] (dx + 128) | (dy + 128) << 8, centre offset = mover - target
    const uint32_t* masks; // [n] orientation mask of kind k in byte k
    const double* mag;     // [kind][n]
    int n, hw, hh;
    int start[kSects + 1]; // group g = entries [start[g], start[g + 1])
    int sect_of[kKinds][kSects];
};
struct WalkListsHost {
    std::vector<uint32_t> meta, masks;
    std::vector<double> mag;
    int n = 0, hw = 0, hh = 0;
    int start[kSects + 1] = {};
    int sect_of[kKinds][kSects] = {};
};

// Tables of the pair formulation of k-5 (sfc_k5_pairs.cu), one device blob: the row-bits ->
// window-word lookup (t_bytes), then the 64 contributor entries.
struct PairTables {
    const unsigned char* blob;
    long long t_bytes;
    int fw, fh, hw, hh;
    uint32_t sect_packed[kKinds]; // sect of kind k fed by sect group g in bits [3g, 3g + 3)
};

// Tables of the large-field formulation of k-5 (sfc_k5_field.cu), one device blob: one byte
// (sect group * K + StepCache slot) per support offset, the quadrant-folded magnitude tables (distinct
// ones only), the orientation-mask word per group.
struct FieldTables {
    const unsigned char* blob;
    int tab_bytes, mag_bytes;
    int fw, fh, hw, hh;
    int ms, mag_stride;             // row stride / size of one folded magnitude table, in doubles
    int mag_of[kKinds];             // magnitude table of kind k
    uint32_t group_of_sect[kKinds]; // sect group feeding sect s of kind k in bits [3s, 3s + 3)
};

// cudaFuncAttributeMaxDynamicSharedMemorySize is state of a (function, device) pair shared by every
// engine of the process: raise it on the CURRENT device when an engine needs more, never lower it.
struct SmemGrant {
    size_t granted[64] = {};
    cudaError_t raise(const void* fn, size_t want, size_t initial = 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
        if (granted[dev] < initial) granted[dev] = initial;
        if (want <= granted[dev]) return cudaSuccess;
        const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
        if (e == cudaSuccess) granted[dev] = want;
        return e;
    }
};

// ---- launchers (defined in the .cu files) --------------------------------------------------
struct K5Launch {
    GridDev g;
    TablesDev t;
    float* dyn;
    const uint8_t* ev;
    Ctl* ctl;
    int chunk_k;
    int advance_tick; // fold "tick += 1" into the kernel (fast path)
    int ev_max;       // k-5: event-count threshold between the scatter and the gather formulation
    int* dense_list;  // k-5: tile ids for the gather kernel (k5_tile_count entries), or nullptr
    int persistent_ctas; // k-5: grid of the persistent gather kernel
    int tile_rows;       // k-5: 8 (default) or 4 rows per tile on the two-kernel path
    int scatter_ctas;    // k-5: grid of the persistent scatter kernel
    TileMarks marks;     // k-5: active-tile list written by k-4 (epoch == nullptr: process every tile)
    int window_path;     // k-5: 1 = window kernel for sparse tiles, 0 = scatter kernel
    WalkLists walk;      // k-5: merged contributor lists (meta == nullptr: the kinds do not share them)
    int listwalk;        // k-5: dense tiles go to the list-walk kernel (1) or the event-walk gather (0)
    int listwalk_only;   // k-5: the list-walk kernel is the only k-5 kernel (every / every active tile)
    int list_cap;        // k-5 gather: events one appended list may hold (0: its capacity; tests lower it)
    PairTables pairs;    // k-5: tables of the pair kernel (blob == nullptr: field not supported)
    int pairs_path;      // k-5: the pair kernel is the k-5 kernel (every / every active tile)
    int pairs_ctas[2];   // k-5: its persistent grid ([1]: the RED variant)
    int listwalk_ctas;   // k-5: persistent grid of the list-walk kernel for this engine's tables
    int window_ctas;     // k-5: ... of the window kernel
    int pairs_red;       // k-5: image += (float)total as a float reduction at the L2 (no image value can be subnormal)
    FieldTables field;   // k-5: tables of the large-field kernel (blob == nullptr: not available)
    int field_path;      // k-5: the large-field kernel is the k-5 kernel
    int field_ctas[2];   // k-5: its persistent grid ([1]: the lazy shape)
    int field_nk, field_warps; // k-5: forced kinds per walk / warps per CTA (0: chosen from the shared-memory budget)
    int field_lazy;      // k-5: partials created on first use (sparse crowds) instead of cleared per block
};
cudaError_t launch_k2_decide(cudaStream_t s, const GridDev& g, const PedArrays& p, const int* occ, const float* stat,
                             const float* dyn, uint8_t* ev, Ctl* ctl, const DecideParams& dp, const SlabDev& slab);
cudaError_t launch_k3_vote(cudaStream_t s, const GridDev& g, const PedArrays& p, const int* occ, Ctl* ctl,
                           const DecideParams& dp, const SlabDev& slab);
cudaError_t launch_k4_move(cudaStream_t s, const GridDev& g, const PedArrays& p, int* occ, uint8_t* ev, Ctl* ctl,
                           unsigned long long* moved_counts, const DebugArrays& dbg, const SlabDev& slab,
                           const TileMarks& marks);

// ---- slab halo exchange (sfc_slab.cu) --------------------------------------------------------
struct HaloRecord {   // 16 bytes: a pedestrian's decision (k-2 -> k-3) or position (k-4 -> next tick)
    int id;
    int a;            // decision: direction          position: x
    double b;         // decision: score              position: y (as an exact double)
};
// Packs records of OWNED pedestrians whose centre lies within `depth` rows of slab edge `edge`
// (0 = low-y edge, 1 = high-y edge) into buf[1..]; buf[0].id receives the count.  kind 0 = decisions,
// 1 = positions.
cudaError_t launch_halo_pack(cudaStream_t s, const GridDev& g, const PedArrays& p, Ctl* ctl, int edge, int kind,
                             int depth, HaloRecord* buf, int capacity);
cudaError_t launch_halo_unpack(cudaStream_t s, const PedArrays& p, Ctl* ctl, int kind, const HaloRecord* buf, int capacity);
cudaError_t launch_clear_events(cudaStream_t s, uint8_t* ev, Ctl* ctl, const SlabDev& slab);
cudaError_t launch_k5_writeback(cudaStream_t s, const K5Launch& a);
int k5_kernels_per_launch(const TablesDev& t, int ev_max);
long long k5_tile_count(const GridDev& g);

// rebuild / rasterize_dynamic.  mode 0: write fresh images to `out` (record layout), no compare;
// mode 1: compare with dyn and record the per-kind drift maxima in ctl; mode 2: overwrite dyn
// unless ctl holds an error.
// Rebuild check pass: tiles whose TileMarks stamp lies outside [stamp_lo, stamp_hi] — the ticks since the previous
// rebuild — are skipped (stamp_lo 0: no skipping).  The caller guarantees the stamps cover that whole span.
struct RebuildSkip {
    TileMarks marks;
    unsigned stamp_lo, stamp_hi;
};
cudaError_t launch_rebuild(cudaStream_t s, const GridDev& g, const TablesDev& t, const PedArrays& p, const int* occ,
                           float* dyn, float* out, Ctl* ctl, int mode, double tolerance, unsigned* changed = nullptr,
                           const RebuildSkip* skip = nullptr);
// `changed`: one bit per rebuild tile (rebuild_tile_count(g) bits).  Mode 1 sets the bit of every tile where a fresh value
// differs from the image bit for bit; mode 2 then skips the tiles whose bit is clear and clears the others' (nullptr: every tile).
long long rebuild_tile_count(const GridDev& g);
cudaError_t launch_drift_verdict(cudaStream_t s, Ctl* ctl, double tolerance);

// debug materialisation of the reference's temporaries
cudaError_t launch_dbg_clear(cudaStream_t s, const DebugArrays& d);
cudaError_t launch_dbg_enroll(cudaStream_t s, const GridDev& g, const PedArrays& p, const DebugArrays& d, Ctl* ctl);
cudaError_t launch_dbg_vote(cudaStream_t s, const DebugArrays& d, int fault_invert);

// layout conversion between the host's per-kind images and the interleaved record buffer
cudaError_t launch_interleave(cudaStream_t s, const float* plane, float* dyn, int kind, long long cells_begin,
                              long long cells, Ctl* ctl);
cudaError_t launch_deinterleave(cudaStream_t s, const float* dyn, float* plane, int kind, long long cells_begin,
                                long long cells);
cudaError_t launch_fill_i8(cudaStream_t s, int8_t* p, long long n, int v);
// -0.0f -> +0.0f over the dynamic images if Ctl::negative_zero is set and a tick of [first, first + ticks) moved anybody
cudaError_t launch_normalize_negative_zero(cudaStream_t s, float* dyn, long long cells, Ctl* ctl, const unsigned long long* moved_counts,
                                           long long first, long long ticks);
cudaError_t launch_occupancy_from_peds(cudaStream_t s, const GridDev& g, const PedArrays& p, int* occ);
cudaError_t launch_tick_advance(cudaStream_t s, Ctl* ctl);
// PedArrays::order from the occupancy grid of an undivided engine (chunk_counts: order_chunks(cells) ints of scratch)
long long order_chunks(long long cells);
cudaError_t launch_order_pedestrians(cudaStream_t s, const GridDev& g, const PedArrays& p, const int* occ, long long cells,
                                     int* chunk_counts, Ctl* ctl);
cudaError_t launch_static_anchor(cudaStream_t s, const GridDev& g, const KindTableDev& t, float* stat, int ax, int ay,
                                 int orientation);
cudaError_t prepare_k5_writeback(int chunk_k, const TablesDev& t);
// window formulation of k-5 (sfc_k5_window.cu)
bool k5_window_supported(const TablesDev& t);
cudaError_t prepare_k5_window(int chunk_k, const TablesDev& t, int ev_max, int sm_count, int* ctas);
cudaError_t launch_k5_window(cudaStream_t s, const K5Launch& a);
// list-walk formulation of k-5 (sfc_k5_listwalk.cu)
bool build_walk_lists(const sfc_tables& t, WalkListsHost* out);
bool k5_listwalk_supported(const WalkLists& w);
cudaError_t prepare_k5_listwalk(int chunk_k, const WalkLists& w, int sm_count, int* ctas);
cudaError_t launch_k5_listwalk(cudaStream_t s, const K5Launch& a, bool from_dense_list);
// pair formulation of k-5 (sfc_k5_pairs.cu)
bool build_pair_tables(const WalkListsHost& w, int chunk_k, PairTables* out, std::vector<unsigned char>* blob);
cudaError_t prepare_k5_pairs(const PairTables& t, int sm_count, int* ctas);
cudaError_t launch_k5_pairs(cudaStream_t s, const K5Launch& a);
// large-field formulation of k-5 (sfc_k5_field.cu)
bool build_field_tables(const WalkListsHost& w, int chunk_k, FieldTables* out, std::vector<unsigned char>* blob);
bool k5_field_supported(const FieldTables& t, int chunk_k, int nk_pref, int warps_pref);
cudaError_t prepare_k5_field(const FieldTables& t, int chunk_k, int nk_pref, int warps_pref, int sm_count, int* ctas);
cudaError_t launch_k5_field(cudaStream_t s, const K5Launch& a);
cudaError_t prepare_rebuild(const TablesDev& t);
// acceptance digest / states_identical on the device (sfc_digest.cu)
size_t digest_scratch_bytes(long long cells, long long peds);
cudaError_t launch_digest(cudaStream_t s, const int* occ, const float* dyn, const int2* center, long long cells, long long peds,
                          void* scratch, unsigned long long* out);
cudaError_t launch_compare(cudaStream_t s, const PedArrays& pa, const PedArrays& pb, const int* oa, const int* ob, const float* sa,
                           const float* sb, const float* da, const float* db, long long cells, unsigned long long* first);

} // namespace sfc
