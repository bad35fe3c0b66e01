// sfc_api.cu — the C ABI (include/socfield_cuda.h) over the sm_100a kernels.
//
// Owns the device-resident SimState, the per-tick temporaries and the CUDA stream / graph that
// sequences k-2 -> k-3 -> k-4 -> k-5 (k-1 does not exist here: nothing needs a full-grid clear).
// There is no CPU path: without a CUDA device sfc_create fails with SFC_E_NO_DEVICE.

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "sfc_internal.cuh"

using namespace sfc;

// Host <-> device bulk copies of the caller's pageable SimState buffers (std::vector storage):
// several host threads each move their slice through their own pair of pinned buffers and their
// own stream, so the CPU memcpy into pinned memory and the PCIe DMA overlap and add up across
// lanes (a single cudaMemcpy from pageable memory is bound by one core's memcpy).
struct Stager {
    static constexpr int kLanes = 8;
    static constexpr size_t kChunk = 4u << 20;
    void* pin[kLanes][2] = {};
    bool busy[kLanes][2] = {};
    cudaStream_t st[kLanes] = {};
    cudaEvent_t ev[kLanes][2] = {};
    cudaEvent_t fence = nullptr;
    bool ready = false;
};

struct sfc_engine {
    sfc_config cfg{};
    GridDev g{};
    DecideParams dp{};
    TablesDev tabs{};
    std::vector<void*> table_allocs;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
    cudaEvent_t ev_step = nullptr, ev_copy = nullptr; // slab groups: "my step is enqueued-complete" / "the halo copies into me are"

    long long cells = 0; // resident su (slab rows + halos)
    int* occ = nullptr;
    float* stat = nullptr;
    float* dyn = nullptr;
    uint8_t* ev = nullptr;
    PedArrays peds{};
    long long ped_capacity = 0;
    Ctl* ctl = nullptr;
    unsigned long long* moved_counts = nullptr;
    long long moved_capacity = 0;
    DebugArrays dbg{};
    float* stage = nullptr; // staging for layout conversion
    long long stage_cells = 0;

    cudaGraphExec_t graph = nullptr;       // one tick: k-2, k-3, k-4, k-5
    cudaGraphExec_t graph_multi = nullptr; // graph_ticks ticks back to back (launch-bound configs: one launch, not graph_ticks)
    int graph_ticks = 10;                  // SFC_GRAPH_TICKS (1: single-tick graphs only)
    bool graph_valid = false;

    // row-slab mode (multi-GPU): halo exchange buffers, [edge 0 = low-y, 1 = high-y][kind 0 = decisions, 1 = positions]
    SlabDev slab{};
    HaloRecord* halo_send[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    HaloRecord* halo_recv[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    int halo_capacity = 0; // records per buffer, header included
    int ped_half_h = 0;    // largest pedestrian half-height of the uploaded population
    int band_count = 0;    // > 1: band-swapped engine (sfc_band_run): g.row0 / g.rows move over the grid
    int band_rows = 0;     // rows of a full band (the last band may be shorter)
    std::vector<uint8_t> band_ev; // host backing of the event map (2 B per su of the whole grid)
    unsigned* rebuild_changed = nullptr; // one bit per rebuild tile: the check pass marks the tiles the commit pass must write
    int* dense_list = nullptr; // k-5 tile ids handed from the scatter to the gather kernel
    int persistent_ctas = 148 * 3;
    int k5_launches = 1;       // kernels per k-5 phase
    int k5_tile_rows = 8;  // tuning knob, SFC_K5_TILE_ROWS (8 or 4)
    int k5_scatter_ctas = 148 * 3; // persistent scatter grid; SFC_K5_SCATTER_CTAS (0 = one CTA per tile)
    int k5_event_max = 64; // tuning knob, overridable with SFC_K5_EVENT_MAX (tests force either k-5 path)
    int k5_window = 0;     // formulation in use: 0 scatter + dense gather kernels, 1 window kernel + dense gather
    int k5_window_pref = -1; // SFC_K5_PATH: "scatter" 0, "window" 1, unset -1 = by crowd density (sfc_upload)
    int k5_window_ok = 0;  // the field geometry fits the window kernel
    int k5_window_event_max = 48; // events per tile region above which the window kernel defers to the dense gather
    TileMarks marks{};     // active-tile list of k-5 (epoch stamps + list) as the kernels see it; epoch == nullptr: off
    TileMarks marks_alloc{}; // ... the allocation (the list is only switched on for sparse crowds, see sfc_upload)
    int k5_active_list = -1; // SFC_K5_ACTIVE_LIST: 0 never, 1 always, -1 by crowd density
    WalkLists walk{};        // merged contributor lists of the list-walk kernel (meta == nullptr: not available)
    int k5_listwalk = 1;     // dense tiles: list-walk kernel (SFC_K5_DENSE=gather: the event-walk gather)
    int k5_listwalk_only = 0; // the list-walk kernel alone (chosen in sfc_upload, or SFC_K5_PATH=listwalk)
    int k5_list_cap = 0;      // SFC_K5_LIST_CAP: forces the large-field gather off its one-list path (tests)
    int k5_path_pref = -1;    // SFC_K5_PATH: 0 scatter, 1 window, 2 listwalk, 3 pairs, -1 by crowd and field (sfc_upload)
    PairTables pairs{};       // tables of the pair kernel (blob == nullptr: the field geometry does not fit it)
    int k5_pairs = 0;         // the pair kernel is the k-5 kernel (chosen in sfc_upload)
    int pairs_ctas[2] = {148, 148};
    int listwalk_ctas = 148, window_ctas = 148; // persistent grids of the list-walk / window kernels for these tables
    int pairs_red = 0;        // its RED variant is exact for the uploaded state (sfc_upload)
    int pairs_red_tables = 0; // ... as far as the field magnitudes go (all >= 2^-40: sums are multiples of 2^-115)
    int pairs_red_pref = -1;  // SFC_K5_RED: 0 never, 1 always (tests), -1 when provably exact
    int negative_zero = 0;    // the uploaded images held a -0.0f (Ctl::negative_zero): runs end with the normalising pass
    double move_rate = 1.0;   // mean over the population of 1 / walk_period (upload)
    double events_per_window = 0.0; // movement events a field window sees per tick: estimated at upload, measured after every run
    long long last_rebuild_tick = -1; // ticks done at the last rebuild whose result the tile stamps have tracked since (-1: none)
    int rebuild_skip = 1;     // SFC_REBUILD_SKIP=0: every rebuild re-rasterizes every tile
    int order_pref = -1;      // per-pedestrian kernels visit the pedestrians in position order: SFC_PED_ORDER=1 / 0, -1: by grid size
    int* order_counts = nullptr; // ordering pass scratch
    long long order_tick = 0; // tick of the last ordering pass
    int k5_crowded = 0;       // crowds: the per-position list walk beats the per-event pair kernel (select_k5_path)
    FieldTables field{};      // tables of the large-field kernel (blob == nullptr: not available for these tables)
    int k5_field = 0;         // the large-field kernel is the k-5 kernel (chosen in sfc_upload)
    int field_ctas[2] = {148, 148}; // its persistent grids ([1]: the lazy shape)
    int field_nk = 0, field_warps = 0; // SFC_K5_FIELD_NK / SFC_K5_FIELD_WARPS: kinds per walk, warps per CTA (0: by shared memory)
    int field_lazy = 0;       // partials created on first use (chosen in sfc_upload from the crowd density)
    int field_lazy_pref = -1; // SFC_K5_FIELD_LAZY: 0 never, 1 always, -1 by crowd density
    int sm_count = 148;
    Stager stager;
    bool uploaded = false;
    long long tick = 0;
    sfc_counters counters{};
    double last_run_ms = 0.0;

    std::string err;
    long long err_tick = -1;
    int err_phase = 0, err_x = 0, err_y = 0;
    double err_value = 0.0;
};

namespace {

constexpr long long kOrderMinPeds = 4096; // smaller crowds are launch-bound: position order buys nothing
constexpr long long kOrderMinCells = 1ll << 28;
constexpr long long kOrderPeriod = 50;    // ticks between ordering passes
constexpr long long kStageCells = 4ll << 20; // 4 Mi su per staging chunk (128 MiB of one image)

int fail(sfc_engine* e, int code, const std::string& msg) {
    e->err = msg;
    return code;
}

int cuda_fail(sfc_engine* e, cudaError_t c, const char* what) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "CUDA error in %s: %s", what, cudaGetErrorString(c));
    e->err = buf;
    return c == cudaErrorMemoryAllocation ? SFC_E_NOMEM : SFC_E_CUDA;
}

#define SFC_CUDA(call)                                            \
    do {                                                          \
        cudaError_t c_ = (call);                                  \
        if (c_ != cudaSuccess) return cuda_fail(e, c_, #call);    \
    } while (0)

template <class T>
cudaError_t dev_alloc(T** p, long long n) {
    return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (size_t)std::max<long long>(n, 1));
}

int upload_table(sfc_engine* e, const sfc_kind_table& src, KindTableDev* dst) {
    if (src.width < 1 || src.height < 1 || src.width % 2 == 0 || src.height % 2 == 0)
        return fail(e, SFC_E_CONFIG, "field_geometry: must be odd x odd");
    if (src.width > 8000 || src.height > 8000) return fail(e, SFC_E_CONFIG, "field_geometry: support too large");
    const size_t n = (size_t)src.width * src.height;
    double* mag = nullptr;
    uint32_t* info = nullptr;
    SFC_CUDA(dev_alloc(&mag, (long long)n));
    e->table_allocs.push_back(mag);
    SFC_CUDA(dev_alloc(&info, (long long)n));
    e->table_allocs.push_back(info);
    SFC_CUDA(cudaMemcpy(mag, src.magnitude, sizeof(double) * n, cudaMemcpyHostToDevice));
    SFC_CUDA(cudaMemcpy(info, src.info, sizeof(uint32_t) * n, cudaMemcpyHostToDevice));
    dst->fw = src.width;
    dst->fh = src.height;
    dst->hw = (src.width - 1) / 2;
    dst->hh = (src.height - 1) / 2;
    dst->mag = mag;
    dst->info = info;
    return SFC_OK;
}

void free_peds(sfc_engine* e) {
    cudaFree(e->peds.center);
    cudaFree(e->peds.gate);
    cudaFree(e->peds.attr);
    cudaFree(e->peds.dir);
    cudaFree(e->peds.score);
    cudaFree(e->peds.won);
    cudaFree(e->peds.moved_dir);
    cudaFree(e->peds.order);
    e->peds = PedArrays{};
    e->ped_capacity = 0;
}

int ensure_peds(sfc_engine* e, long long n) {
    if (n <= e->ped_capacity && e->peds.center) {
        if (n != e->peds.n) e->graph_valid = false; // the captured tick holds the population size (grid sizes, PedArrays::n)
        e->peds.n = n;
        return SFC_OK;
    }
    free_peds(e);
    e->graph_valid = false;
    SFC_CUDA(dev_alloc(&e->peds.center, n));
    SFC_CUDA(dev_alloc(&e->peds.gate, n));
    SFC_CUDA(dev_alloc(&e->peds.attr, n));
    SFC_CUDA(dev_alloc(&e->peds.dir, n));
    SFC_CUDA(dev_alloc(&e->peds.score, n));
    SFC_CUDA(dev_alloc(&e->peds.won, n));
    SFC_CUDA(dev_alloc(&e->peds.moved_dir, n));
    // Position order trades the coalesced reads of the per-pedestrian arrays for neighbouring grid reads.  Measured
    // (profiles/README.md): it pays on grids far beyond the L2 and the TLB reach (config 4: k-2 299 -> 243 us, k-3 129 ->
    // 90 us) and loses where the grid is L2-resident (paper baseline: k-2 47 -> 62 us), so the size of the grid decides.
    const bool ordered = e->order_pref >= 0 ? e->order_pref != 0 : e->cells >= kOrderMinCells;
    if (ordered && n >= (e->order_pref > 0 ? 1 : kOrderMinPeds) && n <= INT_MAX) SFC_CUDA(dev_alloc(&e->peds.order, n));
    e->peds.n = n;
    e->ped_capacity = n;
    return SFC_OK;
}

// Re-list the pedestrians by position (PedArrays::order) — see order_pedestrians in sfc_ped_kernels.cu.  Row slabs
// and bands keep id order: their occupancy holds only their rows.
int enqueue_order(sfc_engine* e, long long tick) {
    if (!e->peds.order || e->slab.active || e->slab.band) return SFC_OK;
    if (!e->order_counts) SFC_CUDA(dev_alloc(&e->order_counts, order_chunks(e->cells)));
    SFC_CUDA(launch_order_pedestrians(e->stream, e->g, e->peds, e->occ, e->cells, e->order_counts, e->ctl));
    e->counters.kernel_launches += 3;
    e->order_tick = tick;
    return SFC_OK;
}

int ensure_moved(sfc_engine* e, long long ticks) {
    if (ticks <= e->moved_capacity) return SFC_OK;
    cudaFree(e->moved_counts);
    e->moved_counts = nullptr;
    e->graph_valid = false;
    const long long cap = std::max<long long>(ticks, 4096);
    SFC_CUDA(dev_alloc(&e->moved_counts, cap));
    e->moved_capacity = cap;
    return SFC_OK;
}

int ensure_stage(sfc_engine* e) {
    if (e->stage) return SFC_OK;
    e->stage_cells = std::min<long long>(e->cells, kStageCells);
    SFC_CUDA(dev_alloc(&e->stage, e->stage_cells * kSects));
    return SFC_OK;
}

bool stager_init(sfc_engine* e) {
    Stager& s = e->stager;
    if (s.ready) return true;
    if (std::getenv("SFC_NO_STAGER")) return false;
    bool ok = cudaEventCreateWithFlags(&s.fence, cudaEventDisableTiming) == cudaSuccess;
    for (int t = 0; t < Stager::kLanes && ok; ++t) {
        ok = cudaStreamCreateWithFlags(&s.st[t], cudaStreamNonBlocking) == cudaSuccess;
        for (int b = 0; b < 2 && ok; ++b)
            ok = cudaHostAlloc(&s.pin[t][b], Stager::kChunk, cudaHostAllocDefault) == cudaSuccess &&
                 cudaEventCreateWithFlags(&s.ev[t][b], cudaEventDisableTiming) == cudaSuccess;
    }
    s.ready = ok;
    return ok;
}

void stager_destroy(sfc_engine* e) {
    Stager& s = e->stager;
    for (int t = 0; t < Stager::kLanes; ++t) {
        if (s.st[t]) cudaStreamSynchronize(s.st[t]);
        for (int b = 0; b < 2; ++b) {
            if (s.pin[t][b]) cudaFreeHost(s.pin[t][b]);
            if (s.ev[t][b]) cudaEventDestroy(s.ev[t][b]);
        }
        if (s.st[t]) cudaStreamDestroy(s.st[t]);
    }
    if (s.fence) cudaEventDestroy(s.fence);
    s = Stager{};
}

// Copies `bytes` between a pageable host buffer and device memory, ordered like a copy enqueued on
// the engine's stream.  to_device: the host buffer may be reused on return and later work on the
// engine's stream sees the data.  Otherwise the host buffer holds the data on return.
cudaError_t bulk_copy(sfc_engine* e, void* dev, void* host, size_t bytes, bool to_device) {
    bool locked = false;
    if (bytes >= (1u << 20)) { // page-locked by its owner (sfc_host_pin): one DMA, no staging
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, host) == cudaSuccess) locked = attr.type == cudaMemoryTypeHost;
        else cudaGetLastError();
    }
    if (locked || bytes < (1u << 20) || !stager_init(e)) {
        cudaError_t c = to_device ? cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, e->stream)
                                  : cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, e->stream);
        if (c == cudaSuccess && !to_device) c = cudaStreamSynchronize(e->stream);
        return c;
    }
    Stager& s = e->stager;
    cudaError_t c = cudaEventRecord(s.fence, e->stream); // the lanes start after what the engine's stream holds so far
    if (c != cudaSuccess) return c;
    std::atomic<int> err{(int)cudaSuccess};
    const size_t per_lane = ((bytes + Stager::kLanes - 1) / Stager::kLanes + 255) & ~(size_t)255;
    auto lane = [&](int t) {
        auto check = [&](cudaError_t r) {
            if (r != cudaSuccess) {
                int none = (int)cudaSuccess;
                err.compare_exchange_strong(none, (int)r);
            }
            return r == cudaSuccess;
        };
        if (!check(cudaSetDevice(e->device)) || !check(cudaStreamWaitEvent(s.st[t], s.fence, 0))) return;
        const size_t begin = std::min(bytes, per_lane * t), end = std::min(bytes, per_lane * (t + 1));
        char* const d = static_cast<char*>(dev);
        char* const h = static_cast<char*>(host);
        size_t prev_off = 0, prev_n = 0;
        int prev_b = -1, i = 0;
        for (size_t off = begin; off < end; off += Stager::kChunk, ++i) {
            const int b = i & 1;
            const size_t n = std::min(Stager::kChunk, end - off);
            if (s.busy[t][b] && !check(cudaEventSynchronize(s.ev[t][b]))) return; // the buffer's last DMA is done
            if (to_device) {
                std::memcpy(s.pin[t][b], h + off, n);
                if (!check(cudaMemcpyAsync(d + off, s.pin[t][b], n, cudaMemcpyHostToDevice, s.st[t]))) return;
            } else {
                if (!check(cudaMemcpyAsync(s.pin[t][b], d + off, n, cudaMemcpyDeviceToHost, s.st[t]))) return;
            }
            if (!check(cudaEventRecord(s.ev[t][b], s.st[t]))) return;
            s.busy[t][b] = true;
            if (!to_device) { // drain the previous chunk while this one is in flight
                if (prev_b >= 0) {
                    if (!check(cudaEventSynchronize(s.ev[t][prev_b]))) return;
                    std::memcpy(h + prev_off, s.pin[t][prev_b], prev_n);
                    s.busy[t][prev_b] = false;
                }
                prev_b = b;
                prev_off = off;
                prev_n = n;
            }
        }
        if (!to_device && prev_b >= 0) {
            if (!check(cudaEventSynchronize(s.ev[t][prev_b]))) return;
            std::memcpy(h + prev_off, s.pin[t][prev_b], prev_n);
            s.busy[t][prev_b] = false;
        }
    };
    std::thread workers[Stager::kLanes - 1];
    for (int t = 1; t < Stager::kLanes; ++t) workers[t - 1] = std::thread(lane, t);
    lane(0);
    for (auto& w : workers) w.join();
    if (err.load() != (int)cudaSuccess) return (cudaError_t)err.load();
    if (to_device) { // later work on the engine's stream waits for every lane's DMA
        for (int t = 0; t < Stager::kLanes; ++t)
            for (int b = 0; b < 2; ++b)
                if (s.busy[t][b]) {
                    c = cudaStreamWaitEvent(e->stream, s.ev[t][b], 0);
                    if (c != cudaSuccess) return c;
                }
    }
    return cudaSuccess;
}

// Contiguous runs of resident rows: (first global row, first local row, row count).  The whole-grid
// engine has one; a slab has its owned rows plus up to two halo runs per side (periodic wrap) or
// fewer (closed boundary: rows beyond the grid do not exist and keep their "empty" initial value).
struct RowSeg {
    int global_row, local_row, rows;
};

std::vector<RowSeg> row_segments(const sfc_engine* e, bool owned_only) {
    std::vector<RowSeg> out;
    const GridDev& g = e->g;
    const int first = owned_only ? 0 : -g.halo, last = owned_only ? g.rows : g.rows + g.halo; // slab-relative
    int run_start = 0, run_global = 0, run_len = 0;
    for (int r = first; r < last; ++r) {
        int y = g.row0 + r;
        bool exists = true;
        if (g.closed) exists = y >= 0 && y < g.H;
        else y = emod(y, g.H);
        if (exists && run_len > 0 && y == run_global + run_len) {
            ++run_len;
            continue;
        }
        if (run_len > 0) out.push_back(RowSeg{run_global, run_start + g.halo, run_len});
        run_len = 0;
        if (exists) {
            run_start = r;
            run_global = y;
            run_len = 1;
        }
    }
    if (run_len > 0) out.push_back(RowSeg{run_global, run_start + g.halo, run_len});
    return out;
}

int ensure_debug(sfc_engine* e) {
    if (e->dbg.enroll_ids) return SFC_OK;
    const long long c = e->cells;
    SFC_CUDA(dev_alloc(&e->dbg.enroll_ids, c * 8));
    SFC_CUDA(dev_alloc(&e->dbg.enroll_scores, c * 8));
    SFC_CUDA(dev_alloc(&e->dbg.winners, c));
    SFC_CUDA(dev_alloc(&e->dbg.moved_from, c));
    SFC_CUDA(dev_alloc(&e->dbg.moved_to, c));
    SFC_CUDA(dev_alloc(&e->dbg.from_mask, c * 3));
    SFC_CUDA(dev_alloc(&e->dbg.to_mask, c * 3));
    e->dbg.cells = c;
    SFC_CUDA(launch_dbg_clear(e->stream, e->dbg));
    e->counters.kernel_launches += 1;
    return SFC_OK;
}

// Pulls the control block back and converts a device-side error into the ABI status.
int check_device_error(sfc_engine* e) {
    Ctl h;
    SFC_CUDA(cudaMemcpyAsync(&h, e->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e->stream));
    SFC_CUDA(cudaStreamSynchronize(e->stream));
    e->tick = h.tick;
    if (h.error_code == 0) return SFC_OK;
    e->err_tick = h.error_tick;
    e->err_phase = h.error_phase;
    e->err_x = h.error_x;
    e->err_y = h.error_y;
    e->err_value = h.error_value;
    char buf[256];
    if (h.error_code == SFC_E_INTEGRITY && h.error_phase == 2) {
        std::snprintf(buf, sizeof buf, "enrollment slot conflict at su (%d,%d)", h.error_x, h.error_y);
    } else if (h.error_code == SFC_E_INTEGRITY && h.error_phase == 5) {
        static const char* names[3] = {"dir-attractive", "dir-repulsive", "recurrent-repulsive"};
        std::snprintf(buf, sizeof buf, "%s image drifted by %s", names[std::clamp(h.error_x, 0, 2)],
                      std::to_string((float)h.error_value).c_str());
    } else if (h.error_phase == 6) {
        std::snprintf(buf, sizeof buf, "device error %d: halo exchange buffer overflow (%g records)", h.error_code, h.error_value);
    } else if (h.error_phase == 4) {
        std::snprintf(buf, sizeof buf, "device error %d in phase 4: event list of the slab overflowed (%g entries)", h.error_code,
                      h.error_value);
    } else {
        std::snprintf(buf, sizeof buf, "device error %d in phase %d%s (%g)", h.error_code, h.error_phase,
                      h.error_phase == 5 ? ": a rebuild tile sees more centres of one id range than its sorted list holds" : "",
                      h.error_value);
    }
    e->err = buf;
    return h.error_code;
}

K5Launch k5_args(sfc_engine* e, int advance) {
    K5Launch l;
    l.g = e->g;
    l.t = e->tabs;
    l.dyn = e->dyn;
    l.ev = e->ev;
    l.ctl = e->ctl;
    l.chunk_k = e->cfg.chunk_k;
    l.advance_tick = advance;
    l.ev_max = e->k5_window ? e->k5_window_event_max : e->k5_event_max;
    l.dense_list = e->dense_list;
    l.persistent_ctas = e->persistent_ctas;
    l.tile_rows = e->k5_tile_rows;
    l.scatter_ctas = e->k5_scatter_ctas;
    l.marks = e->marks;
    l.window_path = e->k5_window;
    l.walk = e->walk;
    l.listwalk = e->k5_listwalk;
    l.listwalk_only = e->k5_listwalk_only;
    l.list_cap = e->k5_list_cap;
    l.pairs = e->pairs;
    l.pairs_path = e->k5_pairs;
    l.pairs_ctas[0] = e->pairs_ctas[0];
    l.pairs_ctas[1] = e->pairs_ctas[1];
    l.pairs_red = e->pairs_red;
    l.field = e->field;
    l.field_path = e->k5_field;
    l.field_ctas[0] = e->field_ctas[0];
    l.field_ctas[1] = e->field_ctas[1];
    l.field_nk = e->field_nk;
    l.field_warps = e->field_warps;
    l.field_lazy = e->field_lazy;
    l.listwalk_ctas = e->listwalk_ctas;
    l.window_ctas = e->window_ctas;
    return l;
}

// Tile stamps repeat with period kEpochPeriod: erase them once per period so that a stamp left by
// a tick exactly one period ago cannot pass for the current one.
int erase_marks_if_due(sfc_engine* e, long long tick) {
    if (e->marks_alloc.epoch && tick > 0 && tick % (long long)kEpochPeriod == 0)
        SFC_CUDA(cudaMemsetAsync(e->marks_alloc.epoch, 0,
                                 sizeof(unsigned) * (size_t)e->marks_alloc.tiles_x * e->marks_alloc.tiles_y, e->stream));
    return SFC_OK;
}

int enqueue_tick_kernels(sfc_engine* e) {
    const DebugArrays none{};
    SFC_CUDA(launch_k2_decide(e->stream, e->g, e->peds, e->occ, e->stat, e->dyn, e->ev, e->ctl, e->dp, e->slab));
    SFC_CUDA(launch_k3_vote(e->stream, e->g, e->peds, e->occ, e->ctl, e->dp, e->slab));
    SFC_CUDA(launch_k4_move(e->stream, e->g, e->peds, e->occ, e->ev, e->ctl, e->moved_counts, none, e->slab, e->marks));
    SFC_CUDA(launch_k5_writeback(e->stream, k5_args(e, 1)));
    return SFC_OK;
}

int enqueue_rebuild(sfc_engine* e, long long now) { // maybe_rebuild body, engine.cpp:540-549; now = ticks done so far
    // (the commit pass only rewrites tiles where the check pass saw a fresh value differ from the image: in a sparse
    // crowd most tiles are all zero before and after)
    unsigned* const changed = e->slab.band ? nullptr : e->rebuild_changed;
    // With the tile stamps on since the previous rebuild (and not erased in between), the check pass leaves tiles alone
    // that no mover has reached since: config 4 re-rasterizes a quarter less of its 1.07e9 su.
    RebuildSkip skip{};
    const long long last = e->last_rebuild_tick, period = (long long)kEpochPeriod;
    if (e->rebuild_skip && e->marks.epoch != nullptr && last >= 0 && last < now && last / period == (now - 1) / period) {
        skip.marks = e->marks;
        skip.stamp_lo = (unsigned)(last % period) + 1u;
        skip.stamp_hi = (unsigned)((now - 1) % period) + 1u;
    }
    SFC_CUDA(launch_rebuild(e->stream, e->g, e->tabs, e->peds, e->occ, e->dyn, nullptr, e->ctl, 1, 0.0, changed, &skip));
    SFC_CUDA(launch_drift_verdict(e->stream, e->ctl, e->cfg.rebuild_tolerance));
    SFC_CUDA(launch_rebuild(e->stream, e->g, e->tabs, e->peds, e->occ, e->dyn, nullptr, e->ctl, 2, 0.0, changed));
    e->counters.kernel_launches += 3;
    e->last_rebuild_tick = changed != nullptr ? now : -1;
    return SFC_OK;
}

int capture_ticks(sfc_engine* e, int ticks, cudaGraphExec_t* out) {
    cudaGraph_t graph = nullptr;
    SFC_CUDA(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    int rc = SFC_OK;
    for (int t = 0; t < ticks && rc == SFC_OK; ++t) rc = enqueue_tick_kernels(e);
    cudaError_t c = cudaStreamEndCapture(e->stream, &graph);
    if (rc != SFC_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (c != cudaSuccess) return cuda_fail(e, c, "cudaStreamEndCapture");
    c = cudaGraphInstantiate(out, graph, 0);
    cudaGraphDestroy(graph);
    if (c != cudaSuccess) return cuda_fail(e, c, "cudaGraphInstantiate");
    return SFC_OK;
}

// The tick as CUDA graphs: every kernel reads the tick from the device-resident Ctl, so a captured
// graph replays tick after tick — and graph_ticks ticks captured back to back replay as one launch.
int build_graph(sfc_engine* e) {
    if (e->graph_valid) return SFC_OK;
    for (cudaGraphExec_t* g : {&e->graph, &e->graph_multi})
        if (*g) {
            cudaGraphExecDestroy(*g);
            *g = nullptr;
        }
    int rc = capture_ticks(e, 1, &e->graph);
    if (rc == SFC_OK && e->graph_ticks > 1) rc = capture_ticks(e, e->graph_ticks, &e->graph_multi);
    if (rc != SFC_OK) return rc;
    e->graph_valid = true;
    return SFC_OK;
}

// Packs the pedestrian attributes on the host (cheap, one pass) and enqueues the copies of the per-pedestrian
// arrays; the staging vectors must outlive the next synchronisation of the engine's stream.
int upload_peds(sfc_engine* e, const sfc_state_view* v, std::vector<int2>* gate, std::vector<uint32_t>* attr, int* max_hh_out) {
    const long long P = v->n_peds;
    gate->resize((size_t)P);
    attr->resize((size_t)P);
    int max_hh = 0;
    double rate = 0.0;
    for (long long i = 0; i < P; ++i) {
        const int hw = (v->foot_w[i] - 1) / 2, hh = (v->foot_h[i] - 1) / 2;
        if (hw > kMaxHalfExtent || hh > kMaxHalfExtent || hw < 0 || hh < 0)
            return fail(e, SFC_E_CONFIG, "footprint: pedestrian footprint exceeds the device limit (4095)");
        max_hh = std::max(max_hh, hh);
        rate += 1.0 / (double)std::max(1, v->walk_period[i]);
        (*gate)[(size_t)i] = make_int2(v->walk_period[i], v->walk_phase[i]);
        (*attr)[(size_t)i] = pack_attr(v->goal_sect[i] & 7, v->orient_attractive[i] & 7, v->orient_repulsive[i] & 7, hw, hh);
    }
    *max_hh_out = max_hh;
    e->move_rate = P > 0 ? rate / (double)P : 1.0;
    {   // movers per tick before anything has been measured: everybody whose gate is open, less the share a crowd blocks
        const double cells = std::max(1.0, (double)e->g.W * (double)e->g.H), rho = (double)P / cells;
        const double movers = (double)P * e->move_rate * std::min(1.0, 1.3 * std::max(0.0, 1.0 - rho));
        e->events_per_window = 2.0 * movers * (double)(e->walk.n + 1) / cells;
        e->k5_crowded = e->events_per_window > (double)(e->walk.n + 1) / 3.0; // (measured: 16 events per 7 x 7 window)
    }
    if (P > 0) {
        SFC_CUDA(cudaMemcpyAsync(e->peds.center, v->center_xy, sizeof(int2) * (size_t)P, cudaMemcpyHostToDevice, e->stream));
        SFC_CUDA(cudaMemcpyAsync(e->peds.gate, gate->data(), sizeof(int2) * (size_t)P, cudaMemcpyHostToDevice, e->stream));
        SFC_CUDA(cudaMemcpyAsync(e->peds.attr, attr->data(), sizeof(uint32_t) * (size_t)P, cudaMemcpyHostToDevice, e->stream));
        SFC_CUDA(cudaMemsetAsync(e->peds.dir, 0xFF, (size_t)P, e->stream));
        SFC_CUDA(cudaMemsetAsync(e->peds.moved_dir, 0xFF, (size_t)P, e->stream));
        SFC_CUDA(cudaMemsetAsync(e->peds.won, 0, (size_t)P, e->stream));
        SFC_CUDA(cudaMemsetAsync(e->peds.score, 0, sizeof(double) * (size_t)P, e->stream));
        e->counters.h2d_bytes += (int64_t)((sizeof(int2) * 2 + sizeof(uint32_t)) * P);
    }
    return SFC_OK;
}

// Chooses the k-5 formulation for a population of P pedestrians (all bit-identical; measured in
// profiles/README.md).  allow_list: the active-tile list (and the window kernel that needs it) may be used.
int select_k5_path(sfc_engine* e, long long P, bool allow_list) {
    if (e->marks_alloc.epoch) {
        // The list pays when most tiles see no mover in a tick: a mover's field box overlaps about
        // (w/32 + 1) x (h/8 + 1) tiles, every pedestrian may move.  Dense crowds skip the bookkeeping.
        const TileMarks& m = e->marks_alloc;
        const long long per_mover = (long long)((2 * m.hw + 1) / kMarkTileW + 2) * ((2 * m.hh + 1) / kMarkTileH + 2);
        const long long n_tiles = (long long)m.tiles_x * m.tiles_y;
        const bool sparse = allow_list && P * per_mover < 2 * n_tiles; // (expected share of active tiles below ~85 %)
        // Which k-5 formulation (all bit-identical; measured in profiles/README.md):
        //   sparse crowd                 -> window kernel over the active-tile list (dense tiles: list walk / gather)
        //   else, fields up to 11 x 11   -> the list-walk kernel alone: per-su cost fixed by the field area, at or
        //                                   below the scatter kernel's from corridor densities up, far below for crowds
        //   else                         -> scatter kernel (+ list walk or event-walk gather for dense tiles)
        //   fields beyond 15 x 15        -> the large-field kernel (every tile; sparse crowds: the window kernel)
        //   crowds on small fields       -> the list walk again: its cost per su is flat, the pair kernel's grows with the
        //                                   events (measured cross-over: 16 events per 7 x 7 window, profiles/k5_crossover.py)
        const bool walk_ok = e->k5_listwalk && k5_listwalk_supported(e->walk) && e->walk.n <= 128;
        const int pairs = e->pairs.blob != nullptr && (e->k5_path_pref == 3 || (e->k5_path_pref < 0 && !(e->k5_crowded && walk_ok)));
        const int window = allow_list && !pairs && e->k5_window_ok && (e->k5_path_pref == 1 || (e->k5_path_pref < 0 && sparse));
        const int field = !pairs && !window && e->field.blob != nullptr &&
                          (e->k5_path_pref == 4 || (e->k5_path_pref < 0 && e->walk.n > 224));
        const int walk_only = !pairs && !window && !field && e->k5_listwalk &&
                              (e->k5_path_pref == 2 || (e->k5_path_pref < 0 && e->walk.n <= 128));
        if (e->k5_path_pref == 4 && !field && std::getenv("SFC_K5_STRICT"))
            return fail(e, SFC_E_CONFIG, "SFC_K5_PATH=field: the large-field kernel does not support these tables / this shape");
        const bool use = allow_list && !field && (window || e->k5_active_list == 1 || (e->k5_active_list < 0 && sparse));
        // the field kernel clears its partials per block unless the crowd is thin: expected events per field window
        const double events_per_window = 2.0 * (double)P * (double)(e->walk.n + 1) / std::max(1.0, (double)e->g.W * (double)e->g.H);
        const int lazy = field && (e->field_lazy_pref >= 0 ? e->field_lazy_pref : events_per_window < 24.0);
        if (use != (e->marks.epoch != nullptr) || window != e->k5_window || walk_only != e->k5_listwalk_only || pairs != e->k5_pairs ||
            field != e->k5_field || lazy != e->field_lazy) {
            if (use != (e->marks.epoch != nullptr)) e->last_rebuild_tick = -1; // (the stamps no longer cover the span since the last rebuild)
            e->marks = use ? m : TileMarks{};
            e->k5_window = window;
            e->k5_listwalk_only = walk_only;
            e->k5_pairs = pairs;
            e->k5_field = field;
            e->field_lazy = lazy;
            e->k5_launches = (walk_only || pairs || field) ? 1 : (window ? 2 : k5_kernels_per_launch(e->tabs, e->k5_event_max));
            e->graph_valid = false;
        }
        // the tick counter may restart: forget every epoch stamp
        SFC_CUDA(cudaMemsetAsync(m.epoch, 0, sizeof(unsigned) * (size_t)n_tiles, e->stream));
    }
    return SFC_OK;
}

} // namespace

extern "C" {

int sfc_abi_version(void) { return SFC_ABI_VERSION; }

int sfc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int sfc_create(const sfc_config* cfg, const sfc_tables* tables, sfc_engine** out, char* err, size_t errlen) {
    auto report = [&](int code, const std::string& msg) {
        if (err && errlen) std::snprintf(err, errlen, "%s", msg.c_str());
        return code;
    };
    *out = nullptr;
    // Engine::Engine validation (engine.cpp:173-174), then the device-side limits
    if (!(cfg->chunk_k == 2 || cfg->chunk_k == 4 || cfg->chunk_k == 8 || cfg->chunk_k == 16))
        return report(SFC_E_CONFIG, "chunk_k: must be 2, 4, 8, or 16");
    if (cfg->density_radius < 0) return report(SFC_E_CONFIG, "density_radius: must be >= 0");
    if (cfg->width < 1) return report(SFC_E_CONFIG, "width: must be >= 1");
    if (cfg->height < 1) return report(SFC_E_CONFIG, "height: must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
        return report(SFC_E_NO_DEVICE, "no CUDA device: the socfield B200 engine has no CPU fallback");
    if (cfg->device < 0 || cfg->device >= ndev) return report(SFC_E_CONFIG, "device: ordinal out of range");

    sfc_engine* e = new (std::nothrow) sfc_engine();
    if (!e) return report(SFC_E_NOMEM, "out of host memory");
    auto bail = [&](int code) {
        const std::string msg = e->err;
        sfc_destroy(e);
        return report(code, msg);
    };
    e->cfg = *cfg;
    e->device = cfg->device;
    if (const char* knob = std::getenv("SFC_GRAPH_TICKS")) e->graph_ticks = std::clamp(std::atoi(knob), 1, 64);
    chain_configure();
    if (const char* knob = std::getenv("SFC_REBUILD_SKIP")) e->rebuild_skip = std::atoi(knob) != 0;
    if (const char* knob = std::getenv("SFC_PED_ORDER")) e->order_pref = std::atoi(knob) != 0;
    if (const char* knob = std::getenv("SFC_K5_TILE_ROWS")) e->k5_tile_rows = std::atoi(knob) == 4 ? 4 : 8;
    if (const char* knob = std::getenv("SFC_K5_PATH")) {
        const std::string path(knob);
        e->k5_path_pref = path == "window" ? 1 : (path == "listwalk" ? 2 : (path == "pairs" ? 3 : (path == "field" ? 4 : 0)));
        e->k5_window_pref = path == "window";
    }
    if (const char* knob = std::getenv("SFC_K5_DENSE")) e->k5_listwalk = std::string(knob) != "gather";
    if (const char* knob = std::getenv("SFC_K5_LIST_CAP")) e->k5_list_cap = std::atoi(knob);
    if (const char* knob = std::getenv("SFC_K5_RED")) e->pairs_red_pref = std::atoi(knob) != 0;
    if (const char* knob = std::getenv("SFC_K5_ACTIVE_LIST")) e->k5_active_list = std::atoi(knob) != 0;
    if (const char* knob = std::getenv("SFC_K5_FIELD_NK")) e->field_nk = std::atoi(knob) == 3 ? 3 : (std::atoi(knob) == 1 ? 1 : 0);
    if (const char* knob = std::getenv("SFC_K5_FIELD_WARPS")) e->field_warps = std::atoi(knob) == 16 ? 16 : (std::atoi(knob) == 8 ? 8 : (std::atoi(knob) == 4 ? 4 : 0));
    if (const char* knob = std::getenv("SFC_K5_FIELD_LAZY")) e->field_lazy_pref = std::atoi(knob) != 0;
    if (cudaSetDevice(e->device) != cudaSuccess) return bail(fail(e, SFC_E_CUDA, "cudaSetDevice failed"));
    e->g.W = cfg->width;
    e->g.H = cfg->height;
    e->g.closed = cfg->closed ? 1 : 0;
    e->g.row0 = cfg->slab_rows > 0 ? cfg->slab_row0 : 0;
    e->g.rows = cfg->slab_rows > 0 ? cfg->slab_rows : cfg->height;
    e->g.halo = 0;
    if (cfg->bands > 1) { // band-swapped engine: the slab window moves over the grid (sfc_band_run)
        if (cfg->slab_rows < 1 || cfg->slab_rows >= cfg->height || cfg->slab_row0 != 0)
            return bail(fail(e, SFC_E_CONFIG, "bands: need 1 <= slab_rows < height and slab_row0 = 0"));
        e->band_count = cfg->bands;
        e->band_rows = cfg->slab_rows;
        e->slab.band = 1;
    }
    if (e->g.rows != cfg->height) { // a proper row slab: resident rows = owned + halo on both sides
        e->slab.active = 1;
        e->g.halo = cfg->slab_halo;
        if (e->g.row0 < 0 || e->g.rows < 1 || e->g.row0 + e->g.rows > cfg->height)
            return bail(fail(e, SFC_E_CONFIG, "slab_rows: slab does not lie inside the grid"));
        if (e->g.halo < 1 || e->g.halo > e->g.rows || e->g.rows + 2 * e->g.halo > cfg->height)
            return bail(fail(e, SFC_E_CONFIG, "slab_halo: need 1 <= halo <= slab_rows and slab_rows + 2*halo <= height"));
    }
    e->dp.w_static = cfg->weight_static;
    e->dp.w_kind[0] = cfg->weight_dir_attractive;
    e->dp.w_kind[1] = cfg->weight_dir_repulsive;
    e->dp.w_kind[2] = cfg->weight_recurrent;
    e->dp.goal_bias = cfg->goal_bias;
    e->dp.regulated = cfg->regulation != 0;
    e->dp.density_radius = cfg->density_radius;
    e->dp.fault_invert = cfg->fault_invert_vote_tiebreak != 0;

    int rc = SFC_OK;
    e->tabs.max_hw = e->tabs.max_hh = 0;
    e->tabs.total_entries = 0;
    for (int k = 0; k < kKinds && rc == SFC_OK; ++k) {
        rc = upload_table(e, tables->kind[k], &e->tabs.k[k]);
        if (rc == SFC_OK) {
            e->tabs.max_hw = std::max(e->tabs.max_hw, e->tabs.k[k].hw);
            e->tabs.max_hh = std::max(e->tabs.max_hh, e->tabs.k[k].hh);
            e->tabs.total_entries += e->tabs.k[k].fw * e->tabs.k[k].fh;
        }
    }
    if (rc != SFC_OK) return bail(rc);
    {   // merged contributor lists for the list-walk kernel, when the three kinds share them
        WalkListsHost h;
        if (build_walk_lists(*tables, &h) && h.n > 0) {
            uint32_t *meta = nullptr, *masks = nullptr;
            double* mag = nullptr;
            bool ok = dev_alloc(&meta, h.n) == cudaSuccess;
            if (ok) e->table_allocs.push_back(meta);
            ok = ok && dev_alloc(&masks, h.n) == cudaSuccess;
            if (ok) e->table_allocs.push_back(masks);
            ok = ok && dev_alloc(&mag, (long long)h.n * kKinds) == cudaSuccess;
            if (ok) e->table_allocs.push_back(mag);
            ok = ok && cudaMemcpy(meta, h.meta.data(), sizeof(uint32_t) * h.meta.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
                 cudaMemcpy(masks, h.masks.data(), sizeof(uint32_t) * h.masks.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
                 cudaMemcpy(mag, h.mag.data(), sizeof(double) * h.mag.size(), cudaMemcpyHostToDevice) == cudaSuccess;
            if (!ok) return bail(fail(e, SFC_E_CUDA, "cudaMalloc / cudaMemcpy (contributor lists)"));
            e->walk.meta = meta;
            e->walk.masks = masks;
            e->walk.mag = mag;
            e->walk.n = h.n;
            e->walk.hw = h.hw;
            e->walk.hh = h.hh;
            std::memcpy(e->walk.start, h.start, sizeof h.start);
            std::memcpy(e->walk.sect_of, h.sect_of, sizeof h.sect_of);
            e->pairs_red_tables = 1;
            for (double m : h.mag)
                if (!(std::fabs(m) >= 0x1p-40 && std::fabs(m) <= 0x1p40)) e->pairs_red_tables = 0;
            std::vector<unsigned char> blob;
            PairTables pt{};
            if (build_pair_tables(h, cfg->chunk_k, &pt, &blob)) {
                unsigned char* dev = nullptr;
                ok = dev_alloc(&dev, (long long)blob.size()) == cudaSuccess;
                if (ok) e->table_allocs.push_back(dev);
                ok = ok && cudaMemcpy(dev, blob.data(), blob.size(), cudaMemcpyHostToDevice) == cudaSuccess;
                if (!ok) return bail(fail(e, SFC_E_CUDA, "cudaMalloc / cudaMemcpy (pair tables)"));
                pt.blob = dev;
                e->pairs = pt;
            }
            FieldTables ft{};
            if (cfg->chunk_k >= 2 && cfg->chunk_k <= 16 && build_field_tables(h, cfg->chunk_k, &ft, &blob)) {
                unsigned char* dev = nullptr;
                ok = dev_alloc(&dev, (long long)blob.size()) == cudaSuccess;
                if (ok) e->table_allocs.push_back(dev);
                ok = ok && cudaMemcpy(dev, blob.data(), blob.size(), cudaMemcpyHostToDevice) == cudaSuccess;
                if (!ok) return bail(fail(e, SFC_E_CUDA, "cudaMalloc / cudaMemcpy (field tables)"));
                ft.blob = dev;
                if (k5_field_supported(ft, cfg->chunk_k, e->field_nk, e->field_warps)) e->field = ft;
                else if (std::getenv("SFC_K5_STRICT")) std::fprintf(stderr, "sfc: field kernel shape unsupported (k %d nk %d warps %d)\n", cfg->chunk_k, e->field_nk, e->field_warps);
            } else if (std::getenv("SFC_K5_STRICT")) {
                std::fprintf(stderr, "sfc: field tables not buildable (n %d hw %d hh %d)\n", h.n, h.hw, h.hh);
            }
        }
    }

    auto cu = [&](cudaError_t c, const char* what) {
        if (c != cudaSuccess && rc == SFC_OK) rc = cuda_fail(e, c, what);
    };
    e->cells = (long long)(e->g.rows + 2 * e->g.halo) * e->g.W;
    cu(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cu(cudaEventCreate(&e->ev_start), "cudaEventCreate");
    cu(cudaEventCreate(&e->ev_stop), "cudaEventCreate");
    cu(dev_alloc(&e->occ, e->cells), "cudaMalloc(occupancy)");
    cu(dev_alloc(&e->stat, e->cells * kSects), "cudaMalloc(static image)");
    cu(dev_alloc(&e->dyn, e->cells * kKinds * kSects), "cudaMalloc(dynamic images)");
    cu(dev_alloc(&e->ev, e->cells * 2), "cudaMalloc(event map)");
    cu(dev_alloc(&e->ctl, 1), "cudaMalloc(ctl)");
    cu(dev_alloc(&e->dense_list, k5_tile_count(e->g)), "cudaMalloc(dense tile list)");
    {
        const long long words = (rebuild_tile_count(e->g) + 31) / 32;
        cu(dev_alloc(&e->rebuild_changed, words), "cudaMalloc(rebuild tile bits)");
        if (rc == SFC_OK) cu(cudaMemset(e->rebuild_changed, 0, sizeof(unsigned) * (size_t)std::max<long long>(words, 1)), "cudaMemset");
    }
    e->k5_window_ok = e->k5_tile_rows == kMarkTileH && k5_window_supported(e->tabs);
    if (e->k5_tile_rows == kMarkTileH) { // active-tile list: 32 x 8 su tiles over the owned rows
        TileMarks& m = e->marks_alloc;
        m.tiles_x = (e->g.W + kMarkTileW - 1) / kMarkTileW;
        m.tiles_y = (e->g.rows + kMarkTileH - 1) / kMarkTileH;
        m.hw = e->tabs.max_hw;
        m.hh = e->tabs.max_hh;
        m.edge_lo = 0;
        m.edge_hi = m.tiles_y;
        if (e->slab.active) { // tiles whose field region reaches into the halo rows
            m.edge_lo = std::min(m.tiles_y, (m.hh + kMarkTileH - 1) / kMarkTileH);
            const int v = e->g.rows - (kMarkTileH - 1) - m.hh;
            m.edge_hi = std::clamp(v <= 0 ? 0 : (v + kMarkTileH - 1) / kMarkTileH, m.edge_lo, m.tiles_y);
        }
        const long long n_tiles = (long long)m.tiles_x * m.tiles_y;
        cu(dev_alloc(&m.epoch, n_tiles), "cudaMalloc(tile epochs)");
        cu(dev_alloc(&m.list, n_tiles), "cudaMalloc(active tile list)");
        if (rc == SFC_OK) cu(cudaMemset(m.epoch, 0, sizeof(unsigned) * (size_t)n_tiles), "cudaMemset");
        // events per tile region above which nearly every address needs the exact K-slot walk:
        // about 4.5 events per field window
        const long long region = (long long)(kMarkTileW + 2 * m.hw) * (kMarkTileH + 2 * m.hh);
        const long long window = (long long)(2 * m.hw + 1) * (2 * m.hh + 1);
        e->k5_window_event_max = (int)std::clamp<long long>(9 * region / (2 * window), 8, 1 << 20);
    }
    if (const char* knob = std::getenv("SFC_K5_EVENT_MAX")) e->k5_event_max = e->k5_window_event_max = std::atoi(knob);
    if (e->slab.active && !e->slab.band) {
        const long long band = (long long)e->g.W * (2 * e->g.halo) + 1;
        e->halo_capacity = (int)std::min<long long>(band, 1 << 18);
        for (int edge = 0; edge < 2; ++edge)
            for (int kind = 0; kind < 2; ++kind) {
                cu(dev_alloc(&e->halo_send[edge][kind], e->halo_capacity), "cudaMalloc(halo send)");
                cu(dev_alloc(&e->halo_recv[edge][kind], e->halo_capacity), "cudaMalloc(halo recv)");
                if (rc == SFC_OK) {
                    cu(cudaMemset(e->halo_send[edge][kind], 0, sizeof(HaloRecord)), "cudaMemset");
                    cu(cudaMemset(e->halo_recv[edge][kind], 0, sizeof(HaloRecord)), "cudaMemset");
                }
            }
        e->slab.ev_capacity = 4ll * e->halo_capacity + 1024;
        cu(dev_alloc(&e->slab.ev_written, e->slab.ev_capacity), "cudaMalloc(event written list)");
    }
    {
        cudaDeviceProp prop{};
        if (cudaGetDeviceProperties(&prop, e->device) == cudaSuccess) {
            e->persistent_ctas = prop.multiProcessorCount * 3;
            e->sm_count = prop.multiProcessorCount;
        }
        e->k5_launches = k5_kernels_per_launch(e->tabs, e->k5_event_max);
        e->k5_scatter_ctas = 1 << 30; // one CTA per tile measured faster than a persistent grid (profiles/README.md)
        if (const char* knob = std::getenv("SFC_K5_SCATTER_CTAS")) e->k5_scatter_ctas = std::atoi(knob) > 0 ? std::atoi(knob) : (1 << 30);
    }
    if (rc != SFC_OK) return bail(rc);
    cu(cudaMemset(e->ctl, 0, sizeof(Ctl)), "cudaMemset");
    cu(cudaMemset(e->occ, 0xFF, sizeof(int) * (size_t)e->cells), "cudaMemset");
    cu(cudaMemset(e->stat, 0, sizeof(float) * (size_t)e->cells * kSects), "cudaMemset");
    cu(cudaMemset(e->dyn, 0, sizeof(float) * (size_t)e->cells * kKinds * kSects), "cudaMemset");
    cu(cudaMemset(e->ev, 0, (size_t)e->cells * 2), "cudaMemset");
    cu(prepare_k5_writeback(cfg->chunk_k, e->tabs), "cudaFuncSetAttribute(k5)");
    cu(prepare_k5_listwalk(cfg->chunk_k, e->walk, e->sm_count, &e->listwalk_ctas), "cudaFuncSetAttribute(k5 list walk)");
    if (e->k5_tile_rows != kMarkTileH || !k5_listwalk_supported(e->walk)) e->k5_listwalk = 0; // (its tiles are 32 x 8)
    if (e->k5_window_ok)
        cu(prepare_k5_window(cfg->chunk_k, e->tabs, e->k5_window_event_max, e->sm_count, &e->window_ctas), "cudaFuncSetAttribute(k5 window)");
    if (e->k5_tile_rows != kMarkTileH) e->pairs.blob = nullptr;
    if (e->pairs.blob) cu(prepare_k5_pairs(e->pairs, e->sm_count, e->pairs_ctas), "cudaFuncSetAttribute(k5 pairs)");
    if (e->field.blob)
        cu(prepare_k5_field(e->field, cfg->chunk_k, e->field_nk, e->field_warps, e->sm_count, e->field_ctas), "cudaFuncSetAttribute(k5 field)");
    cu(prepare_rebuild(e->tabs), "cudaFuncSetAttribute(rebuild)");
    if (rc == SFC_OK) rc = ensure_peds(e, 0);
    if (rc == SFC_OK) rc = ensure_moved(e, 1);
    if (rc != SFC_OK) return bail(rc);
    *out = e;
    return SFC_OK;
}

void sfc_destroy(sfc_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    if (e->graph) cudaGraphExecDestroy(e->graph);
    if (e->graph_multi) cudaGraphExecDestroy(e->graph_multi);
    for (void* p : e->table_allocs) cudaFree(p);
    free_peds(e);
    cudaFree(e->occ);
    cudaFree(e->stat);
    cudaFree(e->dyn);
    cudaFree(e->ev);
    cudaFree(e->order_counts);
    cudaFree(e->ctl);
    cudaFree(e->dense_list);
    cudaFree(e->rebuild_changed);
    stager_destroy(e);
    cudaFree(e->marks_alloc.epoch);
    cudaFree(e->marks_alloc.list);
    for (int edge = 0; edge < 2; ++edge)
        for (int kind = 0; kind < 2; ++kind) {
            cudaFree(e->halo_send[edge][kind]);
            cudaFree(e->halo_recv[edge][kind]);
        }
    cudaFree(e->slab.ev_written);
    cudaFree(e->moved_counts);
    cudaFree(e->stage);
    cudaFree(e->dbg.enroll_ids);
    cudaFree(e->dbg.enroll_scores);
    cudaFree(e->dbg.winners);
    cudaFree(e->dbg.moved_from);
    cudaFree(e->dbg.moved_to);
    cudaFree(e->dbg.from_mask);
    cudaFree(e->dbg.to_mask);
    if (e->ev_step) cudaEventDestroy(e->ev_step);
    if (e->ev_copy) cudaEventDestroy(e->ev_copy);
    if (e->ev_start) cudaEventDestroy(e->ev_start);
    if (e->ev_stop) cudaEventDestroy(e->ev_stop);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

const char* sfc_last_error(const sfc_engine* e) { return e ? e->err.c_str() : "null engine"; }

void sfc_error_detail(const sfc_engine* e, int64_t* tick, int32_t* phase, int32_t* su_x, int32_t* su_y,
                      double* value) {
    if (tick) *tick = e->err_tick;
    if (phase) *phase = e->err_phase;
    if (su_x) *su_x = e->err_x;
    if (su_y) *su_y = e->err_y;
    if (value) *value = e->err_value;
}

int sfc_upload(sfc_engine* e, const sfc_state_view* v) {
    SFC_CUDA(cudaSetDevice(e->device));
    const long long C = e->cells, P = v->n_peds;
    int rc = ensure_peds(e, P);
    if (rc != SFC_OK) return rc;
    rc = ensure_stage(e);
    if (rc != SFC_OK) return rc;
    std::vector<int2> gate;
    std::vector<uint32_t> attr;
    int max_hh = 0;
    const long long W = e->g.W;
    Ctl h{};
    h.tick = v->tick;
    h.run_base = v->tick;
    SFC_CUDA(cudaMemcpyAsync(e->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, e->stream)); // (h lives until the sync below)
    // A view without the dense arrays (occupancy / images NULL) describes a freshly seeded
    // population: the device derives them itself below (no whole-grid host state needed).
    if (!v->occupancy) SFC_CUDA(cudaMemsetAsync(e->occ, 0xFF, sizeof(int) * (size_t)C, e->stream));
    if (!v->static_image) SFC_CUDA(cudaMemsetAsync(e->stat, 0, sizeof(float) * (size_t)C * kSects, e->stream));
    for (const RowSeg& seg : row_segments(e, false)) { // the host arrays cover the whole grid
        const long long hc = (long long)seg.global_row * W, dc = (long long)seg.local_row * W, n_seg = (long long)seg.rows * W;
        if (v->occupancy) {
            SFC_CUDA(bulk_copy(e, e->occ + dc, v->occupancy + hc, sizeof(int) * (size_t)n_seg, true));
            e->counters.h2d_bytes += (int64_t)(sizeof(int) * n_seg);
        }
        if (v->static_image) {
            SFC_CUDA(bulk_copy(e, e->stat + dc * kSects, v->static_image + hc * kSects, sizeof(float) * (size_t)n_seg * kSects, true));
            e->counters.h2d_bytes += (int64_t)(sizeof(float) * n_seg * kSects);
        }
        for (int k = 0; k < kKinds; ++k) {
            if (!v->dyn_images[k]) continue;
            for (long long c0 = 0; c0 < n_seg; c0 += e->stage_cells) {
                const long long n = std::min(e->stage_cells, n_seg - c0);
                SFC_CUDA(bulk_copy(e, e->stage, v->dyn_images[k] + (hc + c0) * kSects, sizeof(float) * (size_t)n * kSects, true));
                SFC_CUDA(launch_interleave(e->stream, e->stage, e->dyn, k, dc + c0, n, e->ctl));
                e->counters.kernel_launches += 1;
                e->counters.h2d_bytes += (int64_t)(sizeof(float) * n * kSects);
            }
        }
    }
    rc = upload_peds(e, v, &gate, &attr, &max_hh);
    if (rc != SFC_OK) return rc;
    if (e->slab.active) {
        // k-4 lists the two event cells of every mover for the next tick's clear: any pedestrian may move
        if (2 * P + 16 > e->slab.ev_capacity) {
            cudaFree(e->slab.ev_written);
            e->slab.ev_written = nullptr;
            e->slab.ev_capacity = 2 * P + 16;
            SFC_CUDA(dev_alloc(&e->slab.ev_written, e->slab.ev_capacity));
        }
        e->ped_half_h = max_hh;
        e->slab.reach = max_hh + 1;
        const int need = 4 * (max_hh + 1) + (e->dp.regulated ? e->dp.density_radius : 0);
        if (e->g.halo < need || e->g.halo < e->tabs.max_hh)
            return fail(e, SFC_E_CONFIG, "slab_halo: too shallow for this population (need max(field half-height, "
                                         "4*(pedestrian half-height+1) + density radius) rows)");
    }
    SFC_CUDA(cudaMemsetAsync(e->ev, 0, (size_t)C * 2, e->stream));
    rc = select_k5_path(e, P, true);
    if (rc != SFC_OK) return rc;
    if (!v->occupancy && P > 0) { // seed_population, scenario.cpp:424
        SFC_CUDA(launch_occupancy_from_peds(e->stream, e->g, e->peds, e->occ));
        e->counters.kernel_launches += 1;
    }
    rc = enqueue_order(e, v->tick);
    if (rc != SFC_OK) return rc;
    int tiny = 0;
    SFC_CUDA(cudaMemcpyAsync(&tiny, &e->ctl->tiny_image, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    SFC_CUDA(cudaMemcpyAsync(&e->negative_zero, &e->ctl->negative_zero, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    SFC_CUDA(cudaStreamSynchronize(e->stream)); // gate/attr staging vectors die here
    {   // float reductions at the L2 flush subnormals: exact only while no image value can be one
        const int red = e->pairs_red_pref >= 0 ? e->pairs_red_pref : (e->pairs_red_tables && !tiny);
        if (red != e->pairs_red) {
            e->pairs_red = red;
            e->graph_valid = false;
        }
    }
    e->tick = v->tick;
    e->uploaded = true;
    e->last_rebuild_tick = -1;
    if (!v->dyn_images[0] || !v->dyn_images[1] || !v->dyn_images[2]) { // rasterize_dynamic, scenario.cpp:427
        if (v->dyn_images[0] || v->dyn_images[1] || v->dyn_images[2])
            return fail(e, SFC_E_STATE, "upload: give all three dynamic images or none");
        return sfc_reset_dynamic_images(e);
    }
    return SFC_OK;
}

int sfc_download(sfc_engine* e, sfc_state_view* v) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "download before upload");
    SFC_CUDA(cudaSetDevice(e->device));
    const long long P = e->peds.n;
    int rc = ensure_stage(e);
    if (rc != SFC_OK) return rc;
    const long long W = e->g.W;
    for (const RowSeg& seg : row_segments(e, true)) { // only the rows this engine owns are authoritative
        const long long hc = (long long)seg.global_row * W, dc = (long long)seg.local_row * W, n_seg = (long long)seg.rows * W;
        if (v->occupancy) {
            SFC_CUDA(bulk_copy(e, e->occ + dc, v->occupancy + hc, sizeof(int) * (size_t)n_seg, false));
            e->counters.d2h_bytes += (int64_t)(sizeof(int) * n_seg);
        }
        for (int k = 0; k < kKinds; ++k) {
            if (!v->dyn_images[k]) continue;
            for (long long c0 = 0; c0 < n_seg; c0 += e->stage_cells) {
                const long long n = std::min(e->stage_cells, n_seg - c0);
                SFC_CUDA(launch_deinterleave(e->stream, e->dyn, e->stage, k, dc + c0, n));
                // (returns with the data on the host: the staging buffer is free for the next chunk)
                SFC_CUDA(bulk_copy(e, e->stage, v->dyn_images[k] + (hc + c0) * kSects, sizeof(float) * (size_t)n * kSects, false));
                e->counters.kernel_launches += 1;
                e->counters.d2h_bytes += (int64_t)(sizeof(float) * n * kSects);
            }
        }
        if (v->static_image) {
            SFC_CUDA(bulk_copy(e, e->stat + dc * kSects, v->static_image + hc * kSects, sizeof(float) * (size_t)n_seg * kSects, false));
            e->counters.d2h_bytes += (int64_t)(sizeof(float) * n_seg * kSects);
        }
    }
    if (v->center_xy && P > 0) {
        if (!e->slab.active) {
            SFC_CUDA(cudaMemcpyAsync(v->center_xy, e->peds.center, sizeof(int2) * (size_t)P, cudaMemcpyDeviceToHost, e->stream));
        } else { // a slab only vouches for the pedestrians whose centre lies in its rows
            std::vector<int2> mine((size_t)P);
            SFC_CUDA(cudaMemcpyAsync(mine.data(), e->peds.center, sizeof(int2) * (size_t)P, cudaMemcpyDeviceToHost, e->stream));
            SFC_CUDA(cudaStreamSynchronize(e->stream));
            for (long long i = 0; i < P; ++i) {
                if (!row_owned(e->g, mine[(size_t)i].y)) continue;
                v->center_xy[2 * i] = mine[(size_t)i].x;
                v->center_xy[2 * i + 1] = mine[(size_t)i].y;
            }
        }
        e->counters.d2h_bytes += (int64_t)(sizeof(int2) * P);
    }
    rc = check_device_error(e); // also refreshes e->tick
    v->tick = e->tick;
    v->n_peds = P;
    (void)rc; // the state is valid to read even after a recorded integrity error
    return SFC_OK;
}

int sfc_run(sfc_engine* e, int64_t ticks, sfc_tick_metrics* metrics, int with_phase_times) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "run before upload");
    if (ticks <= 0) return SFC_OK;
    SFC_CUDA(cudaSetDevice(e->device));
    int rc = ensure_moved(e, ticks);
    if (rc != SFC_OK) return rc;
    SFC_CUDA(cudaMemsetAsync(e->moved_counts, 0, sizeof(unsigned long long) * (size_t)ticks, e->stream));
    const long long base = e->tick;
    SFC_CUDA(cudaMemcpyAsync(&e->ctl->run_base, &base, sizeof(long long), cudaMemcpyHostToDevice, e->stream));
    const long long interval = e->cfg.rebuild_interval;

    std::vector<cudaEvent_t> evs;
    if (with_phase_times) {
        evs.resize((size_t)ticks * 5 + 1);
        for (auto& x : evs) SFC_CUDA(cudaEventCreate(&x));
    } else {
        rc = build_graph(e);
        if (rc != SFC_OK) return rc;
    }
    SFC_CUDA(cudaEventRecord(e->ev_start, e->stream));
    for (long long t = 0; t < ticks;) {
        rc = erase_marks_if_due(e, base + t);
        if (rc != SFC_OK) return rc;
        long long done = 1;
        if (with_phase_times) {
            const DebugArrays none{};
            cudaEvent_t* ev = &evs[(size_t)t * 5];
            SFC_CUDA(cudaEventRecord(ev[0], e->stream));
            // k-1 has no device work: its slot reports zero
            SFC_CUDA(cudaEventRecord(ev[1], e->stream));
            SFC_CUDA(launch_k2_decide(e->stream, e->g, e->peds, e->occ, e->stat, e->dyn, e->ev, e->ctl, e->dp, e->slab));
            SFC_CUDA(cudaEventRecord(ev[2], e->stream));
            SFC_CUDA(launch_k3_vote(e->stream, e->g, e->peds, e->occ, e->ctl, e->dp, e->slab));
            SFC_CUDA(cudaEventRecord(ev[3], e->stream));
            SFC_CUDA(launch_k4_move(e->stream, e->g, e->peds, e->occ, e->ev, e->ctl, e->moved_counts, none, e->slab, e->marks));
            SFC_CUDA(cudaEventRecord(ev[4], e->stream));
            SFC_CUDA(launch_k5_writeback(e->stream, k5_args(e, 1)));
            if (t == ticks - 1) SFC_CUDA(cudaEventRecord(evs[(size_t)ticks * 5], e->stream));
        } else {
            // graph_ticks ticks in one launch when no rebuild and no stamp erasure falls strictly inside them
            const long long n = e->graph_ticks;
            bool multi = e->graph_multi != nullptr && t + n <= ticks;
            if (multi && interval > 0 && (base + t) % interval + n > interval) multi = false;
            if (multi && e->marks_alloc.epoch && (base + t) / (long long)kEpochPeriod != (base + t + n - 1) / (long long)kEpochPeriod) multi = false;
            if (multi) done = n;
            SFC_CUDA(cudaGraphLaunch(multi ? e->graph_multi : e->graph, e->stream));
            e->counters.graph_launches += 1;
        }
        e->counters.kernel_launches += done * (3 + e->k5_launches);
        t += done;
        if (interval > 0 && (base + t) % interval == 0) {
            rc = enqueue_rebuild(e, base + t);
            if (rc != SFC_OK) return rc;
        }
        if (base + t - e->order_tick >= kOrderPeriod) {
            rc = enqueue_order(e, base + t);
            if (rc != SFC_OK) return rc;
        }
    }
    if (e->negative_zero && !e->slab.active) { // (the reference's k-5 turns every -0.0f into +0.0f once anybody moved)
        SFC_CUDA(launch_normalize_negative_zero(e->stream, e->dyn, e->cells, e->ctl, e->moved_counts, 0, ticks));
        e->counters.kernel_launches += 2;
    }
    SFC_CUDA(cudaEventRecord(e->ev_stop, e->stream));
    std::vector<unsigned long long> moved;
    if (metrics) {
        moved.resize((size_t)ticks);
        SFC_CUDA(cudaMemcpyAsync(moved.data(), e->moved_counts, sizeof(unsigned long long) * (size_t)ticks,
                                 cudaMemcpyDeviceToHost, e->stream));
    }
    unsigned long long last_moved = 0;
    SFC_CUDA(cudaMemcpyAsync(&last_moved, e->moved_counts + (ticks - 1), sizeof last_moved, cudaMemcpyDeviceToHost, e->stream));
    rc = check_device_error(e); // synchronises
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e->ev_start, e->ev_stop);
    e->last_run_ms = ms;
    if (rc == SFC_OK && !e->slab.active && e->k5_path_pref < 0) {
        // The crowd tells which small-field kernel suits it: re-choose between runs from the movers of the last tick
        // (with hysteresis around the measured cross-over; both kernels give the same bits).
        e->events_per_window = 2.0 * (double)last_moved * (double)(e->walk.n + 1) / std::max(1.0, (double)e->g.W * (double)e->g.H);
        const double cross = (double)(e->walk.n + 1) / 3.0; // the walk's cost grows with the positions, the pairs' with the events
        const int crowded = e->k5_crowded ? e->events_per_window > 0.8 * cross : e->events_per_window > 1.2 * cross;
        if (crowded != e->k5_crowded) {
            e->k5_crowded = crowded;
            const int rc2 = select_k5_path(e, e->peds.n, true);
            if (rc2 != SFC_OK) return rc2;
        }
    }
    if (metrics) {
        for (long long t = 0; t < ticks; ++t) {
            sfc_tick_metrics& m = metrics[t];
            m.tick = base + t;
            m.moved = (int64_t)moved[(size_t)t];
            for (int p = 0; p < 5; ++p) m.phase_us[p] = 0;
            m.wall_us = (int64_t)(ms * 1000.0 / (double)ticks);
            if (with_phase_times) {
                for (int p = 0; p < 5; ++p) {
                    float pm = 0.0f;
                    cudaEvent_t next = p < 4 ? evs[(size_t)t * 5 + p + 1]
                                             : (t + 1 < ticks ? evs[(size_t)(t + 1) * 5] : evs[(size_t)ticks * 5]);
                    cudaEventElapsedTime(&pm, evs[(size_t)t * 5 + p], next);
                    m.phase_us[p] = (int64_t)(pm * 1000.0f);
                }
                m.wall_us = m.phase_us[0] + m.phase_us[1] + m.phase_us[2] + m.phase_us[3] + m.phase_us[4];
            }
        }
    }
    for (auto& x : evs) cudaEventDestroy(x);
    return rc;
}

int sfc_phase(sfc_engine* e, int phase, int64_t* moved) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "phase before upload");
    SFC_CUDA(cudaSetDevice(e->device));
    int rc = ensure_debug(e);
    if (rc != SFC_OK) return rc;
    switch (phase) {
        case 1: {
            const long long base = e->tick;
            SFC_CUDA(cudaMemcpyAsync(&e->ctl->run_base, &base, sizeof(long long), cudaMemcpyHostToDevice, e->stream));
            SFC_CUDA(cudaMemsetAsync(e->moved_counts, 0, sizeof(unsigned long long), e->stream));
            SFC_CUDA(launch_dbg_clear(e->stream, e->dbg));
            e->counters.kernel_launches += 1;
            break;
        }
        case 2:
            SFC_CUDA(launch_k2_decide(e->stream, e->g, e->peds, e->occ, e->stat, e->dyn, e->ev, e->ctl, e->dp, e->slab));
            SFC_CUDA(launch_dbg_enroll(e->stream, e->g, e->peds, e->dbg, e->ctl));
            e->counters.kernel_launches += 2;
            break;
        case 3:
            rc = erase_marks_if_due(e, e->tick);
            if (rc != SFC_OK) return rc;
            SFC_CUDA(launch_k3_vote(e->stream, e->g, e->peds, e->occ, e->ctl, e->dp, e->slab));
            SFC_CUDA(launch_dbg_vote(e->stream, e->dbg, e->dp.fault_invert));
            e->counters.kernel_launches += 2;
            break;
        case 4:
            SFC_CUDA(launch_k4_move(e->stream, e->g, e->peds, e->occ, e->ev, e->ctl, e->moved_counts, e->dbg, e->slab, e->marks));
            e->counters.kernel_launches += 1;
            break;
        case 5:
            SFC_CUDA(launch_k5_writeback(e->stream, k5_args(e, 0)));
            e->counters.kernel_launches += e->k5_launches;
            if (e->negative_zero && !e->slab.active) {
                SFC_CUDA(launch_normalize_negative_zero(e->stream, e->dyn, e->cells, e->ctl, e->moved_counts, 0, 1));
                e->counters.kernel_launches += 2;
            }
            break;
        case 6: {
            SFC_CUDA(launch_tick_advance(e->stream, e->ctl));
            e->counters.kernel_launches += 1;
            const long long interval = e->cfg.rebuild_interval;
            if (interval > 0 && (e->tick + 1) % interval == 0) {
                rc = enqueue_rebuild(e, e->tick + 1);
                if (rc != SFC_OK) return rc;
            }
            break;
        }
        default: return fail(e, SFC_E_STATE, "phase must be 1..6");
    }
    if (moved) {
        unsigned long long m = 0;
        SFC_CUDA(cudaMemcpyAsync(&m, e->moved_counts, sizeof m, cudaMemcpyDeviceToHost, e->stream));
        SFC_CUDA(cudaStreamSynchronize(e->stream));
        *moved = (int64_t)m;
    }
    return check_device_error(e);
}

int sfc_download_temporaries(sfc_engine* e, sfc_temporaries* out) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "download before upload");
    SFC_CUDA(cudaSetDevice(e->device));
    int rc = ensure_debug(e);
    if (rc != SFC_OK) return rc;
    const long long C = e->cells, P = e->peds.n;
    SFC_CUDA(cudaStreamSynchronize(e->stream));
    if (out->decisions && P > 0) {
        std::vector<int8_t> d((size_t)P);
        SFC_CUDA(cudaMemcpy(d.data(), e->peds.dir, (size_t)P, cudaMemcpyDeviceToHost));
        for (long long i = 0; i < P; ++i) out->decisions[i] = d[(size_t)i];
    }
    if (out->decision_scores && P > 0)
        SFC_CUDA(cudaMemcpy(out->decision_scores, e->peds.score, sizeof(double) * (size_t)P, cudaMemcpyDeviceToHost));
    if (out->enroll_ids) SFC_CUDA(cudaMemcpy(out->enroll_ids, e->dbg.enroll_ids, sizeof(int) * (size_t)C * 8, cudaMemcpyDeviceToHost));
    if (out->enroll_scores)
        SFC_CUDA(cudaMemcpy(out->enroll_scores, e->dbg.enroll_scores, sizeof(double) * (size_t)C * 8, cudaMemcpyDeviceToHost));
    if (out->winners) SFC_CUDA(cudaMemcpy(out->winners, e->dbg.winners, sizeof(int) * (size_t)C, cudaMemcpyDeviceToHost));
    if (out->moved_from) SFC_CUDA(cudaMemcpy(out->moved_from, e->dbg.moved_from, sizeof(int) * (size_t)C, cudaMemcpyDeviceToHost));
    if (out->moved_to) SFC_CUDA(cudaMemcpy(out->moved_to, e->dbg.moved_to, sizeof(int) * (size_t)C, cudaMemcpyDeviceToHost));
    if (out->from_mask) SFC_CUDA(cudaMemcpy(out->from_mask, e->dbg.from_mask, (size_t)C * 3, cudaMemcpyDeviceToHost));
    if (out->to_mask) SFC_CUDA(cudaMemcpy(out->to_mask, e->dbg.to_mask, (size_t)C * 3, cudaMemcpyDeviceToHost));
    return SFC_OK;
}

int sfc_decide(sfc_engine* e, int64_t ped, int32_t* direction, double* score) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "decide before upload");
    if (ped < 0 || ped >= e->peds.n) return fail(e, SFC_E_STATE, "pedestrian index out of range");
    SFC_CUDA(cudaSetDevice(e->device));
    SFC_CUDA(launch_k2_decide(e->stream, e->g, e->peds, e->occ, e->stat, e->dyn, e->ev, e->ctl, e->dp, e->slab));
    e->counters.kernel_launches += 1;
    int8_t d = -1;
    SFC_CUDA(cudaMemcpyAsync(&d, e->peds.dir + ped, 1, cudaMemcpyDeviceToHost, e->stream));
    SFC_CUDA(cudaMemcpyAsync(score, e->peds.score + ped, sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    SFC_CUDA(cudaStreamSynchronize(e->stream));
    *direction = d;
    return SFC_OK;
}

int sfc_rasterize_dynamic(sfc_engine* e, float* out[SFC_KINDS]) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "rasterize before upload");
    SFC_CUDA(cudaSetDevice(e->device));
    int rc = ensure_stage(e);
    if (rc != SFC_OK) return rc;
    float* scratch = nullptr;
    SFC_CUDA(dev_alloc(&scratch, e->cells * kKinds * kSects));
    cudaError_t c = launch_rebuild(e->stream, e->g, e->tabs, e->peds, e->occ, e->dyn, scratch, e->ctl, 0, 0.0);
    e->counters.kernel_launches += 1;
    for (int k = 0; k < kKinds && c == cudaSuccess; ++k) {
        for (long long c0 = 0; c0 < e->cells && c == cudaSuccess; c0 += e->stage_cells) {
            const long long n = std::min(e->stage_cells, e->cells - c0);
            c = launch_deinterleave(e->stream, scratch, e->stage, k, c0, n);
            if (c == cudaSuccess)
                c = cudaMemcpyAsync(out[k] + c0 * kSects, e->stage, sizeof(float) * (size_t)n * kSects, cudaMemcpyDeviceToHost, e->stream);
            if (c == cudaSuccess) c = cudaStreamSynchronize(e->stream);
            e->counters.kernel_launches += 1;
        }
    }
    cudaFree(scratch);
    if (c != cudaSuccess) return cuda_fail(e, c, "sfc_rasterize_dynamic");
    return check_device_error(e);
}

int sfc_reset_dynamic_images(sfc_engine* e) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "rasterize before upload");
    SFC_CUDA(cudaSetDevice(e->device));
    SFC_CUDA(launch_rebuild(e->stream, e->g, e->tabs, e->peds, e->occ, e->dyn, nullptr, e->ctl, 2, 0.0));
    e->counters.kernel_launches += 1;
    return check_device_error(e);
}

int sfc_rasterize_static(sfc_engine* e, int32_t n_tables, const sfc_kind_table* tables, int64_t n_anchors,
                         const sfc_anchor* anchors, const float* base, float* out) {
    SFC_CUDA(cudaSetDevice(e->device));
    std::vector<KindTableDev> dev((size_t)std::max(n_tables, 1));
    const size_t first_alloc = e->table_allocs.size();
    int rc = SFC_OK;
    for (int t = 0; t < n_tables && rc == SFC_OK; ++t) rc = upload_table(e, tables[t], &dev[(size_t)t]);
    if (rc == SFC_OK) {
        cudaError_t c = base ? cudaMemcpyAsync(e->stat, base, sizeof(float) * (size_t)e->cells * kSects,
                                               cudaMemcpyHostToDevice, e->stream)
                             : cudaMemsetAsync(e->stat, 0, sizeof(float) * (size_t)e->cells * kSects, e->stream);
        for (int64_t i = 0; i < n_anchors && c == cudaSuccess; ++i) { // list order = stream order
            if (anchors[i].table < 0 || anchors[i].table >= n_tables) {
                rc = fail(e, SFC_E_CONFIG, "anchor: table index out of range");
                break;
            }
            c = launch_static_anchor(e->stream, e->g, dev[(size_t)anchors[i].table], e->stat, anchors[i].x, anchors[i].y,
                                     anchors[i].orientation);
            e->counters.kernel_launches += 1;
        }
        if (c == cudaSuccess && out && rc == SFC_OK)
            c = cudaMemcpyAsync(out, e->stat, sizeof(float) * (size_t)e->cells * kSects, cudaMemcpyDeviceToHost, e->stream);
        if (c == cudaSuccess) c = cudaStreamSynchronize(e->stream);
        if (c != cudaSuccess) rc = cuda_fail(e, c, "sfc_rasterize_static");
    }
    for (size_t i = first_alloc; i < e->table_allocs.size(); ++i) cudaFree(e->table_allocs[i]);
    e->table_allocs.resize(first_alloc);
    return rc;
}

// ---- row slabs (multi-GPU) -------------------------------------------------------------------

int sfc_slab_halo_rows(int field_half_h, int ped_half_h, int density_radius_if_regulated) {
    return std::max(field_half_h, 4 * (ped_half_h + 1) + density_radius_if_regulated);
}

static bool slab_has_neighbour(const sfc_engine* e, int edge) {
    if (!e->g.closed) return true;
    return edge == 0 ? e->g.row0 > 0 : e->g.row0 + e->g.rows < e->g.H;
}

int sfc_slab_step(sfc_engine* e, int step) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "slab step before upload");
    if (!e->slab.active) return fail(e, SFC_E_STATE, "slab step on a whole-grid engine");
    SFC_CUDA(cudaSetDevice(e->device));
    const DebugArrays none{};
    const int depth = std::min(e->g.halo + e->ped_half_h, e->g.rows);
    switch (step) {
        case 0: // retire last tick's events, decide, publish the decisions of my boundary pedestrians
            SFC_CUDA(launch_clear_events(e->stream, e->ev, e->ctl, e->slab));
            SFC_CUDA(launch_k2_decide(e->stream, e->g, e->peds, e->occ, e->stat, e->dyn, e->ev, e->ctl, e->dp, e->slab));
            for (int edge = 0; edge < 2; ++edge)
                SFC_CUDA(launch_halo_pack(e->stream, e->g, e->peds, e->ctl, edge, 0, depth, e->halo_send[edge][0], e->halo_capacity));
            e->counters.kernel_launches += 7;
            break;
        case 1: { // adopt the neighbours' decisions, vote, move, publish the positions of my boundary pedestrians
            const int rc = erase_marks_if_due(e, e->tick);
            if (rc != SFC_OK) return rc;
        }
            for (int edge = 0; edge < 2; ++edge)
                if (slab_has_neighbour(e, edge))
                    SFC_CUDA(launch_halo_unpack(e->stream, e->peds, e->ctl, 0, e->halo_recv[edge][0], e->halo_capacity));
            SFC_CUDA(launch_k3_vote(e->stream, e->g, e->peds, e->occ, e->ctl, e->dp, e->slab));
            SFC_CUDA(launch_k4_move(e->stream, e->g, e->peds, e->occ, e->ev, e->ctl, e->moved_counts, none, e->slab, e->marks));
            for (int edge = 0; edge < 2; ++edge)
                SFC_CUDA(launch_halo_pack(e->stream, e->g, e->peds, e->ctl, edge, 1, depth, e->halo_send[edge][1], e->halo_capacity));
            e->counters.kernel_launches += 8;
            break;
        case 2: { // adopt the neighbours' positions (their rows of occupancy / events arrived as plain copies), write back
            for (int edge = 0; edge < 2; ++edge)
                if (slab_has_neighbour(e, edge))
                    SFC_CUDA(launch_halo_unpack(e->stream, e->peds, e->ctl, 1, e->halo_recv[edge][1], e->halo_capacity));
            SFC_CUDA(launch_k5_writeback(e->stream, k5_args(e, 1)));
            e->counters.kernel_launches += 2 + e->k5_launches;
            const long long interval = e->cfg.rebuild_interval;
            if (interval > 0 && (e->tick + 1) % interval == 0) {
                const int rc = enqueue_rebuild(e, e->tick + 1);
                if (rc != SFC_OK) return rc;
            }
            e->tick += 1; // host shadow; the device counter advanced inside k-5
            break;
        }
        default: return fail(e, SFC_E_STATE, "slab step must be 0, 1 or 2");
    }
    return SFC_OK;
}

int sfc_slab_buffer(sfc_engine* e, int kind, int edge, int recv, void** ptr, size_t* bytes) {
    if (!e->slab.active || edge < 0 || edge > 1 || kind < 0 || kind > 3) return fail(e, SFC_E_STATE, "no such halo buffer");
    const long long W = e->g.W, halo = e->g.halo, rows = e->g.rows;
    if (kind < 2) {
        *ptr = recv ? e->halo_recv[edge][kind] : e->halo_send[edge][kind];
        *bytes = sizeof(HaloRecord) * (size_t)e->halo_capacity;
        return SFC_OK;
    }
    // dense rows: send = my first / last `halo` owned rows, receive = the halo rows beyond that edge
    const long long send_row = edge == 0 ? halo : rows;           // local row index (owned rows start at `halo`)
    const long long recv_row = edge == 0 ? 0 : halo + rows;
    const long long row = recv ? recv_row : send_row;
    if (kind == 2) {
        *ptr = e->occ + row * W;
        *bytes = sizeof(int) * (size_t)(halo * W);
    } else {
        *ptr = e->ev + 2 * row * W;
        *bytes = (size_t)(2 * halo * W);
    }
    return SFC_OK;
}

void* sfc_stream(sfc_engine* e) { return e ? static_cast<void*>(e->stream) : nullptr; }

int sfc_host_pin(const void* ptr, size_t bytes) {
    if (!ptr || bytes == 0) return -1;
    const cudaError_t c = cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterPortable);
    if (c != cudaSuccess) {
        cudaGetLastError(); // (not sticky; the caller falls back to the staged copy)
        return -1;
    }
    return 0;
}

int sfc_host_unpin(const void* ptr) {
    if (!ptr) return -1;
    const cudaError_t c = cudaHostUnregister(const_cast<void*>(ptr));
    if (c != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return 0;
}

int sfc_slab_finish(sfc_engine* e, int64_t first_tick, int64_t ticks, int64_t* moved) {
    SFC_CUDA(cudaSetDevice(e->device));
    std::vector<unsigned long long> m((size_t)std::max<int64_t>(ticks, 0));
    if (ticks > 0 && moved) {
        SFC_CUDA(cudaMemcpyAsync(m.data(), e->moved_counts + first_tick, sizeof(unsigned long long) * (size_t)ticks,
                                 cudaMemcpyDeviceToHost, e->stream));
    }
    const int rc = check_device_error(e);
    if (moved)
        for (int64_t t = 0; t < ticks; ++t) moved[t] = (int64_t)m[(size_t)t];
    return rc;
}

int sfc_slab_begin(sfc_engine* e, int64_t ticks) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "slab run before upload");
    SFC_CUDA(cudaSetDevice(e->device));
    const int rc = ensure_moved(e, ticks);
    if (rc != SFC_OK) return rc;
    SFC_CUDA(cudaMemsetAsync(e->moved_counts, 0, sizeof(unsigned long long) * (size_t)std::max<int64_t>(ticks, 1), e->stream));
    const long long base = e->tick;
    SFC_CUDA(cudaMemcpyAsync(&e->ctl->run_base, &base, sizeof(long long), cudaMemcpyHostToDevice, e->stream));
    SFC_CUDA(cudaStreamSynchronize(e->stream));
    return SFC_OK;
}

// Single-process driver for N slab engines (same or different devices): the halo exchange is a set
// of peer copies between the engines' buffers.  The multi-process path (one rank per GPU,
// torch.distributed / NCCL send-recv on the same buffers) lives in paper_1803_04782_b200/slabs.py.
int sfc_group_run(sfc_engine** engines, int n, int64_t ticks, sfc_tick_metrics* metrics) {
    if (n < 1) return SFC_E_STATE;
    sfc_engine* e0 = engines[0];
    if (ticks <= 0) return SFC_OK;
    const long long base = e0->tick;
    for (int i = 0; i < n; ++i) {
        const int rc = sfc_slab_begin(engines[i], ticks);
        if (rc != SFC_OK) return rc;
    }
    // Stream-ordered: the host only enqueues.  A copy into slab j waits (event) for the sending slab's
    // step; a slab's next step waits for the copies into it (same stream) and for the copies its
    // neighbours took FROM it (their "copies enqueued" events) — nothing blocks the host until finish.
    for (int i = 0; i < n; ++i) {
        sfc_engine* e = engines[i];
        cudaSetDevice(e->device);
        if (!e->ev_step && cudaEventCreateWithFlags(&e->ev_step, cudaEventDisableTiming) != cudaSuccess)
            return cuda_fail(e0, cudaGetLastError(), "cudaEventCreate(slab step)");
        if (!e->ev_copy && cudaEventCreateWithFlags(&e->ev_copy, cudaEventDisableTiming) != cudaSuccess)
            return cuda_fail(e0, cudaGetLastError(), "cudaEventCreate(slab copy)");
    }
    auto neighbour_of = [&](int i, int edge) { return engines[(i + (edge == 0 ? n - 1 : 1)) % n]; };
    auto exchange = [&](int kind) -> int { // my edge -> the facing edge of the ring neighbour, on the neighbour's stream
        for (int i = 0; i < n; ++i) {
            sfc_engine* e = engines[i];
            for (int edge = 0; edge < 2; ++edge) {
                if (!slab_has_neighbour(e, edge)) continue;
                sfc_engine* nb = neighbour_of(i, edge);
                void *src = nullptr, *dst = nullptr;
                size_t sb = 0, db = 0;
                int rc = sfc_slab_buffer(e, kind, edge, 0, &src, &sb);
                if (rc == SFC_OK) rc = sfc_slab_buffer(nb, kind, 1 - edge, 1, &dst, &db);
                if (rc != SFC_OK || sb != db) return fail(e, SFC_E_STATE, "halo buffers of neighbouring slabs do not match");
                cudaSetDevice(nb->device);
                cudaError_t c = cudaStreamWaitEvent(nb->stream, e->ev_step, 0);
                if (c == cudaSuccess) c = cudaMemcpyPeerAsync(dst, nb->device, src, e->device, sb, nb->stream);
                if (c != cudaSuccess) return cuda_fail(e, c, "cudaMemcpyPeerAsync(halo)");
            }
        }
        return SFC_OK;
    };
    for (int64_t t = 0; t < ticks; ++t) {
        for (int step = 0; step < 3; ++step) {
            for (int i = 0; i < n; ++i) {
                const int rc = sfc_slab_step(engines[i], step);
                if (rc != SFC_OK) return rc;
                const cudaError_t c = cudaEventRecord(engines[i]->ev_step, engines[i]->stream);
                if (c != cudaSuccess) return cuda_fail(e0, c, "cudaEventRecord(slab step)");
            }
            if (step == 2) continue;
            for (int kind = (step == 0 ? 0 : 1); kind <= (step == 0 ? 0 : 3); ++kind) {
                const int rc = exchange(kind);
                if (rc != SFC_OK) return rc;
            }
            for (int i = 0; i < n; ++i) {
                cudaSetDevice(engines[i]->device);
                const cudaError_t c = cudaEventRecord(engines[i]->ev_copy, engines[i]->stream);
                if (c != cudaSuccess) return cuda_fail(e0, c, "cudaEventRecord(halo copies)");
            }
            for (int i = 0; i < n; ++i) // my next step may overwrite what the neighbours are still reading
                for (int edge = 0; edge < 2; ++edge) {
                    if (!slab_has_neighbour(engines[i], edge)) continue;
                    cudaSetDevice(engines[i]->device);
                    const cudaError_t c = cudaStreamWaitEvent(engines[i]->stream, neighbour_of(i, edge)->ev_copy, 0);
                    if (c != cudaSuccess) return cuda_fail(e0, c, "cudaStreamWaitEvent(halo copies)");
                }
        }
    }
    int status = SFC_OK;
    std::vector<int64_t> moved((size_t)ticks), total((size_t)ticks, 0);
    for (int i = 0; i < n; ++i) {
        const int rc = sfc_slab_finish(engines[i], 0, ticks, moved.data());
        if (rc != SFC_OK && status == SFC_OK) {
            status = rc;
            if (engines[i] != e0) { // surface the failing slab's diagnosis on the handle the caller inspects
                e0->err = engines[i]->err;
                e0->err_tick = engines[i]->err_tick;
                e0->err_phase = engines[i]->err_phase;
                e0->err_value = engines[i]->err_value;
            }
        }
        for (int64_t t = 0; t < ticks; ++t) total[(size_t)t] += moved[(size_t)t];
    }
    if (metrics) {
        for (int64_t t = 0; t < ticks; ++t) {
            metrics[t] = sfc_tick_metrics{};
            metrics[t].tick = base + t;
            metrics[t].moved = total[(size_t)t];
        }
    }
    return status;
}

// ---- band-swapped pass (state larger than device memory) --------------------------------------

namespace {

enum { kBandOcc = 1, kBandStat = 2, kBandDyn = 4, kBandEv = 8 };

bool band_window(sfc_engine* e, int b) {
    e->g.row0 = b * e->band_rows;
    e->g.rows = std::min(e->band_rows, e->g.H - e->g.row0);
    return e->g.rows > 0;
}

// Host -> device copy of the current window's rows (owned rows only, or owned + halo).  Rows beyond a
// closed grid do not exist: occupancy "empty", no events there.
int band_load(sfc_engine* e, const sfc_state_view* v, int what, bool owned_only) {
    const long long W = e->g.W, C = (long long)(e->g.rows + 2 * e->g.halo) * W;
    if (what & kBandOcc) SFC_CUDA(cudaMemsetAsync(e->occ, 0xFF, sizeof(int) * (size_t)C, e->stream));
    if (what & kBandEv) SFC_CUDA(cudaMemsetAsync(e->ev, 0, (size_t)C * 2, e->stream));
    for (const RowSeg& seg : row_segments(e, owned_only)) {
        const long long hc = (long long)seg.global_row * W, dc = (long long)seg.local_row * W, n_seg = (long long)seg.rows * W;
        if (what & kBandOcc) {
            SFC_CUDA(bulk_copy(e, e->occ + dc, v->occupancy + hc, sizeof(int) * (size_t)n_seg, true));
            e->counters.h2d_bytes += (int64_t)(sizeof(int) * n_seg);
        }
        if (what & kBandEv) {
            SFC_CUDA(bulk_copy(e, e->ev + 2 * dc, e->band_ev.data() + 2 * hc, (size_t)(2 * n_seg), true));
            e->counters.h2d_bytes += (int64_t)(2 * n_seg);
        }
        if (what & kBandStat) {
            SFC_CUDA(bulk_copy(e, e->stat + dc * kSects, v->static_image + hc * kSects, sizeof(float) * (size_t)n_seg * kSects, true));
            e->counters.h2d_bytes += (int64_t)(sizeof(float) * n_seg * kSects);
        }
        if (what & kBandDyn) {
            for (int k = 0; k < kKinds; ++k)
                for (long long c0 = 0; c0 < n_seg; c0 += e->stage_cells) {
                    const long long n = std::min(e->stage_cells, n_seg - c0);
                    SFC_CUDA(bulk_copy(e, e->stage, v->dyn_images[k] + (hc + c0) * kSects, sizeof(float) * (size_t)n * kSects, true));
                    SFC_CUDA(launch_interleave(e->stream, e->stage, e->dyn, k, dc + c0, n, e->ctl));
                    e->counters.kernel_launches += 1;
                    e->counters.h2d_bytes += (int64_t)(sizeof(float) * n * kSects);
                }
        }
    }
    return SFC_OK;
}

// Device -> host copy of the current window's rows (returns with the data on the host).
int band_store(sfc_engine* e, sfc_state_view* v, int what, bool owned_only) {
    const long long W = e->g.W;
    for (const RowSeg& seg : row_segments(e, owned_only)) {
        const long long hc = (long long)seg.global_row * W, dc = (long long)seg.local_row * W, n_seg = (long long)seg.rows * W;
        if (what & kBandOcc) {
            SFC_CUDA(bulk_copy(e, e->occ + dc, v->occupancy + hc, sizeof(int) * (size_t)n_seg, false));
            e->counters.d2h_bytes += (int64_t)(sizeof(int) * n_seg);
        }
        if (what & kBandEv) {
            SFC_CUDA(bulk_copy(e, e->ev + 2 * dc, e->band_ev.data() + 2 * hc, (size_t)(2 * n_seg), false));
            e->counters.d2h_bytes += (int64_t)(2 * n_seg);
        }
        if (what & kBandDyn) {
            for (int k = 0; k < kKinds; ++k)
                for (long long c0 = 0; c0 < n_seg; c0 += e->stage_cells) {
                    const long long n = std::min(e->stage_cells, n_seg - c0);
                    SFC_CUDA(launch_deinterleave(e->stream, e->dyn, e->stage, k, dc + c0, n));
                    SFC_CUDA(bulk_copy(e, e->stage, v->dyn_images[k] + (hc + c0) * kSects, sizeof(float) * (size_t)n * kSects, false));
                    e->counters.kernel_launches += 1;
                    e->counters.d2h_bytes += (int64_t)(sizeof(float) * n * kSects);
                }
        }
    }
    return SFC_OK;
}

} // namespace

int sfc_band_plan(int32_t width, int32_t height, int32_t halo, int64_t n_peds, int64_t device_bytes, int device) {
    if (device_bytes <= 0) {
        size_t free_b = 0, total_b = 0;
        if (cudaSetDevice(device) != cudaSuccess || cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return -1;
        device_bytes = (int64_t)(free_b - free_b / 16); // keep a margin for staging buffers and tables
    }
    const int64_t per_su = 4 + 32 + 96 + 2 + 1; // occupancy, static image, dynamic images, event map, k-5 work lists
    const int64_t fixed = n_peds * 40 + (512ll << 20); // pedestrian arrays + staging
    for (int bands = 1; bands <= height; ++bands) {
        const int64_t rows = (height + bands - 1) / bands;
        const int64_t resident = bands == 1 ? rows : rows + 2 * halo;
        if (bands > 1 && (rows < halo || rows + 2 * halo > height)) return -1; // bands thinner than the halo: the state cannot be cut further
        if (resident * width * per_su + fixed <= device_bytes) return bands;
    }
    return -1;
}

int sfc_band_run(sfc_engine* e, sfc_state_view* v, int64_t ticks, sfc_tick_metrics* metrics) {
    if (e->band_count < 2) return fail(e, SFC_E_STATE, "band run on an engine created without bands");
    if (!v->occupancy || !v->static_image || !v->dyn_images[0] || !v->dyn_images[1] || !v->dyn_images[2])
        return fail(e, SFC_E_STATE, "band run: the host state must hold every dense array");
    SFC_CUDA(cudaSetDevice(e->device));
    const long long P = v->n_peds, W = e->g.W, H = e->g.H;
    int rc = ensure_peds(e, P);
    if (rc == SFC_OK) rc = ensure_stage(e);
    if (rc == SFC_OK) rc = ensure_moved(e, std::max<int64_t>(ticks, 1));
    if (rc != SFC_OK) return rc;
    std::vector<int2> gate;
    std::vector<uint32_t> attr;
    int max_hh = 0;
    Ctl h{};
    h.tick = v->tick;
    h.run_base = v->tick;
    SFC_CUDA(cudaMemcpyAsync(e->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, e->stream));
    rc = upload_peds(e, v, &gate, &attr, &max_hh);
    if (rc != SFC_OK) return rc;
    const int need = 4 * (max_hh + 1) + (e->dp.regulated ? e->dp.density_radius : 0);
    if (e->g.halo < need || e->g.halo < e->tabs.max_hh)
        return fail(e, SFC_E_CONFIG, "slab_halo: too shallow for this population (need max(field half-height, "
                                     "4*(pedestrian half-height+1) + density radius) rows)");
    e->ped_half_h = max_hh;
    e->slab.reach = 0; // every pedestrian is resident: a band processes exactly the ones whose centre it owns
    band_window(e, 0);
    rc = select_k5_path(e, P, false);
    if (rc != SFC_OK) return rc;
    if (e->pairs_red) { // (float reductions need the upload-time subnormal scan of the whole images: plain read-modify-write here)
        e->pairs_red = 0;
    }
    SFC_CUDA(cudaMemsetAsync(e->moved_counts, 0, sizeof(unsigned long long) * (size_t)std::max<int64_t>(ticks, 1), e->stream));
    SFC_CUDA(cudaStreamSynchronize(e->stream)); // gate / attr staging vectors are consumed
    e->band_ev.assign((size_t)(2 * W * H), 0);
    e->tick = v->tick;
    e->uploaded = true;
    const DebugArrays none{};
    const long long interval = e->cfg.rebuild_interval;
    const int B = e->band_count;
    int status = SFC_OK;
    for (int64_t t = 0; t < ticks && status == SFC_OK; ++t) {
        // pass A: k-2 — decisions (engine.cpp:341-363)
        for (int b = 0; b < B && status == SFC_OK; ++b) {
            if (!band_window(e, b)) break;
            status = band_load(e, v, kBandOcc, false);
            if (status == SFC_OK) status = band_load(e, v, kBandStat | kBandDyn, true);
            if (status != SFC_OK) break;
            SFC_CUDA(launch_k2_decide(e->stream, e->g, e->peds, e->occ, e->stat, e->dyn, e->ev, e->ctl, e->dp, e->slab));
            e->counters.kernel_launches += 1;
        }
        // pass B: k-3 — votes (engine.cpp:365-386)
        for (int b = 0; b < B && status == SFC_OK; ++b) {
            if (!band_window(e, b)) break;
            status = band_load(e, v, kBandOcc, false);
            if (status != SFC_OK) break;
            SFC_CUDA(launch_k3_vote(e->stream, e->g, e->peds, e->occ, e->ctl, e->dp, e->slab));
            e->counters.kernel_launches += 1;
        }
        // pass C: k-4 — moves; occupancy and the tick's events go back band by band, halo rows included
        if (status == SFC_OK) {
            SFC_CUDA(cudaStreamSynchronize(e->stream));
            std::fill(e->band_ev.begin(), e->band_ev.end(), (uint8_t)0);
        }
        for (int b = 0; b < B && status == SFC_OK; ++b) {
            if (!band_window(e, b)) break;
            status = band_load(e, v, kBandOcc | kBandEv, false);
            if (status != SFC_OK) break;
            SFC_CUDA(launch_k4_move(e->stream, e->g, e->peds, e->occ, e->ev, e->ctl, e->moved_counts, none, e->slab, TileMarks{}));
            e->counters.kernel_launches += 1;
            status = band_store(e, v, kBandOcc | kBandEv, false);
        }
        // pass D: k-5 — field write-back (engine.cpp:428-472)
        for (int b = 0; b < B && status == SFC_OK; ++b) {
            if (!band_window(e, b)) break;
            status = band_load(e, v, kBandEv, false);
            if (status == SFC_OK) status = band_load(e, v, kBandDyn, true);
            if (status != SFC_OK) break;
            // (k-4 empties the scatter kernel's hand-off list once per tick; here every band is a k-5 launch of its own)
            SFC_CUDA(cudaMemsetAsync(&e->ctl->dense_count, 0, sizeof(int), e->stream));
            SFC_CUDA(launch_k5_writeback(e->stream, k5_args(e, 0)));
            e->counters.kernel_launches += e->k5_launches;
            status = band_store(e, v, kBandDyn, true);
        }
        if (status != SFC_OK) break;
        SFC_CUDA(launch_tick_advance(e->stream, e->ctl));
        e->counters.kernel_launches += 1;
        e->tick += 1;
        if (interval > 0 && e->tick % interval == 0) { // maybe_rebuild (engine.cpp:538-550): check every band, then commit every band
            for (int pass = 1; pass <= 2 && status == SFC_OK; ++pass) {
                for (int b = 0; b < B && status == SFC_OK; ++b) {
                    if (!band_window(e, b)) break;
                    status = band_load(e, v, kBandOcc, false);
                    if (status == SFC_OK) status = band_load(e, v, kBandDyn, true);
                    if (status != SFC_OK) break;
                    SFC_CUDA(launch_rebuild(e->stream, e->g, e->tabs, e->peds, e->occ, e->dyn, nullptr, e->ctl, pass, 0.0));
                    e->counters.kernel_launches += 1;
                    if (pass == 2) status = band_store(e, v, kBandDyn, true);
                }
                if (pass == 1 && status == SFC_OK) {
                    SFC_CUDA(launch_drift_verdict(e->stream, e->ctl, e->cfg.rebuild_tolerance));
                    e->counters.kernel_launches += 1;
                }
            }
        }
    }
    band_window(e, 0);
    if (status != SFC_OK) return status;
    std::vector<unsigned long long> moved((size_t)std::max<int64_t>(ticks, 0));
    if (ticks > 0)
        SFC_CUDA(cudaMemcpyAsync(moved.data(), e->moved_counts, sizeof(unsigned long long) * (size_t)ticks, cudaMemcpyDeviceToHost, e->stream));
    if (P > 0 && v->center_xy)
        SFC_CUDA(cudaMemcpyAsync(v->center_xy, e->peds.center, sizeof(int2) * (size_t)P, cudaMemcpyDeviceToHost, e->stream));
    rc = check_device_error(e); // synchronises; refreshes e->tick
    v->tick = e->tick;
    if (metrics)
        for (int64_t t = 0; t < ticks; ++t) {
            metrics[t] = sfc_tick_metrics{};
            metrics[t].tick = h.tick + t;
            metrics[t].moved = (int64_t)moved[(size_t)t];
        }
    return rc;
}

int sfc_digest(sfc_engine* e, uint64_t* digest) {
    if (!e->uploaded) return fail(e, SFC_E_STATE, "digest before upload");
    if (e->slab.active) return fail(e, SFC_E_STATE, "digest: whole-grid engines only");
    SFC_CUDA(cudaSetDevice(e->device));
    void* scratch = nullptr;
    SFC_CUDA(cudaMalloc(&scratch, digest_scratch_bytes(e->cells, e->peds.n)));
    unsigned long long* out = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) +
                                                                    (digest_scratch_bytes(e->cells, e->peds.n) - 64));
    cudaError_t c = launch_digest(e->stream, e->occ, e->dyn, e->peds.center, e->cells, e->peds.n, scratch, out);
    unsigned long long h = 0;
    if (c == cudaSuccess) c = cudaMemcpyAsync(&h, out, sizeof h, cudaMemcpyDeviceToHost, e->stream);
    if (c == cudaSuccess) c = cudaStreamSynchronize(e->stream);
    cudaFree(scratch);
    if (c != cudaSuccess) return cuda_fail(e, c, "sfc_digest");
    e->counters.kernel_launches += 2;
    *digest = h;
    return SFC_OK;
}

int sfc_compare(sfc_engine* a, sfc_engine* b, sfc_difference* out) {
    sfc_engine* e = a;
    if (!a->uploaded || !b->uploaded) return fail(e, SFC_E_STATE, "compare before upload");
    if (a->slab.active || b->slab.active || a->device != b->device || a->g.W != b->g.W || a->g.H != b->g.H)
        return fail(e, SFC_E_STATE, "compare: two whole-grid engines of one geometry on one device");
    SFC_CUDA(cudaSetDevice(a->device));
    *out = sfc_difference{};
    int rc = check_device_error(a); // synchronises, refreshes the tick shadows
    if (rc == SFC_OK) rc = check_device_error(b);
    if (rc != SFC_OK && rc != SFC_E_INTEGRITY) return rc;
    if (a->tick != b->tick) {
        out->what = 1;
        return SFC_OK;
    }
    if (a->peds.n != b->peds.n) {
        out->what = 2;
        return SFC_OK;
    }
    unsigned long long* first = nullptr;
    SFC_CUDA(cudaMalloc(reinterpret_cast<void**>(&first), 6 * sizeof(unsigned long long)));
    unsigned long long h[6];
    cudaError_t c = launch_compare(a->stream, a->peds, b->peds, a->occ, b->occ, a->stat, b->stat, a->dyn, b->dyn, a->cells, first);
    if (c == cudaSuccess) c = cudaMemcpyAsync(h, first, sizeof h, cudaMemcpyDeviceToHost, a->stream);
    if (c == cudaSuccess) c = cudaStreamSynchronize(a->stream);
    cudaFree(first);
    if (c != cudaSuccess) return cuda_fail(e, c, "sfc_compare");
    a->counters.kernel_launches += 1;
    for (int w = 0; w < 6; ++w) { // the reference's order: centres, occupancy, static image, dynamic images
        if (h[w] == ~0ull) continue;
        out->what = 3 + w;
        out->index = (int64_t)h[w];
        if (w == 0) {
            int2 ca, cb;
            SFC_CUDA(cudaMemcpy(&ca, a->peds.center + h[w], sizeof ca, cudaMemcpyDeviceToHost));
            SFC_CUDA(cudaMemcpy(&cb, b->peds.center + h[w], sizeof cb, cudaMemcpyDeviceToHost));
            out->ax = ca.x, out->ay = ca.y, out->bx = cb.x, out->by = cb.y;
        } else if (w == 1) {
            SFC_CUDA(cudaMemcpy(&out->ax, a->occ + h[w], sizeof(int), cudaMemcpyDeviceToHost));
            SFC_CUDA(cudaMemcpy(&out->bx, b->occ + h[w], sizeof(int), cudaMemcpyDeviceToHost));
        } else {
            const long long cell = (long long)(h[w] / kSects), sect = (long long)(h[w] % kSects);
            const float* pa = w == 2 ? a->stat + h[w] : a->dyn + (cell * kKinds + (w - 3)) * kSects + sect;
            const float* pb = w == 2 ? b->stat + h[w] : b->dyn + (cell * kKinds + (w - 3)) * kSects + sect;
            SFC_CUDA(cudaMemcpy(&out->av, pa, sizeof(float), cudaMemcpyDeviceToHost));
            SFC_CUDA(cudaMemcpy(&out->bv, pb, sizeof(float), cudaMemcpyDeviceToHost));
        }
        return SFC_OK;
    }
    return SFC_OK;
}

void sfc_get_counters(const sfc_engine* e, sfc_counters* out) {
    *out = e->counters;
    out->k5_path = e->k5_field ? 4 : (e->k5_pairs ? 3 : (e->k5_listwalk_only ? 2 : (e->k5_window ? 1 : 0)));
    out->k5_active_list = e->marks.epoch != nullptr;
}

double sfc_last_run_ms(const sfc_engine* e) { return e->last_run_ms; }

} // extern "C"
