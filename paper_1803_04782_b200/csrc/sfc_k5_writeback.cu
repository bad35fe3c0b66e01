// sfc_k5_writeback.cu — k-5, the field write-back: superpose the movement of every pedestrian
// onto the three dynamic strength images (reference engine.cpp:428-472, the loop that takes
// 63-98 % of the CPU reference's tick).
//
// Reference formulation: for every (su, kind, sect) address walk a precomputed list of F
// contributor offsets, read two mask bytes per offset, accumulate gated +-magnitude terms in
// doubles through a K-slot StepCache (term idx -> slot idx mod K, accumulator.hpp:36-46), fold
// the K slots in slot order, cast to float, add to the image.  6F mask probes per su.
//
// This file holds two of the four bit-identical formulations (the list walk for small fields is
// sfc_k5_listwalk.cu, the warp-per-block kernel for sparse crowds sfc_k5_window.cu) and the
// dispatcher between them (launch_k5_writeback; the engine chooses in sfc_upload):
// the SCATTER kernel for ordinary crowds on fields beyond 11 x 11, and the event-walk GATHER for
// fields beyond 15 x 15 and for tiles the scatter finds crowded there.
//
// A CTA owns a tile of 32 x 8 su.  It stages the tile +
// field-halo region of the 2-byte event map in shared memory once (coalesced row reads) and
// compacts the (few) movement events into a list ordered by (x, then y) with warp ballots — no
// atomics.  That order equals the reference's contributor-list order for every target in the
// tile, because the lists are sorted lexicographically by centre offset (fields.hpp:55-57).
// Zero terms are never materialised (adding +-0.0 to a partial cannot change it), so the work
// is proportional to the number of movers, not to the field area.  Two formulations follow,
// chosen per tile by the number of events in reach:
//
//   SCATTER (sparse tiles, 256 threads): lanes enumerate (event, support offset, kind) triples —
//     fully packed — and add each gated term to a per-address double in shared memory.  An
//     address that receives ONE or TWO terms is order-independent: whichever StepCache slots
//     they fall in, the reference's total is fl(t1 + t2) (IEEE addition is commutative and
//     0.0 + t is exact), so a shared-memory atomic add reproduces it bit for bit.  Addresses with
//     three or more terms (a few per cent of a sparse crowd) go on a work list and are replayed
//     through the exact K-slot order, one address per thread.  Tiles with too many events are
//     appended to a device-side list for the second kernel.
//
//   GATHER (dense tiles, 128 threads, persistent over that list): a warp owns a block of 8 x 4 su,
//     one su per lane, and walks the events in reach with a warp-uniform trip count; only the
//     per-lane "is this offset in the support, which sect, which slot" part diverges.  The K x 8
//     double partials of the kind being processed live in shared memory laid out [slot][thread]
//     (bank = lane: conflict-free for any per-lane slot) and are created lazily under a 64-bit
//     dirty mask; the fold visits only dirty slots (ascending bit order = slot order).
//
// In both, only su that received a term touch HBM: one 32-byte sector per (su, kind).  Nothing is
// read or written for su out of every mover's reach, so sparse crowds move far fewer than the
// dense 192 B/su.
//
// Fields larger than the grid wrap onto themselves (test_engine.cpp:329-340): the region is
// scanned in unwrapped coordinates, so one physical su can appear several times, once per
// periodic image — exactly the reference's while-loop wraps (engine.cpp:450-454).
// Regions too large for shared memory (very large fields) use 32 x 16 tiles, gather only, with the
// region staged in column chunks: the list is sorted, so chunks arrive in order and are appended to
// one list as long as the events fit (else the walks re-stage chunk by chunk).

#include <cstdlib>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kTileW = 32;
constexpr int kBlockW = 8, kBlockH = 4; // su block owned by one warp at a time in the gather (one su per lane)
constexpr int kChunkCells = 2048;       // region cells staged per pass (codes 4 KB + list 16 KB)
constexpr int kTabSmemMax = 768;        // table entries (all kinds) kept in shared memory
constexpr int kReplayCap = 1020;        // scatter: work-list capacity for addresses with >= 3 terms
constexpr int kOboxMax = 512;           // scatter: decoded support offsets of the largest field box
// shared-memory bytes of the scatter: su x 24 addresses x double + three term-count bit planes + work list
constexpr size_t scatter_bytes(int cells) { return (size_t)cells * 24 * 8 + 3 * (size_t)cells * 4 + (kReplayCap + 4) * 4; }

enum { kModeAll = 0, kModeScatter = 1, kModeDense = 2 };

struct K5Args {
    GridDev g;
    TablesDev t;
    float* dyn;
    const uint8_t* ev;
    Ctl* ctl;
    int* dense_list;
    int tiles_x;
    int advance_tick;
    int cap;          // cells staged per pass = event-list capacity
    int list_cap;     // events one list may hold when chunks are appended (<= cap; SFC_K5_LIST_CAP lowers it for tests)
    int rw_max;       // region columns for a full tile
    int tab_smem;     // contributor tables fit in shared memory
    int part_doubles; // size of the partial-sum / scatter region, in doubles
    int ev_max;       // scatter handles tiles with at most this many events in reach
    int n_tiles;      // tiles_x * tiles_y
    TileMarks marks;  // scatter kernel: active-tile list written by k-4 (epoch == nullptr: every tile)
};

struct Smem {
    double* part;
    uint2* evl;
    double* tab_mag;
    uint32_t* tab_info;
    int* colstart;
    uint16_t* codes;
};

__device__ __forceinline__ Smem carve(unsigned char* raw, const K5Args& a) {
    Smem s;
    s.part = reinterpret_cast<double*>(raw);
    s.evl = reinterpret_cast<uint2*>(s.part + a.part_doubles);
    s.tab_mag = reinterpret_cast<double*>(s.evl + a.cap);
    s.tab_info = reinterpret_cast<uint32_t*>(s.tab_mag + (a.tab_smem ? a.t.total_entries : 0));
    s.colstart = reinterpret_cast<int*>(s.tab_info + (a.tab_smem ? ((a.t.total_entries + 1) & ~1) : 0));
    s.codes = reinterpret_cast<uint16_t*>(s.colstart + ((a.rw_max + 2 + 1) & ~1));
    return s;
}

// K: StepCache width.  SG: sects accumulated per gather walk (SG * K <= 64: the dirty set is one
// 64-bit word).  ROWS: block rows per tile (tile height = 4 * ROWS).  NT: threads.
template <int K, int SG, int ROWS, int NT, int MODE>
__device__ void process_tile(const K5Args& a, const Smem& sm, const int tile) {
    constexpr int NW = NT / 32;
    constexpr int NG = kSects / SG;
    constexpr int MH = kBlockH * ROWS;
    static_assert(SG * K <= 64, "dirty mask is one 64-bit word");

    const GridDev g = a.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* const part = sm.part;
    uint2* const evl = sm.evl;
    int* const colstart = sm.colstart;
    uint16_t* const codes = sm.codes;
    const double* const tab_mag = sm.tab_mag;
    const uint32_t* const tab_info = sm.tab_info;

    const int tile_x = tile % a.tiles_x, tile_y = tile / a.tiles_x;
    const int x0 = tile_x * kTileW;
    const int y0 = g.row0 + tile_y * MH; // global row of the tile's first row
    const int nx = min(kTileW, g.W - x0);
    const int ny = min(MH, g.row0 + g.rows - y0);
    const int HW = a.t.max_hw, HH = a.t.max_hh;
    const int RW = nx + 2 * HW, RH = ny + 2 * HH;
    const int xs = x0 - HW, ys = y0 - HH;

    const uint16_t* ev16 = reinterpret_cast<const uint16_t*>(a.ev);
    const int cols_per_pass = max(1, a.cap / RH);
    const bool single_pass = cols_per_pass >= RW;

    // Stages the event codes of region columns [c0, c1) in shared memory (coalesced row reads,
    // column-major store), then compacts the non-zero ones into evl ordered by (x, y).
    // Returns the event count (uniform across the CTA).
    // With base >= 0 the events are APPENDED at evl[base..] and colstart is indexed by region column
    // (chunks arrive in column order, so the list stays sorted); returns -1, writing nothing, when
    // the list would overflow.
    auto build_list = [&](int c0, int c1, int base = -1) -> int {
        const int ncols = c1 - c0;
        const bool append = base >= 0;
        int* const cs = append ? colstart + c0 : colstart; // cs[rc] .. cs[rc + 1]: events of column c0 + rc
        const bool narrow = RW <= g.W; // one conditional add wraps x (wider regions take the general path)
        { // row-major over the chunk (coalesced), eight loads of a thread in flight before the first use
            const int n_cells = ncols * RH;
            const unsigned inv_cols = ncols > 1 ? 0xFFFFFFFFu / (unsigned)ncols + 1u : 0u; // (a one-column chunk: the reciprocal would wrap to 0)
            for (int i0 = 0; i0 < n_cells; i0 += 8 * NT) {
                uint16_t got[8];
                int at[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int i = i0 + q * NT + tid;
                    got[q] = 0;
                    at[q] = -1;
                    if (i < n_cells) {
                        const int ry = ncols > 1 ? (int)__umulhi((unsigned)i, inv_cols) : i; // i / ncols
                        const int rc = i - ry * ncols;
                        at[q] = rc * RH + ry;
                        int x = xs + c0 + rc;
                        long long idx = -1;
                        if (narrow) {
                            const long long row = cell_index(g, 0, ys + ry); // -1: row does not exist
                            if (g.closed) {
                                if (row >= 0 && x >= 0 && x < g.W) idx = row + x;
                            } else if (row >= 0) {
                                x += x < 0 ? g.W : (x >= g.W ? -g.W : 0);
                                idx = row + x;
                            }
                        } else {
                            idx = cell_index(g, x, ys + ry);
                        }
                        if (idx >= 0) got[q] = __ldg(ev16 + idx);
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (at[q] >= 0) codes[at[q]] = got[q];
            }
        }
        __syncthreads();
        for (int rc = warp; rc < ncols; rc += NW) { // per-column counts
            int cnt = 0;
            for (int r0 = 0; r0 < RH; r0 += 32) {
                const int ry = r0 + lane;
                cnt += __popc(__ballot_sync(0xFFFFFFFFu, ry < RH && codes[rc * RH + ry] != 0));
            }
            if (lane == 0) cs[rc + 1] = cnt;
        }
        if (tid == 0) cs[0] = append ? base : 0;
        __syncthreads();
        if (warp == 0) { // inclusive scan of the shifted counts = exclusive column starts
            int carry = append ? base : 0;
            for (int b1 = 1; b1 <= ncols; b1 += 32) {
                const int i = b1 + lane;
                int v = i <= ncols ? cs[i] : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xFFFFFFFFu, v, o);
                    if (lane >= o) v += u;
                }
                if (i <= ncols) cs[i] = v + carry;
                carry += __shfl_sync(0xFFFFFFFFu, v, 31);
            }
        }
        __syncthreads();
        if (append && cs[ncols] > a.list_cap) return -1; // uniform
        for (int rc = warp; rc < ncols; rc += NW) {
            int pos = cs[rc];
            if (cs[rc + 1] == pos) continue;
            for (int r0 = 0; r0 < RH; r0 += 32) {
                const int ry = r0 + lane;
                const uint32_t code = ry < RH ? codes[rc * RH + ry] : 0u;
                const unsigned ballot = __ballot_sync(0xFFFFFFFFu, code != 0);
                if (code != 0)
                    evl[pos + __popc(ballot & ((1u << lane) - 1u))] = make_uint2((uint32_t)(c0 + rc) | ((uint32_t)ry << 16), code);
                pos += __popc(ballot);
            }
        }
        __syncthreads();
        return cs[ncols] - (append ? base : 0);
    };

    int n_events = 0;
    bool one_list = single_pass; // the whole region's events sit in evl, colstart spans the region
    if constexpr (MODE == kModeScatter) {
        // The scatter does not need the events in order (only its rare exact replays do), so the
        // region is read straight from the event map — rows on warps, columns on lanes — and the
        // non-zero cells are appended to a list with a shared-memory counter.
        int* const n_list = colstart;                       // [0]: running count
        uint2* const unsorted = reinterpret_cast<uint2*>(codes + kOboxMax); // [cap]
        if (tid == 0) *n_list = 0;
        __syncthreads();
        // every load of a thread is issued before the first result is used: one L2 round trip, not one per cell
        constexpr int LOADS = (kChunkCells + NT - 1) / NT;
        const bool narrow = RW <= g.W;
        const int ncell = RW * RH;
        uint32_t got[LOADS];
#pragma unroll
        for (int q = 0; q < LOADS; ++q) {
            const int i = q * NT + tid;
            got[q] = 0u;
            if (i < ncell) {
                const int ry = i / RW, rc = i - ry * RW;
                int x = xs + rc;
                long long idx = -1;
                if (narrow) {
                    const long long row = cell_index(g, 0, ys + ry); // -1: row does not exist
                    if (g.closed) {
                        if (row >= 0 && x >= 0 && x < g.W) idx = row + x;
                    } else if (row >= 0) {
                        x += x < 0 ? g.W : (x >= g.W ? -g.W : 0);
                        idx = row + x;
                    }
                } else {
                    idx = cell_index(g, x, ys + ry);
                }
                if (idx >= 0) got[q] = __ldg(ev16 + idx);
            }
        }
#pragma unroll
        for (int q = 0; q < LOADS; ++q) {
            if (got[q] == 0u) continue;
            const int i = q * NT + tid;
            const int ry = i / RW, rc = i - ry * RW;
            unsorted[atomicAdd(n_list, 1)] = make_uint2((uint32_t)rc | ((uint32_t)ry << 16), got[q]);
        }
        __syncthreads();
        n_events = *n_list;
        if (n_events == 0) return; // nobody moved within reach of this tile
        if (n_events > a.ev_max) { // dense tile: hand it to the gather kernel
            if (tid == 0) a.dense_list[atomicAdd(&a.ctl->dense_count, 1)] = tile;
            return;
        }
        // rank sort by (x, y): every region cell appears once, so keys are unique
        for (int i = tid; i < n_events; i += NT) {
            const uint2 mine = unsorted[i];
            const uint32_t key = ((mine.x & 0xFFFFu) << 16) | (mine.x >> 16);
            int rank = 0;
            for (int j = 0; j < n_events; ++j) {
                const uint32_t xj = unsorted[j].x;
                rank += ((((xj & 0xFFFFu) << 16) | (xj >> 16)) < key) ? 1 : 0;
            }
            evl[rank] = mine;
        }
        // support offsets of the largest box, decoded once per CTA: (dx + 128) | (dy + 128) << 8
        const int BW = 2 * HW + 1, BOX = BW * (2 * HH + 1);
        for (int o = tid; o < BOX; o += NT) {
            const int oy = o / BW;
            codes[o] = (uint16_t)((o - oy * BW - HW + 128) | ((oy - HH + 128) << 8));
        }
        __syncthreads();
    } else if (single_pass) {
        n_events = build_list(0, RW);
        if (n_events == 0) return; // nobody moved within reach of this tile
    } else { // large field: stage the region chunk by chunk, keep ONE list if the events fit
        int total = 0;
        one_list = true;
        for (int c0 = 0; c0 < RW; c0 += cols_per_pass) {
            const int n = build_list(c0, min(RW, c0 + cols_per_pass), total);
            __syncthreads();
            if (n < 0) {
                one_list = false;
                break;
            }
            total += n;
        }
        if (one_list) {
            n_events = total;
            if (n_events == 0) return;
        }
    }

    // =========================================================================================
    // SCATTER
    // =========================================================================================
    if constexpr (MODE == kModeScatter) {
        constexpr int CELLS = kTileW * MH;
        double* acc = part;                                                  // [CELLS][24]
        uint32_t* seen1 = reinterpret_cast<uint32_t*>(acc + CELLS * 24);     // [CELLS] addresses with >= 1 term (24-bit masks)
        uint32_t* seen2 = seen1 + CELLS;                                     // [CELLS] ... >= 2 terms
        uint32_t* seen3 = seen2 + CELLS;                                     // [CELLS] ... >= 3 terms
        int* replay = reinterpret_cast<int*>(seen3 + CELLS);                 // [kReplayCap]
        int* n_replay = replay + kReplayCap;
        uint32_t* const touched = seen1;
        {
            float4* z = reinterpret_cast<float4*>(part);
            constexpr int N16 = (CELLS * 24 * 8 + 3 * CELLS * 4) / 16;
            for (int i = tid; i < N16; i += NT) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (tid == 0) *n_replay = 0;
        }
        __syncthreads();
        // threads take (event, support offset) pairs — evenly packed whatever the event count
        const int BW = 2 * HW + 1, BOX = BW * (2 * HH + 1);
        const int pairs = n_events * BOX;
        const float inv_box = 1.0f / (float)BOX;
        for (int pr = tid; pr < pairs; pr += NT) {
            int e = (int)(((float)pr + 0.5f) * inv_box);
            if (e * BOX > pr) --e;
            else if ((e + 1) * BOX <= pr) ++e;
            const uint32_t packed = codes[pr - e * BOX];
            const int dx = (int)(packed & 0xFFu) - 128, dy = (int)(packed >> 8) - 128; // centre offset = mover - target
            if ((dx | dy) == 0) continue;
            const uint2 evt = evl[e];
            const int cx = (int)(evt.x & 0xFFFFu) - dx - HW; // target su
            const int cy = (int)(evt.x >> 16) - dy - HH;
            if (cx < 0 || cx >= nx || cy < 0 || cy >= ny) continue;
            const uint32_t fb = evt.y & 0xFFu, tbyte = (evt.y >> 8) & 0xFFu;
            const int cell = cy * kTileW + cx;
            int tb = 0;
#pragma unroll
            for (int k = 0; k < kKinds; ++k) {
                const KindTableDev& kt = a.t.k[k];
                const int ti = tb + (dy + kt.hh) * kt.fw + dx + kt.hw;
                const bool inside = dx >= -kt.hw && dx <= kt.hw && dy >= -kt.hh && dy <= kt.hh;
                tb += kt.fw * kt.fh;
                if (!inside) continue;
                const uint32_t info = tab_info[ti];
                const uint32_t mask = (info >> 3) & 0xFFu;
                if (mask == 0) continue;
                const int shift = k == 0 ? 0 : (k == 1 ? 3 : 8); // kind 2: orientation 0 of an all-ones mask
                const bool from = (fb & 0x80u) && ((mask >> ((fb >> shift) & 7u)) & 1u);
                const bool to = (tbyte & 0x80u) && ((mask >> ((tbyte >> shift) & 7u)) & 1u);
                if (!from && !to) continue;
                const double mag = tab_mag[ti];
                const int a24 = k * kSects + (int)(info & 7u);
                const uint32_t bit = 1u << a24;
                double* slot = acc + cell * 24 + a24;
                if (from) atomicAdd(slot, -mag);
                if (to) atomicAdd(slot, mag);
                // saturating per-address term count in three bit planes: 1, 2, >= 3
                for (int terms = (from ? 1 : 0) + (to ? 1 : 0); terms > 0; --terms) {
                    if (!(atomicOr(&seen1[cell], bit) & bit)) continue;
                    if (!(atomicOr(&seen2[cell], bit) & bit)) continue;
                    atomicOr(&seen3[cell], bit);
                }
            }
        }
        __syncthreads();
        // addresses with three or more terms: exact K-slot replay, one address per thread
        for (int cell = tid; cell < CELLS; cell += NT) {
            uint32_t m = seen3[cell];
            while (m != 0u) {
                const int a24 = __ffs((int)m) - 1;
                m &= m - 1u;
                const int slot = atomicAdd(n_replay, 1);
                if (slot < kReplayCap) replay[slot] = cell * 24 + a24;
            }
        }
        __syncthreads();
        const int n_rep = *n_replay;
        const bool overflow = n_rep > kReplayCap; // then every thread scans the addresses for its share
        const int rep_items = overflow ? CELLS * 24 : n_rep;
        for (int i = tid; i < rep_items; i += NT) {
            const int addr = overflow ? i : replay[i];
            if (overflow && !((seen3[addr / 24] >> (addr % 24)) & 1u)) continue;
            const int cell = addr / 24, kind = (addr % 24) / kSects, sect = addr % kSects;
            const int tcx = cell % kTileW + HW, tcy = cell / kTileW + HH;
            const KindTableDev& kt = a.t.k[kind];
            int tbase = 0;
            for (int k = 0; k < kind; ++k) tbase += a.t.k[k].fw * a.t.k[k].fh;
            const int shift = kind == 0 ? 0 : (kind == 1 ? 3 : 8);
            double p[K];
            unsigned used = 0;
            for (int e = 0; e < n_events; ++e) { // events in list order = contributor order
                const uint2 evt = evl[e];
                const int dy = (int)(evt.x >> 16) - tcy, dx = (int)(evt.x & 0xFFFFu) - tcx;
                if (dy < -kt.hh || dy > kt.hh || dx < -kt.hw || dx > kt.hw || (dx | dy) == 0) continue;
                const int ti = tbase + (dy + kt.hh) * kt.fw + dx + kt.hw;
                const uint32_t info = tab_info[ti];
                const uint32_t mask = (info >> 3) & 0xFFu;
                if (mask == 0 || (int)(info & 7u) != sect) continue;
                const uint32_t fb = evt.y & 0xFFu, tb = (evt.y >> 8) & 0xFFu;
                const bool from = (fb & 0x80u) && ((mask >> ((fb >> shift) & 7u)) & 1u);
                const bool to = (tb & 0x80u) && ((mask >> ((tb >> shift) & 7u)) & 1u);
                const double mag = tab_mag[ti];
                const uint32_t j2 = (info >> 11) << 1;
#pragma unroll
                for (int half = 0; half < 2; ++half) { // from-term (idx 2j) then to-term (idx 2j+1)
                    if (!(half == 0 ? from : to)) continue;
                    const int slot = (int)((j2 + half) & (K - 1));
                    const double term = half == 0 ? -mag : mag;
#pragma unroll
                    for (int q = 0; q < K; ++q) {
                        if (q != slot) continue;
                        p[q] = ((used >> q) & 1u) ? __dadd_rn(p[q], term) : term;
                    }
                    used |= 1u << slot;
                }
            }
            double total = 0.0; // StepCache::total, slot order
#pragma unroll
            for (int q = 0; q < K; ++q)
                if ((used >> q) & 1u) total = __dadd_rn(total, p[q]);
            acc[addr] = total;
        }
        __syncthreads();
        // apply: one 32-byte sector per touched (su, kind); every load of a thread is issued before
        // the first is consumed
        constexpr int PAIRS = (CELLS * kKinds + NT - 1) / NT;
        float4 v[PAIRS][2];
        uint32_t km[PAIRS];
        float4* rec[PAIRS];
#pragma unroll
        for (int q = 0; q < PAIRS; ++q) {
            const int pr = q * NT + tid, kind = pr / CELLS, cell = pr % CELLS;
            km[q] = pr < CELLS * kKinds ? (touched[cell] >> (kind * kSects)) & 0xFFu : 0u;
            rec[q] = nullptr;
            if (km[q] != 0) {
                const long long gcell = cell_index(g, x0 + cell % kTileW, y0 + cell / kTileW);
                rec[q] = reinterpret_cast<float4*>(a.dyn + gcell * 24 + kind * kSects);
                v[q][0] = rec[q][0];
                v[q][1] = rec[q][1];
            }
        }
#pragma unroll
        for (int q = 0; q < PAIRS; ++q) {
            if (km[q] == 0) continue;
            const int pr = q * NT + tid, kind = pr / CELLS, cell = pr % CELLS;
            const double* ap = acc + cell * 24 + kind * kSects;
            float r[8] = {v[q][0].x, v[q][0].y, v[q][0].z, v[q][0].w, v[q][1].x, v[q][1].y, v[q][1].z, v[q][1].w};
#pragma unroll
            for (int sect = 0; sect < kSects; ++sect)
                if ((km[q] >> sect) & 1u) r[sect] = __fadd_rn(r[sect], __double2float_rn(ap[sect])); // image += (float)total
            rec[q][0] = make_float4(r[0], r[1], r[2], r[3]);
            rec[q][1] = make_float4(r[4], r[5], r[6], r[7]);
        }
        return;
    } else {
        // =====================================================================================
        // GATHER
        // =====================================================================================
        // Walks events [e0, e1) for the su (tcx, tcy) and one kind / sect group, adding each gated
        // term to its StepCache slot.  The loop trip count and the block filter are warp-uniform.
        auto walk = [&](int e0, int e1, int kind, int sg, const KindTableDev& kt, const double* kmag,
                        const uint32_t* kinfo, int tcx, int tcy, int by0r, unsigned long long& dirty) {
            const int shift = kind == 0 ? 0 : (kind == 1 ? 3 : 8);
            for (int e = e0; e < e1; ++e) {
                const uint2 evt = evl[e]; // broadcast read
                const int ery = (int)(evt.x >> 16);
                if (ery < by0r - kt.hh || ery > by0r + kBlockH - 1 + kt.hh) continue; // uniform: out of the block's reach
                const int dy = ery - tcy;
                const int dx = (int)(evt.x & 0xFFFFu) - tcx;
                if (dy < -kt.hh || dy > kt.hh || dx < -kt.hw || dx > kt.hw || (dx | dy) == 0) continue;
                const int ti = (dy + kt.hh) * kt.fw + dx + kt.hw;
                const uint32_t info = kinfo[ti];
                const uint32_t mask = (info >> 3) & 0xFFu;
                if (mask == 0) continue;
                const int sect = info & 7;
                if (SG < kSects && sect / SG != sg) continue;
                const uint32_t fb = evt.y & 0xFFu, tb = (evt.y >> 8) & 0xFFu;
                const bool from = (fb & 0x80u) && ((mask >> ((fb >> shift) & 7u)) & 1u);
                const bool to = (tb & 0x80u) && ((mask >> ((tb >> shift) & 7u)) & 1u);
                if (!from && !to) continue;
                const double mag = kmag[ti];
                const uint32_t j2 = (info >> 11) << 1;
                const int ls = sect % SG;
#pragma unroll
                for (int half = 0; half < 2; ++half) { // from-term (idx 2j) then to-term (idx 2j+1)
                    if (!(half == 0 ? from : to)) continue;
                    const int addr = ls * K + (int)((j2 + half) & (K - 1));
                    const unsigned long long bit = 1ull << addr;
                    double* cellp = part + addr * NT + tid;
                    const double term = half == 0 ? -mag : mag;
                    if (dirty & bit) {
                        *cellp = __dadd_rn(*cellp, term);
                    } else {
                        *cellp = term; // 0.0 + term
                        dirty |= bit;
                    }
                }
            }
        };

        // Folds the dirty slots of one (kind, sect group) into the su's image sector:
        // StepCache::total in slot order (accumulator.hpp:41-46), then image += (float)total.
        auto fold = [&](unsigned long long dirty, float* r) {
            while (dirty != 0ull) {
                const int first = __ffsll((long long)dirty) - 1;
                const int ls = first / K;
                const unsigned long long group = dirty & (((1ull << K) - 1ull) << (ls * K));
                dirty &= ~group;
                unsigned long long rest = group;
                double total = 0.0;
                while (rest != 0ull) {
                    const int addr = __ffsll((long long)rest) - 1;
                    rest &= rest - 1ull;
                    total = __dadd_rn(total, part[addr * NT + tid]);
                }
                const float add = __double2float_rn(total);
#pragma unroll
                for (int q = 0; q < SG; ++q)
                    if (q == ls) r[q] = __fadd_rn(r[q], add);
            }
        };

        constexpr int NBLK = 4 * ROWS; // 8 x 4 blocks per tile: four side by side, ROWS deep
#pragma unroll 1
        for (int b0 = 0; b0 < NBLK; b0 += NW) {
            const int blk = b0 + warp;
            const int bx = (blk % 4) * kBlockW, by = (blk / 4) * kBlockH;
            const bool blk_ok = blk < NBLK && by < ny && bx < nx; // uniform per warp
            if (one_list && !blk_ok) continue; // (chunked mode keeps every warp in the CTA-wide list builds)
            const int cx = bx + (lane % kBlockW), cy = by + (lane / kBlockW); // my su in the tile
            const int tcx = cx + HW, tcy = cy + HH;                             // ... in region coordinates
            const bool in_grid = blk_ok && cx < nx && cy < ny;
            const long long cell = in_grid ? cell_index(g, x0 + cx, y0 + cy) : -1;
            float4* rec = reinterpret_cast<float4*>(a.dyn + (cell < 0 ? 0 : cell) * 24);
            // events that can reach the block lie in a contiguous range of the x-sorted list
            int e_lo = 0, e_hi = n_events;
            if (one_list) {
                e_lo = colstart[max(bx, 0)];
                e_hi = colstart[min(bx + kBlockW + 2 * HW, RW)];
                if (e_lo == e_hi) continue; // uniform
            }

#pragma unroll 1
            for (int kind = 0; kind < kKinds; ++kind) {
                const KindTableDev kt = a.t.k[kind];
                int tbase = 0;
                for (int k = 0; k < kind; ++k) tbase += a.t.k[k].fw * a.t.k[k].fh;
                const double* kmag = a.tab_smem ? tab_mag + tbase : kt.mag;
                const uint32_t* kinfo = a.tab_smem ? tab_info + tbase : kt.info;
#pragma unroll 1
                for (int sg = 0; sg < NG; ++sg) {
                    unsigned long long dirty = 0ull;
                    if (one_list) {
                        if (in_grid) walk(e_lo, e_hi, kind, sg, kt, kmag, kinfo, tcx, tcy, by + HH, dirty);
                    } else { // chunked region: the list is rebuilt per (kind, group)
                        for (int c0 = 0; c0 < RW; c0 += cols_per_pass) {
                            const int n = build_list(c0, min(RW, c0 + cols_per_pass));
                            if (n > 0 && in_grid) walk(0, n, kind, sg, kt, kmag, kinfo, tcx, tcy, by + HH, dirty);
                            __syncthreads();
                        }
                    }
                    if (dirty == 0ull) continue;
                    // one 32-byte sector (or the SG-float part of it) per (su, kind)
                    float r[SG];
                    float* base = reinterpret_cast<float*>(rec) + kind * kSects + sg * SG;
                    if constexpr (SG == 2) {
                        const float2 v = *reinterpret_cast<const float2*>(base);
                        r[0] = v.x; r[1] = v.y;
                    } else {
#pragma unroll
                        for (int q = 0; q < SG / 4; ++q) {
                            const float4 v = reinterpret_cast<const float4*>(base)[q];
                            r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
                        }
                    }
                    fold(dirty, r);
                    if constexpr (SG == 2) {
                        *reinterpret_cast<float2*>(base) = make_float2(r[0], r[1]);
                    } else {
#pragma unroll
                        for (int q = 0; q < SG / 4; ++q)
                            reinterpret_cast<float4*>(base)[q] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                    }
                }
            }
        }
    }
}

template <int K, int SG, int ROWS, int NT, int MODE>
__global__ void __launch_bounds__(NT) k5_writeback_kernel(K5Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    if (MODE != kModeDense && a.advance_tick && blockIdx.x == 0 && tid == 0 && a.ctl->error_code == 0) a.ctl->tick += 1;
    if (a.ctl->error_code != 0) return;
    if (MODE == kModeDense && (int)blockIdx.x >= a.ctl->dense_count) return; // no dense tile for this CTA
    const Smem sm = carve(smem_raw, a);
    if (a.tab_smem) { // contributor tables: one copy per CTA
        int base = 0;
        for (int k = 0; k < kKinds; ++k) {
            const int n = a.t.k[k].fw * a.t.k[k].fh;
            for (int i = tid; i < n; i += NT) {
                sm.tab_mag[base + i] = a.t.k[k].mag[i];
                sm.tab_info[base + i] = a.t.k[k].info[i];
            }
            base += n;
        }
    }
    if (MODE != kModeScatter) __syncthreads(); // (the scatter synchronises after its event collection, before any table use)
    if constexpr (MODE == kModeDense) { // persistent over the tiles the scatter kernel declined
        const int n = a.ctl->dense_count;
        for (int i = blockIdx.x; i < n; i += gridDim.x) {
            process_tile<K, SG, ROWS, NT, MODE>(a, sm, a.dense_list[i]);
            __syncthreads();
        }
    } else if constexpr (MODE == kModeScatter) { // persistent: a CTA strides over the tiles
        if (a.marks.epoch != nullptr) { // ... over the tiles within reach of this tick's movers (TileMarks)
            const int n_edge = tile_edge_count(a.marks);
            const int n_items = n_edge + a.ctl->active_count;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
                int tile;
                if (item < n_edge) { // slab mode: tiles whose region reaches the halo rows
                    const int r = item / a.tiles_x;
                    const int ty = r < a.marks.edge_lo ? r : a.marks.edge_hi + (r - a.marks.edge_lo);
                    tile = ty * a.tiles_x + (item - r * a.tiles_x);
                } else {
                    tile = a.marks.list[item - n_edge];
                }
                process_tile<K, SG, ROWS, NT, MODE>(a, sm, tile);
                __syncthreads();
            }
        } else {
            for (int tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
                process_tile<K, SG, ROWS, NT, MODE>(a, sm, tile);
                __syncthreads();
            }
        }
    } else {
        process_tile<K, SG, ROWS, NT, MODE>(a, sm, blockIdx.x);
    }
}

struct K5Shape {
    size_t smem;
    int cap, rw_max, tab_smem, part_doubles;
};

template <int K, int SG, int ROWS, int NT, int MODE>
K5Shape k5_shape(const TablesDev& t) {
    constexpr int MH = kBlockH * ROWS;
    K5Shape s;
    s.rw_max = kTileW + 2 * t.max_hw;
    const int rh_max = MH + 2 * t.max_hh;
    const int region = s.rw_max * rh_max;
    s.cap = region <= kChunkCells ? region : kChunkCells;
    if (s.cap < rh_max) s.cap = rh_max; // at least one column per pass
    s.cap = (s.cap + 31) & ~31;
    s.tab_smem = t.total_entries <= kTabSmemMax;
    const size_t part_bytes = MODE == kModeScatter ? scatter_bytes(kTileW * kBlockH * ROWS) : sizeof(double) * SG * K * NT;
    s.part_doubles = (int)((part_bytes + 7) / 8);
    size_t b = (size_t)s.part_doubles * 8;
    b += sizeof(uint2) * (size_t)s.cap;
    if (s.tab_smem) b += sizeof(double) * t.total_entries + sizeof(uint32_t) * ((t.total_entries + 1) & ~1);
    b += sizeof(int) * (size_t)((s.rw_max + 2 + 1) & ~1);
    b += sizeof(uint16_t) * (size_t)((s.cap + 1) & ~1);
    if (MODE == kModeScatter) b += sizeof(uint16_t) * kOboxMax + sizeof(uint2) * (size_t)s.cap + 16; // offsets + unsorted list
    s.smem = (b + 127) & ~(size_t)127;
    return s;
}

template <int K, int SG, int ROWS, int NT, int MODE>
cudaError_t launch_one(cudaStream_t stream, const K5Launch& l) {
    constexpr int MH = kBlockH * ROWS;
    const K5Shape sh = k5_shape<K, SG, ROWS, NT, MODE>(l.t);
    K5Args a;
    a.g = l.g;
    a.t = l.t;
    a.dyn = l.dyn;
    a.ev = l.ev;
    a.ctl = l.ctl;
    a.dense_list = l.dense_list;
    a.tiles_x = (l.g.W + kTileW - 1) / kTileW;
    a.advance_tick = l.advance_tick;
    a.cap = sh.cap;
    a.list_cap = l.list_cap > 0 && l.list_cap < sh.cap ? l.list_cap : sh.cap;
    a.rw_max = sh.rw_max;
    a.tab_smem = sh.tab_smem;
    a.part_doubles = sh.part_doubles;
    a.ev_max = l.ev_max;
    a.marks = (MODE == kModeScatter && kBlockH * ROWS == kMarkTileH) ? l.marks : TileMarks{};
    const int tiles_y = (l.g.rows + MH - 1) / MH;
    long long blocks = (long long)a.tiles_x * tiles_y;
    a.n_tiles = (int)blocks;
    if (MODE == kModeDense && blocks > l.persistent_ctas) blocks = l.persistent_ctas;
    if (MODE == kModeScatter && blocks > l.scatter_ctas) blocks = l.scatter_ctas;
    if (MODE == kModeScatter && a.marks.epoch != nullptr && blocks > 4ll * l.persistent_ctas) blocks = 4ll * l.persistent_ctas;
    k5_writeback_kernel<K, SG, ROWS, NT, MODE><<<(unsigned)blocks, NT, sh.smem, stream>>>(a);
    return cudaGetLastError();
}

template <int K, int SG, int ROWS, int NT, int MODE>
cudaError_t prepare_one(const TablesDev& t) {
    static SmemGrant grant; // (one per kernel instantiation)
    return grant.raise(reinterpret_cast<const void*>(k5_writeback_kernel<K, SG, ROWS, NT, MODE>),
                       k5_shape<K, SG, ROWS, NT, MODE>(t).smem);
}

// Small fields (the whole 32 x 8 tile region is staged at once, tables in shared memory): scatter
// + dense gather.  Otherwise 32 x 16 tiles, gather only, chunked staging.
bool two_kernel_path(const TablesDev& t) {
    return (kTileW + 2 * t.max_hw) * (kBlockH * 2 + 2 * t.max_hh) <= kChunkCells && t.total_entries <= kTabSmemMax &&
           (2 * t.max_hw + 1) * (2 * t.max_hh + 1) <= kOboxMax && t.max_hw < 128 && t.max_hh < 128;
}

template <int K, int SG>
cudaError_t prepare_k(const TablesDev& t) {
    cudaError_t e = prepare_one<K, SG, 2, 256, kModeScatter>(t);
    if (e == cudaSuccess) e = prepare_one<K, SG, 2, 128, kModeDense>(t);
    if (e == cudaSuccess) e = prepare_one<K, SG, 1, 256, kModeScatter>(t);
    if (e == cudaSuccess) e = prepare_one<K, SG, 1, 128, kModeDense>(t);
    if (e == cudaSuccess) e = prepare_one<K, SG, 2, 128, kModeAll>(t);
    if (e == cudaSuccess) e = prepare_one<K, SG, 1, 128, kModeAll>(t);
    if (e == cudaSuccess) e = prepare_one<K, SG, 4, 128, kModeAll>(t);
    return e;
}

template <int K, int SG>
cudaError_t launch_k(cudaStream_t s, const K5Launch& l) {
    if (l.pairs_path && l.pairs.blob != nullptr) return launch_k5_pairs(s, l);
    if (l.field_path && l.field.blob != nullptr) return launch_k5_field(s, l);
    const bool walk = l.listwalk && k5_listwalk_supported(l.walk); // dense 32 x 8 tiles: list walk instead of event walk
    if (l.listwalk_only && walk) return launch_k5_listwalk(s, l, false);
    if (l.window_path && k5_window_supported(l.t) && l.dense_list != nullptr) {
        // window kernel over the active tiles; it hands dense tiles (32 x 8) to the dense kernel
        const cudaError_t e = launch_k5_window(s, l);
        if (e != cudaSuccess) return e;
        return walk ? launch_k5_listwalk(s, l, true) : launch_one<K, SG, 2, 128, kModeDense>(s, l);
    }
    // large fields: 32 x 16 tiles (the field halo is staged once per 512 su), gather only
    if (!two_kernel_path(l.t)) return launch_one<K, SG, 4, 128, kModeAll>(s, l);
    if (l.ev_max <= 0 || l.dense_list == nullptr) return launch_one<K, SG, 2, 128, kModeAll>(s, l);
    if (l.tile_rows == 4) { // 32 x 4 tiles: less shared memory per CTA, more CTAs per SM
        const cudaError_t e = launch_one<K, SG, 1, 256, kModeScatter>(s, l);
        if (e != cudaSuccess) return e;
        return launch_one<K, SG, 1, 128, kModeDense>(s, l);
    }
    const cudaError_t e = launch_one<K, SG, 2, 256, kModeScatter>(s, l);
    if (e != cudaSuccess) return e;
    return walk ? launch_k5_listwalk(s, l, true) : launch_one<K, SG, 2, 128, kModeDense>(s, l);
}

} // namespace

// Raises the dynamic shared-memory limits of the variants the engine may launch; done once at
// engine construction so no attribute call lands inside a CUDA-graph capture.
cudaError_t prepare_k5_writeback(int chunk_k, const TablesDev& t) {
    switch (chunk_k) {
        case 2: return prepare_k<2, 8>(t);
        case 4: return prepare_k<4, 8>(t);
        case 8: return prepare_k<8, 8>(t);
        case 16: return prepare_k<16, 4>(t);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k5_writeback(cudaStream_t s, const K5Launch& l) {
    switch (l.chunk_k) {
        case 2: return launch_k<2, 8>(s, l);
        case 4: return launch_k<4, 8>(s, l);
        case 8: return launch_k<8, 8>(s, l);
        case 16: return launch_k<16, 4>(s, l);
        default: return cudaErrorInvalidValue;
    }
}

// Number of kernels one launch_k5_writeback enqueues, and the tile count the dense list must hold.
int k5_kernels_per_launch(const TablesDev& t, int ev_max) { return two_kernel_path(t) && ev_max > 0 ? 2 : 1; }
long long k5_tile_count(const GridDev& g) { return (long long)((g.W + kTileW - 1) / kTileW) * ((g.rows + 3) / 4); }

} // namespace sfc
