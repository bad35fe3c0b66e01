// sfc_k5_pairs.cu — k-5 write-back for small fields (up to 9 su wide, 64 support offsets: the 7 x 7
// fields of BASELINE configs 1, 2, 4 and the paper baseline), every crowd density.
// Reference: k5_writeback_range + StepCache (engine.cpp:428-472, accumulator.hpp:36-46).
//
// The reference evaluates every (su, kind, sect) address by walking that sect's contributor list:
// 6F mask probes per su whether anybody moved or not.  Here the unit of work is a PAIR (su, sect
// group) that actually has a movement event among the group's contributor cells, and a warp works
// on a block of 8 x 4 su with nothing shared between warps but read-only tables (no block barrier,
// no atomics):
//
//   1. stage    the block + field-halo region of the 2-byte event map (<= 16 x 16 cells) is read
//               straight from global memory, two region rows per load; a ballot of "is there an
//               event" gives one bit row per region row.  No event in reach: the block is done.
//   2. window   each lane (one su) turns the bit rows of its field window into ONE 64-bit word laid
//               out [sect group][list position in StepCache slot order] — a table lookup per window
//               row (row bits -> permuted bits), so "does group g see an event" is a byte test and
//               the events of a group come out of a find-first-set loop already in the order the
//               reference folds them.
//   3. compact  the (su, group) pairs with a non-zero byte are listed (warp prefix sum): work is
//               spread evenly over the lanes whatever the crowd looks like.
//   4. fold     a lane takes a pair and visits its events in slot order.  The reference's term
//               idx = 2j (left) / 2j + 1 (arrived) of list position j goes to partial idx mod K, and
//               the partials are summed in slot order; positions j with the same j mod K/2 share
//               their two slots.  Visiting the positions sorted by (j mod K/2, j) therefore needs
//               three doubles per kind: the running total, the class's "left" partial and its
//               "arrived" partial, flushed (total += left; total += arrived) when the class changes.
//               Empty slots hold +0.0 and adding +0.0 changes nothing (the total is never -0.0), so
//               the result is the reference's bit for bit, for every K, with no per-slot storage.
//               image += (float)total as one scalar read-modify-write per touched address — every
//               address belongs to exactly one pair, so plain loads and stores.
//
// The three kinds share the walk (same support and list ranks; a repulsive kind's sect is the
// attractive kind's opposite, so the sect GROUPS coincide — build_walk_lists checks all of it).
// Work items are the eight blocks of every 32 x 8 tile, or of the tiles k-4 listed (TileMarks; the
// stamp carries the blocks within reach), so the cost follows the movers, not the grid.
// Fields larger than the grid wrap onto themselves (test_engine.cpp:329-340): the region is staged
// in unwrapped coordinates, exactly like the reference's while-loop wraps (engine.cpp:450-454).

#include <algorithm>
#include <cstring>
#include <vector>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kBlockW = 8, kBlockH = 4;
constexpr int kPitch = 16;        // staged region row pitch (cells)
constexpr int kRegionRowsMax = 16;
constexpr int kGroupBits = 8;     // window-word bits per sect group
static_assert(kMarkTileW == 4 * kBlockW && kMarkTileH == 2 * kBlockH, "a tile is 4 x 2 blocks");

struct __align__(16) PairEntry {  // one contributor offset, indexed by its window-word bit
    int off_cls;                  // region cell offset dy * kPitch + dx (low 16 bits, signed) | class j mod K/2 << 16
    uint32_t masks;               // orientation mask of kind k in byte k
    double mag[kKinds];
};
static_assert(sizeof(PairEntry) == 32, "two 16-byte loads per entry");

struct WarpScratch {
    uint2 sel[kRegionRowsMax * kPitch];      // per region cell WITH an event: one-hot orientation selectors of the
                                             // "left" (.x) / "arrived" (.y) byte, per kind in the byte lanes (cells
                                             // without an event keep stale words: only cells whose window bit is set are read)
    unsigned long long wm[32];               // window word per su of the block
    uint16_t rb[kRegionRowsMax];             // "has event" bits per region row
    uint8_t wl[32 * kSects];                 // work list: su << 3 | group
};

struct PairArgs {
    GridDev g;
    float* dyn;
    const uint8_t* ev;
    Ctl* ctl;
    TileMarks marks;              // epoch == nullptr: every tile
    const unsigned long long* T;  // [fh << fw] row bits -> window-word bits
    const PairEntry* E;           // [64]
    int fw, fh, hw, hh;
    int rw, rh;                   // block region extent: 8 + 2 hw, 4 + 2 hh
    uint32_t sect_packed[kKinds]; // sect of kind k fed by group g in bits [3g, 3g + 3)
    int tiles_x, n_tiles;
    uint32_t inv_tiles_x;         // floor(2^32 / tiles_x)
    int advance_tick;
};

__device__ __forceinline__ void add_if(double& p, double t, uint32_t flag) { // one predicated DADD
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q add.rn.f64 %0, %0, %1;\n\t}" : "+d"(p) : "d"(t), "r"(flag));
}

// one-hot orientation selectors of an event byte, per kind in the byte lanes (kind 2 is non-directional)
__device__ __forceinline__ uint32_t selector(uint32_t b) { // (branch-free: 0 when bit 7 is clear)
    return ((1u << (b & 7u)) | (256u << ((b >> 3) & 7u)) | 0x10000u) * (b >> 7);
}

// PASSES: staging passes, (4 + 2 hh) / 2 region-row pairs.  RED: image += (float)total as a
// fire-and-forget float reduction at the L2 (round-to-nearest like the reference's add; it flushes
// subnormals, so the engine only selects it when no image value can be subnormal — sfc_upload).
template <int PASSES, bool RED>
__global__ void __launch_bounds__(kThreads, RED ? 4 : 2) k5_pairs_kernel(PairArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // (the tables are constants of the engine: they are staged while k-4 drains)
    const int t_entries = a.fh << a.fw;
    unsigned long long* const sT = reinterpret_cast<unsigned long long*>(smem_raw);
    PairEntry* const sE = reinterpret_cast<PairEntry*>(sT + t_entries);
    WarpScratch* const ws = reinterpret_cast<WarpScratch*>(sE + kSects * kGroupBits) + warp;
    uint32_t* const sSel = reinterpret_cast<uint32_t*>(reinterpret_cast<WarpScratch*>(sE + kSects * kGroupBits) + kWarps); // selector of every event byte
    for (int i = tid; i < 256; i += kThreads) sSel[i] = selector((uint32_t)i);
    for (int i = tid; i < t_entries; i += kThreads) sT[i] = a.T[i];
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.E);
        uint4* dst = reinterpret_cast<uint4*>(sE);
        for (int i = tid; i < kSects * kGroupBits * 2; i += kThreads) dst[i] = src[i];
    }
    __syncthreads();
    chain_wait();
    if (a.advance_tick && blockIdx.x == 0 && tid == 0 && a.ctl->error_code == 0) a.ctl->tick += 1;
    if (a.ctl->error_code != 0) return;

    const GridDev g = a.g;
    const int HW = a.hw, HH = a.hh, RW = a.rw, RH = a.rh;
    const uint32_t vmask = (1u << a.fw) - 1u;
    const uint16_t* const ev16 = reinterpret_cast<const uint16_t*>(a.ev);
    const bool listed = a.marks.epoch != nullptr;
    const int n_edge = listed ? tile_edge_count(a.marks) : 0;
    const long long n_tiles_todo = listed ? (long long)n_edge + a.ctl->active_count : 8ll * a.n_tiles; // (unlisted: items are blocks)
    const long long stride = (long long)gridDim.x * kWarps;
    const int sx = lane & 7, sy = lane >> 3;
    const int c = lane & 15, r0 = lane >> 4; // staging: lanes 0-15 the even region row of a pass, 16-31 the odd one

    // With the active-tile list, work items are TILES (a warp takes every stride-th one) and, within a tile,
    // the blocks some mover's field box touches (the stamp's block bits).  The tile id and stamp of the NEXT tile are loaded while
    // this tile's blocks are processed: the list -> stamp -> region chain of dependent loads is paid once
    // per tile, overlapped, not once per block.
    long long tile_item = (long long)blockIdx.x * kWarps + warp;
    auto tile_of = [&](long long t, uint32_t& mask) -> int { // tile id and its live-block mask
        mask = 0xFFu;
        if (t < n_edge) { // slab mode: tiles whose region reaches the halo rows are always processed
            const int r = (int)t / a.tiles_x;
            const int ty = r < a.marks.edge_lo ? r : a.marks.edge_hi + (r - a.marks.edge_lo);
            return ty * a.tiles_x + ((int)t - r * a.tiles_x);
        }
        const int tile = a.marks.list[t - n_edge];
        mask = (a.marks.epoch[tile] >> 8) & 0xFFu; // blocks within reach of a mover
        return tile;
    };
    int cur_tile = 0, pre_tile = 0;
    uint32_t cur_mask = 0u, pre_mask = 0u;
    bool pre_valid = listed && tile_item < n_tiles_todo;
    if (pre_valid) pre_tile = tile_of(tile_item, pre_mask);

    // Finds the next block that can hold work (inside the grid) and issues the loads of its region: two
    // region rows per pass.
    auto fetch = [&](int& x0, int& y0, uint32_t (&code)[PASSES]) -> bool {
        for (;;) {
            int b, tile;
            if (!listed) { // every block of every tile: spread block by block over the warps of the grid
                if (tile_item >= n_tiles_todo) return false;
                tile = (int)(tile_item >> 3);
                b = (int)(tile_item & 7);
                tile_item += stride;
            } else {
                if (cur_mask == 0u) { // next tile: adopt the prefetched one, start the prefetch of the one after
                    if (!pre_valid) return false;
                    cur_tile = pre_tile;
                    cur_mask = pre_mask;
                    tile_item += stride;
                    pre_valid = tile_item < n_tiles_todo;
                    if (pre_valid) pre_tile = tile_of(tile_item, pre_mask);
                    continue;
                }
                b = __ffs((int)cur_mask) - 1;
                cur_mask &= cur_mask - 1u;
                tile = cur_tile;
            }
            int tile_y = (int)__umulhi((unsigned)tile, a.inv_tiles_x), tile_x = tile - tile_y * a.tiles_x;
            if (tile_x >= a.tiles_x) {
                tile_x -= a.tiles_x;
                tile_y += 1;
            }
            x0 = tile_x * kMarkTileW + (b & 3) * kBlockW;
            y0 = g.row0 + tile_y * kMarkTileH + (b >> 2) * kBlockH;
            if (x0 >= g.W || y0 >= g.row0 + g.rows) continue;
            const int xs = x0 - HW, ys = y0 - HH;
            const int ly0 = ys - g.row0 + g.halo; // local row of the region's first row, if resident unwrapped
            const bool interior = xs >= 0 && xs + RW <= g.W && ys >= 0 && ys + RH <= g.H && ly0 >= 0 &&
                                  ly0 + RH <= g.rows + 2 * g.halo;
            if (interior) {
                const uint16_t* src = ev16 + ((long long)(ly0 + r0) * g.W + xs + c);
                const long long two_rows = 2ll * g.W;
#pragma unroll
                for (int p = 0; p < PASSES; ++p) {
                    code[p] = c < RW ? __ldg(src) : 0u;
                    src += two_rows;
                }
            } else {
#pragma unroll
                for (int p = 0; p < PASSES; ++p) {
                    const long long idx = c < RW ? cell_index(g, xs + c, ys + 2 * p + r0) : -1;
                    code[p] = idx >= 0 ? __ldg(ev16 + idx) : 0u;
                }
            }
            return true;
        }
    };

    // image += (float)total is a read-modify-write of a value nobody else touches: the load is
    // issued when a pair's totals are known and consumed one pair later, behind that pair's work
    float* pend_at[kKinds] = {nullptr, nullptr, nullptr};
    float pend_old[kKinds] = {0.f, 0.f, 0.f}, pend_add[kKinds] = {0.f, 0.f, 0.f};

    int x0 = 0, y0 = 0, nx0 = 0, ny0 = 0;
    uint32_t code[PASSES], next_code[PASSES];
    bool have = fetch(x0, y0, code);
    while (have) {
        // ---- stage: selectors of the event cells, one "has event" bit row per region row ----------
        __syncwarp(); // the previous block's pairs are done with the scratch
        uint32_t rows_nz = 0u;
#pragma unroll
        for (int p = 0; p < PASSES; ++p) {
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, code[p] != 0u);
            if (bal != 0u) { // (warp-uniform)
                if (code[p]) ws->sel[(2 * p + r0) * kPitch + c] = make_uint2(sSel[code[p] & 0xFFu], sSel[code[p] >> 8]);
                if (bal & 0xFFFFu) rows_nz |= 1u << (2 * p);
                if (bal >> 16) rows_nz |= 2u << (2 * p);
            }
            if (lane == 0) *reinterpret_cast<uint32_t*>(&ws->rb[2 * p]) = bal;
        }
        const int bx0 = x0, by0 = y0;
        have = fetch(nx0, ny0, next_code); // the next block's loads fly while this one is processed
        if (rows_nz != 0u) { // somebody moved within reach of this block
            __syncwarp();

            // ---- window word of my su: only region rows with an event contribute --------------------
            const bool valid = bx0 + sx < g.W && by0 + sy < g.row0 + g.rows;
            unsigned long long P = 0ull;
            for (uint32_t m = rows_nz; m; m &= m - 1u) {
                const int r = __ffs(m) - 1, d = r - sy;
                if (d >= 0 && d < a.fh) {
                    const uint32_t v = ((uint32_t)ws->rb[r] >> sx) & vmask;
                    if (v) P |= sT[(d << a.fw) + v];
                }
            }
            if (!valid) P = 0ull;
            ws->wm[lane] = P;

            // ---- list the (su, group) pairs that see an event ---------------------------------------
            uint32_t act; // bit q: byte q of P is non-zero
            {
                const uint32_t lo = (uint32_t)P, hi = (uint32_t)(P >> 32);
                const uint32_t nl = (((lo & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | lo) & 0x80808080u;
                const uint32_t nh = (((hi & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | hi) & 0x80808080u;
                act = (((nl >> 7) * 0x00204081u) >> 21 & 0xFu) | (((nh >> 7) * 0x00204081u) >> 17 & 0xF0u);
            }
            const int cnt = __popc(act);
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int up = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += up;
            }
            const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            int at = incl - cnt;
            while (act) {
                const int q = __ffs(act) - 1;
                act &= act - 1u;
                ws->wl[at++] = (uint8_t)((lane << 3) | q);
            }
            __syncwarp();

            // ---- fold the pairs ----------------------------------------------------------------------
            float* const rec0 = a.dyn + ((long long)(by0 - g.row0 + g.halo) * g.W + bx0) * (kKinds * kSects);
            for (int i = lane; i < total; i += 32) {
                const uint32_t pr = ws->wl[i];
                const int su = (int)(pr >> 3), grp = (int)(pr & 7u);
                uint32_t bits = (uint32_t)(ws->wm[su] >> (kGroupBits * grp)) & 0xFFu;
                const int ux = su & 7, uy = su >> 3;
                const uint2* const centre = ws->sel + (uy + HH) * kPitch + ux + HW;
                const PairEntry* const ent = sE + kGroupBits * grp;
                double tot[kKinds], pf[kKinds], pt[kKinds];
#pragma unroll
                for (int k = 0; k < kKinds; ++k) tot[k] = pf[k] = pt[k] = 0.0;
                int cls = 0;
                while (bits) {
                    const int q = __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const uint4 e0 = *reinterpret_cast<const uint4*>(ent + q);          // off_cls, masks, mag[0]
                    const double2 e1 = *(reinterpret_cast<const double2*>(ent + q) + 1); // mag[1], mag[2]
                    const int off = (int)(short)(e0.x & 0xFFFFu), ecls = (int)(e0.x >> 16);
                    const uint2 sl = centre[off];
                    if (ecls != cls) { // next slot class: fold the finished one, slot 2r then 2r + 1
#pragma unroll
                        for (int k = 0; k < kKinds; ++k) {
                            tot[k] = __dadd_rn(__dadd_rn(tot[k], pf[k]), pt[k]);
                            pf[k] = pt[k] = 0.0;
                        }
                        cls = ecls;
                    }
                    const uint32_t fbits = e0.y & sl.x, tbits = e0.y & sl.y; // gating the six terms is two ANDs
                    const double m0 = __hiloint2double((int)e0.w, (int)e0.z);
                    add_if(pf[0], -m0, fbits & 0xFFu);
                    add_if(pt[0], m0, tbits & 0xFFu);
                    add_if(pf[1], -e1.x, fbits & 0xFF00u);
                    add_if(pt[1], e1.x, tbits & 0xFF00u);
                    add_if(pf[2], -e1.y, fbits & 0xFF0000u);
                    add_if(pt[2], e1.y, tbits & 0xFF0000u);
                }
                float* const rec = rec0 + (uy * g.W + ux) * (kKinds * kSects);
#pragma unroll
                for (int k = 0; k < kKinds; ++k) {
                    if (!RED && pend_at[k]) *pend_at[k] = __fadd_rn(pend_old[k], pend_add[k]); // image += (float)total, engine.cpp:468
                    const double total_k = __dadd_rn(__dadd_rn(tot[k], pf[k]), pt[k]); // StepCache::total
                    const float add = __double2float_rn(total_k);
                    float* const at_k = rec + k * kSects + ((a.sect_packed[k] >> (3 * grp)) & 7u);
                    if (RED) {
                        if (add != 0.0f) atomicAdd(at_k, add); // (result unused: a RED, nothing to wait for)
                    } else {
                        pend_at[k] = nullptr;
                        if (add != 0.0f) {
                            pend_at[k] = at_k;
                            pend_old[k] = *at_k;
                            pend_add[k] = add;
                        }
                    }
                }
            }
        }
        x0 = nx0;
        y0 = ny0;
#pragma unroll
        for (int p = 0; p < PASSES; ++p) code[p] = next_code[p];
    }
    if (!RED) {
#pragma unroll
        for (int k = 0; k < kKinds; ++k)
            if (pend_at[k]) *pend_at[k] = __fadd_rn(pend_old[k], pend_add[k]);
    }
}

struct PairTablesHost {
    std::vector<unsigned long long> T;
    std::vector<PairEntry> E;
    uint32_t sect_packed[kKinds] = {};
    int fw = 0, fh = 0, hw = 0, hh = 0;
};

bool build_host_tables(const WalkListsHost& w, int chunk_k, PairTablesHost* out) {
    if (w.n <= 0 || w.hw > 4 || w.hh > (kRegionRowsMax - kBlockH) / 2) return false;
    const int fw = 2 * w.hw + 1, fh = 2 * w.hh + 1;
    if (((size_t)fh << fw) * sizeof(unsigned long long) > (32u << 10)) return false;
    for (int grp = 0; grp < kSects; ++grp)
        if (w.start[grp + 1] - w.start[grp] > kGroupBits) return false;
    PairTablesHost& t = *out;
    t.fw = fw;
    t.fh = fh;
    t.hw = w.hw;
    t.hh = w.hh;
    t.E.assign((size_t)kSects * kGroupBits, PairEntry{});
    std::vector<int> bit_of((size_t)fw * fh, -1);
    const int half = chunk_k / 2;
    for (int grp = 0; grp < kSects; ++grp) {
        const int len = w.start[grp + 1] - w.start[grp];
        std::vector<int> order((size_t)len);
        for (int j = 0; j < len; ++j) order[(size_t)j] = j;
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return x % half < y % half; }); // (j mod K/2, j)
        for (int q = 0; q < len; ++q) {
            const int j = order[(size_t)q], i = w.start[grp] + j;
            const int dx = (int)(w.meta[(size_t)i] & 0xFFu) - 128, dy = (int)((w.meta[(size_t)i] >> 8) & 0xFFu) - 128;
            PairEntry& e = t.E[(size_t)grp * kGroupBits + q];
            e.off_cls = (int)(((uint32_t)(dy * kPitch + dx) & 0xFFFFu) | ((uint32_t)(j % half) << 16));
            e.masks = w.masks[(size_t)i];
            for (int k = 0; k < kKinds; ++k) e.mag[k] = w.mag[(size_t)k * w.n + i];
            bit_of[(size_t)(dy + w.hh) * fw + dx + w.hw] = grp * kGroupBits + q;
        }
    }
    t.T.assign((size_t)fh << fw, 0ull);
    for (int d = 0; d < fh; ++d)
        for (uint32_t v = 0; v < (1u << fw); ++v) {
            unsigned long long bits = 0ull;
            for (int i = 0; i < fw; ++i)
                if (((v >> i) & 1u) && bit_of[(size_t)d * fw + i] >= 0) bits |= 1ull << bit_of[(size_t)d * fw + i];
            t.T[((size_t)d << fw) + v] = bits;
        }
    for (int k = 0; k < kKinds; ++k) {
        t.sect_packed[k] = 0u;
        for (int grp = 0; grp < kSects; ++grp) t.sect_packed[k] |= (uint32_t)(w.sect_of[k][grp] & 7) << (3 * grp);
    }
    return true;
}

size_t pairs_smem(const PairTables& t) {
    return (((size_t)t.fh << t.fw) * sizeof(unsigned long long) + sizeof(PairEntry) * kSects * kGroupBits +
            sizeof(WarpScratch) * kWarps + 256 * sizeof(uint32_t) + 15) & ~(size_t)15;
}

} // namespace

bool build_pair_tables(const WalkListsHost& w, int chunk_k, PairTables* out, std::vector<unsigned char>* blob) {
    PairTablesHost h;
    if (!build_host_tables(w, chunk_k, &h)) return false;
    const size_t t_bytes = h.T.size() * sizeof(unsigned long long), e_bytes = h.E.size() * sizeof(PairEntry);
    blob->assign(t_bytes + e_bytes, 0);
    std::memcpy(blob->data(), h.T.data(), t_bytes);
    std::memcpy(blob->data() + t_bytes, h.E.data(), e_bytes);
    *out = PairTables{};
    out->fw = h.fw;
    out->fh = h.fh;
    out->hw = h.hw;
    out->hh = h.hh;
    out->t_bytes = (long long)t_bytes;
    for (int k = 0; k < kKinds; ++k) out->sect_packed[k] = h.sect_packed[k];
    return true;
}

// Raises the kernel's dynamic shared-memory limit on the CURRENT device (the attribute is per
// device) and sizes the persistent grid.
template <int PASSES>
cudaError_t prepare_one(size_t smem, int sm_count, int* ctas) { // ctas[0]: plain read-modify-write, ctas[1]: RED
    static SmemGrant grant[2]; // (per kernel instantiation)
    cudaError_t e = grant[0].raise(reinterpret_cast<const void*>(k5_pairs_kernel<PASSES, false>), smem);
    if (e == cudaSuccess) e = grant[1].raise(reinterpret_cast<const void*>(k5_pairs_kernel<PASSES, true>), smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k5_pairs_kernel<PASSES, false>, kThreads, smem);
    if (e != cudaSuccess) return e;
    ctas[0] = sm_count * (per_sm > 0 ? per_sm : 1);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k5_pairs_kernel<PASSES, true>, kThreads, smem);
    if (e != cudaSuccess) return e;
    ctas[1] = sm_count * (per_sm > 0 ? per_sm : 1);
    return cudaSuccess;
}

template <int PASSES>
void launch_one(cudaStream_t s, const PairArgs& a, bool red, unsigned blocks, size_t smem) {
    if (red) launch_chained(k5_pairs_kernel<PASSES, true>, dim3(blocks), dim3(kThreads), smem, s, a);
    else launch_chained(k5_pairs_kernel<PASSES, false>, dim3(blocks), dim3(kThreads), smem, s, a);
}

cudaError_t prepare_k5_pairs(const PairTables& t, int sm_count, int* ctas) {
    const size_t smem = pairs_smem(t);
    switch (2 + t.hh) {
        case 2: return prepare_one<2>(smem, sm_count, ctas);
        case 3: return prepare_one<3>(smem, sm_count, ctas);
        case 4: return prepare_one<4>(smem, sm_count, ctas);
        case 5: return prepare_one<5>(smem, sm_count, ctas);
        case 6: return prepare_one<6>(smem, sm_count, ctas);
        case 7: return prepare_one<7>(smem, sm_count, ctas);
        case 8: return prepare_one<8>(smem, sm_count, ctas);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k5_pairs(cudaStream_t s, const K5Launch& l) {
    const PairTables& t = l.pairs;
    PairArgs a;
    a.g = l.g;
    a.dyn = l.dyn;
    a.ev = l.ev;
    a.ctl = l.ctl;
    a.marks = l.marks;
    a.T = reinterpret_cast<const unsigned long long*>(t.blob);
    a.E = reinterpret_cast<const PairEntry*>(t.blob + t.t_bytes);
    a.fw = t.fw;
    a.fh = t.fh;
    a.hw = t.hw;
    a.hh = t.hh;
    a.rw = kBlockW + 2 * t.hw;
    a.rh = kBlockH + 2 * t.hh;
    for (int k = 0; k < kKinds; ++k) a.sect_packed[k] = t.sect_packed[k];
    a.tiles_x = (l.g.W + kMarkTileW - 1) / kMarkTileW;
    a.n_tiles = a.tiles_x * ((l.g.rows + kMarkTileH - 1) / kMarkTileH);
    a.inv_tiles_x = (uint32_t)std::min<unsigned long long>(0x100000000ull / (unsigned long long)a.tiles_x, 0xFFFFFFFFull);
    a.advance_tick = l.advance_tick;
    const bool red = l.pairs_red != 0;
    long long blocks = l.pairs_ctas[red ? 1 : 0] > 0 ? l.pairs_ctas[red ? 1 : 0] : 148;
    if (a.marks.epoch == nullptr && blocks > a.n_tiles) blocks = a.n_tiles; // one CTA covers a tile per round
    if (blocks < 1) blocks = 1;
    const size_t smem = pairs_smem(t);
    switch (2 + t.hh) {
        case 2: launch_one<2>(s, a, red, (unsigned)blocks, smem); break;
        case 3: launch_one<3>(s, a, red, (unsigned)blocks, smem); break;
        case 4: launch_one<4>(s, a, red, (unsigned)blocks, smem); break;
        case 5: launch_one<5>(s, a, red, (unsigned)blocks, smem); break;
        case 6: launch_one<6>(s, a, red, (unsigned)blocks, smem); break;
        case 7: launch_one<7>(s, a, red, (unsigned)blocks, smem); break;
        case 8: launch_one<8>(s, a, red, (unsigned)blocks, smem); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

} // namespace sfc
