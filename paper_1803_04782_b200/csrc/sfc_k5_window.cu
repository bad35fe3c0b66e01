// sfc_k5_window.cu — k-5 write-back for sparse-to-moderate crowds (reference engine.cpp:428-472).
//
// The reference evaluates, for every (su, kind, sect) address, a list of F contributor offsets
// against the movement log: 6F probes per su whether anybody moved or not.  Here the unit of work
// is a WARP on a block of 8 x 4 su, taken from the tick's active-tile list (TileMarks, written by
// k-4: only the 32 x 8 tiles within field reach of a mover exist for this kernel; a tile is eight
// blocks).  Everything a warp touches is private to it — no block barriers, no atomics on the data
// path, nothing shared between warps but the read-only tables:
//
//   1. stage    the block + field-halo region of the 2-byte event map is read straight from global
//               memory (L1 / L2 hits: the map is small and neighbouring blocks overlap); the codes
//               go to the warp's shared memory, "is there an event" into one 64-bit word per region
//               column, and every event is appended to the warp's event list.
//   2. scatter  event by event (warp-uniform loop): the lanes enumerate the su of the block inside
//               the event's field box — all distinct, so plain shared-memory read-modify-writes —
//               and add the gated +-magnitudes of the three kinds to per-(su, kind, sect) doubles,
//               counting terms per address in three bit planes (>= 1, >= 2, >= 3 terms).
//               One or two terms per address are order-independent — whichever StepCache slots
//               they fall in, the reference's total is fl(t1 + t2) (IEEE addition commutes and
//               0.0 + t is exact) — so the event order does not matter here.
//   3. replay   an address with three or more terms is re-walked by the lane that owns the su
//               through the exact K-slot order (term idx -> slot idx mod K, slots folded in order,
//               accumulator.hpp:36-46): the lane slides over the column words of its window and
//               visits the set bits in (dx, dy) lexicographic order, which is the reference's
//               contributor-list order (fields.hpp:55-57).
//   4. apply    image += (float)total on the touched 32-byte sectors only.
//
// Tiles with many movers in reach (k-4 counts them in the tile's stamp) would have nearly every
// address re-walked: they are handed, whole, to the persistent dense gather kernel of
// sfc_k5_writeback.cu.
//
// Fields larger than the grid wrap onto themselves (test_engine.cpp:329-340): the region is staged
// in unwrapped coordinates, so one physical su can appear several times, exactly like the
// reference's while-loop wraps (engine.cpp:450-454).

#include <algorithm>
#include <cstdlib>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kWarps = 8;            // warps per CTA, each on its own blocks
constexpr int kThreads = kWarps * 32;
constexpr int kBlockW = 8, kBlockH = 4; // su block owned by one warp at a time (one su per lane)
constexpr int kBlocksPerTile = (kMarkTileW / kBlockW) * (kMarkTileH / kBlockH);
constexpr int kTabSmemMax = 768;     // table entries (all kinds) kept in shared memory
constexpr int kEvlCap = 48;          // event-list capacity per block (beyond it: every address is re-walked)
static_assert(kMarkTileW == 4 * kBlockW && kMarkTileH == 2 * kBlockH, "a tile is 4 x 2 blocks");

struct WinArgs {
    GridDev g;
    TablesDev t;
    float* dyn;
    const uint8_t* ev;
    Ctl* ctl;
    TileMarks marks;
    int* dense_list;
    int use_list;
    int mover_max;  // tiles with more movers in reach go to the dense gather
    int advance_tick;
    int rwb;        // block region columns: 8 + 2 * max_hw
    int rwp;        // row pitch of the staged codes (u16 units)
    int rhb;        // block region rows: 4 + 2 * max_hh (<= 64)
    int warp_bytes; // shared memory per warp
    int table_bytes;
};

struct WinShape {
    size_t smem;
    int rwb, rwp, rhb, warp_bytes, table_bytes, tab_smem;
};

bool same_box(const TablesDev& t) { // the three kinds share one field geometry
    return t.k[0].hw == t.k[1].hw && t.k[1].hw == t.k[2].hw && t.k[0].hh == t.k[1].hh && t.k[1].hh == t.k[2].hh;
}

constexpr int kAccBytes = kKinds * kSects * 32 * 8; // per warp: [kind * 8 + sect][lane] doubles
constexpr int kCntBytes = 32 * 16;                  // per warp: term-count bit planes per su

WinShape win_shape(const TablesDev& t) {
    WinShape s;
    s.rwb = kBlockW + 2 * t.max_hw;
    s.rwp = (s.rwb + 1) & ~1;
    s.rhb = kBlockH + 2 * t.max_hh;
    s.tab_smem = t.total_entries <= kTabSmemMax;
    s.table_bytes = s.tab_smem ? (int)(sizeof(double) * t.total_entries + sizeof(uint32_t) * 2 * ((t.total_entries + 3) & ~3)) : 0;
    s.table_bytes = (s.table_bytes + 15) & ~15;
    int wb = kAccBytes + kCntBytes;                         // accumulators + term counters
    wb += (int)sizeof(uint4) * kEvlCap;                     // event list
    wb += (int)sizeof(unsigned long long) * s.rwb;          // column words
    wb += (int)sizeof(long long) * s.rhb;                   // su index of each region row
    wb += 16;                                               // event counter
    wb += (int)sizeof(uint16_t) * s.rwp * s.rhb;            // event codes
    s.warp_bytes = (wb + 15) & ~15;
    s.smem = (size_t)s.table_bytes + (size_t)kWarps * s.warp_bytes;
    return s;
}

// One term (or the from/to pair of one cell) lands on the addresses in `m` (bit = kind * 8 + sect):
// saturating per-address term counts kept as three bit planes (>= 1, >= 2, >= 3 terms).
__device__ __forceinline__ void count_terms(uint4& planes, uint32_t m) {
    planes.z |= planes.y & m;
    planes.y |= planes.x & m;
    planes.x |= m;
}

// An event cell of a block's region: remember it in its column word and list it with the su of the
// block inside the largest field box around it.
__device__ __forceinline__ void list_event(unsigned long long* colw, uint4* evl, int* n_list, int c, int ry, uint32_t code, int HW,
                                        int HH, int bnx, int bny) {
    atomicOr(&colw[c], 1ull << ry);
    const int tx0 = max(c - 2 * HW, 0), tx1 = min(c, bnx - 1);
    const int ty0 = max(ry - 2 * HH, 0), ty1 = min(ry, bny - 1);
    if (tx1 < tx0 || ty1 < ty0) return;
    const uint32_t fb = code & 0xFFu, tb = code >> 8;
    const bool hf = fb & 0x80u, ht = tb & 0x80u;
    // per kind: orientation index of the from / to byte, 8 = no such event (bit 8 of an 8-bit
    // orientation mask is never set); kind 2 is non-directional: orientation 0
    const uint32_t f0 = hf ? (fb & 7u) : 8u, f1 = hf ? ((fb >> 3) & 7u) : 8u, f2 = hf ? 0u : 8u;
    const uint32_t t0 = ht ? (tb & 7u) : 8u, t1 = ht ? ((tb >> 3) & 7u) : 8u, t2 = ht ? 0u : 8u;
    const int at = atomicAdd(n_list, 1); // the scatter does not care about event order
    if (at < kEvlCap)
        evl[at] = make_uint4((uint32_t)c | ((uint32_t)ry << 9) | ((uint32_t)tx0 << 15) | ((uint32_t)tx1 << 18) |
                                 ((uint32_t)ty0 << 21) | ((uint32_t)ty1 << 23),
                             f0 | (t0 << 4) | (f1 << 8) | (t1 << 12) | (f2 << 16) | (t2 << 20),
                             hf ? ((1u << f0) | (256u << f1) | 0x10000u) : 0u, // selectors into the combined mask word
                             ht ? ((1u << t0) | (256u << t1) | 0x10000u) : 0u);
}

// FAST: the three kinds share one field geometry and the tables sit in shared memory — the common
// case (the scenario format has one field_geometry).  One combined word per offset then carries the
// sects and the orientation masks of all kinds, so gating the six possible terms of an (event, su)
// pair is two ANDs.
template <int K, bool TAB_SMEM, bool FAST>
__global__ void __launch_bounds__(kThreads, 3) k5_window_kernel(WinArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (a.advance_tick && blockIdx.x == 0 && tid == 0 && a.ctl->error_code == 0) a.ctl->tick += 1;
    if (a.ctl->error_code != 0) return;

    double* const s_mag = reinterpret_cast<double*>(smem_raw);
    uint32_t* const s_info = reinterpret_cast<uint32_t*>(s_mag + (TAB_SMEM ? a.t.total_entries : 0));
    uint32_t* const s_combo = s_info + (TAB_SMEM ? a.t.total_entries : 0); // [fw * fh] (FAST only)
    if (TAB_SMEM) { // contributor tables: one copy per CTA
        int base = 0;
        for (int k = 0; k < kKinds; ++k) {
            const int n = a.t.k[k].fw * a.t.k[k].fh;
            for (int i = tid; i < n; i += kThreads) {
                s_mag[base + i] = a.t.k[k].mag[i];
                s_info[base + i] = a.t.k[k].info[i];
            }
            base += n;
        }
        if (FAST) { // mask(kind 0) | mask(kind 1) << 8 | (kind 2 gated on orientation 0) << 16 | the three sects from bit 17
            const int n = a.t.k[0].fw * a.t.k[0].fh;
            for (int i = tid; i < n; i += kThreads) {
                const uint32_t i0 = a.t.k[0].info[i], i1 = a.t.k[1].info[i], i2 = a.t.k[2].info[i];
                const uint32_t m0 = (i0 >> 3) & 0xFFu, m1 = (i1 >> 3) & 0xFFu, m2 = (i2 >> 3) & 1u;
                s_combo[i] = m0 | (m1 << 8) | (m2 << 16) | ((i0 & 7u) << 17) | ((i1 & 7u) << 20) | ((i2 & 7u) << 23);
            }
        }
        __syncthreads(); // the only block barrier
    }
    unsigned char* const mine_smem = smem_raw + a.table_bytes + (size_t)warp * a.warp_bytes;
    double* const acc = reinterpret_cast<double*>(mine_smem) + lane;                              // [kind * 8 + sect] * 32
    uint4* const cnt = reinterpret_cast<uint4*>(mine_smem + kAccBytes);                           // [su of the block]
    uint4* const evl = cnt + 32;                                                                  // [kEvlCap]
    unsigned long long* const colw = reinterpret_cast<unsigned long long*>(evl + kEvlCap);       // [rwb]
    long long* const rowoff = reinterpret_cast<long long*>(colw + a.rwb);                         // [rhb] su index of the row's x = 0, -1 none
    int* const n_list = reinterpret_cast<int*>(rowoff + a.rhb);                                   // [4]
    uint16_t* const codes = reinterpret_cast<uint16_t*>(n_list + 4);                              // [rhb][rwp]

    const GridDev g = a.g;
    const int HW = a.t.max_hw, HH = a.t.max_hh;
    const int RWB = a.rwb, RWP = a.rwp;
    const bool narrow = RWB <= g.W; // one conditional add wraps x
    const unsigned long long hmask = (2 * HH + 1) >= 64 ? ~0ull : ((1ull << (2 * HH + 1)) - 1ull);
    const uint16_t* const ev16 = reinterpret_cast<const uint16_t*>(a.ev);
    const int tiles_x = a.marks.tiles_x;
    const int n_edge = a.use_list ? tile_edge_count(a.marks) : 0;
    const long long n_items =
        (long long)kBlocksPerTile * (a.use_list ? n_edge + a.ctl->active_count : tiles_x * a.marks.tiles_y);
    const unsigned stamp = a.ctl->epoch;
    const int tb1 = a.t.k[0].fw * a.t.k[0].fh, tb2 = tb1 + a.t.k[1].fw * a.t.k[1].fh; // table bases of kinds 1, 2
    const unsigned inv_rwb = 0xFFFFFFFFu / (unsigned)RWB + 1u;
    const int lx = lane & (kBlockW - 1), ly = lane >> 3; // my su in the block

    for (long long item = (long long)blockIdx.x * kWarps + warp; item < n_items; item += (long long)gridDim.x * kWarps) {
        const int titem = (int)(item / kBlocksPerTile), blk = (int)(item - (long long)titem * kBlocksPerTile);
        int tile;
        if (!a.use_list) {
            tile = titem;
        } else if (titem < n_edge) { // slab mode: tiles whose region reaches the halo rows
            const int r = titem / tiles_x;
            const int ty = r < a.marks.edge_lo ? r : a.marks.edge_hi + (r - a.marks.edge_lo);
            tile = ty * tiles_x + (titem - r * tiles_x);
        } else {
            tile = a.marks.list[titem - n_edge];
        }
        if (a.use_list && titem >= n_edge) { // a listed tile: k-4 counted the movers and noted the blocks within reach
            const unsigned word = a.marks.epoch[tile];
            if ((word >> 16) == stamp) {
                if (a.mover_max < (int)kMarkCountMax && (int)(word & kMarkCountMax) > a.mover_max) { // dense: exact kernel
                    if (blk == 0 && lane == 0) a.dense_list[atomicAdd(&a.ctl->dense_count, 1)] = tile;
                    continue;
                }
                if (!((word >> (8 + blk)) & 1u)) continue; // no mover's field box touches this block
            }
        }
        const int tile_y = tile / tiles_x, tile_x = tile - tile_y * tiles_x;
        const int bx0 = tile_x * kMarkTileW + (blk & 3) * kBlockW;             // first su column of my block
        const int by0 = g.row0 + tile_y * kMarkTileH + (blk >> 2) * kBlockH;   // ... global row
        const int bnx = min(kBlockW, g.W - bx0), bny = min(kBlockH, g.row0 + g.rows - by0);
        if (bnx <= 0 || bny <= 0) continue; // the block lies outside the grid (partial tile)
        const int RH = bny + 2 * HH;
        const int xs = bx0 - HW, ys = by0 - HH;

        // ---- stage ---------------------------------------------------------------------------
        __syncwarp(); // the previous block is done with the staging buffers
        for (int ry = lane; ry < RH; ry += 32) rowoff[ry] = cell_index(g, 0, ys + ry); // -1: no such row / not resident
        for (int c = lane; c < RWB; c += 32) colw[c] = 0ull;
        if (lane == 0) *n_list = 0;
        __syncwarp();
        auto found = [&](int c, int ry, uint32_t code) { list_event(colw, evl, n_list, c, ry, code, HW, HH, bnx, bny); };
        auto column_x = [&](int c) -> int { // physical x of a region column, -1 when it does not exist
            int x = xs + c;
            if (g.closed) return (x >= 0 && x < g.W) ? x : -1;
            if (narrow) return x + (x < 0 ? g.W : (x >= g.W ? -g.W : 0));
            return emod(x, g.W);
        };
        {
            const int n_cells = RWB * RH;
            for (int i0 = 0; i0 < n_cells; i0 += 8 * 32) {
                uint32_t got[8];
                int cq[8], rq[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) { // the loads of the chunk fly together
                    const int i = i0 + q * 32 + lane;
                    got[q] = 0u;
                    cq[q] = -1;
                    if (i < n_cells) {
                        rq[q] = (int)__umulhi((unsigned)i, inv_rwb); // i / RWB
                        cq[q] = i - rq[q] * RWB;
                        const int x = column_x(cq[q]);
                        const long long ro = rowoff[rq[q]];
                        if (ro >= 0 && x >= 0) got[q] = __ldg(ev16 + ro + x);
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (cq[q] < 0) continue;
                    codes[rq[q] * RWP + cq[q]] = (uint16_t)got[q];
                    if (got[q] != 0u) found(cq[q], rq[q], got[q]);
                }
            }
        }
        __syncwarp();
        const int n_events = *n_list;
        if (n_events == 0) continue; // nobody within reach of this block
        const bool mine = lx < bnx && ly < bny;
        uint4 planes = make_uint4(0u, 0u, 0u, 0u);

        if (n_events <= kEvlCap) {
            // ---- scatter ---------------------------------------------------------------------
#pragma unroll
            for (int i = 0; i < kKinds * kSects; ++i) acc[i * 32] = 0.0;
            cnt[lane] = make_uint4(0u, 0u, 0u, 0u);
            __syncwarp();
            for (int e = 0; e < n_events; ++e) {
                const uint4 evt = evl[e]; // broadcast
                const int tx0 = (int)((evt.x >> 15) & 7u), tx1 = (int)((evt.x >> 18) & 7u);
                const int ty0 = (int)((evt.x >> 21) & 3u), ty1 = (int)((evt.x >> 23) & 3u);
                const int w = tx1 - tx0 + 1, h = ty1 - ty0 + 1;
                const int ec = (int)(evt.x & 511u), er = (int)((evt.x >> 9) & 63u);
                // at most 8 x 4 su: one pass, lane i -> (i % w, i / w)
                const int iy = (lane >= w) + (lane >= 2 * w) + (lane >= 3 * w);
                if (lane < w * h) {
                    const int tx = tx0 + lane - iy * w, ty = ty0 + iy;
                    const int dx = ec - HW - tx, dy = er - HH - ty; // centre offset = mover - target
                    const int su = ty * kBlockW + tx;
                    double* const my = acc - lane + su; // accumulators of that su
                    if (FAST) {
                        const int tl = (dy + HH) * (2 * HW + 1) + dx + HW;
                        const uint32_t combo = s_combo[tl];
                        const uint32_t fbits = combo & evt.z, tbits = combo & evt.w; // gated terms, all kinds
                        if ((fbits | tbits) != 0u) { // (else: the centre offset, offsets outside the support, other orientations)
                            uint32_t mf = 0u, mt = 0u;
#pragma unroll
                            for (int k = 0; k < kKinds; ++k) {
                                const uint32_t km = k == 0 ? 0xFFu : (k == 1 ? 0xFF00u : 0x10000u);
                                const bool from = fbits & km, to = tbits & km;
                                const int a24 = k * kSects + (int)((combo >> (17 + 3 * k)) & 7u); // (a repulsive kind points the other way)
                                if (from) mf |= 1u << a24;
                                if (to) mt |= 1u << a24;
                                // one or two terms in all: the plain sum IS the reference's total; more: replayed below
                                if (from != to) {
                                    const double mag = s_mag[(k == 0 ? 0 : (k == 1 ? tb1 : tb2)) + tl];
                                    my[a24 * 32] = __dadd_rn(my[a24 * 32], from ? -mag : mag); // (-mag + mag would add +0.0)
                                }
                            }
                            uint4 pl = cnt[su];
                            count_terms(pl, mf);
                            count_terms(pl, mt);
                            cnt[su] = pl;
                        }
                    } else {
                        uint4 pl = cnt[su];
                        int tbase = 0;
#pragma unroll
                        for (int k = 0; k < kKinds; ++k) {
                            const KindTableDev& kt = a.t.k[k];
                            const int tb = tbase;
                            tbase += kt.fw * kt.fh;
                            if (dx < -kt.hw || dx > kt.hw || dy < -kt.hh || dy > kt.hh) continue;
                            const int tl = (dy + kt.hh) * kt.fw + dx + kt.hw;
                            const uint32_t info = TAB_SMEM ? s_info[tb + tl] : __ldg(kt.info + tl);
                            const uint32_t mask = (info >> 3) & 0xFFu;
                            const bool from = (mask >> ((evt.y >> (8 * k)) & 15u)) & 1u, to = (mask >> ((evt.y >> (8 * k + 4)) & 15u)) & 1u;
                            if (!from && !to) continue; // (also the centre offset and offsets outside the support: mask 0)
                            const int a24 = k * kSects + (int)(info & 7u);
                            if (from != to) {
                                const double mag = TAB_SMEM ? s_mag[tb + tl] : __ldg(kt.mag + tl);
                                my[a24 * 32] = __dadd_rn(my[a24 * 32], from ? -mag : mag);
                            }
                            if (from) count_terms(pl, 1u << a24);
                            if (to) count_terms(pl, 1u << a24);
                        }
                        cnt[su] = pl;
                    }
                }
                __syncwarp(); // the next event may touch the same su from another lane
            }
            if (mine) planes = cnt[lane];
        } else if (mine) {
            // more events than the list holds (a crowded block of a tile k-4 could not count, e.g. at a
            // slab edge): every address of every su goes through the exact walk
            planes.x = planes.z = 0xFFFFFFu;
        }

        // ---- replay + apply (lane: my su) ------------------------------------------------------
        if (__ballot_sync(0xFFFFFFFFu, planes.x != 0u) == 0u) continue; // nothing reached this block
        float4 v[kKinds][2];
        float4* rec = nullptr;
        if (planes.x != 0u) { // request the touched sectors now: they fly while the replay runs
            rec = reinterpret_cast<float4*>(a.dyn + (rowoff[ly + HH] + bx0 + lx) * (kKinds * kSects));
#pragma unroll
            for (int k = 0; k < kKinds; ++k) {
                if (((planes.x >> (8 * k)) & 0xFFu) == 0u) continue;
                v[k][0] = rec[2 * k];
                v[k][1] = rec[2 * k + 1];
            }
        }
        {
            uint32_t m3 = planes.z; // addresses with three or more terms: exact K-slot order
            while (m3 != 0u) {
                const int a24 = __ffs((int)m3) - 1;
                m3 &= m3 - 1u;
                const int kind = a24 >> 3, sect = a24 & 7;
                const KindTableDev& kt = a.t.k[kind];
                const int tb = kind == 0 ? 0 : (kind == 1 ? tb1 : tb2);
                const int shift = kind == 0 ? 0 : (kind == 1 ? 3 : 8); // kind 2: orientation 0 of an all-ones mask
                double p[K];
                unsigned used = 0u;
                int cc = HW - kt.hw - 1;
                const int cc_last = HW + kt.hw;
                unsigned long long bits = 0ull;
                for (;;) { // my window's events, column by column, rows ascending
                    while (bits == 0ull && cc < cc_last) {
                        ++cc;
                        bits = (colw[lx + cc] >> ly) & hmask;
                    }
                    if (bits == 0ull) break;
                    const int dyp = __ffsll((long long)bits) - 1;
                    bits &= bits - 1ull;
                    const int dx = cc - HW, dy = dyp - HH;
                    if (dy < -kt.hh || dy > kt.hh) continue;
                    const int tl = (dy + kt.hh) * kt.fw + dx + kt.hw;
                    const uint32_t info = TAB_SMEM ? s_info[tb + tl] : __ldg(kt.info + tl);
                    const uint32_t mask = (info >> 3) & 0xFFu;
                    if (mask == 0u || (int)(info & 7u) != sect) continue;
                    const uint32_t code = codes[(ly + dyp) * RWP + lx + cc];
                    const uint32_t fb = code & 0xFFu, tbyte = code >> 8;
                    const bool from = (fb & 0x80u) && ((mask >> ((fb >> shift) & 7u)) & 1u);
                    const bool to = (tbyte & 0x80u) && ((mask >> ((tbyte >> shift) & 7u)) & 1u);
                    if (!from && !to) continue;
                    const double mag = TAB_SMEM ? s_mag[tb + tl] : __ldg(kt.mag + tl);
                    const uint32_t j2 = (info >> 11) << 1;
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) { // from-term (idx 2j) then to-term (idx 2j+1)
                        if (!(hf == 0 ? from : to)) continue;
                        const int slot = (int)((j2 + hf) & (K - 1));
                        const double term = hf == 0 ? -mag : mag;
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
                acc[a24 * 32] = total;
            }
        }
        if (planes.x != 0u) { // image += (float)total, one 32-byte sector per touched (su, kind)
#pragma unroll
            for (int k = 0; k < kKinds; ++k) {
                const uint32_t km = (planes.x >> (8 * k)) & 0xFFu;
                if (km == 0u) continue;
                float f[8] = {v[k][0].x, v[k][0].y, v[k][0].z, v[k][0].w, v[k][1].x, v[k][1].y, v[k][1].z, v[k][1].w};
#pragma unroll
                for (int sct = 0; sct < kSects; ++sct)
                    if ((km >> sct) & 1u) f[sct] = __fadd_rn(f[sct], __double2float_rn(acc[(k * kSects + sct) * 32]));
                rec[2 * k] = make_float4(f[0], f[1], f[2], f[3]);
                rec[2 * k + 1] = make_float4(f[4], f[5], f[6], f[7]);
            }
        }
    }
}

template <int K, bool TAB_SMEM, bool FAST>
cudaError_t prepare_one(const WinShape& sh, int sm_count, int* ctas) {
    static SmemGrant grant; // (one per kernel instantiation)
    cudaError_t e = grant.raise(reinterpret_cast<const void*>(k5_window_kernel<K, TAB_SMEM, FAST>), sh.smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k5_window_kernel<K, TAB_SMEM, FAST>, kThreads, sh.smem);
    if (e != cudaSuccess) return e;
    *ctas = sm_count * (per_sm > 0 ? per_sm : 1);
    return cudaSuccess;
}

template <int K>
cudaError_t prepare_k(const TablesDev& t, int /*ev_max*/, int sm_count, int* ctas) {
    const WinShape sh = win_shape(t);
    if (sh.tab_smem && same_box(t)) return prepare_one<K, true, true>(sh, sm_count, ctas);
    return sh.tab_smem ? prepare_one<K, true, false>(sh, sm_count, ctas) : prepare_one<K, false, false>(sh, sm_count, ctas);
}

template <int K>
cudaError_t launch_k(cudaStream_t stream, const K5Launch& l) {
    const WinShape sh = win_shape(l.t);
    WinArgs a;
    a.g = l.g;
    a.t = l.t;
    a.dyn = l.dyn;
    a.ev = l.ev;
    a.ctl = l.ctl;
    a.marks = l.marks;
    a.dense_list = l.dense_list;
    a.use_list = l.marks.epoch != nullptr;
    a.mover_max = l.ev_max < 0 ? 0 : l.ev_max / 2; // a mover is two events
    a.advance_tick = l.advance_tick;
    a.rwb = sh.rwb;
    a.rwp = sh.rwp;
    a.rhb = sh.rhb;
    a.warp_bytes = sh.warp_bytes;
    a.table_bytes = sh.table_bytes;
    static const int knob = std::getenv("SFC_K5_WINDOW_CTAS") ? std::atoi(std::getenv("SFC_K5_WINDOW_CTAS")) : 0;
    long long blocks = (long long)l.marks.tiles_x * l.marks.tiles_y * kBlocksPerTile / kWarps + 1;
    const int cap = knob > 0 ? knob : (l.window_ctas > 0 ? l.window_ctas : 148);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (sh.tab_smem && same_box(l.t))
        k5_window_kernel<K, true, true><<<(unsigned)blocks, kThreads, sh.smem, stream>>>(a);
    else if (sh.tab_smem)
        k5_window_kernel<K, true, false><<<(unsigned)blocks, kThreads, sh.smem, stream>>>(a);
    else
        k5_window_kernel<K, false, false><<<(unsigned)blocks, kThreads, sh.smem, stream>>>(a);
    return cudaGetLastError();
}

} // namespace

// The window kernel keeps one 64-bit word per region column (4 + 2*hh rows) and packs region
// coordinates into 9 + 6 bits; larger fields take the chunked gather of sfc_k5_writeback.cu.
bool k5_window_supported(const TablesDev& t) {
    if (kBlockH + 2 * t.max_hh > 64 || kBlockW + 2 * t.max_hw > 512) return false;
    return win_shape(t).smem <= 220 * 1024;
}

cudaError_t prepare_k5_window(int chunk_k, const TablesDev& t, int ev_max, int sm_count, int* ctas) {
    if (!k5_window_supported(t)) return cudaSuccess;
    switch (chunk_k) {
        case 2: return prepare_k<2>(t, ev_max, sm_count, ctas);
        case 4: return prepare_k<4>(t, ev_max, sm_count, ctas);
        case 8: return prepare_k<8>(t, ev_max, sm_count, ctas);
        case 16: return prepare_k<16>(t, ev_max, sm_count, ctas);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k5_window(cudaStream_t s, const K5Launch& l) {
    switch (l.chunk_k) {
        case 2: return launch_k<2>(s, l);
        case 4: return launch_k<4>(s, l);
        case 8: return launch_k<8>(s, l);
        case 16: return launch_k<16>(s, l);
        default: return cudaErrorInvalidValue;
    }
}

} // namespace sfc
