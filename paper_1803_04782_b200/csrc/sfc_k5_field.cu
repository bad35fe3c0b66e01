// sfc_k5_field.cu — k-5 write-back for LARGE fields (beyond 15 x 15: BASELINE configs 3 and 5,
// the paper's 21^2 ... 77^2 sweep), every crowd density.
// Reference: k5_writeback_range + StepCache (engine.cpp:428-472, accumulator.hpp:36-46).
//
// The reference walks, for every (su, kind, sect) address, that sect's contributor list (F offsets,
// two mask probes each) and adds the gated terms to K f64 partials: term idx -> partial idx mod K,
// idx = 2 j for the "left" term and 2 j + 1 for the "arrived" term of list position j; partials
// folded in slot order, cast to float, added to the image.  Here the non-zero terms are found from
// the EVENTS instead:
//
//   tile      a CTA of NW warps owns a tile of NW blocks of 8 x 2 su (32 x 2 / 32 x 4 / 32 x 8 su), one
//             block per warp for the whole life of the tile.  A su is served by TWO lanes: lane l < 16
//             adds its "left" terms (even StepCache slots), lane l + 16 its "arrived" terms (odd slots)
//             — the two never share a partial, so a warp consumes one left event and one arrived event
//             per step and needs half the partials per lane: twice the warps for the same shared memory.
//   stage     the tile + field-halo region of the 2-byte event map is read once with 16-byte loads
//             (eight cells); cells somebody left / arrived at set a bit in per-column bit maps in shared
//             memory.  A popcount scan over the columns gives every event its place in the (x, y)-sorted
//             left / arrived event lists — the reference's contributor-list order for every su of the
//             tile, because the lists are sorted lexicographically by centre offset (fields.hpp:55-57).
//   stream    the lists are materialised in column chunks of at most `cap` events each (normally one
//             chunk) and walked by every warp with a WARP-UNIFORM trip count: lanes differ only in the
//             offset they see.  Per (event, lane): one table byte (sect group * K + StepCache slot), one
//             orientation-mask word per group, the magnitude from a quadrant-folded f64 table (|dx|,
//             |dy|: the magnitudes are symmetric, checked on the host) — all in shared memory — then one
//             f64 read-modify-write per gated term on the lane's own partials, laid out
//             [kind][group][slot / 2][lane] (bank = lane: conflict-free whatever the slot).  The
//             partials persist across chunks, so nothing is ever re-staged; the three kinds share one
//             walk (NK = 3) when their partials fit, else one walk per kind (NK = 1).
//   fold      StepCache::total per (kind, sect) in slot order — alternating between the su's two lanes'
//             partials —, image += (float)total; each lane of the pair folds four sects of every kind.
//
// Zero terms are never materialised (x + +-0.0 = x), empty partials hold +0.0 (0.0 + p = p, and a
// partial is never -0.0), so the bits are the reference's.  LAZY variants (thin crowds) create a
// partial on its first term under a per-lane dirty mask instead of clearing all of them per block.
// Fields larger than the grid wrap onto themselves: the region is staged in unwrapped coordinates
// (engine.cpp:450-454).

#include <algorithm>
#include <cstring>
#include <vector>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kBlockW = 8, kBlockH = 2;
constexpr int kTileW = 32;
constexpr int kMaxThreads = 512;
constexpr size_t kSmemLimit = 227u << 10;
constexpr uint32_t kNoEntry = 0xFFu;

// One movement event as the walks see it (8 bytes): a cell somebody LEFT (term -magnitude, StepCache
// idx 2 j) or ARRIVED at (term +magnitude, idx 2 j + 1) — the two kinds live in separate lists.
//   x: one-hot orientation selectors, kind k in byte k (kind 2: bit 16) | region row << 17
//   y: region column
typedef uint2 FieldEvent;

struct FieldArgs {
    GridDev g;
    float* dyn;
    const uint8_t* ev;
    Ctl* ctl;
    const unsigned char* blob;    // tab8 | mag tables | lut
    int tab_bytes, mag_bytes;
    int fw, fh, hw, hh, ms;       // ms: row stride of a folded magnitude table (doubles)
    int mag_stride;               // doubles per magnitude table
    int mag_of[kKinds];           // magnitude table of kind k
    uint32_t group_of_sect[kKinds]; // sect group feeding sect s of kind k in bits [3s, 3s + 3)
    int tiles_x, n_tiles, tile_h;
    int rw_max, nwords;           // region columns of a full tile; 32-bit words per column bit map
    int cs_ints;                  // ints of the column-start block (two arrays of rw_max + 2; at least one per region row)
    int cap;                      // entries per list chunk (each of the two lists)
    int advance_tick;
    int vec_ok;                   // 16-byte event-map loads are aligned (W % 8 == 0)
};

__device__ __forceinline__ uint32_t selector(uint32_t b) { // one-hot orientation per kind byte, 0 without an event
    return ((1u << (b & 7u)) | (256u << ((b >> 3) & 7u)) | 0x10000u) * (b >> 7);
}

// ONE_MAG: the kinds of a walk share one magnitude table (always true for NK == 1).
template <int K, int NK, bool LAZY, bool ONE_MAG>
__global__ void __launch_bounds__(NK == 3 ? 256 : kMaxThreads) k5_field_kernel(FieldArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int KH = K / 2;                // partials per (kind, group) and lane: the even or the odd slots
    constexpr int KO = kSects * KH * 32;     // partial doubles per kind and warp
#ifndef SFC_FIELD_EV
#define SFC_FIELD_EV (LAZY ? 2 : (NK == 3 ? 8 : 4))
#endif
    constexpr int EV = SFC_FIELD_EV;         // events a lane looks up before it folds any of them
    constexpr int PW = NK * KO;              // ... per warp
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5;

    // ---- shared memory ------------------------------------------------------------------------
    double* const part_all = reinterpret_cast<double*>(smem_raw);
    double* const smag = part_all + (size_t)NW * PW;
    FieldEvent* const evl = reinterpret_cast<FieldEvent*>(smag + a.mag_bytes / 8); // [left: cap | arrived: cap]
    uint32_t* const colbits = reinterpret_cast<uint32_t*>(evl + 2 * a.cap);        // [column][left words | arrived words]
    int* const colstart = reinterpret_cast<int*>(colbits + a.rw_max * 2 * a.nwords); // [left: rw_max + 2 | arrived: rw_max + 2]
    uint32_t* const lut = reinterpret_cast<uint32_t*>(colstart + a.cs_ints);
    int* const rowlocal = colstart; // staging only (before the scan writes colstart): resident row of each region row, -1: no such row
    uint8_t* const tab8 = reinterpret_cast<uint8_t*>(lut + kSects);
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(a.blob);
        uint32_t* dst = reinterpret_cast<uint32_t*>(tab8);
        for (int i = tid; i < a.tab_bytes / 4; i += NT) dst[i] = src[i];
        const double* msrc = reinterpret_cast<const double*>(a.blob + a.tab_bytes);
        for (int i = tid; i < a.mag_bytes / 8; i += NT) smag[i] = msrc[i];
        if (tid < kSects) lut[tid] = reinterpret_cast<const uint32_t*>(a.blob + a.tab_bytes + a.mag_bytes)[tid];
    }
    __syncthreads();
    chain_wait(); // (the tables above are constants of the engine, staged while k-4 drains)
    if (a.advance_tick && blockIdx.x == 0 && tid == 0 && a.ctl->error_code == 0) a.ctl->tick += 1;
    if (a.ctl->error_code != 0) return;

    const GridDev g = a.g;
    const int HW = a.hw, HH = a.hh, FW = a.fw, MS = a.ms, NWORDS = a.nwords, CW = 2 * a.nwords;
    const int CS = a.rw_max + 2; // stride between the two column-start arrays
    const uint16_t* const ev16 = reinterpret_cast<const uint16_t*>(a.ev);
    double* const part = part_all + (size_t)warp * PW + lane;
    const int half = lane >> 4;                        // 0: this lane adds "left" terms, 1: "arrived" terms
    const int bx = (warp & 3) * kBlockW, by = (warp >> 2) * kBlockH;
    const int sx = lane & 7, sy = (lane >> 3) & 1;
    const int flip = half ? 0 : (int)0x80000000u;      // left: -magnitude

    for (int tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int tile_y = tile / a.tiles_x, tile_x = tile - tile_y * a.tiles_x;
        const int x0 = tile_x * kTileW, y0 = g.row0 + tile_y * a.tile_h;
        const int nx = min(kTileW, g.W - x0), ny = min(a.tile_h, g.row0 + g.rows - y0);
        const int RW = nx + 2 * HW, RH = ny + 2 * HH;
        const int xs = x0 - HW, ys = y0 - HH;

        // ---- stage: per-column bit maps of the region's events ---------------------------------
        for (int i = tid; i < RW * CW; i += NT) colbits[i] = 0u;
        for (int ry = tid; ry < RH; ry += NT) {
            const long long at = cell_index(g, 0, ys + ry);
            rowlocal[ry] = at < 0 ? -1 : (int)(at / g.W);
        }
        __syncthreads();
        {
            const int gx0 = (xs >> 3) * 8; // (arithmetic shift: floor for negative xs)
            const int NG = (xs + RW - gx0 + 7) >> 3;
            const int items = RH * NG;
            const unsigned inv_ng = NG > 1 ? 0xFFFFFFFFu / (unsigned)NG + 1u : 0u; // i / NG for i < 2^16
            constexpr int Q = 4;
            for (int i0 = 0; i0 < items; i0 += Q * NT) {
                uint4 got[Q];
                int at_ry[Q], at_gx[Q];
                bool slow[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const int i = i0 + q * NT + tid;
                    got[q] = make_uint4(0u, 0u, 0u, 0u);
                    at_ry[q] = -1;
                    slow[q] = false;
                    if (i < items) {
                        const int ry = NG > 1 ? (int)__umulhi((unsigned)i, inv_ng) : i;
                        const int gx = gx0 + 8 * (i - ry * NG);
                        at_ry[q] = ry;
                        at_gx[q] = gx;
                        const long long row = (long long)rowlocal[ry] * g.W; // negative: the row does not exist / is not resident
                        if (row < 0) {
                            at_ry[q] = -1;
                        } else if (a.vec_ok && gx >= 0 && gx + 8 <= g.W) {
                            got[q] = __ldg(reinterpret_cast<const uint4*>(ev16 + row + gx));
                        } else {
                            slow[q] = true;
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    if (at_ry[q] < 0) continue;
                    const int ry = at_ry[q], gx = at_gx[q];
                    const uint32_t bit = 1u << (ry & 31);
                    uint32_t* const word = colbits + (ry >> 5);
                    if (slow[q]) { // group across the grid's x edge, or an unaligned row: cell by cell
#pragma unroll 1
                        for (int i = 0; i < 8; ++i) {
                            const int col = gx + i - xs;
                            if (col < 0 || col >= RW) continue;
                            const long long idx = cell_index(g, gx + i, ys + ry);
                            const uint32_t code = idx >= 0 ? (uint32_t)__ldg(ev16 + idx) : 0u;
                            if (code & 0xFFu) atomicOr(word + col * CW, bit);
                            if (code >> 8) atomicOr(word + col * CW + NWORDS, bit);
                        }
                    } else if ((got[q].x | got[q].y | got[q].z | got[q].w) != 0u) {
                        const uint32_t w4[4] = {got[q].x, got[q].y, got[q].z, got[q].w};
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const uint32_t code = (w4[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
                            const int col = gx + i - xs;
                            if (code != 0u && col >= 0 && col < RW) {
                                if (code & 0xFFu) atomicOr(word + col * CW, bit);
                                if (code >> 8) atomicOr(word + col * CW + NWORDS, bit);
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (warp < 2) { // exclusive column starts of the left (warp 0) and arrived (warp 1) lists: popcount scans
            for (int t = warp; t < 2; t += NW) {
                int* const cs = colstart + t * CS;
                int carry = 0;
                for (int c0 = 0; c0 < RW; c0 += 32) {
                    const int c = c0 + lane;
                    int v = 0;
                    if (c < RW)
                        for (int w = 0; w < NWORDS; ++w) v += __popc(colbits[c * CW + t * NWORDS + w]);
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int u = __shfl_up_sync(0xFFFFFFFFu, v, o);
                        if (lane >= o) v += u;
                    }
                    if (c < RW) cs[c + 1] = v + carry;
                    carry += __shfl_sync(0xFFFFFFFFu, v, 31);
                }
                if (lane == 0) cs[0] = 0;
            }
        }
        __syncthreads();
        const int n_left = colstart[RW], n_arrived = colstart[CS + RW];
        if (n_left + n_arrived == 0) { // nobody moved within reach of this tile (uniform)
            __syncthreads();           // (the next tile's row table reuses the column-start block every thread just read)
            continue;
        }

        // ---- my block --------------------------------------------------------------------------
        const bool blk_ok = bx < nx && by < ny; // uniform per warp
        const int cx = bx + sx, cy = by + sy;
        const bool in_grid = blk_ok && cx < nx && cy < ny;
        const int tcx = cx + HW, tcy = cy + HH; // my su in region coordinates
        const int col_lo = bx, col_hi = min(bx + kBlockW + 2 * HW, RW); // region columns within the block's reach
        const bool blk_live = blk_ok && (colstart[col_hi] > colstart[col_lo] || colstart[CS + col_hi] > colstart[CS + col_lo]);
        const bool single = n_left <= a.cap && n_arrived <= a.cap;
        // table byte of the offset (event - my su): tabp[ry * FW + rc]; one magnitude row per |dy|
        const uint8_t* const tabp = tab8 + ((HH - tcy) * FW + (HW - tcx));
        const unsigned span_x = 2u * (unsigned)HW, span_y = 2u * (unsigned)HH;
        const FieldEvent* const my_list = evl + half * a.cap;
        const int* const my_cs = colstart + half * CS;
        // my half (four sects) of my su's 96-byte record
        float* const rec = a.dyn + (in_grid ? cell_index(g, x0 + cx, y0 + cy) : 0) * (kKinds * kSects) + 4 * half;

#pragma unroll 1
        for (int kp = 0; kp < kKinds / NK; ++kp) {
            unsigned long long dirty[NK]; // LAZY: partials created so far, bit = group * K/2 + slot / 2
            bool any = false;
            const double* mtab[NK]; // kind k's magnitude table
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                mtab[k] = smag + a.mag_of[NK == 1 ? kp : k] * a.mag_stride;
                dirty[k] = 0ull;
            }
            const uint32_t kmask = NK == 3 ? 0x1FFFFu : (kp == 0 ? 0xFFu : (kp == 1 ? 0xFF00u : 0x10000u));
            if (!LAZY && blk_live) {
#pragma unroll 8
                for (int i = 0; i < NK * kSects * KH; ++i) part[i * 32] = 0.0;
            }
            // thin crowds (latency-bound): the image sectors this pass will update are requested now and consumed after the walks
            float4 old[NK];
#pragma unroll
            for (int k = 0; k < NK; ++k)
                old[k] = LAZY && blk_live && in_grid ? *reinterpret_cast<const float4*>(rec + (NK == 1 ? kp : k) * kSects) : make_float4(0.f, 0.f, 0.f, 0.f);

            int c0 = 0;
            while (c0 < RW) {
                int c1 = RW;
                const int base_l = colstart[c0], base_a = colstart[CS + c0];
                if (n_left - base_l > a.cap || n_arrived - base_a > a.cap) {
                    c1 = c0 + 1;
                    while (c1 < RW && colstart[c1 + 1] - base_l <= a.cap && colstart[CS + c1 + 1] - base_a <= a.cap) ++c1;
                }
                if (!(single && kp > 0)) { // (a single chunk is listed once and kept for every kind pass)
                    if (!single) __syncthreads(); // the previous chunk's walks are done with the lists
                    const int items = (c1 - c0) * CW; // (column, left / arrived, word)
                    for (int i = tid; i < items; i += NT) {
                        const int c = c0 + i / CW, tw = i - (c - c0) * CW, t = tw >= NWORDS ? 1 : 0, w = tw - t * NWORDS;
                        uint32_t bits = colbits[c * CW + tw];
                        if (bits == 0u) continue;
                        int pos = colstart[t * CS + c] - (t ? base_a : base_l);
                        for (int q = 0; q < w; ++q) pos += __popc(colbits[c * CW + t * NWORDS + q]);
                        FieldEvent* const out = evl + t * a.cap;
                        while (bits != 0u) {
                            const int ry = w * 32 + __ffs((int)bits) - 1;
                            bits &= bits - 1u;
                            const long long idx = cell_index(g, xs + c, ys + ry);
                            const uint32_t code = idx >= 0 ? (uint32_t)__ldg(ev16 + idx) : 0u;
                            out[pos++] = make_uint2(selector(t ? code >> 8 : code & 0xFFu) | ((uint32_t)ry << 17), (uint32_t)c);
                        }
                    }
                    __syncthreads();
                }

                // ---- walk the chunk's events within my block's reach: one left and one arrived event per step
                const int lo = max(c0, col_lo), hi = min(c1, col_hi);
                if (blk_live && lo < hi) {
                    const int my_base = half ? base_a : base_l;
                    const int e0 = my_cs[lo] - my_base, e1 = my_cs[hi] - my_base;
                    const int len = e1 - e0;
                    const int steps = max(__shfl_sync(0xFFFFFFFFu, len, 0), __shfl_sync(0xFFFFFFFFu, len, 16));
#pragma unroll 1
                    for (int i = 0; i < steps; i += EV) {
                        // EV events per trip: every table lookup is in flight before any event's partials are touched
                        FieldEvent fe[EV];
                        uint32_t info[EV];
#pragma unroll
                        for (int h = 0; h < EV; ++h) {
                            const int e = e0 + i + h;
                            fe[h] = my_list[min(e, a.cap - 1)];
                            const int u = (int)fe[h].y - tcx, v = (int)(fe[h].x >> 17) - tcy;
                            const bool ok = e < e1 && in_grid && (unsigned)(u + HW) <= span_x && (unsigned)(v + HH) <= span_y;
                            info[h] = ok ? (uint32_t)tabp[(int)(fe[h].x >> 17) * FW + (int)fe[h].y] : kNoEntry;
                        }
#pragma unroll
                        for (int h = 0; h < EV; ++h) {
                            if (info[h] == kNoEntry) continue;
                            const int grp = (int)info[h] / K;
                            const uint32_t gate = lut[grp] & fe[h].x & kmask; // byte k non-zero: kind k's term is live
                            if (gate == 0u) continue;
                            const int mi = abs((int)(fe[h].x >> 17) - tcy) * MS + abs((int)fe[h].y - tcx);
                            const int pidx = (int)(info[h] >> 1); // group * K/2 + slot / 2
                            double* const p = part + pidx * 32;
                            double mk[NK];
                            {
                                const double m = mtab[0][mi];
                                mk[0] = __hiloint2double(__double2hiint(m) ^ flip, __double2loint(m));
                            }
#pragma unroll
                            for (int k = 1; k < NK; ++k) {
                                if (ONE_MAG) {
                                    mk[k] = mk[0];
                                } else {
                                    const double m = mtab[k][mi];
                                    mk[k] = __hiloint2double(__double2hiint(m) ^ flip, __double2loint(m));
                                }
                            }
                            any = true;
#pragma unroll
                            for (int k = 0; k < NK; ++k) {
                                const uint32_t live = NK == 1 ? gate : gate & (k == 0 ? 0xFFu : (k == 1 ? 0xFF00u : 0x10000u));
                                if (live == 0u) continue;
                                if (LAZY) {
                                    const unsigned long long bit = 1ull << pidx;
                                    const double old = (dirty[k] & bit) ? p[k * KO] : 0.0;
                                    p[k * KO] = __dadd_rn(old, mk[k]);
                                    dirty[k] |= bit;
                                } else {
                                    p[k * KO] = __dadd_rn(p[k * KO], mk[k]);
                                }
                            }
                        }
                    }
                }
                c0 = c1;
            }

            // ---- fold: StepCache::total in slot order, image += (float)total -------------------
            // Slot 2 q lives with the su's "left" lane, slot 2 q + 1 with its "arrived" lane; each lane
            // of the pair folds four sects of every kind (one 16-byte sector half).
            __syncwarp(); // the partner lane's partials are read below
            const int any_other = __shfl_xor_sync(0xFFFFFFFFu, (int)any, 16);
            const bool any_su = any || any_other != 0;
            unsigned long long d_left[NK], d_arrived[NK];
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, dirty[k], 16);
                d_left[k] = half ? other : dirty[k];
                d_arrived[k] = half ? dirty[k] : other;
            }
            if (in_grid && any_su) {
                const double* const pl = part - 16 * half; // the pair's "left" lane column (the "arrived" one is 16 further)
    #pragma unroll
                for (int k = 0; k < NK; ++k) {
                    const int kind = NK == 1 ? kp : k;
                    if (LAZY && (d_left[k] | d_arrived[k]) == 0ull) continue;
                    float4* const r4 = reinterpret_cast<float4*>(rec + kind * kSects);
                    const float4 v = LAZY ? old[k] : *r4;
                    float r[4] = {v.x, v.y, v.z, v.w};
                    const uint32_t gos = a.group_of_sect[kind] >> (12 * half);
    #pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int grp = (int)((gos >> (3 * j)) & 7u);
                        const double* const p = pl + k * KO + grp * (KH * 32);
                        double total = 0.0;
                        if (LAZY) {
                            uint32_t ml = (uint32_t)(d_left[k] >> (grp * KH)) & ((1u << KH) - 1u);
                            uint32_t ma = (uint32_t)(d_arrived[k] >> (grp * KH)) & ((1u << KH) - 1u);
                            if ((ml | ma) == 0u) continue;
    #pragma unroll
                            for (int q = 0; q < KH; ++q) { // slot order: 2 q, 2 q + 1
                                if ((ml >> q) & 1u) total = __dadd_rn(total, p[q * 32]);
                                if ((ma >> q) & 1u) total = __dadd_rn(total, p[q * 32 + 16]);
                            }
                        } else {
    #pragma unroll
                            for (int q = 0; q < KH; ++q) {
                                total = __dadd_rn(total, p[q * 32]);
                                total = __dadd_rn(total, p[q * 32 + 16]);
                            }
                        }
                        r[j] = __fadd_rn(r[j], __double2float_rn(total)); // engine.cpp:468
                    }
                    *r4 = make_float4(r[0], r[1], r[2], r[3]);
                }
            }
            __syncwarp(); // (the next pass rewrites partials the partner lane may still be folding)
        }
        __syncthreads(); // every walk is done before the next tile restages colbits / the lists
    }
}

// ---- host: tables -------------------------------------------------------------------------------

struct FieldShape {
    size_t smem;
    int nk, warps, cap, rw_max, nwords, tile_h;
};

int cs_ints(int rw_max, int rh_max) { return (std::max(2 * (rw_max + 2), rh_max) + 1) & ~1; }

size_t fixed_bytes(const FieldTables& t, int tile_h) {
    const int rw_max = kTileW + 2 * t.hw, rh_max = tile_h + 2 * t.hh;
    const int nwords = (rh_max + 31) / 32;
    return (size_t)t.mag_bytes + sizeof(uint32_t) * (size_t)rw_max * 2 * nwords + sizeof(int) * (size_t)cs_ints(rw_max, rh_max) +
           sizeof(uint32_t) * kSects + (size_t)t.tab_bytes + 16;
}

// Chooses kinds per walk, warps per CTA (a warp owns 8 x 2 su: tile height = warps / 2) and the list
// capacity for these tables and chunk width (nk_pref / warps_pref > 0 force a choice; tests and tuning).
bool field_shape(const FieldTables& t, int chunk_k, int nk_pref, int warps_pref, bool lazy, FieldShape* out) {
    if (t.blob == nullptr) return false;
    // crowds (partials cleared per block): one walk for the three kinds; thin crowds (lazy partials): the
    // small shape, several CTAs per SM, so one CTA's staging overlaps another's walks
    static const int eager_order[5][2] = {{3, 8}, {1, 16}, {1, 8}, {3, 4}, {1, 4}}; // (three kinds never run on 16 warps: launch bounds)
    static const int lazy_order[5][2] = {{1, 8}, {1, 4}, {1, 16}, {3, 8}, {3, 4}};
    for (const auto& cand : lazy ? lazy_order : eager_order) {
        const int nk = cand[0], warps = cand[1];
        if (nk_pref > 0 && nk != nk_pref) continue;
        if (warps_pref > 0 && warps != warps_pref) continue;
        const int tile_h = kBlockH * (warps / 4);
        const size_t part = sizeof(double) * (size_t)warps * nk * kSects * (chunk_k / 2) * 32;
        const size_t fixed = fixed_bytes(t, tile_h);
        const int rh_max = tile_h + 2 * t.hh;
        const size_t per_cap = 2 * sizeof(FieldEvent); // one entry in each of the two lists
        if (part + fixed + per_cap * (size_t)std::max(128, rh_max) > kSmemLimit) continue;
        long long cap = (long long)((kSmemLimit - part - fixed) / per_cap);
        const long long region = (long long)(kTileW + 2 * t.hw) * rh_max;
        // (thin crowds: short lists keep the CTA small enough for three per SM; longer regions stream in chunks)
        cap = std::min<long long>(cap, std::min<long long>(region, lazy ? std::max(256, rh_max) : std::max(1024, rh_max)));
        if (cap < rh_max) continue; // one column must always fit a chunk
        out->nk = nk;
        out->warps = warps;
        out->tile_h = tile_h;
        out->cap = (int)cap;
        out->rw_max = kTileW + 2 * t.hw;
        out->nwords = (rh_max + 31) / 32;
        out->smem = (part + fixed + per_cap * (size_t)cap + 127) & ~(size_t)127;
        return true;
    }
    return false;
}

template <int K, int NK, bool LAZY, bool ONE_MAG>
cudaError_t prepare_one(size_t smem, int threads, int sm_count, int* ctas) {
    static SmemGrant grant; // (one per kernel instantiation)
    cudaError_t e = grant.raise(reinterpret_cast<const void*>(k5_field_kernel<K, NK, LAZY, ONE_MAG>), smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k5_field_kernel<K, NK, LAZY, ONE_MAG>, threads, smem);
    if (e != cudaSuccess) return e;
    *ctas = sm_count * (per_sm > 0 ? per_sm : 1);
    return cudaSuccess;
}

bool shares_magnitudes(const FieldTables& t) { return t.mag_of[1] == t.mag_of[0] && t.mag_of[2] == t.mag_of[0]; }

template <int K>
cudaError_t prepare_k(const FieldShape& sh, bool lazy, bool one_mag, int sm_count, int* ctas) {
    const int threads = sh.warps * 32;
    if (sh.nk == 3) {
        if (one_mag)
            return lazy ? prepare_one<K, 3, true, true>(sh.smem, threads, sm_count, ctas)
                        : prepare_one<K, 3, false, true>(sh.smem, threads, sm_count, ctas);
        return lazy ? prepare_one<K, 3, true, false>(sh.smem, threads, sm_count, ctas)
                    : prepare_one<K, 3, false, false>(sh.smem, threads, sm_count, ctas);
    }
    return lazy ? prepare_one<K, 1, true, true>(sh.smem, threads, sm_count, ctas) : prepare_one<K, 1, false, true>(sh.smem, threads, sm_count, ctas);
}

template <int K>
void launch_k(cudaStream_t s, const FieldArgs& a, const FieldShape& sh, bool lazy, bool one_mag, unsigned blocks) {
    const int threads = sh.warps * 32;
    if (sh.nk == 3) {
        if (one_mag) {
            if (lazy) launch_chained(k5_field_kernel<K, 3, true, true>, dim3(blocks), dim3(threads), sh.smem, s, a);
            else launch_chained(k5_field_kernel<K, 3, false, true>, dim3(blocks), dim3(threads), sh.smem, s, a);
        } else {
            if (lazy) launch_chained(k5_field_kernel<K, 3, true, false>, dim3(blocks), dim3(threads), sh.smem, s, a);
            else launch_chained(k5_field_kernel<K, 3, false, false>, dim3(blocks), dim3(threads), sh.smem, s, a);
        }
    } else {
        if (lazy) launch_chained(k5_field_kernel<K, 1, true, true>, dim3(blocks), dim3(threads), sh.smem, s, a);
        else launch_chained(k5_field_kernel<K, 1, false, true>, dim3(blocks), dim3(threads), sh.smem, s, a);
    }
}

} // namespace

// Builds the shared-walk tables of the field kernel from the merged contributor lists: one byte per
// support offset — sect group * K + the StepCache slot of the offset's "left" term (2 * rank mod K) —, the orientation masks per group, and the magnitudes
// folded onto one quadrant.  Returns false — the kernel is then not used — when a mask is not a
// function of the sect group, a magnitude table is not symmetric, or the field is out of range.
bool build_field_tables(const WalkListsHost& w, int chunk_k, FieldTables* out, std::vector<unsigned char>* blob) {
    *out = FieldTables{};
    if (w.n <= 0 || w.hw > 127 || w.hh > 127) return false; // (list entries: row < 2^15, table index within int)
    const int fw = 2 * w.hw + 1, fh = 2 * w.hh + 1;
    std::vector<uint8_t> tab((size_t)fw * fh, (uint8_t)kNoEntry);
    uint32_t lut[kSects];
    bool lut_set[kSects] = {};
    int ms = w.hw + 1;
    while (ms % 16 != 8) ++ms; // rows of eight doubles land on alternating halves of the banks
    const int mag_stride = ms * (w.hh + 1);
    std::vector<double> mags; // distinct magnitude tables
    int mag_of[kKinds], nm = 0;
    for (int k = 0; k < kKinds; ++k) {
        std::vector<double> q((size_t)mag_stride, 0.0);
        std::vector<char> have((size_t)mag_stride, 0);
        for (int grp = 0; grp < kSects; ++grp)
            for (int i = w.start[grp]; i < w.start[grp + 1]; ++i) {
                const int dx = (int)(w.meta[(size_t)i] & 0xFFu) - 128, dy = (int)((w.meta[(size_t)i] >> 8) & 0xFFu) - 128;
                const size_t at = (size_t)std::abs(dy) * ms + std::abs(dx);
                const double m = w.mag[(size_t)k * w.n + i];
                if (have[at] && std::memcmp(&q[at], &m, sizeof m) != 0) return false; // not symmetric
                q[at] = m;
                have[at] = 1;
            }
        int same = -1;
        for (int j = 0; j < nm && same < 0; ++j)
            if (std::memcmp(mags.data() + (size_t)j * mag_stride, q.data(), sizeof(double) * mag_stride) == 0) same = j;
        if (same < 0) {
            mags.insert(mags.end(), q.begin(), q.end());
            same = nm++;
        }
        mag_of[k] = same;
    }
    for (int grp = 0; grp < kSects; ++grp) {
        const int len = w.start[grp + 1] - w.start[grp];
        for (int j = 0; j < len; ++j) {
            const int i = w.start[grp] + j;
            const int dx = (int)(w.meta[(size_t)i] & 0xFFu) - 128, dy = (int)((w.meta[(size_t)i] >> 8) & 0xFFu) - 128;
            if (std::abs(dx) > w.hw || std::abs(dy) > w.hh) return false;
            tab[(size_t)(dy + w.hh) * fw + dx + w.hw] = (uint8_t)(grp * chunk_k + ((2 * j) & (chunk_k - 1))); // partial of its "left" term
            if (!lut_set[grp]) {
                lut[grp] = w.masks[(size_t)i];
                lut_set[grp] = true;
            } else if (lut[grp] != w.masks[(size_t)i]) {
                return false; // orientation masks must depend on the sect group alone
            }
        }
        if (!lut_set[grp]) lut[grp] = 0u;
        if (lut[grp] >> 24) return false;
        // kind 2 is gated by selector bit 16 (orientation 0 of byte 2): its mask must hold that bit or be empty.
        // Only bits 0..16 stay in the word: the list entries carry the event's position from bit 17 up.
        if (((lut[grp] >> 16) & 0xFFu) != 0u && !((lut[grp] >> 16) & 1u)) return false;
        lut[grp] &= 0x1FFFFu;
    }
    const size_t tab_bytes = (tab.size() + 15) & ~(size_t)15;
    const size_t mag_bytes = mags.size() * sizeof(double);
    blob->assign(tab_bytes + mag_bytes + sizeof lut, 0);
    std::memcpy(blob->data(), tab.data(), tab.size());
    std::memcpy(blob->data() + tab_bytes, mags.data(), mag_bytes);
    std::memcpy(blob->data() + tab_bytes + mag_bytes, lut, sizeof lut);
    out->fw = fw;
    out->fh = fh;
    out->hw = w.hw;
    out->hh = w.hh;
    out->ms = ms;
    out->mag_stride = mag_stride;
    out->tab_bytes = (int)tab_bytes;
    out->mag_bytes = (int)mag_bytes;
    for (int k = 0; k < kKinds; ++k) {
        out->mag_of[k] = mag_of[k];
        out->group_of_sect[k] = 0u;
        for (int grp = 0; grp < kSects; ++grp) out->group_of_sect[k] |= (uint32_t)grp << (3 * (w.sect_of[k][grp] & 7));
    }
    return true;
}

bool k5_field_supported(const FieldTables& t, int chunk_k, int nk_pref, int warps_pref) {
    FieldShape sh;
    return field_shape(t, chunk_k, nk_pref, warps_pref, false, &sh) && field_shape(t, chunk_k, nk_pref, warps_pref, true, &sh);
}

// ctas[0]: persistent grid of the eager shape, ctas[1]: of the lazy shape
cudaError_t prepare_k5_field(const FieldTables& t, int chunk_k, int nk_pref, int warps_pref, int sm_count, int* ctas) {
    for (int lazy = 0; lazy < 2; ++lazy) {
        FieldShape sh;
        if (!field_shape(t, chunk_k, nk_pref, warps_pref, lazy != 0, &sh)) return cudaErrorInvalidValue;
        cudaError_t e = cudaErrorInvalidValue;
        switch (chunk_k) {
            case 2: e = prepare_k<2>(sh, lazy != 0, shares_magnitudes(t), sm_count, ctas + lazy); break;
            case 4: e = prepare_k<4>(sh, lazy != 0, shares_magnitudes(t), sm_count, ctas + lazy); break;
            case 8: e = prepare_k<8>(sh, lazy != 0, shares_magnitudes(t), sm_count, ctas + lazy); break;
            case 16: e = prepare_k<16>(sh, lazy != 0, shares_magnitudes(t), sm_count, ctas + lazy); break;
            default: break;
        }
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_k5_field(cudaStream_t s, const K5Launch& l) {
    const FieldTables& t = l.field;
    FieldShape sh;
    if (!field_shape(t, l.chunk_k, l.field_nk, l.field_warps, l.field_lazy != 0, &sh)) return cudaErrorInvalidValue;
    FieldArgs a;
    a.g = l.g;
    a.dyn = l.dyn;
    a.ev = l.ev;
    a.ctl = l.ctl;
    a.blob = t.blob;
    a.tab_bytes = t.tab_bytes;
    a.mag_bytes = t.mag_bytes;
    a.fw = t.fw;
    a.fh = t.fh;
    a.hw = t.hw;
    a.hh = t.hh;
    a.ms = t.ms;
    a.mag_stride = t.mag_stride;
    for (int k = 0; k < kKinds; ++k) {
        a.mag_of[k] = t.mag_of[k];
        a.group_of_sect[k] = t.group_of_sect[k];
    }
    a.tile_h = sh.tile_h;
    a.tiles_x = (l.g.W + kTileW - 1) / kTileW;
    a.n_tiles = a.tiles_x * ((l.g.rows + sh.tile_h - 1) / sh.tile_h);
    a.rw_max = sh.rw_max;
    a.nwords = sh.nwords;
    a.cs_ints = cs_ints(sh.rw_max, sh.tile_h + 2 * t.hh);
    a.cap = l.list_cap > 0 ? std::clamp(l.list_cap, sh.tile_h + 2 * t.hh, sh.cap) : sh.cap;
    a.advance_tick = l.advance_tick;
    a.vec_ok = l.g.W % 8 == 0;
    long long blocks = l.field_ctas[l.field_lazy ? 1 : 0] > 0 ? l.field_ctas[l.field_lazy ? 1 : 0] : 148;
    if (blocks > a.n_tiles) blocks = a.n_tiles;
    if (blocks < 1) blocks = 1;
    switch (l.chunk_k) {
        case 2: launch_k<2>(s, a, sh, l.field_lazy != 0, shares_magnitudes(t), (unsigned)blocks); break;
        case 4: launch_k<4>(s, a, sh, l.field_lazy != 0, shares_magnitudes(t), (unsigned)blocks); break;
        case 8: launch_k<8>(s, a, sh, l.field_lazy != 0, shares_magnitudes(t), (unsigned)blocks); break;
        case 16: launch_k<16>(s, a, sh, l.field_lazy != 0, shares_magnitudes(t), (unsigned)blocks); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

} // namespace sfc
