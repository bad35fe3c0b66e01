// sfc_k5_field.cu — k-5 write-back for LARGE fields (beyond 15 x 15: BASELINE configs 3 and 5,
// the paper's 21^2 ... 77^2 sweep), every crowd density.
// Reference: k5_writeback_range + StepCache (engine.cpp:428-472, accumulator.hpp:36-46).
//
// The reference walks, for every (su, kind, sect) address, that sect's contributor list (F offsets,
// two mask probes each) and adds the gated terms to K f64 partials: term idx -> partial idx mod K,
// idx = 2 j (left) / 2 j + 1 (arrived) for list position j; partials folded in slot order, cast to
// float, added to the image.  Here the non-zero terms are found from the EVENTS instead:
//
//   tile      a CTA of NW warps owns a tile of NW blocks of 8 x 4 su (32 x 4 or 32 x 8 su), one
//             block per warp, one su per lane, for the whole life of the tile.
//   stage     the tile + field-halo region of the 2-byte event map is read once with 16-byte loads
//             (eight cells); cells with an event set a bit in a per-column bit map in shared memory.
//             A popcount scan over the columns gives every event its place in the (x, y)-sorted
//             event list — the reference's contributor-list order for every su of the tile, because
//             the lists are sorted lexicographically by centre offset (fields.hpp:55-57).
//   stream    the list is materialised in column chunks of at most `cap` events (normally one
//             chunk) and walked by every warp with a WARP-UNIFORM trip count: lanes differ only in
//             the offset they see.  Per (event, lane): one table byte (sect group * K + StepCache
//             slot), one orientation-mask word per group, the magnitude from a quadrant-folded f64
//             table (|dx|, |dy|: the magnitudes are symmetric, checked on the host) — all in shared
//             memory — then one f64 read-modify-write per gated term on the lane's own partials,
//             laid out [kind][group][slot][lane] (bank = lane: conflict-free whatever the slot).
//             The partials persist across chunks, so nothing is ever re-staged; the three kinds
//             share one walk (NK = 3) when their partials fit, else one walk per kind (NK = 1).
//   fold      StepCache::total per touched (kind, sect) in slot order, image += (float)total, one
//             32-byte sector per touched (su, kind).
//
// Zero terms are never materialised (x + +-0.0 = x), empty partials hold +0.0 (0.0 + p = p, and a
// partial is never -0.0), so the bits are the reference's.  LAZY variants (sparse crowds) create a
// partial on its first term under a per-lane dirty mask instead of clearing all of them per block.
// Fields larger than the grid wrap onto themselves: the region is staged in unwrapped coordinates
// (engine.cpp:450-454).

#include <algorithm>
#include <cstring>
#include <vector>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kBlockW = 8, kBlockH = 4;
constexpr int kTileW = 32;
constexpr int kMaxThreads = 256;
constexpr size_t kSmemLimit = 227u << 10;
constexpr uint32_t kNoEntry = 0xFFu;

// One movement event as the walks see it: a cell somebody LEFT (term -magnitude, StepCache idx 2 j)
// or ARRIVED at (term +magnitude, idx 2 j + 1).  A cell with both yields two entries.
struct __align__(16) FieldEvent {
    uint32_t sel; // one-hot orientation selectors, kind k in byte k (kind 2: bit 16) | arrived << 31
    int lin;      // ry * fw + rc: the uniform part of the table index
    int rc, ry;   // region column / row
};

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
    int cap;                      // entries per list chunk
    int advance_tick;
    int vec_ok;                   // 16-byte event-map loads are aligned (W % 8 == 0)
};

__device__ __forceinline__ uint32_t selector(uint32_t b) { // one-hot orientation per kind byte, 0 without an event
    return ((1u << (b & 7u)) | (256u << ((b >> 3) & 7u)) | 0x10000u) * (b >> 7);
}

template <int K>
struct Log2K {
    static constexpr int value = K == 2 ? 1 : (K == 4 ? 2 : (K == 8 ? 3 : 4));
};

template <int K, int NK, bool LAZY>
__global__ void __launch_bounds__(kMaxThreads) k5_field_kernel(FieldArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int PW = NK * kSects * K * 32;   // partial doubles per warp
    constexpr int KO = kSects * K * 32;        // ... per kind
    constexpr int DW = (kSects * K + 63) / 64; // dirty words per kind
    constexpr int LOGK = Log2K<K>::value;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5;
    if (a.advance_tick && blockIdx.x == 0 && tid == 0 && a.ctl->error_code == 0) a.ctl->tick += 1;
    if (a.ctl->error_code != 0) return;

    // ---- shared memory ------------------------------------------------------------------------
    double* const part_all = reinterpret_cast<double*>(smem_raw);
    double* const smag = part_all + (size_t)NW * PW;
    FieldEvent* const evl = reinterpret_cast<FieldEvent*>(smag + a.mag_bytes / 8);
    uint32_t* const colbits = reinterpret_cast<uint32_t*>(evl + a.cap); // [column][left words | arrived words]
    int* const colstart = reinterpret_cast<int*>(colbits + a.rw_max * 2 * a.nwords);
    uint32_t* const lut = reinterpret_cast<uint32_t*>(colstart + a.rw_max + 2);
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

    const GridDev g = a.g;
    const int HW = a.hw, HH = a.hh, FW = a.fw, MS = a.ms, NWORDS = a.nwords, CW = 2 * a.nwords;
    const uint16_t* const ev16 = reinterpret_cast<const uint16_t*>(a.ev);
    double* const part = part_all + (size_t)warp * PW + lane;
    const int bx = (warp & 3) * kBlockW, by = (warp >> 2) * kBlockH;
    const int sx = lane & 7, sy = lane >> 3;

    for (int tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int tile_y = tile / a.tiles_x, tile_x = tile - tile_y * a.tiles_x;
        const int x0 = tile_x * kTileW, y0 = g.row0 + tile_y * a.tile_h;
        const int nx = min(kTileW, g.W - x0), ny = min(a.tile_h, g.row0 + g.rows - y0);
        const int RW = nx + 2 * HW, RH = ny + 2 * HH;
        const int xs = x0 - HW, ys = y0 - HH;

        // ---- stage: per-column bit maps of the region's events ---------------------------------
        for (int i = tid; i < RW * CW; i += NT) colbits[i] = 0u;
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
                        const long long row = cell_index(g, 0, ys + ry); // -1: the row does not exist / is not resident
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
        if (warp == 0) { // exclusive column starts: scan of the per-column entry counts
            int carry = 0;
            for (int c0 = 0; c0 < RW; c0 += 32) {
                const int c = c0 + lane;
                int v = 0;
                if (c < RW)
                    for (int w = 0; w < CW; ++w) v += __popc(colbits[c * CW + w]);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xFFFFFFFFu, v, o);
                    if (lane >= o) v += u;
                }
                if (c < RW) colstart[c + 1] = v + carry;
                carry += __shfl_sync(0xFFFFFFFFu, v, 31);
            }
            if (lane == 0) colstart[0] = 0;
        }
        __syncthreads();
        const int n_total = colstart[RW];
        if (n_total == 0) continue; // nobody moved within reach of this tile (uniform; colbits untouched until the next sync)

        // ---- my block --------------------------------------------------------------------------
        const bool blk_ok = bx < nx && by < ny; // uniform per warp
        const int cx = bx + sx, cy = by + sy;
        const bool in_grid = blk_ok && cx < nx && cy < ny;
        const int tcx = cx + HW, tcy = cy + HH; // my su in region coordinates
        const int col_lo = bx, col_hi = min(bx + kBlockW + 2 * HW, RW); // region columns within the block's reach
        const bool blk_live = blk_ok && colstart[col_hi] > colstart[col_lo];
        const bool single = n_total <= a.cap;
        // table word of the offset (event - my su): tabp[event.lin]; one magnitude row per |dy|
        const uint8_t* const tabp = tab8 + ((HH - tcy) * FW + (HW - tcx));
        const unsigned span_x = 2u * (unsigned)HW, span_y = 2u * (unsigned)HH;

#pragma unroll 1
        for (int kp = 0; kp < kKinds / NK; ++kp) {
            unsigned long long dirty[NK][DW];
            bool any = false;
            const double* mtab[NK]; // kind k's magnitude table
#pragma unroll
            for (int k = 0; k < NK; ++k) mtab[k] = smag + a.mag_of[NK == 1 ? kp : k] * a.mag_stride;
            const bool one_mag = NK == 1 || (mtab[1] == mtab[0] && mtab[2] == mtab[0]); // (uniform)
            const uint32_t kmask = NK == 3 ? 0x1FFFFu : (kp == 0 ? 0xFFu : (kp == 1 ? 0xFF00u : 0x10000u));
#pragma unroll
            for (int k = 0; k < NK; ++k)
#pragma unroll
                for (int w = 0; w < DW; ++w) dirty[k][w] = 0ull;
            if (!LAZY && blk_live) {
#pragma unroll 8
                for (int i = 0; i < NK * kSects * K; ++i) part[i * 32] = 0.0;
            }

            int c0 = 0;
            while (c0 < RW) {
                int c1 = RW;
                const int base = colstart[c0];
                if (n_total - base > a.cap) {
                    c1 = c0 + 1;
                    while (c1 < RW && colstart[c1 + 1] - base <= a.cap) ++c1;
                }
                if (!(single && kp > 0)) { // (a single chunk is listed once and kept for every kind pass)
                    if (!single) __syncthreads(); // the previous chunk's walks are done with evl
                    const int items = (c1 - c0) * NWORDS;
                    for (int i = tid; i < items; i += NT) {
                        const int c = c0 + i / NWORDS, w = i - (c - c0) * NWORDS;
                        const uint32_t bf = colbits[c * CW + w], bt = colbits[c * CW + NWORDS + w];
                        uint32_t bits = bf | bt;
                        if (bits == 0u) continue;
                        int pos = colstart[c] - base;
                        for (int q = 0; q < w; ++q) pos += __popc(colbits[c * CW + q]) + __popc(colbits[c * CW + NWORDS + q]);
                        while (bits != 0u) {
                            const int r = __ffs((int)bits) - 1, ry = w * 32 + r;
                            bits &= bits - 1u;
                            const long long idx = cell_index(g, xs + c, ys + ry);
                            const uint32_t code = idx >= 0 ? (uint32_t)__ldg(ev16 + idx) : 0u;
                            FieldEvent fe;
                            fe.lin = ry * FW + c;
                            fe.rc = c;
                            fe.ry = ry;
                            if ((bf >> r) & 1u) {
                                fe.sel = selector(code & 0xFFu);
                                evl[pos++] = fe;
                            }
                            if ((bt >> r) & 1u) {
                                fe.sel = selector(code >> 8) | 0x80000000u;
                                evl[pos++] = fe;
                            }
                        }
                    }
                    __syncthreads();
                }

                // ---- walk the chunk's events within my block's reach ---------------------------
                const int lo = max(c0, col_lo), hi = min(c1, col_hi);
                if (blk_live && lo < hi) {
                    const int e0 = colstart[lo] - base, e1 = colstart[hi] - base;
                    auto lookup = [&](const FieldEvent& fe) -> uint32_t {
                        const bool ok = in_grid && (unsigned)(fe.rc - tcx + HW) <= span_x && (unsigned)(fe.ry - tcy + HH) <= span_y;
                        return ok ? (uint32_t)tabp[fe.lin] : kNoEntry;
                    };
#pragma unroll 1
                    for (int e = e0; e < e1; e += 2) {
                        // two events per trip: both table lookups are in flight before either event's partials are touched
                        FieldEvent fe[2];
                        uint32_t info[2];
                        fe[0] = evl[e];
                        fe[1] = evl[min(e + 1, e1 - 1)];
                        info[0] = lookup(fe[0]);
                        info[1] = e + 1 < e1 ? lookup(fe[1]) : kNoEntry;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if (info[h] == kNoEntry) continue;
                            const FieldEvent cur = fe[h];
                            const uint32_t gate = lut[info[h] >> LOGK] & cur.sel & kmask; // byte k non-zero: kind k's term is live
                            if (gate == 0u) continue;
                            const int arrived = (int)(cur.sel >> 31);
                            const int mi = abs(cur.ry - tcy) * MS + abs(cur.rc - tcx);
                            const int flip = (int)(~cur.sel & 0x80000000u); // left: -magnitude
                            const int pidx = (int)info[h] + arrived;        // group * K + slot
                            double* const p = part + pidx * 32;
                            double mk[NK];
                            {
                                const double m = mtab[0][mi];
                                mk[0] = __hiloint2double(__double2hiint(m) ^ flip, __double2loint(m));
                            }
#pragma unroll
                            for (int k = 1; k < NK; ++k) {
                                if (one_mag) {
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
                                    const unsigned long long bit = 1ull << (pidx & 63);
                                    if (DW == 1 || pidx < 64) {
                                        const double old = (dirty[k][0] & bit) ? p[k * KO] : 0.0;
                                        p[k * KO] = __dadd_rn(old, mk[k]);
                                        dirty[k][0] |= bit;
                                    } else {
                                        const double old = (dirty[k][DW - 1] & bit) ? p[k * KO] : 0.0;
                                        p[k * KO] = __dadd_rn(old, mk[k]);
                                        dirty[k][DW - 1] |= bit;
                                    }
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
            if (!in_grid || !any) continue;
            const long long cell = cell_index(g, x0 + cx, y0 + cy);
            float* const rec = a.dyn + cell * (kKinds * kSects);
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const int kind = NK == 1 ? kp : k;
                if (LAZY) {
                    bool none = true;
#pragma unroll
                    for (int w = 0; w < DW; ++w) none = none && dirty[k][w] == 0ull;
                    if (none) continue;
                }
                float4* const r4 = reinterpret_cast<float4*>(rec + kind * kSects);
                const float4 v0 = r4[0], v1 = r4[1];
                float r[kSects] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                const uint32_t gos = a.group_of_sect[kind];
#pragma unroll
                for (int s = 0; s < kSects; ++s) {
                    const int grp = (int)((gos >> (3 * s)) & 7u);
                    const double* const p = part + k * KO + grp * (K * 32);
                    double total = 0.0;
                    if (LAZY) {
                        const int bit0 = grp * K;
                        const unsigned long long d = (DW == 1 || bit0 < 64) ? dirty[k][0] : dirty[k][DW - 1];
                        uint32_t gm = (uint32_t)(d >> (bit0 & 63)) & ((1u << K) - 1u);
                        if (gm == 0u) continue;
                        while (gm != 0u) { // slot order
                            const int q = __ffs((int)gm) - 1;
                            gm &= gm - 1u;
                            total = __dadd_rn(total, p[q * 32]);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < K; ++q) total = __dadd_rn(total, p[q * 32]);
                    }
                    r[s] = __fadd_rn(r[s], __double2float_rn(total)); // engine.cpp:468
                }
                r4[0] = make_float4(r[0], r[1], r[2], r[3]);
                r4[1] = make_float4(r[4], r[5], r[6], r[7]);
            }
        }
        __syncthreads(); // every walk is done before the next tile restages colbits / evl
    }
}

// ---- host: tables -------------------------------------------------------------------------------

struct FieldShape {
    size_t smem;
    int nk, warps, cap, rw_max, nwords, tile_h;
};

size_t fixed_bytes(const FieldTables& t, int tile_h) {
    const int rw_max = kTileW + 2 * t.hw, rh_max = tile_h + 2 * t.hh;
    const int nwords = (rh_max + 31) / 32;
    return (size_t)t.mag_bytes + sizeof(uint32_t) * (size_t)rw_max * 2 * nwords + sizeof(int) * (size_t)(rw_max + 2) +
           sizeof(uint32_t) * kSects + (size_t)t.tab_bytes + 16;
}

// Chooses kinds per walk, warps per CTA and the list capacity for these tables and chunk width:
// (nk_pref / warps_pref > 0 force a choice; tests and tuning).
bool field_shape(const FieldTables& t, int chunk_k, int nk_pref, int warps_pref, bool lazy, FieldShape* out) {
    if (t.blob == nullptr) return false;
    // crowds (partials cleared per block): one walk for the three kinds; thin crowds (lazy partials): the
    // small shape, several CTAs per SM, so one CTA's staging overlaps another's walks
    static const int eager_order[4][2] = {{3, 4}, {1, 8}, {1, 4}, {3, 8}};
    static const int lazy_order[4][2] = {{1, 4}, {1, 8}, {3, 4}, {3, 8}};
    for (const auto& cand : lazy ? lazy_order : eager_order) {
        const int nk = cand[0], warps = cand[1];
        if (nk == 3 && chunk_k > 8) continue;
        if (nk_pref > 0 && nk != nk_pref) continue;
        if (warps_pref > 0 && warps != warps_pref) continue;
        const int tile_h = kBlockH * (warps / 4);
        const size_t part = sizeof(double) * (size_t)warps * nk * kSects * chunk_k * 32;
        const size_t fixed = fixed_bytes(t, tile_h);
        const int rh_max = tile_h + 2 * t.hh;
        if (part + fixed + sizeof(FieldEvent) * (size_t)std::max(256, 2 * rh_max) > kSmemLimit) continue;
        long long cap = (long long)((kSmemLimit - part - fixed) / sizeof(FieldEvent));
        const long long region = (long long)(kTileW + 2 * t.hw) * rh_max;
        // (thin crowds: a short list keeps the CTA small enough for three per SM; longer regions stream in chunks)
        cap = std::min<long long>(cap, std::min<long long>(2 * region, lazy ? std::max(256, 2 * rh_max) : std::max(1024, 2 * rh_max)));
        if (cap < 2 * rh_max) continue; // one column must always fit a chunk
        out->nk = nk;
        out->warps = warps;
        out->tile_h = tile_h;
        out->cap = (int)cap;
        out->rw_max = kTileW + 2 * t.hw;
        out->nwords = (rh_max + 31) / 32;
        out->smem = (part + fixed + sizeof(FieldEvent) * (size_t)cap + 127) & ~(size_t)127;
        return true;
    }
    return false;
}

template <int K, int NK, bool LAZY>
cudaError_t prepare_one(size_t smem, int threads, int sm_count, int* ctas) {
    static SmemGrant grant; // (one per kernel instantiation)
    cudaError_t e = grant.raise(reinterpret_cast<const void*>(k5_field_kernel<K, NK, LAZY>), smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k5_field_kernel<K, NK, LAZY>, threads, smem);
    if (e != cudaSuccess) return e;
    *ctas = sm_count * (per_sm > 0 ? per_sm : 1);
    return cudaSuccess;
}

template <int K>
cudaError_t prepare_k(const FieldShape& sh, bool lazy, int sm_count, int* ctas) {
    const int threads = sh.warps * 32;
    if (sh.nk == 3) {
        if constexpr (K <= 8)
            return lazy ? prepare_one<K, 3, true>(sh.smem, threads, sm_count, ctas) : prepare_one<K, 3, false>(sh.smem, threads, sm_count, ctas);
        else
            return cudaErrorInvalidValue;
    }
    return lazy ? prepare_one<K, 1, true>(sh.smem, threads, sm_count, ctas) : prepare_one<K, 1, false>(sh.smem, threads, sm_count, ctas);
}

template <int K>
void launch_k(cudaStream_t s, const FieldArgs& a, const FieldShape& sh, bool lazy, unsigned blocks) {
    const int threads = sh.warps * 32;
    if (sh.nk == 3) {
        if constexpr (K <= 8) {
            if (lazy) k5_field_kernel<K, 3, true><<<blocks, threads, sh.smem, s>>>(a);
            else k5_field_kernel<K, 3, false><<<blocks, threads, sh.smem, s>>>(a);
        }
    } else {
        if (lazy) k5_field_kernel<K, 1, true><<<blocks, threads, sh.smem, s>>>(a);
        else k5_field_kernel<K, 1, false><<<blocks, threads, sh.smem, s>>>(a);
    }
}

} // namespace

// Builds the shared-walk tables of the field kernel from the merged contributor lists: one byte per
// support offset — sect group * K + the StepCache slot of the offset's "left" term (2 * rank mod K) —, the orientation masks per group, and the magnitudes
// folded onto one quadrant.  Returns false — the kernel is then not used — when a mask is not a
// function of the sect group, a magnitude table is not symmetric, or the field is out of range.
bool build_field_tables(const WalkListsHost& w, int chunk_k, FieldTables* out, std::vector<unsigned char>* blob) {
    *out = FieldTables{};
    if (w.n <= 0 || w.hw > 127 || w.hh > 127) return false;
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
            case 2: e = prepare_k<2>(sh, lazy != 0, sm_count, ctas + lazy); break;
            case 4: e = prepare_k<4>(sh, lazy != 0, sm_count, ctas + lazy); break;
            case 8: e = prepare_k<8>(sh, lazy != 0, sm_count, ctas + lazy); break;
            case 16: e = prepare_k<16>(sh, lazy != 0, sm_count, ctas + lazy); break;
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
    a.cap = l.list_cap > 0 ? std::clamp(l.list_cap, 2 * (sh.tile_h + 2 * t.hh), sh.cap) : sh.cap;
    a.advance_tick = l.advance_tick;
    a.vec_ok = l.g.W % 8 == 0;
    long long blocks = l.field_ctas[l.field_lazy ? 1 : 0] > 0 ? l.field_ctas[l.field_lazy ? 1 : 0] : 148;
    if (blocks > a.n_tiles) blocks = a.n_tiles;
    if (blocks < 1) blocks = 1;
    switch (l.chunk_k) {
        case 2: launch_k<2>(s, a, sh, l.field_lazy != 0, (unsigned)blocks); break;
        case 4: launch_k<4>(s, a, sh, l.field_lazy != 0, (unsigned)blocks); break;
        case 8: launch_k<8>(s, a, sh, l.field_lazy != 0, (unsigned)blocks); break;
        case 16: launch_k<16>(s, a, sh, l.field_lazy != 0, (unsigned)blocks); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

} // namespace sfc
