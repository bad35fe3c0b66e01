// sfc_k5_listwalk.cu — k-5 write-back for dense crowds on small fields: the reference's own
// formulation (engine.cpp:428-472), one su per lane.
//
// For every (su, kind, sect) address the reference walks that sect's contributor list in order,
// term idx = 2j (left) / 2j + 1 (arrived) for the j-th contributor, partial = idx mod K, partials
// folded in slot order (accumulator.hpp:36-46).  The slot depends on the LIST POSITION only, so a
// walk unrolled by K / 2 positions has compile-time slots: the K partials of an address live in
// registers, every lane of a warp runs the same instruction stream (one su each, 32 su of a tile
// row), and the result is the reference's bit for bit with no replay, no atomics, no sorting —
// whatever the number of movers.  Adding +-0.0 never changes a partial, so positions where no lane
// of the warp sees an event are skipped with one ballot.
//
// The three kinds share the walk when they have the same support and list ranks (they do whenever
// they share a field geometry: a repulsive kind's sect is the attractive kind's opposite, so the
// sect GROUPS of offsets coincide): one event-code load per position serves six gated terms.
//
// A CTA takes a 32 x 8 su tile — from the dense-tile list the scatter / window kernel filled, or
// every (active) tile when this is the only k-5 kernel — stages tile + field halo of the event map
// in shared memory (coalesced, loads batched), and warp w walks row w.  Cost per su is 6F gated
// adds at most, independent of the crowd: the dense-crowd path for fields up to 15 x 15.

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kThreads = 256;
constexpr int kListSmemMax = 256; // merged list entries kept in shared memory (15 x 15 fields: 224)

struct LwArgs {
    GridDev g;
    WalkLists w;
    float* dyn;
    const uint8_t* ev;
    Ctl* ctl;
    TileMarks marks;       // every-tile mode: active-tile list (epoch == nullptr: all tiles)
    const int* dense_list; // dense-list mode: tiles handed over by the scatter / window kernel
    int from_dense_list;
    int advance_tick;
    int tiles_x, n_tiles;
    int rwf, rwp, rh;      // region columns, code row pitch (u16), region rows of a full tile
    int list_smem;
};

// p += t when flag != 0, as ONE predicated DADD (the compiler's if-conversion would emit an
// unconditional add followed by two selects per 64-bit partial).
__device__ __forceinline__ void add_if(double& p, double t, uint32_t flag) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q add.rn.f64 %0, %0, %1;\n\t}" : "+d"(p) : "d"(t), "r"(flag));
}

template <int K, bool LIST_SMEM>
__global__ void __launch_bounds__(kThreads) k5_listwalk_kernel(LwArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const int n = a.w.n;
    float* const tot = reinterpret_cast<float*>(smem_raw);                          // [kind * 8 + sect][kThreads]
    double* const s_mag = reinterpret_cast<double*>(tot + kKinds * kSects * kThreads); // [n][4]: kinds 0..2 (+ pad): one 16 B + one 8 B load
    int2* const s_ent = reinterpret_cast<int2*>(s_mag + (LIST_SMEM ? 4 * n : 0));    // [n] (cell offset dy * pitch + dx, masks)
    long long* const rowoff = reinterpret_cast<long long*>(s_ent + (LIST_SMEM ? n : 0)); // [rh]
    // per region cell: one-hot orientation selectors of the event that left it (.x) / arrived at it (.y),
    // per kind in the byte lanes of the mask words (kind 2 is non-directional: orientation 0); 0 = no event
    uint2* const sel = reinterpret_cast<uint2*>(rowoff + a.rh);                      // [rh][rwp]
    if (LIST_SMEM) {
        for (int i = tid; i < n; i += kThreads) {
            const uint32_t m = a.w.meta[i];
            s_ent[i] = make_int2(((int)((m >> 8) & 0xFFu) - 128) * a.rwp + ((int)(m & 0xFFu) - 128), (int)a.w.masks[i]);
            for (int k = 0; k < kKinds; ++k) s_mag[4 * i + k] = a.w.mag[k * n + i];
            s_mag[4 * i + 3] = 0.0;
        }
    }
    chain_wait(); // (the walk list above is a constant of the engine, staged while k-4 drains)
    if (!a.from_dense_list && a.advance_tick && blockIdx.x == 0 && tid == 0 && a.ctl->error_code == 0) a.ctl->tick += 1;
    if (a.ctl->error_code != 0) return;

    const GridDev g = a.g;
    const int HW = a.w.hw, HH = a.w.hh;
    const int RWF = a.rwf, RWP = a.rwp;
    const bool narrow = RWF <= g.W;
    const uint16_t* const ev16 = reinterpret_cast<const uint16_t*>(a.ev);
    const unsigned inv_rwf = 0xFFFFFFFFu / (unsigned)RWF + 1u;
    int n_items, n_edge = 0;
    if (a.from_dense_list) {
        n_items = a.ctl->dense_count;
    } else if (a.marks.epoch != nullptr) {
        n_edge = tile_edge_count(a.marks);
        n_items = n_edge + a.ctl->active_count;
    } else {
        n_items = a.n_tiles;
    }

    for (int item = (int)blockIdx.x; item < n_items; item += (int)gridDim.x) {
        int tile;
        if (a.from_dense_list) {
            tile = a.dense_list[item];
        } else if (a.marks.epoch == nullptr) {
            tile = item;
        } else if (item < n_edge) { // slab mode: tiles whose region reaches the halo rows
            const int r = item / a.tiles_x;
            const int ty = r < a.marks.edge_lo ? r : a.marks.edge_hi + (r - a.marks.edge_lo);
            tile = ty * a.tiles_x + (item - r * a.tiles_x);
        } else {
            tile = a.marks.list[item - n_edge];
        }
        const int tile_y = tile / a.tiles_x, tile_x = tile - tile_y * a.tiles_x;
        const int x0 = tile_x * kMarkTileW;
        const int y0 = g.row0 + tile_y * kMarkTileH;
        const int nx = min(kMarkTileW, g.W - x0);
        const int ny = min(kMarkTileH, g.row0 + g.rows - y0);
        const int RH = ny + 2 * HH;
        const int xs = x0 - HW, ys = y0 - HH;

        // ---- stage (CTA) ---------------------------------------------------------------------
        __syncthreads(); // the previous tile is done with codes / rowoff (and the lists are loaded)
        for (int ry = tid; ry < RH; ry += kThreads) rowoff[ry] = cell_index(g, 0, ys + ry); // -1: no such row / not resident
        __syncthreads();
        bool any = false;
        {
            const int n_cells = RWF * RH;
            for (int i0 = 0; i0 < n_cells; i0 += 4 * kThreads) {
                uint32_t got[4];
                int at[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) { // the loads of the chunk fly together
                    const int i = i0 + q * kThreads + tid;
                    got[q] = 0u;
                    at[q] = -1;
                    if (i < n_cells) {
                        const int ry = (int)__umulhi((unsigned)i, inv_rwf); // i / RWF
                        const int c = i - ry * RWF;
                        at[q] = ry * RWP + c;
                        int x = xs + c;
                        if (g.closed) {
                            if (x < 0 || x >= g.W) x = -1;
                        } else if (narrow) {
                            x += x < 0 ? g.W : (x >= g.W ? -g.W : 0);
                        } else {
                            x = emod(x, g.W);
                        }
                        const long long ro = rowoff[ry];
                        if (ro >= 0 && x >= 0) got[q] = __ldg(ev16 + ro + x);
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (at[q] >= 0) {
                        const uint32_t fb = got[q] & 0xFFu, tb = got[q] >> 8;
                        sel[at[q]] = make_uint2((fb & 0x80u) ? ((1u << (fb & 7u)) | (256u << ((fb >> 3) & 7u)) | 0x10000u) : 0u,
                                                (tb & 0x80u) ? ((1u << (tb & 7u)) | (256u << ((tb >> 3) & 7u)) | 0x10000u) : 0u);
                        any |= got[q] != 0u;
                    }
            }
        }
        if (__syncthreads_or(any ? 1 : 0) == 0) continue; // nobody moved within reach of this tile

        // ---- walk (lane: one su of tile row `warp`) -------------------------------------------
        const bool valid = lane < nx && warp < ny;
        const uint2* const centre = sel + (warp + HH) * RWP + lane + HW; // my su in the staged region
        bool touched = false;
#pragma unroll 1
        for (int grp = 0; grp < kSects; ++grp) {
            double p[kKinds][K];
#pragma unroll
            for (int k = 0; k < kKinds; ++k)
#pragma unroll
                for (int q = 0; q < K; ++q) p[k][q] = 0.0;
            const int j_end = a.w.start[grp + 1];
            for (int j0 = a.w.start[grp]; j0 < j_end; j0 += K / 2) {
#pragma unroll
                for (int u = 0; u < K / 2; ++u) { // list position j0 + u: term idx 2u (left), 2u + 1 (arrived) mod K
                    const int j = j0 + u;
                    if (j >= j_end) break; // uniform
                    int off;      // cell offset of the contributor: centre offset = mover - target
                    uint32_t mk;  // orientation mask of kind k in byte k
                    if (LIST_SMEM) {
                        const int2 ent = s_ent[j];
                        off = ent.x;
                        mk = (uint32_t)ent.y;
                    } else {
                        const uint32_t m = __ldg(a.w.meta + j);
                        off = ((int)((m >> 8) & 0xFFu) - 128) * RWP + ((int)(m & 0xFFu) - 128);
                        mk = __ldg(a.w.masks + j);
                    }
                    const uint2 c = valid ? centre[off] : make_uint2(0u, 0u);
                    if (__ballot_sync(0xFFFFFFFFu, (c.x | c.y) != 0u) == 0u) continue; // zero terms never change a partial
                    const uint32_t fbits = mk & c.x, tbits = mk & c.y; // gating the six terms is two ANDs
                    double mg[kKinds];
                    if (LIST_SMEM) {
                        const double2 m01 = *reinterpret_cast<const double2*>(s_mag + 4 * j);
                        mg[0] = m01.x;
                        mg[1] = m01.y;
                        mg[2] = s_mag[4 * j + 2];
                    } else {
#pragma unroll
                        for (int k = 0; k < kKinds; ++k) mg[k] = __ldg(a.w.mag + k * n + j);
                    }
#pragma unroll
                    for (int k = 0; k < kKinds; ++k) {
                        add_if(p[k][2 * u], -mg[k], fbits & (0xFFu << (8 * k)));
                        add_if(p[k][2 * u + 1], mg[k], tbits & (0xFFu << (8 * k)));
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kKinds; ++k) {
                double total = 0.0; // StepCache::total, slot order
#pragma unroll
                for (int q = 0; q < K; ++q) total = __dadd_rn(total, p[k][q]);
                const float add = __double2float_rn(total);
                tot[(k * kSects + a.w.sect_of[k][grp]) * kThreads + tid] = add;
                touched |= add != 0.0f;
            }
        }

        // ---- apply: image += (float)total, one 32-byte sector per touched (su, kind) ------------
        if (valid && touched) {
            float4* const rec = reinterpret_cast<float4*>(a.dyn + (rowoff[warp + HH] + x0 + lane) * (kKinds * kSects));
#pragma unroll
            for (int k = 0; k < kKinds; ++k) {
                float t[8];
                bool nz = false;
#pragma unroll
                for (int s = 0; s < kSects; ++s) {
                    t[s] = tot[(k * kSects + s) * kThreads + tid];
                    nz |= t[s] != 0.0f;
                }
                if (!nz) continue;
                const float4 v0 = rec[2 * k], v1 = rec[2 * k + 1];
                rec[2 * k] = make_float4(__fadd_rn(v0.x, t[0]), __fadd_rn(v0.y, t[1]), __fadd_rn(v0.z, t[2]), __fadd_rn(v0.w, t[3]));
                rec[2 * k + 1] = make_float4(__fadd_rn(v1.x, t[4]), __fadd_rn(v1.y, t[5]), __fadd_rn(v1.z, t[6]), __fadd_rn(v1.w, t[7]));
            }
        }
    }
}

struct LwShape {
    size_t smem;
    int rwf, rwp, rh, list_smem;
};

LwShape lw_shape(const WalkLists& w) {
    LwShape s;
    s.rwf = kMarkTileW + 2 * w.hw;
    s.rwp = (s.rwf + 1) & ~1;
    s.rh = kMarkTileH + 2 * w.hh;
    s.list_smem = w.n <= kListSmemMax;
    size_t b = sizeof(float) * kKinds * kSects * kThreads;
    if (s.list_smem) b += sizeof(double) * 4 * w.n + sizeof(int2) * w.n;
    b += sizeof(long long) * s.rh;
    b += sizeof(uint2) * (size_t)s.rwp * s.rh;
    s.smem = (b + 15) & ~(size_t)15;
    return s;
}

template <int K>
cudaError_t prepare_one(const WalkLists& w, int sm_count, int* ctas) {
    static SmemGrant grant; // (one per kernel instantiation)
    const LwShape sh = lw_shape(w);
    cudaError_t e = grant.raise(reinterpret_cast<const void*>(k5_listwalk_kernel<K, true>), sh.smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k5_listwalk_kernel<K, true>, kThreads, sh.smem);
    if (e != cudaSuccess) return e;
    *ctas = sm_count * (per_sm > 0 ? per_sm : 1);
    return cudaSuccess;
}

template <int K>
cudaError_t launch_one(cudaStream_t stream, const K5Launch& l, bool from_dense_list) {
    const LwShape sh = lw_shape(l.walk);
    LwArgs a;
    a.g = l.g;
    a.w = l.walk;
    a.dyn = l.dyn;
    a.ev = l.ev;
    a.ctl = l.ctl;
    a.marks = from_dense_list ? TileMarks{} : l.marks;
    a.dense_list = l.dense_list;
    a.from_dense_list = from_dense_list ? 1 : 0;
    a.advance_tick = l.advance_tick;
    a.tiles_x = (l.g.W + kMarkTileW - 1) / kMarkTileW;
    a.n_tiles = a.tiles_x * ((l.g.rows + kMarkTileH - 1) / kMarkTileH);
    a.rwf = sh.rwf;
    a.rwp = sh.rwp;
    a.rh = sh.rh;
    a.list_smem = sh.list_smem;
    long long blocks = a.n_tiles;
    if (blocks > l.listwalk_ctas) blocks = l.listwalk_ctas;
    if (blocks < 1) blocks = 1;
    return launch_chained(k5_listwalk_kernel<K, true>, dim3((unsigned)blocks), dim3(kThreads), sh.smem, stream, a); // (supported lists always fit: kListSmemMax)
}

} // namespace

// Builds the merged per-sect-group contributor lists from the three kind tables (host copies).
// Returns false — the list walk is then not used — when the kinds do not share support and ranks.
bool build_walk_lists(const sfc_tables& t, WalkListsHost* out) {
    const int fw = t.kind[0].width, fh = t.kind[0].height;
    for (int k = 1; k < kKinds; ++k)
        if (t.kind[k].width != fw || t.kind[k].height != fh) return false;
    if (fw > 255 || fh > 255) return false;
    const int hw = (fw - 1) / 2, hh = (fh - 1) / 2;
    struct Entry {
        int sect0, rank, dx, dy, at;
    };
    std::vector<Entry> entries;
    for (int dy = -hh; dy <= hh; ++dy)
        for (int dx = -hw; dx <= hw; ++dx) {
            const int at = (dy + hh) * fw + dx + hw;
            const uint32_t i0 = t.kind[0].info[at];
            const bool in0 = ((i0 >> 3) & 0xFFu) != 0u;
            for (int k = 1; k < kKinds; ++k) {
                const uint32_t ik = t.kind[k].info[at];
                if ((((ik >> 3) & 0xFFu) != 0u) != in0) return false;  // different support
                if (in0 && (ik >> 11) != (i0 >> 11)) return false;      // different list rank
            }
            if (in0) entries.push_back(Entry{(int)(i0 & 7u), (int)(i0 >> 11), dx, dy, at});
        }
    std::sort(entries.begin(), entries.end(),
              [](const Entry& x, const Entry& y) { return x.sect0 != y.sect0 ? x.sect0 < y.sect0 : x.rank < y.rank; });
    WalkListsHost& w = *out;
    w.n = (int)entries.size();
    w.hw = hw;
    w.hh = hh;
    w.meta.assign((size_t)w.n, 0u);
    w.masks.assign((size_t)w.n, 0u);
    w.mag.assign((size_t)w.n * kKinds, 0.0);
    for (int s = 0; s <= kSects; ++s) w.start[s] = 0;
    for (int k = 0; k < kKinds; ++k)
        for (int s = 0; s < kSects; ++s) w.sect_of[k][s] = -1;
    for (int i = 0; i < w.n; ++i) {
        const Entry& e = entries[(size_t)i];
        if (i > 0 && entries[(size_t)i - 1].sect0 == e.sect0 && entries[(size_t)i - 1].rank + 1 != e.rank) return false;
        if ((i == 0 || entries[(size_t)i - 1].sect0 != e.sect0) && e.rank != 0) return false; // ranks must be 0, 1, 2, ...
        w.start[e.sect0 + 1] += 1;
        w.meta[(size_t)i] = (uint32_t)(e.dx + 128) | ((uint32_t)(e.dy + 128) << 8);
        for (int k = 0; k < kKinds; ++k) {
            const uint32_t ik = t.kind[k].info[e.at];
            w.masks[(size_t)i] |= ((ik >> 3) & 0xFFu) << (8 * k);
            w.mag[(size_t)k * w.n + i] = t.kind[k].magnitude[e.at];
            int& mapped = w.sect_of[k][e.sect0];
            if (mapped < 0) mapped = (int)(ik & 7u);
            if (mapped != (int)(ik & 7u)) return false; // a group of kind 0 must be one group of kind k
        }
    }
    for (int s = 0; s < kSects; ++s) w.start[s + 1] += w.start[s];
    for (int k = 0; k < kKinds; ++k) { // the map must be a permutation (empty groups take the unused sects)
        bool used[kSects] = {};
        for (int s = 0; s < kSects; ++s)
            if (w.sect_of[k][s] >= 0) {
                if (used[w.sect_of[k][s]]) return false;
                used[w.sect_of[k][s]] = true;
            }
        for (int s = 0; s < kSects; ++s)
            if (w.sect_of[k][s] < 0)
                for (int q = 0; q < kSects; ++q)
                    if (!used[q]) {
                        w.sect_of[k][s] = q;
                        used[q] = true;
                        break;
                    }
    }
    return true;
}

// Fields up to 15 x 15 (the per-su cost grows with the field area whatever the crowd).
bool k5_listwalk_supported(const WalkLists& w) { return w.meta != nullptr && w.n > 0 && w.n <= kListSmemMax; }

cudaError_t prepare_k5_listwalk(int chunk_k, const WalkLists& w, int sm_count, int* ctas) {
    if (!k5_listwalk_supported(w)) return cudaSuccess;
    switch (chunk_k) {
        case 2: return prepare_one<2>(w, sm_count, ctas);
        case 4: return prepare_one<4>(w, sm_count, ctas);
        case 8: return prepare_one<8>(w, sm_count, ctas);
        case 16: return prepare_one<16>(w, sm_count, ctas);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k5_listwalk(cudaStream_t s, const K5Launch& l, bool from_dense_list) {
    switch (l.chunk_k) {
        case 2: return launch_one<2>(s, l, from_dense_list);
        case 4: return launch_one<4>(s, l, from_dense_list);
        case 8: return launch_one<8>(s, l, from_dense_list);
        case 16: return launch_one<16>(s, l, from_dense_list);
        default: return cudaErrorInvalidValue;
    }
}

} // namespace sfc
