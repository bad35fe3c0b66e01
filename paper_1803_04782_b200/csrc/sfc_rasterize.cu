// sfc_rasterize.cu — from-scratch rasterisation of the strength images on the device:
//   * rebuild / rasterize_dynamic (reference engine.cpp:158-168 -> fields.cpp:152-160), used by
//     the periodic drift check and image replacement (engine.cpp:538-550) and by seeding;
//   * rasterize_static (fields.cpp:162-168) for openings and obstacles.
//
// The reference scatters: for pedestrian 0, 1, 2, ... add (float)|strength| into every su of the
// field's support.  Float addition is order dependent, so a bit-identical result needs the same
// per-address order: ascending pedestrian id, and for one pedestrian whose field wraps onto
// itself, ascending row-major support offset.  Here it is a gather with that order made
// explicit: a CTA collects the pedestrian centres inside its tile + field-halo region, sorts
// them by (id, -y, -x) in shared memory (bitonic network on 64-bit keys), and every su walks
// the sorted list adding the table magnitudes in float — atomics-free and bit-exact.

#include <algorithm>
#include <cstdlib>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kTileW = 32;
constexpr int kRbThreads = 128;
constexpr int kRbTileH = kRbThreads / kTileW;
constexpr int kRbMaxEntries = 8192; // sorted-list capacity per tile (64 KB of keys)

struct RbArgs {
    GridDev g;
    TablesDev t;
    PedArrays p;
    const int* occ;
    float* dyn;
    float* out;
    Ctl* ctl;
    int tiles_x;
    int mode;
    int cap; // power of two
    unsigned* changed; // one bit per tile, or nullptr (see launch_rebuild)
    RebuildSkip skip;  // check pass: tiles no mover has reached since the previous rebuild are left alone
    int rw_full, dr_full, dc_full; // region width of a full-width tile and the scan's (row, column) step for it
    unsigned inv_rw_full;          // tid / rw_full = umulhi(tid, inv_rw_full) for tid < 2^16
};

// MODE 0: rasterize into `out`; 1: check pass (compare, drift, "changed" bits); 2: commit pass (replace the images).
// (A compile-time mode: the commit pass does not carry the check pass's prefetched records in registers.)
template <int MODE>
__global__ void __launch_bounds__(kRbThreads) rebuild_kernel(RbArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw); // [cap]
    float* acc = reinterpret_cast<float*>(keys + a.cap);                           // [24][NT]
    __shared__ int s_count;
    __shared__ float s_drift[kKinds][kRbThreads / 32];

    const GridDev g = a.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (MODE == 2 && a.ctl->error_code != 0) return;
    const int tile_x = blockIdx.x, tile_y = blockIdx.y; // (a 2-D grid: no division)
    const unsigned tile = (unsigned)tile_y * (unsigned)a.tiles_x + (unsigned)tile_x;
    if (MODE == 2 && a.changed != nullptr) { // the check pass found this tile's images equal to the fresh ones, bit for bit
        const unsigned word = a.changed[tile >> 5], bit = 1u << (tile & 31);
        if (!(word & bit)) return; // (uniform)
    }

    if (MODE == 1 && a.skip.stamp_lo != 0u) {
        // k-4 stamps every tile within field reach of a mover with the tick (TileMarks).  A tile not stamped since the
        // previous rebuild has seen no k-5 write, and every pedestrian whose field reaches it stands where it stood then:
        // its images are the fresh ones of that rebuild, bit for bit — nothing to compare, nothing to commit (its
        // "changed" bit stays clear).  Slab edge tiles also depend on pedestrians only the halo rows show: never skipped.
        const int mty = tile_y * kRbTileH / kMarkTileH;
        if (mty >= a.skip.marks.edge_lo && mty < a.skip.marks.edge_hi) {
            const unsigned stamp = a.skip.marks.epoch[mty * a.skip.marks.tiles_x + tile_x] >> 16;
            if (stamp < a.skip.stamp_lo || stamp > a.skip.stamp_hi) return; // (uniform)
        }
    }
    const int x0 = tile_x * kTileW, y0 = g.row0 + tile_y * kRbTileH;
    const int nx = min(kTileW, g.W - x0), ny = min(kRbTileH, g.row0 + g.rows - y0);
    const int HW = a.t.max_hw, HH = a.t.max_hh;
    const int RW = nx + 2 * HW, RH = ny + 2 * HH;
    const int xs = x0 - HW, ys = y0 - HH;
    const int lx = tid % kTileW, ly = tid / kTileW;
    const bool active = lx < nx && ly < ny;
    const int tcx = lx + HW, tcy = ly + HH;

    bool have_acc = false; // (most tiles of a sparse crowd see no centre: their sums are never materialised)
    // check pass: the su's record is requested now and compared after the region has been scanned and summed
    const long long my_cell = active ? cell_index(g, x0 + lx, y0 + ly) : 0;
    float4 old[6];
#pragma unroll
    for (int v = 0; v < 6; ++v)
        old[v] = (active && MODE == 1) ? reinterpret_cast<const float4*>(a.dyn + my_cell * 24)[v] : make_float4(0.f, 0.f, 0.f, 0.f);

    // The centres of the region are taken in ROUNDS of ascending id ranges: one round over every id when
    // they fit the sorted list (the usual case), else as many equal id ranges as bring a range's expected
    // share under half the capacity — per-address order is ascending id either way, so the float sums are
    // the reference's.  (Ids are handed out in placement order, i.e. uniformly over the grid.)
    int rounds = 1;
    for (int round = 0; round < rounds; ++round) {
        const long long id_lo = rounds == 1 ? 0 : a.p.n * round / rounds, id_hi = rounds == 1 ? a.p.n : a.p.n * (round + 1) / rounds;
        __syncthreads(); // (the previous round's walk is done with the keys)
        if (tid == 0) s_count = 0;
        __syncthreads();
        // collect the pedestrian centres of the region (any order; sorted below); (row, column) of a thread's cells
        // advance incrementally — no division, one wrap per axis
        const bool narrow = RW <= g.W; // (a field wider than the grid wraps more than once: the general path)
        auto consider_id = [&](int id, int wx, int wy, int ryi, int rxi) {
            if (id < id_lo || id >= id_hi) return; // (empty su hold -1)
            const int2 c = a.p.center[id];
            if (c.x != wx || c.y != wy) return; // a footprint su, not the centre
            const int pos = atomicAdd(&s_count, 1);
            if (pos < a.cap) {
                const uint32_t attr = a.p.attr[id];
                keys[pos] = ((unsigned long long)(uint32_t)id << 32) | ((unsigned long long)(8191 - ryi) << 19) |
                            ((unsigned long long)(8191 - rxi) << 6) | (unsigned long long)((attr >> 3) & 0x3Fu);
            }
        };
        auto consider = [&](long long idx, int wx, int wy, int ryi, int rxi) { consider_id(a.occ[idx], wx, wy, ryi, rxi); };
        {
            // (the divisions by the region width are done on the host for full-width tiles)
            const bool full = RW == a.rw_full;
            const int dr = full ? a.dr_full : kRbThreads / RW, dc = full ? a.dc_full : kRbThreads - dr * RW;
            int ryi = full ? (int)__umulhi((unsigned)tid, a.inv_rw_full) : tid / RW, rxi = tid - ryi * RW;
            const int ly0 = ys - g.row0 + g.halo; // local row of the region's first row, if it is resident unwrapped
            if (narrow && xs >= 0 && xs + RW <= g.W && ys >= 0 && ys + RH <= g.H && ly0 >= 0 && ly0 + RH <= g.rows + 2 * g.halo) {
                // the region lies inside the grid and inside the resident rows (nearly every tile): plain indexing
                // (four cells per trip: the occupancy loads of a trip are in flight together — a 7 x 7 field's region is
                // three cells per thread, one round trip instead of three)
                const long long base = (long long)ly0 * g.W + xs;
                while (ryi < RH) {
                    int id[4], by[4], bx[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        id[q] = kNoPed;
                        by[q] = bx[q] = 0;
                        if (ryi < RH) {
                            if (rxi >= RW) {
                                rxi -= RW;
                                ++ryi;
                            }
                            if (ryi < RH) {
                                id[q] = a.occ[base + (long long)ryi * g.W + rxi];
                                by[q] = ryi;
                                bx[q] = rxi;
                            }
                            rxi += dc;
                            ryi += dr;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) consider_id(id[q], xs + bx[q], ys + by[q], by[q], bx[q]);
                }
            } else {
                for (; ryi < RH; rxi += dc, ryi += dr) {
                    if (rxi >= RW) {
                        rxi -= RW;
                        if (++ryi >= RH) break;
                    }
                    int wx = xs + rxi, wy = ys + ryi;
                    long long idx;
                    if (narrow) {
                        const long long row = cell_index(g, 0, wy); // -1: the row does not exist / is not resident
                        if (row < 0) continue;
                        if (g.closed) {
                            if (wx < 0 || wx >= g.W) continue;
                        } else {
                            wx += wx < 0 ? g.W : (wx >= g.W ? -g.W : 0);
                        }
                        idx = row + wx;
                    } else {
                        idx = cell_index(g, wx, wy);
                        if (idx < 0) continue;
                        if (!g.closed) wx = emod(wx, g.W);
                    }
                    if (!g.closed) wy = emod(wy, g.H);
                    consider(idx, wx, wy, ryi, rxi);
                }
            }
        }
        __syncthreads();
        const int n = s_count;
        if (n > a.cap) {
            if (rounds == 1) { // too many centres for one sorted list: split the id range and start over
                rounds = min(4096, 2 * ((n + a.cap - 1) / a.cap));
                round = -1;
                continue;
            }
            if (tid == 0) raise_error(a.ctl, SFC_E_STATE, 5, x0, y0, (double)n);
            return;
        }
        // bitonic sort of the first pow2 >= n keys (padding keys are all-ones)
        int m = 1;
        while (m < n) m <<= 1;
        if (m > n) {
            for (int i = n + tid; i < m; i += kRbThreads) keys[i] = ~0ull;
            __syncthreads();
        }
        for (int k = 2; k <= m; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < m; i += kRbThreads) {
                    const int partner = i ^ j;
                    if (partner > i) {
                        const unsigned long long ka = keys[i], kb = keys[partner];
                        const bool up = (i & k) == 0;
                        if ((ka > kb) == up) {
                            keys[i] = kb;
                            keys[partner] = ka;
                        }
                    }
                }
                __syncthreads();
            }
        }

        if (n > 0 && !have_acc) { // (a thread's sums are its own column: no barrier needed)
#pragma unroll
            for (int q = 0; q < kKinds * kSects; ++q) acc[q * kRbThreads + tid] = 0.0f;
            have_acc = true;
        }
        if (active && n > 0) {
            for (int e = 0; e < n; ++e) {
                const unsigned long long key = keys[e];
                const int ry = 8191 - (int)((key >> 19) & 0x1FFF), rx = 8191 - (int)((key >> 6) & 0x1FFF);
                const int dx = rx - tcx, dy = ry - tcy; // centre offset = centre - target
                if ((dx | dy) == 0) continue;
                const uint32_t orients = (uint32_t)(key & 0x3F);
#pragma unroll
                for (int kind = 0; kind < kKinds; ++kind) {
                    const KindTableDev kt = a.t.k[kind];
                    if (dx < -kt.hw || dx > kt.hw || dy < -kt.hh || dy > kt.hh) continue;
                    const int ti = (dy + kt.hh) * kt.fw + dx + kt.hw;
                    const uint32_t info = __ldg(kt.info + ti);
                    const uint32_t mask = (info >> 3) & 0xFFu;
                    const int orient = kind == 0 ? (orients & 7) : (kind == 1 ? ((orients >> 3) & 7) : 0);
                    if (!((mask >> orient) & 1u)) continue;
                    float* slot = acc + (kind * kSects + (info & 7)) * kRbThreads + tid;
                    *slot = __fadd_rn(*slot, __double2float_rn(__ldg(kt.mag + ti))); // += (float)s.norm()
                }
            }
        }
    }

    float drift[kKinds] = {0.0f, 0.0f, 0.0f};
    bool differs = false;
    if (active) { // the su's 96-byte record as six 16-byte accesses
        float4* const rec = reinterpret_cast<float4*>((MODE == 0 ? a.out : a.dyn) + my_cell * 24);
        bool blank = false; // nothing in reach and the record is all +0.0f: equal, no drift
        if (MODE == 1 && !have_acc) {
            uint32_t any_bits = 0u;
#pragma unroll
            for (int v = 0; v < 6; ++v)
                any_bits |= __float_as_uint(old[v].x) | __float_as_uint(old[v].y) | __float_as_uint(old[v].z) | __float_as_uint(old[v].w);
            blank = any_bits == 0u;
        }
        if (MODE == 1 && !blank) {
#pragma unroll
            for (int v = 0; v < 6; ++v) {
                const float o[4] = {old[v].x, old[v].y, old[v].z, old[v].w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int q = 4 * v + c;
                    const float fresh = have_acc ? acc[q * kRbThreads + tid] : 0.0f;
                    const float d = fabsf(o[c] - fresh);
                    if (drift[q / 8] < d) drift[q / 8] = d; // std::max(worst, d): a NaN never wins
                    differs = differs || __float_as_uint(o[c]) != __float_as_uint(fresh);
                }
            }
        } else if (MODE != 1) {
#pragma unroll
            for (int v = 0; v < 6; ++v)
                rec[v] = have_acc ? make_float4(acc[(4 * v) * kRbThreads + tid], acc[(4 * v + 1) * kRbThreads + tid],
                                                acc[(4 * v + 2) * kRbThreads + tid], acc[(4 * v + 3) * kRbThreads + tid])
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    if (a.changed != nullptr) { // the tile's "commit needed" bit: set by the check pass, consumed by the commit pass
        if (MODE == 1) {
            if (__any_sync(0xFFFFFFFFu, differs) && lane == 0) atomicOr(&a.changed[tile >> 5], 1u << (tile & 31));
        } else if (MODE == 2) {
            __syncthreads(); // (every thread of the CTA has read the word)
            if (tid == 0) atomicAnd(&a.changed[tile >> 5], ~(1u << (tile & 31)));
        }
    }
    if (MODE == 1) { // max_abs_difference (fields.cpp:144-150) reduced warp -> CTA -> grid
        const bool some = __any_sync(0xFFFFFFFFu, drift[0] > 0.0f || drift[1] > 0.0f || drift[2] > 0.0f);
#pragma unroll
        for (int k = 0; k < kKinds; ++k) {
            float v = drift[k];
            if (some) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
            }
            if (lane == 0) s_drift[k][warp] = v;
        }
        __syncthreads();
        if (tid < kKinds) {
            float v = 0.0f;
            for (int w = 0; w < kRbThreads / 32; ++w) v = fmaxf(v, s_drift[tid][w]);
            if (v > 0.0f) atomicMax(&a.ctl->drift_bits[tid], __float_as_uint(v)); // non-negative floats order as uints
        }
    }
}

__global__ void drift_verdict_kernel(Ctl* ctl, double tolerance) { // engine.cpp:541-548
    if (ctl->error_code != 0) return;
    for (int k = 0; k < kKinds; ++k) {
        const float drift = __uint_as_float(ctl->drift_bits[k]);
        if ((double)drift > tolerance) {
            raise_error(ctl, SFC_E_INTEGRITY, 5, k, 0, (double)drift);
            break;
        }
    }
    for (int k = 0; k < kKinds; ++k) ctl->drift_bits[k] = 0u;
}

// One anchored static field (rasterize_into, fields.cpp:152-160) as a per-target gather: the
// thread owning target su t adds the field's strength once per periodic image of t inside the
// support, images in row-major offset order.
__global__ void static_anchor_kernel(GridDev g, KindTableDev kt, float* stat, int ax, int ay, int bw, int bh,
                                     int orientation) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= bw * bh) return;
    const int by = i / bw, bx = i - by * bw;
    // first unwrapped target of this thread's residue class, then its periodic images
    const int ux0 = ax - kt.hw + bx, uy0 = ay - kt.hh + by;
    const long long idx = cell_index(g, ux0, uy0);
    if (idx < 0) return; // clipped under a closed boundary
    const int stepx = g.closed ? (kt.fw + 1) : g.W, stepy = g.closed ? (kt.fh + 1) : g.H;
    for (int uy = uy0; uy <= ay + kt.hh; uy += stepy) {
        for (int ux = ux0; ux <= ax + kt.hw; ux += stepx) {
            const int dx = ax - ux, dy = ay - uy; // centre offset = anchor - target
            if ((dx | dy) == 0) continue;
            const int ti = (dy + kt.hh) * kt.fw + dx + kt.hw;
            const uint32_t info = kt.info[ti];
            const uint32_t mask = (info >> 3) & 0xFFu;
            if (mask == 0 || (orientation >= 0 && !((mask >> orientation) & 1u))) continue;
            float* slot = stat + idx * kSects + (info & 7);
            *slot = __fadd_rn(*slot, __double2float_rn(kt.mag[ti]));
        }
    }
}

int next_pow2(int v) {
    int m = 32;
    while (m < v) m <<= 1;
    return m;
}

} // namespace

namespace {
int rebuild_cap(const TablesDev& t) {
    const int region = (kTileW + 2 * t.max_hw) * (kRbTileH + 2 * t.max_hh);
    return next_pow2(region < kRbMaxEntries ? region : kRbMaxEntries);
}
size_t rebuild_smem(const TablesDev& t) {
    return sizeof(unsigned long long) * (size_t)rebuild_cap(t) + sizeof(float) * 24 * kRbThreads;
}
} // namespace

// Raises the dynamic shared-memory limit ahead of time (must not happen inside a graph capture).
cudaError_t prepare_rebuild(const TablesDev& t) {
    static SmemGrant grant[3];
    cudaError_t e = grant[0].raise(reinterpret_cast<const void*>(rebuild_kernel<0>), rebuild_smem(t), 48 * 1024);
    if (e == cudaSuccess) e = grant[1].raise(reinterpret_cast<const void*>(rebuild_kernel<1>), rebuild_smem(t), 48 * 1024);
    if (e == cudaSuccess) e = grant[2].raise(reinterpret_cast<const void*>(rebuild_kernel<2>), rebuild_smem(t), 48 * 1024);
    // the passes are latency-bound on small CTAs: ask for the largest shared-memory carve-out so that shared memory
    // does not cap the resident CTAs below what the registers allow (a hint; failure is harmless)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(rebuild_kernel<0>), cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(rebuild_kernel<1>), cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(rebuild_kernel<2>), cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    (void)cudaGetLastError();
    return e;
}

long long rebuild_tile_count(const GridDev& g) { return (long long)((g.W + kTileW - 1) / kTileW) * ((g.rows + kRbTileH - 1) / kRbTileH); }

cudaError_t launch_rebuild(cudaStream_t s, const GridDev& g, const TablesDev& t, const PedArrays& p, const int* occ,
                           float* dyn, float* out, Ctl* ctl, int mode, double /*tolerance*/, unsigned* changed, const RebuildSkip* skip) {
    RbArgs a;
    a.g = g;
    a.t = t;
    a.p = p;
    a.occ = occ;
    a.dyn = dyn;
    a.out = out;
    a.ctl = ctl;
    a.mode = mode;
    a.changed = changed;
    a.skip = (skip != nullptr && mode == 1 && changed != nullptr && skip->marks.epoch != nullptr) ? *skip : RebuildSkip{};
    a.tiles_x = (g.W + kTileW - 1) / kTileW;
    a.rw_full = kTileW + 2 * t.max_hw;
    a.dr_full = kRbThreads / a.rw_full;
    a.dc_full = kRbThreads - a.dr_full * a.rw_full;
    a.inv_rw_full = 0xFFFFFFFFu / (unsigned)a.rw_full + 1u;
    a.cap = rebuild_cap(t);
    if (const char* knob = std::getenv("SFC_REBUILD_CAP")) // (tests: a short sorted list forces the id-range rounds)
        a.cap = std::min(a.cap, next_pow2(std::max(1, std::atoi(knob))));
    const size_t smem = rebuild_smem(t);
    const int tiles_y = (g.rows + kRbTileH - 1) / kRbTileH;
    if (tiles_y > 65535) return cudaErrorInvalidConfiguration; // (262 140 rows per slab / band)
    const dim3 grid((unsigned)a.tiles_x, (unsigned)tiles_y);
    if (mode == 0) rebuild_kernel<0><<<grid, kRbThreads, smem, s>>>(a);
    else if (mode == 1) rebuild_kernel<1><<<grid, kRbThreads, smem, s>>>(a);
    else rebuild_kernel<2><<<grid, kRbThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_drift_verdict(cudaStream_t s, Ctl* ctl, double tolerance) {
    drift_verdict_kernel<<<1, 1, 0, s>>>(ctl, tolerance);
    return cudaGetLastError();
}

cudaError_t launch_static_anchor(cudaStream_t s, const GridDev& g, const KindTableDev& t, float* stat, int ax, int ay,
                                 int orientation) {
    // one thread per residue class of target su: the whole support box, or the whole grid
    // extent along an axis where the support is at least as wide as a periodic grid
    const int bw = (!g.closed && t.fw > g.W) ? g.W : t.fw;
    const int bh = (!g.closed && t.fh > g.H) ? g.H : t.fh;
    const int n = bw * bh;
    static_anchor_kernel<<<(n + 127) / 128, 128, 0, s>>>(g, t, stat, ax, ay, bw, bh, orientation);
    return cudaGetLastError();
}

} // namespace sfc
