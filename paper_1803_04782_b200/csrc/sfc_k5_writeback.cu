// sfc_k5_writeback.cu — k-5, the field write-back: superpose the movement of every pedestrian
// onto the three dynamic strength images (reference engine.cpp:428-472, the loop that takes
// 63-98 % of the CPU reference's tick).
//
// Reference formulation: for every (su, kind, sect) address walk a precomputed list of F
// contributor offsets, read two mask bytes per offset, accumulate gated +-magnitude terms in
// doubles through a K-slot StepCache (term idx -> slot idx mod K, accumulator.hpp:36-46), fold
// the K slots in slot order, cast to float, add to the image.  6F mask probes per su.
//
// B200 formulation (bit-identical results):
//   * One CTA owns a 32 x TH tile of su.  It scans the tile + field-halo region of the 2-byte
//     event map ONCE, compacting the (few) movement events into a shared-memory list ordered
//     by (x, then y).  That order equals the reference's contributor-list order for every
//     target in the tile, because the lists are sorted lexicographically by centre offset
//     (fields.hpp:55-57) — so walking the list front to back feeds every StepCache slot its
//     terms in the reference's order.  Zero terms are never materialised: adding +-0.0 to a
//     partial cannot change it.
//   * Each thread owns one su.  Its K x (sects per pass) double partials live in shared memory
//     laid out [slot][thread] (bank = thread: conflict-free for any per-lane slot), created
//     lazily under a dirty bitmask so untouched addresses cost nothing.
//   * The tile's 96-byte su records move HBM -> shared -> HBM with cp.async.bulk (TMA 1-D bulk
//     copies, one per tile row, mbarrier completion), issued before the gather so the copy
//     overlaps the arithmetic.  A tile whose region holds no event is skipped without touching
//     the images; rows of a tile that received no term are not written back.
//
// Fields larger than the grid wrap onto themselves (test_engine.cpp:329-340): the region is
// scanned in unwrapped coordinates, so one physical su can appear several times, once per
// periodic image — exactly the reference's while-loop wraps (engine.cpp:450-454).

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kTileW = 32;
constexpr int kTabSmemMax = 1024; // table entries (all kinds) kept in shared memory

struct K5Args {
    GridDev g;
    TablesDev t;
    float* dyn;
    const uint8_t* ev;
    Ctl* ctl;
    int tiles_x;
    int advance_tick;
    int tab_smem;  // tables fit in shared memory
    int cap;       // event-list capacity (entries)
    int rw_max;    // region columns for a full tile
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// K: StepCache width.  NT: threads = su per tile (32 x NT/32).  SG: sects accumulated per pass
// (SG * K <= 64 so the dirty set is one 64-bit word).
template <int K, int NT, int SG>
__global__ void __launch_bounds__(NT) k5_writeback_kernel(K5Args a) {
    constexpr int TH = NT / kTileW;
    constexpr int NW = NT / 32;
    static_assert(SG * K <= 64, "dirty mask is one 64-bit word");
    extern __shared__ __align__(128) unsigned char smem_raw[];

    const GridDev g = a.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (a.advance_tick && blockIdx.x == 0 && tid == 0 && a.ctl->error_code == 0) a.ctl->tick += 1;
    if (a.ctl->error_code != 0) return;

    // ---- shared memory carve-up ----
    double* part = reinterpret_cast<double*>(smem_raw);                       // [SG*K][NT]
    float* tile = reinterpret_cast<float*>(part + SG * K * NT);               // [NT][24], 128-B aligned
    uint2* evl = reinterpret_cast<uint2*>(tile + NT * 24);                    // [cap]
    int* colstart = reinterpret_cast<int*>(evl + a.cap);                      // [rw_max + 2]
    double* tab_mag = reinterpret_cast<double*>(colstart + ((a.rw_max + 2 + 1) & ~1)); // [entries] if tab_smem
    uint32_t* tab_info = reinterpret_cast<uint32_t*>(tab_mag + (a.tab_smem ? a.t.total_entries : 0));
    int* warp_cnt = reinterpret_cast<int*>(tab_info + (a.tab_smem ? ((a.t.total_entries + 1) & ~1) : 0)); // [2][NW]
    uint64_t* bar = reinterpret_cast<uint64_t*>(warp_cnt + 2 * NW + ((2 * NW) & 1));
    int* row_dirty = reinterpret_cast<int*>(bar + 1); // [TH]

    const int tile_x = blockIdx.x % a.tiles_x, tile_y = blockIdx.x / a.tiles_x;
    const int x0 = tile_x * kTileW;
    const int y0 = g.row0 + tile_y * TH; // global row of the tile's first row
    const int nx = min(kTileW, g.W - x0);
    const int ny = min(TH, g.row0 + g.rows - y0);
    const int HW = a.t.max_hw, HH = a.t.max_hh;
    const int RW = nx + 2 * HW, RH = ny + 2 * HH;
    const int xs = x0 - HW, ys = y0 - HH;
    const int lx = tid % kTileW, ly = tid / kTileW;
    const bool active = lx < nx && ly < ny;
    const int tcx = lx + HW, tcy = ly + HH; // my su in region coordinates

    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < TH) row_dirty[tid] = 0;
    if (a.tab_smem) {
        int base = 0;
        for (int k = 0; k < kKinds; ++k) {
            const int n = a.t.k[k].fw * a.t.k[k].fh;
            for (int i = tid; i < n; i += NT) {
                tab_mag[base + i] = a.t.k[k].mag[i];
                tab_info[base + i] = a.t.k[k].info[i];
            }
            base += n;
        }
    }
    __syncthreads();

    const uint16_t* ev16 = reinterpret_cast<const uint16_t*>(a.ev);
    const int cols_per_pass = max(1, a.cap / RH);
    const bool single_pass = cols_per_pass >= RW;

    // Compacts the events of region columns [c0, c1) into evl, ordered by (x, y); leaves
    // colstart[c - c0] = index of the first event with column >= c.  Returns the count.
    auto build_list = [&](int c0, int c1) -> int {
        const int ncols = c1 - c0;
        for (int i = tid; i <= ncols; i += NT) colstart[i] = 0;
        __syncthreads();
        const int ncell = ncols * RH;
        int running = 0;
        int parity = 0;
        for (int base = 0; base < ncell; base += NT, parity ^= 1) {
            const int i = base + tid;
            uint32_t code = 0;
            int rxi = 0, ryi = 0;
            if (i < ncell) {
                rxi = c0 + i / RH;
                ryi = i - (rxi - c0) * RH;
                const long long idx = cell_index(g, xs + rxi, ys + ryi);
                if (idx >= 0) code = ev16[idx];
            }
            const unsigned ballot = __ballot_sync(0xFFFFFFFFu, code != 0);
            if (lane == 0) warp_cnt[parity * NW + warp] = __popc(ballot);
            __syncthreads();
            int before = 0, total = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const int c = warp_cnt[parity * NW + w];
                before += w < warp ? c : 0;
                total += c;
            }
            if (code != 0) {
                const int pos = running + before + __popc(ballot & ((1u << lane) - 1u));
                evl[pos] = make_uint2((uint32_t)rxi | ((uint32_t)ryi << 16), code);
                atomicAdd(&colstart[rxi - c0 + 1], 1); // per-column counts, shifted by one
            }
            running += total;
        }
        __syncthreads();
        if (warp == 0) { // inclusive scan of the shifted counts = exclusive starts
            int carry = 0;
            for (int base = 0; base <= ncols; base += 32) {
                const int i = base + lane;
                int v = i <= ncols ? colstart[i] : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xFFFFFFFFu, v, o);
                    if (lane >= o) v += u;
                }
                if (i <= ncols) colstart[i] = v + carry;
                carry += __shfl_sync(0xFFFFFFFFu, v, 31);
            }
        }
        __syncthreads();
        return running;
    };

    auto issue_tile_load = [&]() {
        if (tid == 0) {
            mbar_expect_tx(bar, (uint32_t)(ny * nx * 96));
            for (int r = 0; r < ny; ++r) {
                const long long cell = cell_index(g, x0, y0 + r);
                bulk_g2s(tile + r * kTileW * 24, a.dyn + cell * 24, (uint32_t)(nx * 96), bar);
            }
        }
    };

    int n_events = 0;
    if (single_pass) {
        n_events = build_list(0, RW);
        if (n_events == 0) return; // nobody moved within reach of this tile
    }
    issue_tile_load();

    bool touched = false;
    bool tile_ready = false;

#pragma unroll 1
    for (int kind = 0; kind < kKinds; ++kind) {
        const KindTableDev kt = a.t.k[kind];
        int tbase = 0;
        for (int k = 0; k < kind; ++k) tbase += a.t.k[k].fw * a.t.k[k].fh;
        const double* kmag = a.tab_smem ? tab_mag + tbase : kt.mag;
        const uint32_t* kinfo = a.tab_smem ? tab_info + tbase : kt.info;
#pragma unroll 1
        for (int sg = 0; sg < kSects / SG; ++sg) {
            unsigned long long dirty = 0ull;
            auto walk = [&](int c0, int c1) {
                if (!active) return;
                const int lo_c = min(max(tcx - kt.hw, c0), c1), hi_c = min(max(tcx + kt.hw + 1, c0), c1);
                const int lo = colstart[lo_c - c0], hi = colstart[hi_c - c0];
                for (int e = lo; e < hi; ++e) {
                    const uint2 evt = evl[e];
                    const int dy = (int)(evt.x >> 16) - tcy;
                    if (dy < -kt.hh || dy > kt.hh) continue;
                    const int dx = (int)(evt.x & 0xFFFFu) - tcx;
                    if ((dx | dy) == 0) continue;
                    const int ti = (dy + kt.hh) * kt.fw + dx + kt.hw;
                    const uint32_t info = kinfo[ti];
                    const uint32_t mask = (info >> 3) & 0xFFu;
                    if (mask == 0) continue;
                    const int sect = info & 7;
                    if (SG < kSects && sect / SG != sg) continue;
                    const int ls = sect % SG;
                    const uint32_t j2 = (info >> 11) << 1;
                    const double mag = kmag[ti];
                    const uint32_t fb = evt.y & 0xFFu, tb = (evt.y >> 8) & 0xFFu;
                    const int shift = kind == 0 ? 0 : (kind == 1 ? 3 : 8); // kind 2: orientation 0 of an all-ones mask
#pragma unroll
                    for (int half = 0; half < 2; ++half) { // from-term (idx 2j) then to-term (idx 2j+1)
                        const uint32_t b = half == 0 ? fb : tb;
                        if (!(b & 0x80u)) continue;
                        const int orient = (int)((b >> shift) & 7u);
                        if (!((mask >> orient) & 1u)) continue;
                        const int slot = (int)((j2 + half) & (K - 1));
                        const int addr = ls * K + slot;
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

            if (single_pass) {
                walk(0, RW);
            } else {
                for (int c0 = 0; c0 < RW; c0 += cols_per_pass) {
                    const int c1 = min(RW, c0 + cols_per_pass);
                    const int n = build_list(c0, c1);
                    if (n > 0) walk(c0, c1);
                    __syncthreads(); // list is rebuilt next iteration
                }
            }

            if (dirty != 0ull) {
                if (!tile_ready) {
                    mbar_wait(bar, 0);
                    tile_ready = true;
                }
                touched = true;
                // vector access to my su record: 96-byte stride across lanes is 2-way conflicted
                // for 128-bit accesses but 8-way for scalars
                float* rec = tile + tid * 24 + kind * kSects + sg * SG;
                float r[SG];
                if constexpr (SG == 2) {
                    const float2 v = *reinterpret_cast<const float2*>(rec);
                    r[0] = v.x; r[1] = v.y;
                } else {
#pragma unroll
                    for (int q = 0; q < SG / 4; ++q) {
                        const float4 v = reinterpret_cast<const float4*>(rec)[q];
                        r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
                    }
                }
#pragma unroll
                for (int ls = 0; ls < SG; ++ls) {
                    const unsigned m = (unsigned)((dirty >> (ls * K)) & ((1ull << K) - 1ull));
                    if (m == 0) continue;
                    double total = 0.0; // StepCache::total, slot order (accumulator.hpp:41-46)
#pragma unroll
                    for (int slot = 0; slot < K; ++slot) {
                        if ((m >> slot) & 1u) total = __dadd_rn(total, part[(ls * K + slot) * NT + tid]);
                    }
                    r[ls] = __fadd_rn(r[ls], __double2float_rn(total)); // image += (float)total
                }
                if constexpr (SG == 2) {
                    *reinterpret_cast<float2*>(rec) = make_float2(r[0], r[1]);
                } else {
#pragma unroll
                    for (int q = 0; q < SG / 4; ++q)
                        reinterpret_cast<float4*>(rec)[q] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                }
            }
        }
    }

    if (touched) row_dirty[ly] = 1;
    if (!tile_ready) mbar_wait(bar, 0); // the bulk loads must land before the CTA may exit
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
        bool any = false;
        for (int r = 0; r < ny; ++r) {
            if (!row_dirty[r]) continue;
            const long long cell = cell_index(g, x0, y0 + r);
            bulk_s2g(a.dyn + cell * 24, tile + r * kTileW * 24, (uint32_t)(nx * 96));
            any = true;
        }
        if (any) bulk_commit_wait_read();
    }
}

struct K5Shape {
    size_t smem;
    int cap, rw_max, tab_smem;
};

template <int K, int NT, int SG>
K5Shape k5_shape(const TablesDev& t) {
    constexpr int TH = NT / kTileW;
    K5Shape s;
    s.rw_max = kTileW + 2 * t.max_hw;
    const int rh_max = TH + 2 * t.max_hh;
    s.cap = 1024;
    if (s.cap < rh_max) s.cap = (rh_max + 31) & ~31;
    s.tab_smem = t.total_entries <= kTabSmemMax;
    size_t b = 0;
    b += sizeof(double) * SG * K * NT;
    b += sizeof(float) * NT * 24;
    b += sizeof(uint2) * (size_t)s.cap;
    b += sizeof(int) * (size_t)((s.rw_max + 2 + 1) & ~1);
    if (s.tab_smem) b += sizeof(double) * t.total_entries + sizeof(uint32_t) * ((t.total_entries + 1) & ~1);
    b += sizeof(int) * (2 * (NT / 32) + ((2 * (NT / 32)) & 1));
    b += sizeof(uint64_t);
    b += sizeof(int) * TH;
    s.smem = (b + 127) & ~(size_t)127;
    return s;
}

template <int K, int NT, int SG>
cudaError_t launch_variant(cudaStream_t stream, const K5Launch& l) {
    constexpr int TH = NT / kTileW;
    const K5Shape sh = k5_shape<K, NT, SG>(l.t);
    K5Args a;
    a.g = l.g;
    a.t = l.t;
    a.dyn = l.dyn;
    a.ev = l.ev;
    a.ctl = l.ctl;
    a.tiles_x = (l.g.W + kTileW - 1) / kTileW;
    a.advance_tick = l.advance_tick;
    a.tab_smem = sh.tab_smem;
    a.cap = sh.cap;
    a.rw_max = sh.rw_max;
    const int tiles_y = (l.g.rows + TH - 1) / TH;
    const long long blocks = (long long)a.tiles_x * tiles_y;
    k5_writeback_kernel<K, NT, SG><<<(unsigned)blocks, NT, sh.smem, stream>>>(a);
    return cudaGetLastError();
}

template <int K, int NT, int SG>
cudaError_t prepare_variant(const TablesDev& t) {
    return cudaFuncSetAttribute(k5_writeback_kernel<K, NT, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)k5_shape<K, NT, SG>(t).smem);
}

} // namespace

// Raises the dynamic shared-memory limit of the variant sfc_create will launch; done once at
// engine construction so no attribute call lands inside a CUDA-graph capture.
cudaError_t prepare_k5_writeback(int chunk_k, const TablesDev& t) {
    switch (chunk_k) {
        case 2: return prepare_variant<2, 128, 8>(t);
        case 4: return prepare_variant<4, 128, 8>(t);
        case 8: return prepare_variant<8, 128, 8>(t);
        case 16: return prepare_variant<16, 128, 4>(t);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k5_writeback(cudaStream_t s, const K5Launch& l) {
    switch (l.chunk_k) {
        case 2: return launch_variant<2, 128, 8>(s, l);
        case 4: return launch_variant<4, 128, 8>(s, l);
        case 8: return launch_variant<8, 128, 8>(s, l);
        case 16: return launch_variant<16, 128, 4>(s, l);
        default: return cudaErrorInvalidValue;
    }
}

size_t k5_smem_bytes(int chunk_k, const TablesDev& t) {
    switch (chunk_k) {
        case 2: return k5_shape<2, 128, 8>(t).smem;
        case 4: return k5_shape<4, 128, 8>(t).smem;
        case 8: return k5_shape<8, 128, 8>(t).smem;
        default: return k5_shape<16, 128, 4>(t).smem;
    }
}

} // namespace sfc
