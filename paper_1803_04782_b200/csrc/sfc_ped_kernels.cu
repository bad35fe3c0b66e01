// sfc_ped_kernels.cu — per-pedestrian phases of the tick: k-2 decide, k-3 vote, k-4 move.
//
// k-2 follows the reference's decide_core arithmetic exactly (engine.cpp:289-324): double
// precision, products and sums individually rounded (__dmul_rn/__dadd_rn — the reference binary
// contains no FMA), the 19-comparator sort network with ties to the lower sect (engine.cpp:31-50).
//
// k-3/k-4 do NOT materialise the reference's 96-byte-per-su EnrollmentTable.  Under v_max = 1
// the only pedestrian that can register for su c through slot d is the occupant of c - step(d)
// (engine.hpp:45-48), so the winner test for a newly covered su is an 8-neighbour gather on
// the occupancy grid plus the per-pedestrian decision arrays: same result, no per-su
// temporaries, no atomics, no full-grid clear (the reference's k-1).

#include <atomic>
#include <climits>
#include <cstdlib>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr int kPedThreads = 128;

__device__ __forceinline__ int sect_distance(int a, int b) { // fields.cpp:62-65
    int d = (a - b) & 7;
    return d < 8 - d ? d : 8 - d;
}

// Visits the su a step in `dir` would newly cover (engine.cpp:271-287: the cells of the new
// footprint the old footprint does not already cover form an L: one column if the step has an
// x component, one row if it has a y component).  fn(x, y) gets unwrapped global coordinates
// and returns false to stop early.  Returns false if stopped.
template <class Fn>
__device__ __forceinline__ bool for_new_cells(int cx, int cy, int rw, int rh, int dir, Fn&& fn) {
    const int ux = step_dx(dir), uy = step_dy(dir);
    const int ncx = cx + ux, ncy = cy + uy;
    if (ux != 0) {
        const int ox = ux > 0 ? rw : -rw;
        for (int oy = -rh; oy <= rh; ++oy)
            if (!fn(ncx + ox, ncy + oy)) return false;
    }
    if (uy != 0) {
        const int oy = uy > 0 ? rh : -rh;
        const int skip = ux != 0 ? (ux > 0 ? rw : -rw) : (rw + 1); // corner already visited
        for (int ox = -rw; ox <= rw; ++ox) {
            if (ox == skip) continue;
            if (!fn(ncx + ox, ncy + oy)) return false;
        }
    }
    return true;
}

// The pedestrian thread t of a per-pedestrian kernel works on.  Pedestrians are seeded at random su, so in id order
// every thread of a warp reads its own sectors of the images and of the occupancy grid; PedArrays::order lists
// the ids by centre in row-major order as of the last ordering pass (order_pedestrians below), which puts
// neighbours in one warp.  Ids stay the tie-break everywhere (engine.cpp:375-378), so the order a tick visits
// the pedestrians in cannot change its result.
__device__ __forceinline__ long long ped_of_thread(const PedArrays& p, const Ctl* ctl, long long t) {
    return (p.order != nullptr && ctl->order_ok != 0) ? (long long)p.order[t] : t;
}

// One compare-exchange of the sort network on (score, sect) pairs: keep the better key first —
// higher score, lower sect on ties (engine.cpp:34-41).
__device__ __forceinline__ void cex(double& sa, int& ia, double& sb, int& ib) {
    const bool swap = (sa < sb) || (sa == sb && ia > ib);
    const double ts = swap ? sb : sa;
    const int ti = swap ? ib : ia;
    sb = swap ? sa : sb;
    ib = swap ? ia : ib;
    sa = ts;
    ia = ti;
}

// (The three per-pedestrian phases are device functions of the thread's index.  Running all three in ONE launch for
// a crowd of one CTA — CTA barriers instead of launches — was measured and is slower: config 1, 29.1 against 25.4 us a
// tick; the phases are chains of dependent loads, and four CTAs on four SMs hide them better than one.)
__device__ __forceinline__ void k2_decide_body(long long t, const GridDev& g, const PedArrays& p, const int* occ, const float* __restrict__ stat,
                                               const float* dyn, uint8_t* ev, Ctl* ctl, const DecideParams& dp, const SlabDev& slab) {
    if (t >= p.n) return;
    if (ctl->error_code != 0) return;
    const long long i = ped_of_thread(p, ctl, t);
    const int2 c = p.center[i];
    if (!row_owned(g, c.y)) return;
    const uint32_t attr = p.attr[i];

    // Retire the previous tick's movement events of this pedestrian (the reference clears its
    // whole MovementLog in k-1, engine.cpp:335-339; here only the two touched su are reset).
    const int md = slab.active ? -1 : p.moved_dir[i]; // (slabs clear their event cells from a written-list instead)
    if (md >= 0) {
        const long long to = cell_index(g, c.x, c.y);
        const long long from = cell_index(g, c.x - step_dx(md), c.y - step_dy(md));
        ev[2 * to + 1] = 0;
        if (from >= 0) ev[2 * from] = 0;
        p.moved_dir[i] = -1;
    }

    int8_t out_dir = kStill;
    double out_score = 0.0;

    const int2 gate = p.gate[i];
    const long long tick = ctl->tick;
    if (tick % gate.x == gate.y) { // walk gate, engine.cpp:291
        const int rw = attr_half_w(attr), rh = attr_half_h(attr);
        double gfac = 1.0;
        if (dp.regulated) { // local_density (grid.cpp:58-72) + regulate (engine.cpp:242-248)
            int occupied = 0, window = 0;
            const int r = dp.density_radius;
            for (int oy = -r; oy <= r; ++oy) {
                for (int ox = -r; ox <= r; ++ox) {
                    const long long idx = cell_index(g, c.x + ox, c.y + oy);
                    if (idx < 0) continue;
                    ++window;
                    occupied += occ[idx] != kNoPed;
                }
            }
            const double rho = window == 0 ? 0.0 : __ddiv_rn((double)occupied, (double)window);
            gfac = fmax(0.1, __dsub_rn(1.0, rho));
        }

        const long long base = cell_index(g, c.x, c.y);
        const float4* sp = reinterpret_cast<const float4*>(stat + base * kSects);
        const float4* dq = reinterpret_cast<const float4*>(dyn + base * (kKinds * kSects));
        float img[4][8];
        {
            const float4 a = __ldg(sp), b = __ldg(sp + 1);
            img[0][0] = a.x; img[0][1] = a.y; img[0][2] = a.z; img[0][3] = a.w;
            img[0][4] = b.x; img[0][5] = b.y; img[0][6] = b.z; img[0][7] = b.w;
#pragma unroll
            for (int k = 0; k < kKinds; ++k) {
                const float4 u = dq[2 * k], v = dq[2 * k + 1];
                img[k + 1][0] = u.x; img[k + 1][1] = u.y; img[k + 1][2] = u.z; img[k + 1][3] = u.w;
                img[k + 1][4] = v.x; img[k + 1][5] = v.y; img[k + 1][6] = v.z; img[k + 1][7] = v.w;
            }
        }
        const int goal = attr_goal(attr);
        double s[8];
        int o[8];
#pragma unroll
        for (int sect = 0; sect < 8; ++sect) {
            double raw = __dmul_rn(dp.w_static, (double)img[0][sect]);
#pragma unroll
            for (int k = 0; k < kKinds; ++k) raw = __dadd_rn(raw, __dmul_rn(dp.w_kind[k], (double)img[k + 1][sect]));
            const int dist = sect_distance(sect, goal);
            const double kcos = dist == 0 ? 1.0 : (dist == 1 ? 0.70710678118654752440 : 0.0);
            s[sect] = __dadd_rn(__dmul_rn(gfac, raw), __dmul_rn(dp.goal_bias, kcos));
            o[sect] = sect;
        }
        // sort8_desc, engine.cpp:42-48
        cex(s[0], o[0], s[1], o[1]); cex(s[2], o[2], s[3], o[3]); cex(s[0], o[0], s[2], o[2]);
        cex(s[1], o[1], s[3], o[3]); cex(s[1], o[1], s[2], o[2]);
        cex(s[4], o[4], s[5], o[5]); cex(s[6], o[6], s[7], o[7]); cex(s[4], o[4], s[6], o[6]);
        cex(s[5], o[5], s[7], o[7]); cex(s[5], o[5], s[6], o[6]);
        cex(s[0], o[0], s[4], o[4]); cex(s[1], o[1], s[5], o[5]); cex(s[1], o[1], s[4], o[4]);
        cex(s[2], o[2], s[6], o[6]); cex(s[3], o[3], s[7], o[7]); cex(s[3], o[3], s[6], o[6]);
        cex(s[2], o[2], s[4], o[4]); cex(s[3], o[3], s[5], o[5]); cex(s[3], o[3], s[4], o[4]);

        if ((rw | rh) == 0) {
            // 1 x 1 pedestrian: a step newly covers exactly the neighbour su.  All eight neighbours are
            // read at once (one memory round trip) instead of one per rejected candidate.
            int nb[8];
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                const long long idx = cell_index(g, c.x + step_dx(d), c.y + step_dy(d));
                nb[d] = idx >= 0 ? occ[idx] : 0; // off a closed grid: never empty
            }
            unsigned free_dirs = 0u;
#pragma unroll
            for (int d = 0; d < 8; ++d) free_dirs |= (nb[d] == kNoPed ? 1u : 0u) << d;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (out_dir != kStill) break;
                if (s[r] <= 0.0) break; // sorted: no later direction qualifies (engine.cpp:319)
                if ((free_dirs >> o[r]) & 1u) { // move_cells_empty, engine.cpp:256-269
                    out_dir = (int8_t)o[r];
                    out_score = s[r];
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (out_dir != kStill) break;
                if (s[r] <= 0.0) break; // sorted: no later direction qualifies (engine.cpp:319)
                const bool ok = for_new_cells(c.x, c.y, rw, rh, o[r], [&](int x, int y) {
                    const long long idx = cell_index(g, x, y);
                    return idx >= 0 && occ[idx] == kNoPed; // move_cells_empty, engine.cpp:256-269
                });
                if (ok) {
                    out_dir = (int8_t)o[r];
                    out_score = s[r];
                }
            }
        }
    }
    p.dir[i] = out_dir;
    p.score[i] = out_score;
}

__global__ void __launch_bounds__(kPedThreads)
k2_decide_kernel(GridDev g, PedArrays p, const int* __restrict__ occ, const float* __restrict__ stat,
                 const float* __restrict__ dyn, uint8_t* __restrict__ ev, Ctl* ctl, DecideParams dp, SlabDev slab) {
    chain_release(p.n <= kChainReleasePeds);
    chain_wait();
    k2_decide_body((long long)blockIdx.x * blockDim.x + threadIdx.x, g, p, occ, stat, dyn, ev, ctl, dp, slab);
}

__device__ __forceinline__ void k3_vote_body(long long t, const GridDev& g, const PedArrays& p, const int* occ, Ctl* ctl, int fault,
                                             const SlabDev& slab) {
    if (t == 0) { // k-4 rebuilds the active-tile list of k-5 every tick
        ctl->active_count = 0;
        ctl->epoch = (unsigned)(ctl->tick % kEpochPeriod) + 1u;
    }
    if (t >= p.n) return;
    if (ctl->error_code != 0) return;
    const long long i = ped_of_thread(p, ctl, t);
    const int d = p.dir[i];
    if (d < 0) return;
    const int2 c = p.center[i];
    if (!row_within(g, c.y, slab.reach)) return; // owned, or a neighbour's pedestrian that can touch my rows
    const uint32_t attr = p.attr[i];
    const double my = p.score[i];
    // engine.cpp:365-386 restated per claimant: I win su c iff no other registrant of c beats
    // (score, then lower id — higher id under the fault hook).
    if ((attr_half_w(attr) | attr_half_h(attr)) == 0) {
        // 1 x 1 pedestrian: one claimed su.  Its eight neighbours' occupants, then their decisions, then
        // the rivals' scores are each read as one batch: three memory round trips instead of up to 24.
        const int x = c.x + step_dx(d), y = c.y + step_dy(d);
        int q[8];
#pragma unroll
        for (int slot = 0; slot < 8; ++slot) {
            const long long idx = cell_index(g, x - step_dx(slot), y - step_dy(slot));
            q[slot] = idx >= 0 ? occ[idx] : kNoPed;
        }
        int qd[8];
#pragma unroll
        for (int slot = 0; slot < 8; ++slot) qd[slot] = (q[slot] >= 0 && q[slot] != (int)i) ? (int)p.dir[q[slot]] : -2;
        // the reference's scan of the su's slots in slot order (first registrant seeds the best, then strictly
        // greater score, then the id tie-break): kept as a scan so that NaN scores order exactly as there
        double theirs[8];
#pragma unroll
        for (int slot = 0; slot < 8; ++slot) theirs[slot] = qd[slot] == slot ? p.score[q[slot]] : 0.0;
        int best_id = kNoPed;
        double best = 0.0;
#pragma unroll
        for (int slot = 0; slot < 8; ++slot) {
            const bool me = slot == d;
            if (!me && qd[slot] != slot) continue; // not a registrant of my su
            const int id = me ? (int)i : q[slot];
            const double score = me ? my : theirs[slot];
            bool better = best_id == kNoPed || score > best;
            if (!better && score == best) better = fault ? id > best_id : id < best_id;
            if (better) {
                best_id = id;
                best = score;
            }
        }
        p.won[i] = best_id == (int)i ? 1 : 0;
        return;
    }
    const bool won = for_new_cells(c.x, c.y, attr_half_w(attr), attr_half_h(attr), d, [&](int x, int y) {
        int best_id = kNoPed;
        double best = 0.0;
#pragma unroll
        for (int slot = 0; slot < 8; ++slot) { // (slot order, as the reference scans them)
            int id;
            double score;
            if (slot == d) {
                id = (int)i;
                score = my;
            } else {
                const long long idx = cell_index(g, x - step_dx(slot), y - step_dy(slot));
                if (idx < 0) continue;
                id = occ[idx];
                if (id < 0 || id == (int)i) continue;
                if (p.dir[id] != slot) continue;
                score = p.score[id];
            }
            bool better = best_id == kNoPed || score > best;
            if (!better && score == best) better = fault ? id > best_id : id < best_id;
            if (better) {
                best_id = id;
                best = score;
            }
        }
        return best_id == (int)i;
    });
    p.won[i] = won ? 1 : 0;
}

// Splits the unwrapped interval [lo, hi] of one axis into at most two intervals of wrapped
// coordinates relative to `origin`, clipped to [0, owned): n = extent of the axis (W or H).
// Returns the number of intervals written to out[][2].
__device__ __forceinline__ int wrapped_intervals(int lo, int hi, int n, bool closed, int origin, int owned, int out[2][2]) {
    int cnt = 0;
    auto push = [&](int a, int b) { // relative coordinates, clip to the owned range
        a = max(a, 0);
        b = min(b, owned - 1);
        if (a <= b) {
            out[cnt][0] = a;
            out[cnt][1] = b;
            ++cnt;
        }
    };
    if (closed) {
        push(max(lo, 0) - origin, min(hi, n - 1) - origin);
    } else if (hi - lo + 1 >= n) {
        push(0, owned - 1);
    } else {
        const int a = emod(lo - origin, n), b = a + (hi - lo);
        push(a, min(b, n - 1));
        if (b >= n) push(0, b - n);
    }
    return cnt;
}

// Lists every k-5 tile within field reach of a mover's old or new centre (TileMarks).
constexpr int kFirstsMax = 4; // tiles one mover can be the first to stamp before it appends them itself (7 x 7 fields: at most 2 x 2)

// `firsts` / `n_firsts`: tiles this mover stamped first this tick; the caller appends them to the list with one
// atomic per WARP (every first of a tick bumps the same counter).
__device__ __forceinline__ void mark_tiles(const GridDev& g, const TileMarks& m, Ctl* ctl, unsigned epoch, int fx, int fy, int ux,
                                           int uy, bool slab_active, int (&firsts)[kFirstsMax], int& n_firsts) {
    int xr[2][2], yr[2][2];
    const int nxr = wrapped_intervals(min(fx, fx + ux) - m.hw, max(fx, fx + ux) + m.hw, g.W, g.closed != 0, 0, g.W, xr);
    const int nyr = wrapped_intervals(min(fy, fy + uy) - m.hh, max(fy, fy + uy) + m.hh, g.H, g.closed != 0, g.row0, g.rows, yr);
    for (int iy = 0; iy < nyr; ++iy)
        for (int ty = yr[iy][0] / kMarkTileH; ty <= yr[iy][1] / kMarkTileH; ++ty) {
            if (slab_active && (ty < m.edge_lo || ty >= m.edge_hi)) continue; // edge tiles are always processed
            // rows of 8 x 4 blocks of this tile the reach rectangle touches (a tile is 2 block rows x 4 block columns)
            const int by0 = (max(yr[iy][0], ty * kMarkTileH) - ty * kMarkTileH) >> 2;
            const int by1 = (min(yr[iy][1], ty * kMarkTileH + kMarkTileH - 1) - ty * kMarkTileH) >> 2;
            const unsigned rows = (by0 == 0 ? 0x0Fu : 0u) | (by1 == 1 ? 0xF0u : 0u);
            for (int ix = 0; ix < nxr; ++ix)
                for (int tx = xr[ix][0] / kMarkTileW; tx <= xr[ix][1] / kMarkTileW; ++tx) {
                    const int bx0 = (max(xr[ix][0], tx * kMarkTileW) - tx * kMarkTileW) >> 3;
                    const int bx1 = (min(xr[ix][1], tx * kMarkTileW + kMarkTileW - 1) - tx * kMarkTileW) >> 3;
                    const unsigned cols = ((2u << bx1) - (1u << bx0)) * 0x11u; // block columns bx0..bx1 in both block rows
                    const unsigned blocks = rows & cols;
                    const int t = ty * m.tiles_x + tx;
                    // stamp the tile, add its blocks within reach, count this mover; the first mover of the tick lists the tile
                    unsigned old = *reinterpret_cast<volatile unsigned*>(m.epoch + t);
                    for (;;) {
                        const bool current = (old >> 16) == epoch;
                        const unsigned n = current ? min((old & kMarkCountMax) + 1u, kMarkCountMax) : 1u;
                        const unsigned b = (current ? (old >> 8) & 0xFFu : 0u) | blocks;
                        const unsigned prev = atomicCAS(m.epoch + t, old, (epoch << 16) | (b << 8) | n);
                        if (prev == old) {
                            if (!current) {
                                if (n_firsts < kFirstsMax) firsts[n_firsts++] = t;
                                else m.list[atomicAdd(&ctl->active_count, 1)] = t; // (large fields: more tiles than the buffer holds)
                            }
                            break;
                        }
                        old = prev;
                    }
                }
        }
}

__global__ void __launch_bounds__(kPedThreads)
k3_vote_kernel(GridDev g, PedArrays p, const int* __restrict__ occ, Ctl* ctl, int fault, SlabDev slab) {
    chain_release(p.n <= kChainReleasePeds);
    chain_wait();
    k3_vote_body((long long)blockIdx.x * blockDim.x + threadIdx.x, g, p, occ, ctl, fault, slab);
}

// (every thread of the warp comes here, pedestrian or not: the tail is warp-collective)
__device__ __forceinline__ void k4_move_body(long long t, const GridDev& g, const PedArrays& p, int* occ, uint8_t* ev, Ctl* ctl,
                                             unsigned long long* moved_counts, const DebugArrays& dbg, const SlabDev& slab,
                                             const TileMarks& marks) {
    bool moved = false;
    int firsts[kFirstsMax], n_firsts = 0;
    if (t == 0) ctl->dense_count = 0; // k-5's dense-tile list starts empty every tick
    if (t < p.n && ctl->error_code == 0) {
        const long long i = ped_of_thread(p, ctl, t);
        const int d = p.dir[i];
        const int2 c = p.center[i];
        if (d >= 0 && p.won[i] && row_within(g, c.y, slab.reach)) {
            const uint32_t attr = p.attr[i];
            const int rw = attr_half_w(attr), rh = attr_half_h(attr);
            const int ux = step_dx(d), uy = step_dy(d);
            // release the su the new footprint no longer covers (engine.cpp:403-409): the mirror
            // image of the newly covered L, taken around the old centre
            if (ux != 0) {
                const int ox = ux > 0 ? -rw : rw;
                for (int oy = -rh; oy <= rh; ++oy) {
                    const long long idx = cell_index(g, c.x + ox, c.y + oy);
                    if (idx >= 0) occ[idx] = kNoPed;
                }
            }
            if (uy != 0) {
                const int oy = uy > 0 ? -rh : rh;
                for (int ox = -rw; ox <= rw; ++ox) {
                    const long long idx = cell_index(g, c.x + ox, c.y + oy);
                    if (idx >= 0) occ[idx] = kNoPed;
                }
            }
            for_new_cells(c.x, c.y, rw, rh, d, [&](int x, int y) { // engine.cpp:410
                const long long idx = cell_index(g, x, y);
                if (idx >= 0) occ[idx] = (int)i;
                return true;
            });
            int nx = c.x + ux, ny = c.y + uy;
            if (!g.closed) {
                nx = emod(nx, g.W);
                ny = emod(ny, g.H);
            }
            p.center[i] = make_int2(nx, ny);
            const long long from = cell_index(g, c.x, c.y), to = cell_index(g, nx, ny);
            const uint8_t code = event_code(attr);
            if (from >= 0) ev[2 * from] = code;
            if (to >= 0) ev[2 * to + 1] = code;
            p.moved_dir[i] = (int8_t)d;
            if (marks.epoch) mark_tiles(g, marks, ctl, ctl->epoch, c.x, c.y, ux, uy, slab.active != 0, firsts, n_firsts);
            if (slab.band) {
                p.won[i] = 0;
            } else if (slab.active) { // remember the event cells for next tick's clear
                const int at = atomicAdd(&ctl->ev_written_count, 2);
                if (at + 1 < slab.ev_capacity) {
                    slab.ev_written[at] = from >= 0 ? 2 * from : -1;
                    slab.ev_written[at + 1] = to >= 0 ? 2 * to + 1 : -1;
                } else { // (sized for two entries per resident pedestrian at upload: cannot happen)
                    raise_error(ctl, SFC_E_STATE, 4, nx, ny, (double)at);
                }
            }
            if (dbg.moved_from) { // MovementLog as the reference shapes it (engine.cpp:412-423)
                dbg.moved_from[from] = (int)i;
                dbg.moved_to[to] = (int)i;
                for (int k = 0; k < kKinds; ++k) {
                    const uint8_t mask = k < 2 ? (uint8_t)(1u << attr_orient(attr, k)) : (uint8_t)0xFF;
                    dbg.from_mask[(long long)k * dbg.cells + from] = mask;
                    dbg.to_mask[(long long)k * dbg.cells + to] = mask;
                }
            }
            moved = row_owned(g, c.y); // a neighbour's pedestrian is counted by its owner
        }
    }
    // tiles stamped first by this warp's movers go on the active-tile list with one counter bump per warp
    if (marks.epoch != nullptr && __any_sync(0xFFFFFFFFu, n_firsts != 0)) {
        const int lane = threadIdx.x & 31;
        int incl = n_firsts;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int up = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= d) incl += up;
        }
        const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        int base = 0;
        if (lane == 31) base = atomicAdd(&ctl->active_count, total);
        base = __shfl_sync(0xFFFFFFFFu, base, 31) + incl - n_firsts;
#pragma unroll
        for (int q = 0; q < kFirstsMax; ++q)
            if (q < n_firsts) marks.list[base + q] = firsts[q];
    }
    // TickMetrics::moved: one atomic per warp
    const unsigned ballot = __ballot_sync(0xFFFFFFFFu, moved);
    if ((threadIdx.x & 31) == 0 && ballot != 0) {
        atomicAdd(&moved_counts[ctl->tick - ctl->run_base], (unsigned long long)__popc(ballot));
    }
}

__global__ void __launch_bounds__(kPedThreads)
k4_move_kernel(GridDev g, PedArrays p, int* __restrict__ occ, uint8_t* __restrict__ ev, Ctl* ctl,
               unsigned long long* __restrict__ moved_counts, DebugArrays dbg, SlabDev slab, TileMarks marks) {
    chain_release(p.n <= kChainReleasePeds);
    chain_wait();
    k4_move_body((long long)blockIdx.x * blockDim.x + threadIdx.x, g, p, occ, ev, ctl, moved_counts, dbg, slab, marks);
}

// ---- reference-shaped temporaries for the Inspector path -----------------------------------

__global__ void dbg_clear_kernel(DebugArrays d) { // k-1, engine.cpp:335-339
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.cells) return;
    for (int s = 0; s < 8; ++s) {
        d.enroll_ids[i * 8 + s] = kNoPed;
        d.enroll_scores[i * 8 + s] = 0.0;
    }
    d.winners[i] = kNoPed;
    d.moved_from[i] = kNoPed;
    d.moved_to[i] = kNoPed;
    for (int k = 0; k < kKinds; ++k) {
        d.from_mask[(long long)k * d.cells + i] = 0;
        d.to_mask[(long long)k * d.cells + i] = 0;
    }
}

__global__ void dbg_enroll_kernel(GridDev g, PedArrays p, DebugArrays d, Ctl* ctl) { // engine.cpp:346-361
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const int dir = p.dir[i];
    if (dir < 0) return;
    const int2 c = p.center[i];
    const uint32_t attr = p.attr[i];
    const double score = p.score[i];
    for_new_cells(c.x, c.y, attr_half_w(attr), attr_half_h(attr), dir, [&](int x, int y) {
        const long long idx = cell_index(g, x, y);
        if (idx < 0) return true;
        const int prev = atomicCAS(&d.enroll_ids[idx * 8 + dir], kNoPed, (int)i);
        if (prev != kNoPed) {
            raise_error(ctl, SFC_E_INTEGRITY, 2, emod(x, g.W), emod(y, g.H), 0.0);
        } else {
            d.enroll_scores[idx * 8 + dir] = score;
        }
        return true;
    });
}

__global__ void dbg_vote_kernel(DebugArrays d, int fault) { // engine.cpp:365-386
    const long long su = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (su >= d.cells) return;
    int best_id = kNoPed;
    double best_score = 0.0;
    for (int slot = 0; slot < 8; ++slot) {
        const int id = d.enroll_ids[su * 8 + slot];
        if (id == kNoPed) continue;
        const double score = d.enroll_scores[su * 8 + slot];
        bool better = best_id == kNoPed || score > best_score;
        if (!better && score == best_score) better = fault ? id > best_id : id < best_id;
        if (better) {
            best_id = id;
            best_score = score;
        }
    }
    d.winners[su] = best_id;
}

// Non-zero image values below this magnitude could produce subnormal sums (see Ctl::tiny_image).
constexpr float kTinyImage = 2.0194839e-28f; // 2^-92

__global__ void interleave_kernel(const float* __restrict__ plane, float* __restrict__ dyn, int kind, long long cells, Ctl* ctl) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; // one float4 (half a su record slot)
    if (t >= cells * 2) return;
    const long long cell = t >> 1;
    const int half = (int)(t & 1);
    const float4 v = reinterpret_cast<const float4*>(plane)[t];
    reinterpret_cast<float4*>(dyn)[cell * 6 + kind * 2 + half] = v;
    const float lo = fminf(fminf(v.x != 0.f ? fabsf(v.x) : 1.f, v.y != 0.f ? fabsf(v.y) : 1.f),
                           fminf(v.z != 0.f ? fabsf(v.z) : 1.f, v.w != 0.f ? fabsf(v.w) : 1.f));
    if (lo < kTinyImage && ctl->tiny_image == 0) ctl->tiny_image = 1;
    const bool nz = __float_as_uint(v.x) == 0x80000000u || __float_as_uint(v.y) == 0x80000000u || __float_as_uint(v.z) == 0x80000000u ||
                    __float_as_uint(v.w) == 0x80000000u;
    if (nz && ctl->negative_zero == 0) ctl->negative_zero = 1;
}

// See Ctl::negative_zero.  x + (+0.0f) = x for every x but -0.0f, so the reference's unconditional add is this pass.
__global__ void normalize_negative_zero_kernel(float* __restrict__ dyn, long long n4, const Ctl* ctl,
                                               const unsigned long long* __restrict__ moved_counts, long long first, long long ticks) {
    if (ctl->negative_zero == 0 || ctl->error_code != 0) return;
    bool moved = false;
    for (long long t = 0; t < ticks && !moved; ++t) moved = moved_counts[first + t] != 0ull;
    if (!moved) return;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 v = reinterpret_cast<float4*>(dyn)[i];
        const bool nz = __float_as_uint(v.x) == 0x80000000u || __float_as_uint(v.y) == 0x80000000u || __float_as_uint(v.z) == 0x80000000u ||
                        __float_as_uint(v.w) == 0x80000000u;
        if (!nz) continue;
        v.x = __fadd_rn(v.x, 0.0f);
        v.y = __fadd_rn(v.y, 0.0f);
        v.z = __fadd_rn(v.z, 0.0f);
        v.w = __fadd_rn(v.w, 0.0f);
        reinterpret_cast<float4*>(dyn)[i] = v;
    }
}

__global__ void negative_zero_done_kernel(Ctl* ctl, const unsigned long long* __restrict__ moved_counts, long long first, long long ticks) {
    if (ctl->negative_zero == 0 || ctl->error_code != 0) return;
    for (long long t = 0; t < ticks; ++t)
        if (moved_counts[first + t] != 0ull) {
            ctl->negative_zero = 0;
            return;
        }
}

__global__ void deinterleave_kernel(const float* __restrict__ dyn, float* __restrict__ plane, int kind, long long cells) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cells * 2) return;
    const long long cell = t >> 1;
    const int half = (int)(t & 1);
    reinterpret_cast<float4*>(plane)[t] = reinterpret_cast<const float4*>(dyn)[cell * 6 + kind * 2 + half];
}

// OccupancyGrid of a freshly seeded population (scenario.cpp:424): every su of a footprint holds its
// pedestrian's id.  Footprints of a valid population are disjoint, so the writes do not collide.
__global__ void occupancy_from_peds_kernel(GridDev g, PedArrays p, int* __restrict__ occ) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const int2 c = p.center[i];
    const uint32_t attr = p.attr[i];
    const int rw = attr_half_w(attr), rh = attr_half_h(attr);
    for (int oy = -rh; oy <= rh; ++oy)
        for (int ox = -rw; ox <= rw; ++ox) {
            const long long idx = cell_index(g, c.x + ox, c.y + oy);
            if (idx >= 0) occ[idx] = (int)i;
        }
}

__global__ void fill_i8_kernel(int8_t* p, long long n, int v) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = (int8_t)v;
}

__global__ void tick_advance_kernel(Ctl* ctl) {
    if (ctl->error_code == 0) ctl->tick += 1;
}

inline unsigned blocks_for(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    return (unsigned)(b < 1 ? 1 : b);
}

// ---- ordering pass: PedArrays::order = ids by centre, row-major ------------------------------
// The occupancy grid already is the pedestrians sorted by position: a compaction of the su that hold a centre,
// taken in flat order, is the list.  Three launches (count per chunk, scan, write), run at upload and every
// kOrderPeriod ticks — pedestrians move one su per tick, so the order stays nearly sorted in between.
constexpr int kOrdThreads = 256;
constexpr int kOrdChunk = 4096; // su per block

__device__ __forceinline__ bool centre_at(const GridDev& g, const PedArrays& p, const int* __restrict__ occ, long long su,
                                          long long cells, int& id) {
    id = su < cells ? occ[su] : kNoPed;
    if (id < 0) return false;
    const int2 c = p.center[id];
    return cell_index(g, c.x, c.y) == su; // (a footprint's other su carry the id too)
}

__global__ void __launch_bounds__(kOrdThreads)
order_count_kernel(GridDev g, PedArrays p, const int* __restrict__ occ, long long cells, int* __restrict__ counts) {
    __shared__ int warp_n[kOrdThreads / 32];
    const long long base = (long long)blockIdx.x * kOrdChunk;
    int n = 0, id;
#pragma unroll 4
    for (int r = 0; r < kOrdChunk / kOrdThreads; ++r) n += centre_at(g, p, occ, base + r * kOrdThreads + threadIdx.x, cells, id) ? 1 : 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) n += __shfl_xor_sync(0xFFFFFFFFu, n, d);
    if ((threadIdx.x & 31) == 0) warp_n[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        int total = 0;
        for (int w = 0; w < kOrdThreads / 32; ++w) total += warp_n[w];
        counts[blockIdx.x] = total;
    }
}

// counts -> exclusive starts, in place (one CTA); the list is used only if it holds every pedestrian exactly once
__global__ void __launch_bounds__(1024) order_scan_kernel(int* __restrict__ counts, long long n_chunks, long long population, Ctl* ctl) {
    __shared__ long long part[1024];
    const long long per = (n_chunks + 1023) / 1024;
    const long long lo = min(n_chunks, threadIdx.x * per), hi = min(n_chunks, lo + per);
    long long sum = 0;
    for (long long i = lo; i < hi; ++i) sum += counts[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
        const long long v = (int)threadIdx.x >= d ? part[threadIdx.x - d] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    long long run = part[threadIdx.x] - sum;
    for (long long i = lo; i < hi; ++i) {
        const int c = counts[i];
        counts[i] = (int)min(run, (long long)INT_MAX);
        run += c;
    }
    if (threadIdx.x == 1023) ctl->order_ok = part[1023] == population ? 1 : 0;
}

__global__ void __launch_bounds__(kOrdThreads)
order_write_kernel(GridDev g, PedArrays p, const int* __restrict__ occ, long long cells, const int* __restrict__ starts,
                   const Ctl* ctl) {
    __shared__ int warp_n[2][kOrdThreads / 32];
    if (ctl->order_ok == 0) return;
    const long long base = (long long)blockIdx.x * kOrdChunk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int run = starts[blockIdx.x];
    for (int r = 0; r < kOrdChunk / kOrdThreads; ++r) {
        int id;
        const bool here = centre_at(g, p, occ, base + r * kOrdThreads + threadIdx.x, cells, id);
        const unsigned ballot = __ballot_sync(0xFFFFFFFFu, here);
        if (lane == 0) warp_n[r & 1][warp] = __popc(ballot);
        __syncthreads(); // (double-buffered counts: one barrier per round)
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kOrdThreads / 32; ++w) {
            const int c = warp_n[r & 1][w];
            before += w < warp ? c : 0;
            total += c;
        }
        if (here) p.order[run + before + __popc(ballot & ((1u << lane) - 1u))] = id;
        run += total;
    }
}

} // namespace

cudaError_t launch_k2_decide(cudaStream_t s, const GridDev& g, const PedArrays& p, const int* occ, const float* stat,
                             const float* dyn, uint8_t* ev, Ctl* ctl, const DecideParams& dp, const SlabDev& slab) {
    return launch_chained(k2_decide_kernel, dim3(blocks_for(p.n, kPedThreads)), dim3(kPedThreads), 0, s, g, p, occ, stat, dyn, ev, ctl, dp, slab);
}

cudaError_t launch_k3_vote(cudaStream_t s, const GridDev& g, const PedArrays& p, const int* occ, Ctl* ctl,
                           const DecideParams& dp, const SlabDev& slab) {
    return launch_chained(k3_vote_kernel, dim3(blocks_for(p.n, kPedThreads)), dim3(kPedThreads), 0, s, g, p, occ, ctl, dp.fault_invert, slab);
}

cudaError_t launch_k4_move(cudaStream_t s, const GridDev& g, const PedArrays& p, int* occ, uint8_t* ev, Ctl* ctl,
                           unsigned long long* moved_counts, const DebugArrays& dbg, const SlabDev& slab,
                           const TileMarks& marks) {
    return launch_chained(k4_move_kernel, dim3(blocks_for(p.n, kPedThreads)), dim3(kPedThreads), 0, s, g, p, occ, ev, ctl, moved_counts, dbg, slab, marks);
}

cudaError_t launch_dbg_clear(cudaStream_t s, const DebugArrays& d) {
    dbg_clear_kernel<<<blocks_for(d.cells, 256), 256, 0, s>>>(d);
    return cudaGetLastError();
}

cudaError_t launch_dbg_enroll(cudaStream_t s, const GridDev& g, const PedArrays& p, const DebugArrays& d, Ctl* ctl) {
    dbg_enroll_kernel<<<blocks_for(p.n, 256), 256, 0, s>>>(g, p, d, ctl);
    return cudaGetLastError();
}

cudaError_t launch_dbg_vote(cudaStream_t s, const DebugArrays& d, int fault_invert) {
    dbg_vote_kernel<<<blocks_for(d.cells, 256), 256, 0, s>>>(d, fault_invert);
    return cudaGetLastError();
}

cudaError_t launch_interleave(cudaStream_t s, const float* plane, float* dyn, int kind, long long cells_begin,
                              long long cells, Ctl* ctl) {
    interleave_kernel<<<blocks_for(cells * 2, 256), 256, 0, s>>>(plane, dyn + cells_begin * (kKinds * kSects), kind, cells, ctl);
    return cudaGetLastError();
}

cudaError_t launch_deinterleave(cudaStream_t s, const float* dyn, float* plane, int kind, long long cells_begin,
                                long long cells) {
    deinterleave_kernel<<<blocks_for(cells * 2, 256), 256, 0, s>>>(dyn + cells_begin * (kKinds * kSects), plane, kind, cells);
    return cudaGetLastError();
}

cudaError_t launch_occupancy_from_peds(cudaStream_t s, const GridDev& g, const PedArrays& p, int* occ) {
    occupancy_from_peds_kernel<<<blocks_for(p.n, 256), 256, 0, s>>>(g, p, occ);
    return cudaGetLastError();
}

cudaError_t launch_fill_i8(cudaStream_t s, int8_t* p, long long n, int v) {
    fill_i8_kernel<<<blocks_for(n, 256), 256, 0, s>>>(p, n, v);
    return cudaGetLastError();
}

cudaError_t launch_normalize_negative_zero(cudaStream_t s, float* dyn, long long cells, Ctl* ctl, const unsigned long long* moved_counts,
                                           long long first, long long ticks) {
    const long long n4 = cells * (kKinds * kSects / 4);
    const int blocks = (int)std::min<long long>((n4 + 255) / 256, 148 * 8);
    normalize_negative_zero_kernel<<<std::max(blocks, 1), 256, 0, s>>>(dyn, n4, ctl, moved_counts, first, ticks);
    negative_zero_done_kernel<<<1, 1, 0, s>>>(ctl, moved_counts, first, ticks);
    return cudaGetLastError();
}

cudaError_t launch_tick_advance(cudaStream_t s, Ctl* ctl) {
    tick_advance_kernel<<<1, 1, 0, s>>>(ctl);
    return cudaGetLastError();
}

namespace {
std::atomic<int> g_chain{-1}; // -1: not read yet
}

// (read again whenever an engine is created, so a process can switch between engines — tests do)
void chain_configure() {
    const char* knob = std::getenv("SFC_CHAIN");
    g_chain.store(knob == nullptr || std::atoi(knob) != 0 ? 1 : 0, std::memory_order_relaxed);
}

bool chain_enabled() {
    if (g_chain.load(std::memory_order_relaxed) < 0) chain_configure();
    return g_chain.load(std::memory_order_relaxed) != 0;
}

long long order_chunks(long long cells) { return (cells + kOrdChunk - 1) / kOrdChunk; }

cudaError_t launch_order_pedestrians(cudaStream_t s, const GridDev& g, const PedArrays& p, const int* occ, long long cells,
                                     int* chunk_counts, Ctl* ctl) {
    const long long n_chunks = order_chunks(cells);
    if (n_chunks == 0 || p.order == nullptr) return cudaSuccess;
    order_count_kernel<<<(unsigned)n_chunks, kOrdThreads, 0, s>>>(g, p, occ, cells, chunk_counts);
    order_scan_kernel<<<1, 1024, 0, s>>>(chunk_counts, n_chunks, p.n, ctl);
    order_write_kernel<<<(unsigned)n_chunks, kOrdThreads, 0, s>>>(g, p, occ, cells, chunk_counts, ctl);
    return cudaGetLastError();
}

} // namespace sfc
