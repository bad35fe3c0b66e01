// sfc_slab.cu — row-slab decomposition across GPUs: the sparse half of the per-tick halo exchange.
//
// The SU grid is split into contiguous row slabs, one per engine (one per GPU); a pedestrian is
// owned by the slab that holds its centre.  Every coupling of the tick is short range, so a slab
// only talks to its two ring neighbours.  Dense state — occupancy rows and event-map
// rows next to an edge — is exchanged as plain contiguous row ranges (no kernel needed).  The
// kernels here move the per-pedestrian part:
//   kind 0, after k-2: (id, direction, score) of my pedestrians near the edge, so the neighbour can
//                      evaluate the vote for its own claimants and, redundantly, for mine that
//                      step into its rows;
//   kind 1, after k-4: (id, x, y) of my pedestrians near the edge, so the neighbour's centre array
//                      stays exact for every pedestrian inside its halo.
// Per-pedestrian arrays are indexed by global id on every engine, so unpacking is a scatter.
// All tie-breaks of the model are on pedestrian id, never on ownership, so the decomposition does
// not change any result (tests/test_gpu_slabs.py compares N slabs with the undivided grid).

#include "sfc_internal.cuh"

namespace sfc {

namespace {

__global__ void halo_pack_kernel(GridDev g, PedArrays p, Ctl* ctl, int edge, int kind, int depth, HaloRecord* buf,
                                 int capacity) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const int2 c = p.center[i];
    if (!row_owned(g, c.y)) return;
    int ly = c.y - g.row0;
    if (!g.closed) ly = emod(ly, g.H);
    const bool near = edge == 0 ? ly < depth : ly >= g.rows - depth;
    if (!near) return;
    const int at = atomicAdd(&ctl->halo_counts[edge * 2 + kind], 1) + 1; // slot 0 is the header
    if (at >= capacity) {
        raise_error(ctl, SFC_E_STATE, 6, edge, kind, (double)at);
        return;
    }
    HaloRecord r;
    r.id = (int)i;
    if (kind == 0) {
        r.a = p.dir[i];
        r.b = p.score[i];
    } else {
        r.a = c.x;
        r.b = (double)c.y;
    }
    buf[at] = r;
}

__global__ void halo_header_kernel(Ctl* ctl, int edge, int kind, HaloRecord* buf, int capacity) {
    int n = ctl->halo_counts[edge * 2 + kind];
    if (n > capacity - 1) n = capacity - 1;
    buf[0].id = n;
    buf[0].a = kind;
    buf[0].b = 0.0;
    ctl->halo_counts[edge * 2 + kind] = 0;
}

__global__ void halo_unpack_kernel(PedArrays p, int kind, const HaloRecord* buf, int capacity) {
    const int n = min(buf[0].id, capacity - 1);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const HaloRecord r = buf[i + 1];
    if (r.id < 0 || r.id >= p.n) return;
    if (kind == 0) {
        p.dir[r.id] = (int8_t)r.a;
        p.score[r.id] = r.b;
    } else {
        p.center[r.id] = make_int2(r.a, (int)r.b);
    }
}

__global__ void clear_events_kernel(uint8_t* ev, Ctl* ctl, SlabDev slab) {
    const long long n = min((long long)ctl->ev_written_count, slab.ev_capacity);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long at = slab.ev_written[i];
        if (at >= 0) ev[at] = 0;
    }
}

__global__ void clear_events_done_kernel(Ctl* ctl) { ctl->ev_written_count = 0; }

} // namespace

cudaError_t launch_halo_pack(cudaStream_t s, const GridDev& g, const PedArrays& p, Ctl* ctl, int edge, int kind,
                             int depth, HaloRecord* buf, int capacity) {
    const unsigned blocks = (unsigned)((p.n + 255) / 256 > 0 ? (p.n + 255) / 256 : 1);
    halo_pack_kernel<<<blocks, 256, 0, s>>>(g, p, ctl, edge, kind, depth, buf, capacity);
    halo_header_kernel<<<1, 1, 0, s>>>(ctl, edge, kind, buf, capacity);
    return cudaGetLastError();
}

cudaError_t launch_halo_unpack(cudaStream_t s, const PedArrays& p, Ctl* /*ctl*/, int kind, const HaloRecord* buf,
                               int capacity) {
    halo_unpack_kernel<<<(unsigned)((capacity + 255) / 256), 256, 0, s>>>(p, kind, buf, capacity);
    return cudaGetLastError();
}

cudaError_t launch_clear_events(cudaStream_t s, uint8_t* ev, Ctl* ctl, const SlabDev& slab) {
    clear_events_kernel<<<64, 256, 0, s>>>(ev, ctl, slab);
    clear_events_done_kernel<<<1, 1, 0, s>>>(ctl);
    return cudaGetLastError();
}

} // namespace sfc
