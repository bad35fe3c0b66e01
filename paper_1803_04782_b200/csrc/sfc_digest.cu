// sfc_digest.cu — the acceptance digest and states_identical on the device.
//
// Digest: FNV-1a over occupancy bytes -> the three dynamic images -> the centres as int32 pairs,
// exactly the reference's state_digest (tests/acceptance/acceptance_main.cpp:39-58), without
// bringing the state to the host (config 4 holds 107 GB of it).
//
// FNV-1a is a serial recurrence, h <- (h ^ b) * p mod 2^64, and the XOR makes it non-linear — but
// only through the LOW BYTE of h: h ^ b = h + ((l ^ b) - l) with l = h mod 256, and the low byte
// of the next h depends on l and b alone.  So over any run of n bytes
//     h_out = p^n * (h_in - l_in) + R[l_in],      R[l] = FNV-1a over the run started from h = l,
// i.e. a run is summarised by 256 hashes.  Kernel 1 cuts the stream into runs and computes that
// table per run, one thread per starting low byte (the run's bytes staged through shared memory
// and broadcast); kernel 2, one thread, chains the runs.  256 x the serial work, all of it
// parallel: 100 MB of state (config 2) in a few milliseconds, bit-identical to the CPU loop.
//
// states_identical (engine.cpp:103-156): first difference between two device-resident states in
// the reference's order — centres, occupancy, static image, dynamic images — found with one
// min-reduction per array.

#include <algorithm>
#include <vector>

#include "sfc_internal.cuh"

namespace sfc {

namespace {

constexpr unsigned long long kFnvPrime = 1099511628211ull;
constexpr unsigned long long kFnvBasis = 14695981039346656037ull;
constexpr int kTileBytes = 4096; // bytes of a run staged per pass

struct DigestArgs {
    const int* occ;
    const float* dyn;
    const int2* center;
    long long seg_bytes[5];   // occupancy, image 0, 1, 2, centres
    long long seg_chunk0[6];  // first run of each segment (prefix sums)
    long long run_bytes;      // bytes per run (multiple of 32; the last run of a segment is shorter)
    unsigned long long* table; // [runs][256]
    long long runs;
};

// byte `o` (multiple of 4) of segment `seg` as a little-endian word
__device__ __forceinline__ uint32_t stream_word(const DigestArgs& a, int seg, long long o) {
    if (seg == 0) return (uint32_t)a.occ[o >> 2];
    if (seg == 4) return reinterpret_cast<const uint32_t*>(a.center)[o >> 2];
    // image plane seg - 1, host layout [cell][8] floats: the device keeps [cell][kind][8]
    const long long cell = o >> 5;
    return __float_as_uint(a.dyn[(cell * kKinds + (seg - 1)) * kSects + ((o >> 2) & 7)]);
}

__global__ void __launch_bounds__(256) digest_runs_kernel(DigestArgs a) {
    __shared__ uint32_t tile[kTileBytes / 4];
    const long long run = blockIdx.x;
    int seg = 0;
    while (seg < 4 && run >= a.seg_chunk0[seg + 1]) ++seg;
    const long long begin = (run - a.seg_chunk0[seg]) * a.run_bytes;
    const long long end = min(begin + a.run_bytes, a.seg_bytes[seg]);
    unsigned long long h = threadIdx.x; // this thread's starting low byte
    for (long long t0 = begin; t0 < end; t0 += kTileBytes) {
        const int n = (int)min((long long)kTileBytes, end - t0); // multiple of 4
        __syncthreads();
        for (int w = threadIdx.x; w < n / 4; w += blockDim.x) tile[w] = stream_word(a, seg, t0 + 4ll * w);
        __syncthreads();
        for (int w = 0; w < n / 4; ++w) {
            const uint32_t v = tile[w];
            h = (h ^ (v & 0xFFu)) * kFnvPrime;
            h = (h ^ ((v >> 8) & 0xFFu)) * kFnvPrime;
            h = (h ^ ((v >> 16) & 0xFFu)) * kFnvPrime;
            h = (h ^ (v >> 24)) * kFnvPrime;
        }
    }
    a.table[run * 256 + threadIdx.x] = h;
}

__device__ unsigned long long pow_prime(long long n) {
    unsigned long long r = 1ull, b = kFnvPrime;
    for (; n > 0; n >>= 1) {
        if (n & 1) r *= b;
        b *= b;
    }
    return r;
}

__global__ void digest_chain_kernel(DigestArgs a, unsigned long long* out) {
    unsigned long long h = kFnvBasis;
    const unsigned long long full = pow_prime(a.run_bytes);
    for (int seg = 0; seg < 5; ++seg) {
        const long long first = a.seg_chunk0[seg], last = a.seg_chunk0[seg + 1] - 1;
        for (long long run = first; run <= last; ++run) {
            const long long n = run < last ? a.run_bytes : a.seg_bytes[seg] - (last - first) * a.run_bytes;
            const unsigned long long l = h & 0xFFull;
            h = (run < last ? full : pow_prime(n)) * (h - l) + a.table[run * 256 + l];
        }
    }
    *out = h;
}

// ---- states_identical ------------------------------------------------------------------------

struct CompareArgs {
    const int2 *ca, *cb;
    const int *oa, *ob;
    const float *sa, *sb, *da, *db;
    long long peds, cells;
    unsigned long long* first; // [6]: centres, occupancy, static, dyn 0..2 — smallest differing index (~0: none)
};

__global__ void compare_kernel(CompareArgs a) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.peds) {
        const int2 x = a.ca[i], y = a.cb[i];
        if (x.x != y.x || x.y != y.y) atomicMin(&a.first[0], (unsigned long long)i);
    }
    if (i >= a.cells) return;
    if (a.oa[i] != a.ob[i]) atomicMin(&a.first[1], (unsigned long long)i);
    const uint32_t* sa = reinterpret_cast<const uint32_t*>(a.sa) + i * kSects;
    const uint32_t* sb = reinterpret_cast<const uint32_t*>(a.sb) + i * kSects;
    for (int s = 0; s < kSects; ++s)
        if (sa[s] != sb[s]) { // bit comparison, like the reference's memcmp
            atomicMin(&a.first[2], (unsigned long long)(i * kSects + s));
            break;
        }
    const uint32_t* da = reinterpret_cast<const uint32_t*>(a.da) + i * (kKinds * kSects);
    const uint32_t* db = reinterpret_cast<const uint32_t*>(a.db) + i * (kKinds * kSects);
    for (int k = 0; k < kKinds; ++k)
        for (int s = 0; s < kSects; ++s)
            if (da[k * kSects + s] != db[k * kSects + s]) {
                atomicMin(&a.first[3 + k], (unsigned long long)(i * kSects + s));
                break;
            }
}

} // namespace

// scratch: caller-provided device buffer of digest_scratch_bytes(cells, peds) bytes; out: device u64
long long digest_runs(long long cells, long long peds, long long* run_bytes) {
    const long long total = cells * 4 + cells * 96 + peds * 8;
    long long rb = 16 << 10;
    while ((total + rb - 1) / rb > 32768) rb *= 2; // at most ~32k runs (+ one short run per segment)
    *run_bytes = rb;
    const long long seg[5] = {cells * 4, cells * 32, cells * 32, cells * 32, peds * 8};
    long long runs = 0;
    for (long long s : seg) runs += (s + rb - 1) / rb;
    return runs;
}

size_t digest_scratch_bytes(long long cells, long long peds) {
    long long rb = 0;
    return (size_t)digest_runs(cells, peds, &rb) * 256 * sizeof(unsigned long long) + 64;
}

cudaError_t launch_digest(cudaStream_t s, const int* occ, const float* dyn, const int2* center, long long cells, long long peds,
                          void* scratch, unsigned long long* out) {
    DigestArgs a;
    a.occ = occ;
    a.dyn = dyn;
    a.center = center;
    a.runs = digest_runs(cells, peds, &a.run_bytes);
    const long long seg[5] = {cells * 4, cells * 32, cells * 32, cells * 32, peds * 8};
    a.seg_chunk0[0] = 0;
    for (int i = 0; i < 5; ++i) {
        a.seg_bytes[i] = seg[i];
        a.seg_chunk0[i + 1] = a.seg_chunk0[i] + (seg[i] + a.run_bytes - 1) / a.run_bytes;
    }
    a.table = static_cast<unsigned long long*>(scratch);
    if (a.runs > 0) digest_runs_kernel<<<(unsigned)a.runs, 256, 0, s>>>(a);
    digest_chain_kernel<<<1, 1, 0, s>>>(a, out);
    return cudaGetLastError();
}

cudaError_t launch_compare(cudaStream_t s, const PedArrays& pa, const PedArrays& pb, const int* oa, const int* ob, const float* sa,
                           const float* sb, const float* da, const float* db, long long cells, unsigned long long* first) {
    cudaError_t c = cudaMemsetAsync(first, 0xFF, 6 * sizeof(unsigned long long), s);
    if (c != cudaSuccess) return c;
    CompareArgs a;
    a.ca = pa.center;
    a.cb = pb.center;
    a.oa = oa;
    a.ob = ob;
    a.sa = sa;
    a.sb = sb;
    a.da = da;
    a.db = db;
    a.peds = std::min(pa.n, pb.n);
    a.cells = cells;
    a.first = first;
    const long long n = std::max(a.peds, a.cells);
    if (n > 0) compare_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

} // namespace sfc
