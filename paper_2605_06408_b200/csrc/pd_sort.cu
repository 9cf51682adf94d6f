// pd_sort.cu -- own device primitives for the two HBM-bound library steps of the path (SURVEY.md
// §8(a) a4, a13): an LSD radix sort of (u64 Morton key, u32 id) pairs and an exclusive scan of int32
// counts into int64 CSR offsets.
//
// Radix sort: 8-bit digits, one pass per digit, each pass = histogram -> digit-major scan -> stable
// scatter.  A block owns a tile of TILE keys; within a tile, keys are ranked stably in rounds of
// THREADS keys: __match_any_sync gives each key its peers (same digit) in its warp, per-warp digit
// counts in shared memory give the offset of earlier warps, and a running per-digit count carries
// the offset of earlier rounds.  Passes whose digit is constant over all keys are skipped.
#include <cuda_runtime.h>
#include <stdint.h>

#include "pd_bvh.cuh"

namespace pd {
namespace {

constexpr int RADIX = 256;
constexpr int SORT_THREADS = 256;
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int SORT_ITEMS = 16;
constexpr int TILE = SORT_THREADS * SORT_ITEMS;  // keys per block

inline unsigned nblocks(int64_t n, int per) { return (unsigned)((n + per - 1) / per); }

__device__ __forceinline__ unsigned lanemask_lt_s() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Per-tile digit histogram; hist is digit-major: hist[d * nb + b].  Also ORs/ANDs all keys so the
// host can skip passes whose digit never varies.
__global__ void __launch_bounds__(SORT_THREADS) k_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                       uint32_t* __restrict__ hist, int nb) {
    __shared__ uint32_t h[RADIX];
    for (int d = threadIdx.x; d < RADIX; d += SORT_THREADS) h[d] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * TILE;
#pragma unroll 4
    for (int i = 0; i < SORT_ITEMS; ++i) {
        int64_t k = base + (int64_t)i * SORT_THREADS + threadIdx.x;
        if (k < n) atomicAdd(&h[(keys[k] >> shift) & (RADIX - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RADIX; d += SORT_THREADS) hist[(size_t)d * nb + blockIdx.x] = h[d];
}

// Exclusive scan of row blockIdx.x of the digit-major histogram (length m), in place; row total to
// totals[blockIdx.x].
__global__ void __launch_bounds__(1024) k_scan_rows(uint32_t* __restrict__ hist, int64_t m, uint32_t* __restrict__ totals) {
    uint32_t* a = hist + (size_t)blockIdx.x * m;
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = 0; base < m; base += 1024) {
        int64_t i = base + threadIdx.x;
        uint32_t v = i < m ? a[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t s = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;  // inclusive
        }
        __syncthreads();
        uint32_t excl = carry + (wid ? warp_sums[wid - 1] : 0u) + x - v;
        if (i < m) a[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

// Exclusive scan of the RADIX digit totals (one block of RADIX threads).
__global__ void __launch_bounds__(RADIX) k_scan_totals(uint32_t* __restrict__ totals) {
    __shared__ uint32_t t[RADIX];
    t[threadIdx.x] = totals[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int d = 0; d < RADIX; ++d) {
            uint32_t v = t[d];
            t[d] = run;
            run += v;
        }
    }
    __syncthreads();
    totals[threadIdx.x] = t[threadIdx.x];
}

// Stable scatter of one tile.
__global__ void __launch_bounds__(SORT_THREADS) k_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                          uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                          int64_t n, int shift, const uint32_t* __restrict__ offs, int nb,
                                                          const uint32_t* __restrict__ dbase) {
    __shared__ uint32_t base_d[RADIX];          // global start of digit d for this tile
    __shared__ uint32_t run[RADIX];             // keys of digit d already placed by earlier rounds
    __shared__ uint16_t wcnt[SORT_WARPS][RADIX]; // per-warp digit counts of the current round
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < RADIX; d += SORT_THREADS) {
        base_d[d] = dbase[d] + offs[(size_t)d * nb + blockIdx.x];
        run[d] = 0;
        for (int w = 0; w < SORT_WARPS; ++w) wcnt[w][d] = 0;
    }
    __syncthreads();
    int64_t tile = (int64_t)blockIdx.x * TILE;
    for (int r = 0; r < SORT_ITEMS; ++r) {
        int64_t k = tile + (int64_t)r * SORT_THREADS + threadIdx.x;
        bool valid = k < n;
        uint64_t key = valid ? kin[k] : 0ull;
        uint32_t val = valid ? vin[k] : 0u;
        int d = valid ? (int)((key >> shift) & (RADIX - 1)) : RADIX + lane;  // idle lanes never match
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int intra = __popc(peers & lanemask_lt_s());
        if (valid && intra == 0) wcnt[wid][d] = (uint16_t)__popc(peers);
        __syncthreads();
        if (valid) {
            uint32_t off = run[d];
            for (int w = 0; w < wid; ++w) off += wcnt[w][d];
            uint32_t pos = base_d[d] + off + intra;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
        for (int dd = threadIdx.x; dd < RADIX; dd += SORT_THREADS) {
            uint32_t s = 0;
            for (int w = 0; w < SORT_WARPS; ++w) {
                s += wcnt[w][dd];
                wcnt[w][dd] = 0;
            }
            run[dd] += s;
        }
        __syncthreads();
    }
}

// OR and AND of all keys (to skip passes whose digit is constant).
__global__ void k_key_bits(const uint64_t* __restrict__ keys, int64_t n, unsigned long long* __restrict__ orand) {
    uint64_t o = 0, a = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        o |= k;
        a &= k;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, s);
        a &= __shfl_xor_sync(0xffffffffu, a, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&orand[0], (unsigned long long)o);
        atomicAnd(&orand[1], (unsigned long long)a);
    }
}

// ---- exclusive scan of int32 counts into int64 offsets[n+1] (3 phases)
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int64_t block_incl_scan(int64_t v, int64_t* warp_sums) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    int64_t r = x + (wid ? warp_sums[wid - 1] : 0);
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_tile_sums(const int32_t* __restrict__ cnt, int64_t n, int64_t* __restrict__ sums) {
    __shared__ int64_t ws[32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i)
        if (base + i < n) s += cnt[base + i];
    int64_t incl = block_incl_scan(s, ws);
    if (threadIdx.x == SCAN_THREADS - 1) sums[blockIdx.x] = incl;
}

__global__ void __launch_bounds__(1024) k_scan_sums(int64_t* __restrict__ sums, int64_t m) {
    __shared__ int64_t ws[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b = 0; b < m; b += blockDim.x) {
        int64_t i = b + threadIdx.x;
        int64_t v = i < m ? sums[i] : 0;
        int64_t incl = block_incl_scan(v, ws);
        int64_t c = carry;
        if (i < m) sums[i] = c + incl - v;  // exclusive
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = c + incl;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_tile_scan(const int32_t* __restrict__ cnt, int64_t n, const int64_t* __restrict__ sums,
                                                            int64_t* __restrict__ offsets) {
    __shared__ int64_t ws[32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int32_t v[SCAN_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = base + i < n ? cnt[base + i] : 0;
        s += v[i];
    }
    int64_t run = block_incl_scan(s, ws) - s + sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        run += v[i];
        if (base + i < n) offsets[base + i + 1] = run;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) offsets[0] = 0;
}

}  // namespace

// Temp layout: [hist u32 RADIX*nb][orand u64 x2 | totals u32 RADIX][ping-pong keys u64 n][vals u32 n]
cudaError_t sort_pairs(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                       int64_t n, void* temp, size_t* temp_bytes, cudaStream_t st, int* launches) {
    const int nb = (int)nblocks(n, TILE);
    size_t hist_bytes = ((size_t)RADIX * nb * sizeof(uint32_t) + 255) & ~(size_t)255;
    size_t need = hist_bytes + 2048 + (size_t)n * sizeof(uint64_t) + (size_t)n * sizeof(uint32_t) + 256;
    if (!temp) {
        *temp_bytes = need;
        return cudaSuccess;
    }
    if (*temp_bytes < need) return cudaErrorInvalidValue;
    char* t = (char*)temp;
    uint32_t* hist = (uint32_t*)t;
    unsigned long long* orand = (unsigned long long*)(t + hist_bytes);
    uint32_t* totals = (uint32_t*)(t + hist_bytes + 256);
    uint64_t* kbuf = (uint64_t*)(t + hist_bytes + 2048);
    uint32_t* vbuf = (uint32_t*)(kbuf + n);
    // which digits vary?
    unsigned long long init[2] = {0ull, ~0ull};
    cudaMemcpyAsync(orand, init, sizeof(init), cudaMemcpyHostToDevice, st);
    k_key_bits<<<592, 256, 0, st>>>(keys_in, n, orand);
    unsigned long long h[2];
    cudaMemcpyAsync(h, orand, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    const uint64_t vary = h[0] ^ h[1];
    int passes[8], np = 0;
    for (int p = 0; p < 8; ++p)
        if ((vary >> (8 * p)) & 0xffull) passes[np++] = p;
    if (launches) *launches += 1;
    if (np == 0) {  // all keys equal: the (stable) identity order
        cudaMemcpyAsync(keys_out, keys_in, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(vals_out, vals_in, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
        return cudaGetLastError();
    }
    // ping-pong so that the last pass lands in keys_out
    const uint64_t* ksrc = keys_in;
    const uint32_t* vsrc = vals_in;
    for (int q = 0; q < np; ++q) {
        bool last_to_out = ((np - 1 - q) % 2) == 0;
        uint64_t* kdst = last_to_out ? keys_out : kbuf;
        uint32_t* vdst = last_to_out ? vals_out : vbuf;
        int shift = 8 * passes[q];
        k_hist<<<nb, SORT_THREADS, 0, st>>>(ksrc, n, shift, hist, nb);
        k_scan_rows<<<RADIX, 1024, 0, st>>>(hist, nb, totals);
        k_scan_totals<<<1, RADIX, 0, st>>>(totals);
        k_scatter<<<nb, SORT_THREADS, 0, st>>>(ksrc, vsrc, kdst, vdst, n, shift, hist, nb, totals);
        if (launches) *launches += 4;
        ksrc = kdst;
        vsrc = vdst;
    }
    return cudaGetLastError();
}

cudaError_t scan_counts(const int32_t* cnt, int64_t* offsets, int64_t n, void* temp, size_t* temp_bytes,
                        cudaStream_t st, int* launches) {
    const int nb = (int)nblocks(n, SCAN_TILE);
    size_t need = (size_t)(nb + 1) * sizeof(int64_t);
    if (!temp) {
        *temp_bytes = need;
        return cudaSuccess;
    }
    if (n <= 0) {
        cudaMemsetAsync(offsets, 0, sizeof(int64_t), st);
        return cudaGetLastError();
    }
    int64_t* sums = (int64_t*)temp;
    k_tile_sums<<<nb, SCAN_THREADS, 0, st>>>(cnt, n, sums);
    k_scan_sums<<<1, 1024, 0, st>>>(sums, nb);
    k_tile_scan<<<nb, SCAN_THREADS, 0, st>>>(cnt, n, sums, offsets);
    if (launches) *launches += 3;
    return cudaGetLastError();
}

}  // namespace pd
