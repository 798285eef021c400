// Exact top-m selection over unique u64 keys (score desc, id asc encoded, common.cuh).
//
// MSB-first radix select with 8-bit digits: each pass histograms the keys that
// share the already-fixed high digits, picks the digit d holding the m-th
// largest key and stops as soon as d's bucket is exactly the remainder.  The
// threshold T it returns satisfies |{key >= T}| == m, so "keep key >= T" is the
// top-m set (CandidatePool.top / frontier top-ef, pool.py:49-55, search.py:258-259).
#pragma once
#include "common.cuh"

// Find digit d in hist[256] (descending) with cnt(>d) < rem <= cnt(>=d); warp-wide.
// Returns d; *gt = cnt(>d), *eq = hist[d].
__device__ __forceinline__ int warp_pick_digit(const uint32_t *hist, uint32_t rem, uint32_t *gt,
                                               uint32_t *eq) {
    const int lane = threadIdx.x & 31;
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) { c[b] = hist[lane * 8 + b]; sum += c[b]; }
    uint32_t incl = sum; // inclusive suffix sum over lanes >= lane
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        uint32_t t = __shfl_down_sync(0xffffffffu, incl, off);
        if (lane + off < 32) incl += t;
    }
    uint32_t acc = incl - sum;
    int found = -1;
    uint32_t g = 0, e = 0;
#pragma unroll
    for (int b = 7; b >= 0; --b) {
        if (found < 0 && acc < rem && rem <= acc + c[b]) { found = lane * 8 + b; g = acc; e = c[b]; }
        acc += c[b];
    }
    const uint32_t who = __ballot_sync(0xffffffffu, found >= 0);
    const int src = __ffs(who) - 1;
    *gt = __shfl_sync(0xffffffffu, g, src);
    *eq = __shfl_sync(0xffffffffu, e, src);
    return __shfl_sync(0xffffffffu, found, src);
}

__device__ __forceinline__ uint64_t high_mask(int shift) {
    return shift >= 56 ? 0ull : (~0ull << (shift + 8));
}

// Warp-cooperative: threshold of the top m among keys[0..n) (n > m >= 1).
// hist: this warp's 256-entry shared histogram.
static __device__ uint64_t warp_select_threshold(const uint64_t *keys, int n, int m, uint32_t *hist) {
    const int lane = threadIdx.x & 31;
    uint64_t prefix = 0;
    uint32_t rem = (uint32_t)m;
    for (int shift = 56; shift >= 0; shift -= 8) {
        const uint64_t hm = high_mask(shift);
        for (int b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        for (int i = lane; i < n; i += 32) {
            const uint64_t k = keys[i];
            if (((k ^ prefix) & hm) == 0) atomicAdd(&hist[(k >> shift) & 255], 1u);
        }
        __syncwarp();
        uint32_t gt, eq;
        const int d = warp_pick_digit(hist, rem, &gt, &eq);
        __syncwarp();
        rem -= gt;
        prefix |= (uint64_t)d << shift;
        if (eq == rem) break;
    }
    return prefix;
}

// CTA-cooperative version (all GR_NT threads call it).  hist: 256 shared u32;
// bcast: 4 shared u32 scratch.
template <int NT = GR_NT>
static __device__ uint64_t cta_select_threshold(const uint64_t *keys, int n, int m, uint32_t *hist,
                                         uint32_t *bcast) {
    const int tid = threadIdx.x;
    uint64_t prefix = 0;
    uint32_t rem = (uint32_t)m;
    for (int shift = 56; shift >= 0; shift -= 8) {
        const uint64_t hm = high_mask(shift);
        for (int b = tid; b < 256; b += NT) hist[b] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += NT) {
            const uint64_t k = keys[i];
            if (((k ^ prefix) & hm) == 0) atomicAdd(&hist[(k >> shift) & 255], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            uint32_t gt, eq;
            const int d = warp_pick_digit(hist, rem, &gt, &eq);
            if (tid == 0) { bcast[0] = (uint32_t)d; bcast[1] = gt; bcast[2] = eq; }
        }
        __syncthreads();
        const uint32_t d = bcast[0], gt = bcast[1], eq = bcast[2];
        __syncthreads();
        rem -= gt;
        prefix |= (uint64_t)d << shift;
        if (eq == rem) break;
    }
    return prefix;
}

// CTA bitonic sort, descending by key, of n entries (keys, vals) in shared memory
// padded to cap (power of two >= n).  Padding keys are 0 (below every real key).
template <int NT = GR_NT>
static __device__ void cta_sort_desc(uint64_t *keys, int32_t *vals, int n, int cap) {
    for (int i = n + threadIdx.x; i < cap; i += NT) { keys[i] = 0ull; vals[i] = -1; }
    __syncthreads();
    for (int size = 2; size <= cap; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < cap; i += NT) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = (i & size) == 0;
                    const uint64_t a = keys[i], b = keys[j];
                    if (desc ? (a < b) : (a > b)) {
                        keys[i] = b; keys[j] = a;
                        const int32_t t = vals[i]; vals[i] = vals[j]; vals[j] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Bitonic sort (descending) by a group of GT threads synchronised with named barrier `bar`
// (bar >= 1; barrier 0 is __syncthreads).  gtid: thread index inside the group.
template <int GT>
static __device__ void group_sort_desc(uint64_t *keys, int32_t *vals, int n, int cap, int gtid, int bar) {
    auto sync = [&]() {
        if constexpr (GT == 32) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(GT) : "memory");
    };
    for (int i = n + gtid; i < cap; i += GT) { keys[i] = 0ull; vals[i] = -1; }
    sync();
    for (int size = 2; size <= cap; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = gtid; i < cap; i += GT) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = (i & size) == 0;
                    const uint64_t a = keys[i], b = keys[j];
                    if (desc ? (a < b) : (a > b)) {
                        keys[i] = b; keys[j] = a;
                        const int32_t t = vals[i]; vals[i] = vals[j]; vals[j] = t;
                    }
                }
            }
            sync();
        }
    }
}
