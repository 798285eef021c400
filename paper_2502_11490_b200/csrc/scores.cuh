// Traversal-only score tables (SURVEY.md §8(b) "test scorers").
//
// The reference's own search tests drive c_hipanns with `euclidean_scorer`
// (search.py:73-81: -sqrt(einsum('ij,ij->i', v - q, v - q)) in fp64) or with ad-hoc
// ScoreFns.  Here such a scorer is a table of fp64 scores [Q][n_items] indexed by item
// id, built on the device (gr_scores_euclid) or uploaded (gr_scores_create).  The
// traversal kernel (search_kernel.cuh, MODE 2) orders items by a u32 per-query DENSE
// RANK of the fp64 score (equal scores -> equal code, -0.0 == +0.0), so the
// (score desc, id asc) order of the fp64 values is reproduced exactly inside the
// kernel's u64 keys (code << 32 | ~id rank); returned scores are the fp64 table values.
#pragma once
#include <cub/block/block_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "common.cuh"

// fp64 -> orderable u64 (ascending numeric order), -0.0 canonicalised to +0.0
__device__ __forceinline__ uint64_t f64_orderable(double d) {
    if (d == 0.0) d = 0.0;
    const uint64_t u = (uint64_t)__double_as_longlong(d);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// numpy 2.3 einsum('ij,ij->i') fp64 order (oracle sqnorm_rows_f64):
// two lanes; per 8-element block p: acc = a0^2 + (a1^2 + (a2^2 + (a3^2 + acc))) with lane l
// taking element p + 2t + l; zero-padded pairs for the remainder; result acc0 + acc1.
// Separately rounded multiply and add (no FMA contraction).
__global__ void euclid_table_kernel(const double *__restrict__ vec, int64_t n, int dim,
                                    const double *__restrict__ qry, int64_t Q,
                                    double *__restrict__ out, int *__restrict__ bad) {
    const int64_t total = n * Q;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = t / n, i = t % n;
        const double *v = vec + i * dim, *u = qry + q * dim;
        double acc0 = 0.0, acc1 = 0.0;
        const int nb = dim / 8;
        for (int b = 0; b < nb; ++b) {
            const int p = 8 * b;
            double d[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) d[j] = __dsub_rn(v[p + j], u[p + j]);
            // lane 0: elements p, p+2, p+4, p+6; lane 1: p+1, p+3, p+5, p+7
            double s0 = __dadd_rn(__dmul_rn(d[6], d[6]), acc0);
            double s1 = __dadd_rn(__dmul_rn(d[7], d[7]), acc1);
            s0 = __dadd_rn(__dmul_rn(d[4], d[4]), s0);
            s1 = __dadd_rn(__dmul_rn(d[5], d[5]), s1);
            s0 = __dadd_rn(__dmul_rn(d[2], d[2]), s0);
            s1 = __dadd_rn(__dmul_rn(d[3], d[3]), s1);
            acc0 = __dadd_rn(__dmul_rn(d[0], d[0]), s0);
            acc1 = __dadd_rn(__dmul_rn(d[1], d[1]), s1);
        }
        for (int p = 8 * nb; p < dim; p += 2) {
            const double d0 = __dsub_rn(v[p], u[p]);
            const double d1 = p + 1 < dim ? __dsub_rn(v[p + 1], u[p + 1]) : 0.0;
            acc0 = __dadd_rn(__dmul_rn(d0, d0), acc0);
            acc1 = __dadd_rn(__dmul_rn(d1, d1), acc1);
        }
        const double s = -__dsqrt_rn(__dadd_rn(acc0, acc1));
        if (isnan(s)) atomicOr(bad, 1);
        out[t] = s;
    }
}

__global__ void table_keys_kernel(const double *__restrict__ tab, int64_t total,
                                  uint64_t *__restrict__ keys, int32_t *__restrict__ idx,
                                  int64_t n, int *__restrict__ bad) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const double v = tab[t];
        if (isnan(v)) atomicOr(bad, 1);
        keys[t] = f64_orderable(v);
        idx[t] = (int32_t)(t % n);
    }
}

// one CTA per query row: sorted ascending keys -> dense rank + 1 scattered to code[row][idx]
template <int NT>
__global__ void __launch_bounds__(NT) dense_rank_kernel(const uint64_t *__restrict__ skeys,
                                                        const int32_t *__restrict__ sidx,
                                                        int64_t n, uint32_t *__restrict__ code) {
    using Scan = cub::BlockScan<uint32_t, NT>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t carry;
    const int64_t row = blockIdx.x;
    const uint64_t *k = skeys + row * n;
    const int32_t *ix = sidx + row * n;
    uint32_t *c = code + row * n;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += NT) {
        const int64_t i = base + threadIdx.x;
        const uint32_t flag = (i < n && i > 0 && k[i] != k[i - 1]) ? 1u : 0u;
        uint32_t incl, total;
        Scan(tmp).InclusiveSum(flag, incl, total);
        const uint32_t r = carry + incl;
        if (i < n) c[ix[i]] = r + 1u;
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
}

// Build codes[Q][n] (u32 dense ranks, higher = better score) from a device fp64 table.
// Returns cudaError; *bad (device int) gets 1 if any score is NaN.
inline cudaError_t build_score_codes(const double *tab, int64_t Q, int64_t n, uint32_t *codes,
                                     int *bad, cudaStream_t st) {
    const int64_t total = Q * n;
    uint64_t *keys = nullptr, *skeys = nullptr;
    int32_t *idx = nullptr, *sidx = nullptr;
    int64_t *offs = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t r) { if (e == cudaSuccess) e = r; return e == cudaSuccess; };
    if (chk(cudaMalloc(&keys, total * 8)) && chk(cudaMalloc(&skeys, total * 8)) &&
        chk(cudaMalloc(&idx, total * 4)) && chk(cudaMalloc(&sidx, total * 4)) &&
        chk(cudaMalloc(&offs, (Q + 1) * 8))) {
        const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
        table_keys_kernel<<<grid, 256, 0, st>>>(tab, total, keys, idx, n, bad);
        std::vector<int64_t> h(Q + 1);
        for (int64_t q = 0; q <= Q; ++q) h[q] = q * n;
        if (chk(cudaMemcpyAsync(offs, h.data(), (Q + 1) * 8, cudaMemcpyHostToDevice, st)) &&
            chk(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp_bytes, keys, skeys, idx, sidx,
                                                     total, Q, offs, offs + 1, st)) &&
            chk(cudaMalloc(&tmp, tmp_bytes)) &&
            chk(cub::DeviceSegmentedSort::SortPairs(tmp, tmp_bytes, keys, skeys, idx, sidx, total,
                                                     Q, offs, offs + 1, st))) {
            dense_rank_kernel<256><<<(unsigned)Q, 256, 0, st>>>(skeys, sidx, n, codes);
            chk(cudaGetLastError());
            chk(cudaStreamSynchronize(st));  // h and the temporaries are freed below
        }
    }
    cudaFree(keys); cudaFree(skeys); cudaFree(idx); cudaFree(sidx); cudaFree(offs); cudaFree(tmp);
    return e;
}
