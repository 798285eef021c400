// Shared device-side definitions for the GMP-GR HiPANNS hot path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#define GR_MAX_MLP 6
#define GR_MAX_LAYERS 8
#define GR_NT 256          // threads per CTA
#define GR_NW (GR_NT / 32) // warps per CTA
#define GR_PT 32           // pairs per scoring tile (4 per warp)

// ---------------------------------------------------------------------------
// Exact-fp32 reduction order (numpy einsum, metric.py:30-32).
//
// A K-wide dot product is consumed in float4 "chunks".  numpy accumulates four
// SSE lanes; inside each 16-element block it adds chunk 3, then 2, 1, 0 to the
// lane accumulators (acc = a_t*b_t + acc, separately rounded); the tail chunks
// (zero-padded) follow in ascending order; the result is (l0+l1)+(l2+l3).
// So the whole reduction is "acc4 += x4[c]*w4[c]" over chunks c taken in the
// PROCESSING ORDER perm(j):  j < 4*floor(K/16): 4*(j/4) + 3 - j%4, else j.
// perm is an involution.  Weights and activations are stored in processing
// order so every kernel runs the same uniform loop.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int chunk_perm(int j, int K) {
    int nfull4 = (K / 16) * 4;
    return j < nfull4 ? ((j & ~3) + 3 - (j & 3)) : j;
}
__host__ __device__ __forceinline__ int n_chunks(int K) { return (K + 3) / 4; }

__device__ __forceinline__ void mac4(float4 &a, const float4 x, const float4 w) {
    a.x = __fadd_rn(__fmul_rn(x.x, w.x), a.x);
    a.y = __fadd_rn(__fmul_rn(x.y, w.y), a.y);
    a.z = __fadd_rn(__fmul_rn(x.z, w.z), a.z);
    a.w = __fadd_rn(__fmul_rn(x.w, w.w), a.w);
}
// mac4 in packed f32x2 instructions (FFMA2 + FADD2, half the issue slots): the product is
// fma(x, w, nz) with nz = -0.0 passed at run time -- exactly fl(x * w) for every x, w (the
// -0 addend changes neither a rounded product nor the sign of a zero one) -- and ptxas,
// which does not know nz, cannot contract it with the add as it does mul.rn.f32x2 +
// add.rn.f32x2.  Same per-lane arithmetic and order as mac4: a = fl(fl(x * w) + a).
__device__ __forceinline__ void mac4x2(float4 &a, const float4 x, const float4 w, float nz) {
    auto pk = [](float lo, float hi) {
        return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
    };
    const unsigned long long z2 = pk(nz, nz);
    unsigned long long p0, p1, s0, s1;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p0) : "l"(pk(x.x, x.y)), "l"(pk(w.x, w.y)), "l"(z2));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p1) : "l"(pk(x.z, x.w)), "l"(pk(w.z, w.w)), "l"(z2));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s0) : "l"(p0), "l"(pk(a.x, a.y)));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s1) : "l"(p1), "l"(pk(a.z, a.w)));
    a = make_float4(__uint_as_float((uint32_t)s0), __uint_as_float((uint32_t)(s0 >> 32)),
                    __uint_as_float((uint32_t)s1), __uint_as_float((uint32_t)(s1 >> 32)));
}
__device__ __forceinline__ float hsum4(const float4 a) {
    return __fadd_rn(__fadd_rn(a.x, a.y), __fadd_rn(a.z, a.w));
}
// np.maximum(v, 0) on this numpy returns +0.0 for v = -0.0 (SSE maxps operand order)
__device__ __forceinline__ float relu_np(float v) { return v > 0.0f ? v : 0.0f; }

// (score desc, id asc) total order as one u64: orderable(score) << 32 | ~rank.
// -0.0 is canonicalised to +0.0 (Python compares them equal, pool.py:32-39).
__host__ __device__ __forceinline__ uint32_t f32_orderable(float f) {
    if (f == 0.0f) f = 0.0f;
#ifdef __CUDA_ARCH__
    uint32_t u = __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
#endif
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float orderable_f32(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
#ifdef __CUDA_ARCH__
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}
__device__ __forceinline__ uint64_t make_key(float score, uint32_t rank) {
    return ((uint64_t)f32_orderable(score) << 32) | (uint64_t)(~rank);
}

// Device copy of the metric MLP in processing order.
struct DevModel {
    int n_mlp, relu, d_h, Z;
    int dims[GR_MAX_MLP + 1];
    int nch[GR_MAX_MLP + 1];     // input chunks of layer m (m == n_mlp: attention)
    const float4 *W[GR_MAX_MLP]; // [nch[m]][dims[m+1]] in processing order
    const float *b[GR_MAX_MLP];  // [dims[m+1]]
    const float4 *A;             // [nch[n_mlp]] attention in processing order
    int pre_ch;                  // layer-0 chunks that see only h_u (4 * floor(d_h/16))
    // tensor-core operands (tc_scorer.cuh), present when the model has the TcMlp shape
    const void *tcB;             // bf16 hi/lo core-matrix images: W0 item half, W1
    const float *tcMisc;         // b1[64] | W2[Z][64] | b2[4] | attention[4]
    int tc_ok;
    const void *exBlock;         // exact weight block in FixedMlp/ExactQ layout (fixed shapes)
};

// Device graph: layer 0 as fixed-width rows padded with -1 (no count reads);
// upper layers compacted to the nodes of level >= 1 via up_row.
struct DevGraph {
    int n_layers;
    int64_t n;
    int32_t entry;
    const int32_t *adj[GR_MAX_LAYERS]; // layer 0: [n][ld0]; l>=1: [n_up][ld_l]
    int ld[GR_MAX_LAYERS];             // row stride (>= degree cap, multiple of 4)
    int deg[GR_MAX_LAYERS];            // degree cap
    const int32_t *up_row;             // [n] row in upper-layer arrays, -1 if level 0
    const int64_t *ids;                // [n] item id per slot
    const int32_t *rows;               // [n] embedding row per slot (nullptr: slot)
    const uint32_t *rank;              // [n] tie-break rank (nullptr: slot)
};

__device__ __forceinline__ const int32_t *graph_row(const DevGraph &g, int layer, int32_t s) {
    if (layer == 0) return g.adj[0] + (int64_t)s * g.ld[0];
    int32_t r = __ldg(g.up_row + s);
    return r < 0 ? nullptr : g.adj[layer] + (int64_t)r * g.ld[layer];
}
__device__ __forceinline__ uint32_t slot_rank(const DevGraph &g, int32_t s) {
    return g.rank ? __ldg(g.rank + s) : (uint32_t)s;
}
__device__ __forceinline__ int64_t slot_row(const DevGraph &g, int32_t s) {
    return g.rows ? (int64_t)__ldg(g.rows + s) : (int64_t)s;
}

struct DevItems {
    const float *emb; // [n][ld] fp32, ld multiple of 4 (16-byte rows)
    int64_t n;
    int d, ld;
    const uint16_t *hl; // [n][2d] bf16 bits: hi = bf16(x), lo = bf16(x - hi) (d % 64 == 0), or null
    int hl_by_slot;     // hl rows indexed by graph slot (graph-owned copy) instead of item row
};
