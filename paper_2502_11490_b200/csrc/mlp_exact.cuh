// Exact-fp32 metric MLP over a tile of GR_PT (user, item) pairs, on CUDA cores.
//
// Reproduces relevance_batch (metric.py:102-154) bit-for-bit: every affine output
// is the numpy-einsum reduction (common.cuh) of its input row, + bias (fp32 add),
// ReLU = np.maximum(v, 0) between layers, final attention dot without bias.
// __fmul_rn/__fadd_rn are never contracted into FMA.
//
// Activations live in shared memory in processing order ([pair][chunk] float4,
// odd row stride so per-pair lane mappings are bank-conflict free); weights live
// in shared memory as [chunk][out] float4 so a warp's 32 lanes (32 outputs) read
// 512 contiguous bytes.  Big layers: warp w owns pairs 4w..4w+3 (activation
// reads are warp broadcasts), lane owns outputs lane and lane+32 -> 8 outputs,
// 32 fp32 lane accumulators per thread.  Narrow layers (O <= 16): one thread per
// (pair, output).
#pragma once
#include "common.cuh"

struct TileSmem {
    float4 *x0;       // [GR_PT][ldx0]
    int ldx0;
    float4 *h[2];     // [GR_PT][ldh]
    int ldh;
    float *score;     // [GR_PT]
};

// store y for (pair p, output o) of a layer whose output width is O into the
// next activation buffer (processing order of a K = O wide input)
__device__ __forceinline__ void store_act(float4 *X, int ld, int p, int o, int O, float y) {
    int j = chunk_perm(o >> 2, O);
    reinterpret_cast<float *>(X)[((int64_t)p * ld + j) * 4 + (o & 3)] = y;
}

// One affine layer: Y[p][o] = bias[o] + dot(X[p], W[o]) (+ReLU), for all GR_PT pairs.
// `init` (nullable) holds a per-output starting accumulator (hoisted h_u blocks).
// Writes outputs (and zero padding up to a multiple of 4) with store_act.
__device__ __forceinline__ void mlp_layer(const float4 *__restrict__ X, int ldx, int nch,
                                          const float4 *__restrict__ W, int O,
                                          const float *__restrict__ bias,
                                          const float4 *__restrict__ init, bool relu,
                                          float4 *Y, int ldy) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int Opad = (O + 3) & ~3;
    if (O > 16) {
        for (int og = 0; og < Opad; og += 64) {
            const int o0 = og + lane, o1 = og + lane + 32;
            const bool v0 = o0 < O, v1 = o1 < O;
            float4 a[4][2];
            float4 i0 = make_float4(0.f, 0.f, 0.f, 0.f), i1 = i0;
            if (init) {
                if (v0) i0 = init[o0];
                if (v1) i1 = init[o1];
            }
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) { a[pp][0] = i0; a[pp][1] = i1; }
            const float4 *xr = X + (warp * 4) * ldx;
#pragma unroll 2
            for (int j = 0; j < nch; ++j) {
                const float4 w0 = v0 ? W[j * O + o0] : make_float4(0.f, 0.f, 0.f, 0.f);
                const float4 w1 = v1 ? W[j * O + o1] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int pp = 0; pp < 4; ++pp) {
                    const float4 x = xr[pp * ldx + j];
                    mac4(a[pp][0], x, w0);
                    mac4(a[pp][1], x, w1);
                }
            }
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) {
                const int p = warp * 4 + pp;
                if (o0 < Opad) {
                    float y = 0.f;
                    if (v0) { y = __fadd_rn(hsum4(a[pp][0]), bias[o0]); if (relu) y = relu_np(y); }
                    store_act(Y, ldy, p, o0, O, y);
                }
                if (o1 < Opad) {
                    float y = 0.f;
                    if (v1) { y = __fadd_rn(hsum4(a[pp][1]), bias[o1]); if (relu) y = relu_np(y); }
                    store_act(Y, ldy, p, o1, O, y);
                }
            }
        }
    } else {
        // narrow layer: thread per (pair, output); lanes = pairs, so W reads broadcast
        for (int t = tid; t < GR_PT * Opad; t += GR_NT) {
            const int p = t % GR_PT, o = t / GR_PT;
            float y = 0.f;
            if (o < O) {
                float4 a = init ? init[o] : make_float4(0.f, 0.f, 0.f, 0.f);
                const float4 *xr = X + p * ldx;
                for (int j = 0; j < nch; ++j) mac4(a, xr[j], W[j * O + o]);
                y = __fadd_rn(hsum4(a), bias[o]);
                if (relu) y = relu_np(y);
            }
            store_act(Y, ldy, p, o, O, y);
        }
    }
}

// Run layers 0..n_mlp-1 and the attention dot on the tile whose layer-0 input is in
// S.x0 (chunks [pre_ch, nch0) of the pair vector when `init` holds the hoisted user
// accumulators, else all chunks).  W0 points at the layer-0 weights matching x0.
// Writes S.score[p]; returns (via flag) whether any final-layer value was non-finite.
__device__ __forceinline__ void mlp_tile(const DevModel &M, const TileSmem &S,
                                         const float4 *const *Wm, const float *const *bm,
                                         const float4 *sA, const float4 *W0, int x0_nch,
                                         const float4 *init, int n_valid, int *nonfinite) {
    const float4 *X = S.x0;
    int ldx = S.ldx0, nch = x0_nch;
    int cur = 0;
    for (int m = 0; m < M.n_mlp; ++m) {
        const bool last = (m == M.n_mlp - 1);
        float4 *Y = S.h[cur];
        mlp_layer(X, ldx, nch, m == 0 ? W0 : Wm[m], M.dims[m + 1], bm[m], m == 0 ? init : nullptr,
                  (!last) && M.relu, Y, S.ldh);
        __syncthreads();
        X = Y;
        ldx = S.ldh;
        nch = M.nch[m + 1];
        cur ^= 1;
    }
    // final-layer finiteness check (metric.py:134-135) + attention (metric.py:150-154)
    const int Z = M.Z;
    for (int p = threadIdx.x; p < GR_PT; p += GR_NT) {
        const float4 *zr = X + p * ldx;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        bool bad = false;
        for (int j = 0; j < nch; ++j) {
            const float4 z = zr[j];
            mac4(a, z, sA[j]);
            bad |= !(isfinite(z.x) && isfinite(z.y) && isfinite(z.z) && isfinite(z.w));
        }
        S.score[p] = hsum4(a);
        if (bad && p < n_valid) atomicOr(nonfinite, 1);
    }
    (void)Z;
}
