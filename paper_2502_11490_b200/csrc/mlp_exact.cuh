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

// ---------------------------------------------------------------------------
// Compile-time-shaped variant for the BASELINE model family
// (create_model(d, d, Z, hidden=(64, 64)), metric.py:229-267; evalharness.py:77):
// d_h = D_H (multiple of 16, user half hoisted), H0 = H1 = 64, Z outputs.  All smem
// offsets are immediates, every output is valid, loops fully unrolled: the inner loop
// is 6 LDS.128 + 64 FMUL/FADD per chunk.
// ---------------------------------------------------------------------------
template <int D_H, int Z>
struct FixedMlp {
    static_assert(D_H % 16 == 0, "hoisting needs whole 16-element user blocks");
    static constexpr int H = 64;
    static constexpr int NCH0 = D_H / 4;     // item-half chunks of layer 0
    static constexpr int NCHH = H / 4;       // hidden-layer input chunks
    static constexpr int NCHZ = (Z + 3) / 4; // attention chunks
    static constexpr int LDX0 = NCH0 | 1;
    static constexpr int LDH = NCHH | 1;
    // float4 offsets inside the fixed block
    static constexpr int OFF_W0 = 0;
    static constexpr int OFF_W1 = OFF_W0 + NCH0 * H;
    static constexpr int OFF_W2 = OFF_W1 + NCHH * H;
    static constexpr int OFF_A = OFF_W2 + NCHH * Z;
    static constexpr int OFF_B0 = OFF_A + NCHZ;
    static constexpr int OFF_B1 = OFF_B0 + H / 4;
    static constexpr int OFF_B2 = OFF_B1 + H / 4;
    static constexpr int OFF_ACC0 = OFF_B2 + NCHZ;
    static constexpr int OFF_X0 = OFF_ACC0 + H;
    static constexpr int OFF_H0 = OFF_X0 + GR_PT * LDX0;
    static constexpr int OFF_H1 = OFF_H0 + GR_PT * LDH;
    static constexpr int OFF_Z = OFF_H1 + GR_PT * LDH;
    static constexpr int LDZ = NCHZ | 1;
    static constexpr int OFF_SCORE = OFF_Z + GR_PT * LDZ;
    static constexpr int TOTAL = OFF_SCORE + GR_PT / 4; // float4 units

    // layer with O = 64 outputs: warp w -> pairs 4w..4w+3, lane -> outputs lane, lane+32
    template <int NCH, int LDX, bool HAS_INIT>
    static __device__ __forceinline__ void big(const float4 *__restrict__ X,
                                               const float4 *__restrict__ W,
                                               const float *__restrict__ bias,
                                               const float4 *__restrict__ init,
                                               float *__restrict__ Y) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        float4 a[4][2];
        float4 i0 = make_float4(0.f, 0.f, 0.f, 0.f), i1 = i0;
        if (HAS_INIT) { i0 = init[lane]; i1 = init[lane + 32]; }
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) { a[pp][0] = i0; a[pp][1] = i1; }
        const float4 *xr = X + warp * 4 * LDX;
        const float4 *wr = W + lane;
#pragma unroll 8
        for (int j = 0; j < NCH; ++j) {
            const float4 w0 = wr[j * H], w1 = wr[j * H + 32];
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) {
                const float4 x = xr[pp * LDX + j];
                mac4(a[pp][0], x, w0);
                mac4(a[pp][1], x, w1);
            }
        }
        // epilogue: bias, ReLU, store in the next layer's processing order (K = 64)
        const float b0 = bias[lane], b1 = bias[lane + 32];
        const int j0 = chunk_perm(lane >> 2, H) * 4 + (lane & 3);
        const int j1 = chunk_perm((lane + 32) >> 2, H) * 4 + (lane & 3);
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
            const int p = warp * 4 + pp;
            Y[p * LDH * 4 + j0] = relu_np(__fadd_rn(hsum4(a[pp][0]), b0));
            Y[p * LDH * 4 + j1] = relu_np(__fadd_rn(hsum4(a[pp][1]), b1));
        }
    }

    // run the tile with weights/buffers at explicit addresses (smem or global weights)
    static __device__ __forceinline__ void tile_p(const float4 *W0, const float4 *W1,
                                                  const float4 *W2, const float4 *A,
                                                  const float *b0, const float *b1,
                                                  const float *b2, const float4 *acc0,
                                                  float4 *x0, float4 *h0, float4 *h1, float *zb,
                                                  float *score, int n_valid, int *nonfinite) {
        big<NCH0, LDX0, true>(x0, W0, b0, acc0, reinterpret_cast<float *>(h0));
        __syncthreads();
        big<NCHH, LDH, false>(h0, W1, b1, nullptr, reinterpret_cast<float *>(h1));
        __syncthreads();
        if (threadIdx.x < GR_PT * Z) {
            const int p = threadIdx.x % GR_PT, o = threadIdx.x / GR_PT;
            const float4 *hr = h1 + p * LDH;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NCHH; ++j) mac4(acc, hr[j], W2[j * Z + o]);
            zb[p * LDZ * 4 + o] = __fadd_rn(hsum4(acc), b2[o]);
        }
        __syncthreads();
        if (threadIdx.x < GR_PT) {
            const int p = threadIdx.x;
            const float *z = zb + p * LDZ * 4;
            bool bad = false;
#pragma unroll
            for (int o = 0; o < Z; ++o) bad |= !isfinite(z[o]);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NCHZ; ++j) {
                const int c = chunk_perm(j, Z);
                float e[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) e[u] = (4 * c + u < Z) ? z[4 * c + u] : 0.f;
                mac4(acc, make_float4(e[0], e[1], e[2], e[3]), A[j]);
            }
            score[p] = hsum4(acc);
            if (bad && p < n_valid) atomicOr(nonfinite, 1);
        }
    }

    // run the tile: x0 holds item halves in processing order (user half hoisted into acc0)
    static __device__ __forceinline__ void tile(float4 *base, int n_valid, int *nonfinite) {
        tile_p(base + OFF_W0, base + OFF_W1, base + OFF_W2, base + OFF_A,
               reinterpret_cast<const float *>(base + OFF_B0),
               reinterpret_cast<const float *>(base + OFF_B1),
               reinterpret_cast<const float *>(base + OFF_B2), base + OFF_ACC0, base + OFF_X0,
               base + OFF_H0, base + OFF_H1, reinterpret_cast<float *>(base + OFF_Z),
               reinterpret_cast<float *>(base + OFF_SCORE), n_valid, nonfinite);
    }
};
