// Persistent hop-synchronous C-HiPANNS kernel (exact-fp32 scoring fused in).
//
// One CTA runs one query at a time and pulls the next query index from a global
// counter (persistent grid = SMs x resident CTAs).  Semantics = the reference
// c_hipanns in deterministic mode (search.py:194-286) via its hop-synchronous
// restatement (SURVEY.md §8(a'), pinned by oracle/):
//
//   init   claim {entry} + N_top(entry), score them            (search.py:235-236)
//   layer  seeds = top-kp of everything scored (the pool)      (search.py:239)
//   hop    expand every searcher's frontier rows; a node goes to the lowest
//          searcher index listing it (lock-step claim order, search.py:261-265);
//          score all fresh claims in one dense batch; each searcher keeps the
//          top-ef of its own claims (search.py:258-259); dead searchers stay dead.
//
// Claims use a per-CTA-slot u64 tag array over all slots (epoch-stamped, never
// cleared): tag = epoch<<32 | (0xFFFFFFFE - searcher) while a hop is claiming
// (atomicMax keeps the LOWEST searcher index), epoch<<32 | 0xFFFFFFFF once owned.
// A tag below epoch<<32 means "unclaimed in this query".  One atomic per
// neighbour read; owners are resolved after a CTA barrier.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "mlp_exact.cuh"
#include "select.cuh"
#include "tc_scorer.cuh"

struct SearchArgs {
    DevGraph g;
    DevModel M;
    DevItems it;
    const float *users; // [Q][d_h]
    int64_t Q;
    int k, kp, hops, ef;
    int64_t *out_ids;
    double *out_scores;
    int32_t *out_count;
    int64_t *out_stats;
    // per-slot scratch
    uint32_t *tags;    // [slots][n] epoch-stamped claim tags
    uint32_t *epochs;  // [slots]
    int32_t *f_slot;   // [slots][2][capF]
    int32_t *f_srch;   // [slots][2][capF]
    int32_t *surv_v;   // [slots][capS]
    int32_t *surv_i;   // [slots][capS]
    int32_t *fr_v;     // [slots][capS]
    int32_t *fr_i;     // [slots][capS]
    uint64_t *fr_key;  // [slots][capS]
    int32_t *seg_v;    // [slots][capS]
    uint64_t *seg_key; // [slots][capS]
    uint64_t *pool_key; // [slots][2][capP]
    int32_t *pool_slot; // [slots][2][capP]
    int32_t *pool_meta; // [slots][2][capP]: eval hop << 1 | exact (tensor-core mode)
    unsigned long long *counters; // [0] exact re-scores, [1] tensor-core scores,
                                  // [2] band violations, [3] max |approx - exact| / band (f32 bits)
    float band_rel, band_abs;     // refinement band: |s - T| <= band_rel*|T| + band_abs
    unsigned long long *phase_cycles; // nullable: per-phase SM cycles (instrumentation)
    int64_t capF, capS, capP;
    int *queue;
    int *nonfinite;
    int *band_viol;  // violations since the last status read (tensor-core mode certificate)
    // shared-memory layout (byte offsets into dynamic smem)
    int off_w0, off_w[GR_MAX_MLP], off_b[GR_MAX_MLP], off_A, off_acc0, off_x0, off_h0, off_h1,
        off_score, off_hist, off_sortk, off_sortv, off_kp;
    int ldx0, ldh, sortcap;
    // MODE 2 (traversal-only score table, scores.cuh): codes / fp64 scores [Q][tab_n] by item id
    const uint32_t *tab_code;
    const double *tab_f64;
    int64_t tab_n;
    // tensor-core pipeline A-operand loader: TMA tile::gather4 over the bf16 hi/lo item table
    // (GMPGR_TMA), else per-thread cp.async
    int tma;
    CUtensorMap hl_map;
    // duo kernel (search_duo.cuh): two units per CTA, bitset visited state
    int unit0, unit_stride, off_misc, off_tmemp;  // shared-memory plan (bytes)
    int32_t *cont_v, *cont_i;  // [units][capS] contested touches
    uint64_t *hash;            // [units][hash_cap] (query, node) -> survivor index
    int64_t hash_cap;
    uint32_t *vis;             // [units * G][vis_words]: 1 visited bit per node
    int64_t vis_words;
    int32_t *vlog;             // [units * G][log_cap]: claimed nodes of the running query
    int log_cap;
    // streamed host calls (gr_search): users arrive in chunks while the kernel runs; a unit
    // waits until *avail >= the end of its batch, and counts finished queries per chunk of
    // chunk_q queries into qdone[] (the copy-out stream waits on those counters)
    const int *avail;
    int *qdone;
    int chunk_q;
    float negz;  // -0.0f: the run-time addend of the packed exact products (common.cuh mac4x2)
    int off_exw0;       // duo MODE 1: shared-memory copy of the exact layer-0 (item half) weights
    float4 *acc0g;      // duo MODE 1: [units][G][64] hoisted user halves (global; MODE 0 keeps them in smem)
};

// Tensor-core mode certificate (run time).  The refinement argument (see below) needs
// |approx - exact| < band/2 for every item.  Every exact re-score sees both values: it
// records the largest ratio |approx - exact| / band(exact) and counts ratios above 1/2 in
// the CTA's shared accumulators (bc[0] = count, bc[1] = max ratio as f32 bits); the host
// re-runs the batch in exact mode when any violation was seen (gr_search).
__device__ __forceinline__ void band_record(unsigned *bc, uint64_t approx_key, float exact,
                                            float band_rel, float band_abs) {
    const float ap = orderable_f32((uint32_t)(approx_key >> 32));
    const float r = fabsf(ap - exact) / (band_rel * fabsf(exact) + band_abs);
    if (!(r == r)) return;  // non-finite scores are reported by the nonfinite flag
    if (r > 0.5f) atomicAdd(bc, 1u);
    atomicMax(bc + 1, __float_as_uint(r));
}
__device__ __forceinline__ void band_flush(const unsigned *bc, unsigned long long *counters,
                                           int *band_viol) {
    if (bc[0]) {
        atomicAdd(counters + 2, (unsigned long long)bc[0]);
        atomicAdd(band_viol, (int)bc[0]);
    }
    if (bc[1]) atomicMax(counters + 3, (unsigned long long)bc[1]);
}

struct CtaState {
    int q;
    uint32_t epoch;
    int wrap;
    int nF, nS, nFresh, nPool, nPool2, nFn;
    int pool_cur, f_cur;
    uint64_t poolT, hopmax, best;
    int besthop;
    int64_t per_layer[GR_MAX_LAYERS];
    int64_t rows, nbrs;
    uint32_t bcast[4];
};

// u32 tag = epoch (20 bits) << 12 | code: claim code 0xFFE - searcher (atomicMax keeps the
// lowest searcher), 0xFFF = owned.  A tag below epoch << 12 is "unclaimed in this query".
// Epochs wrap every 2^20 - 1 queries per slot: the slot's array is then cleared (tag_epoch).
#define GR_EPOCH_MAX ((1u << 20) - 1u)
__device__ __forceinline__ uint32_t claim_code(uint32_t epoch, int i) {
    return (epoch << 12) | (0xFFEu - (uint32_t)i);
}
__device__ __forceinline__ uint32_t done_code(uint32_t epoch) { return (epoch << 12) | 0xFFFu; }
// next epoch of a slot; on wrap the whole CTA clears that slot's tag array (rare)
__device__ __forceinline__ uint32_t next_epoch(uint32_t *epochs, int64_t slot, uint32_t *tags,
                                               int64_t n, int *wrap_flag) {
    uint32_t e = epochs[slot] + 1u;
    if (e > GR_EPOCH_MAX) { e = 1u; *wrap_flag = 1; }
    epochs[slot] = e;
    return e;
}

// warp-aggregated append of (v, i) when ok; returns nothing
__device__ __forceinline__ void warp_append2(bool ok, int32_t v, int32_t i, int *counter,
                                             int32_t *dv, int32_t *di) {
    const int lane = threadIdx.x & 31;
    const unsigned mask = __ballot_sync(0xffffffffu, ok);
    if (!mask) return;
    int base = 0;
    if (lane == 0) base = atomicAdd(counter, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (ok) {
        const int pos = base + __popc(mask & ((1u << lane) - 1u));
        dv[pos] = v;
        di[pos] = i;
    }
}

// DH > 0 selects the compile-time-shaped scorer FixedMlp<DH, ZZ> (host lays out smem to match)
// MODE 0: exact-fp32 scoring of every claim.  MODE 1 (DH > 0): tcgen05 split-bf16 scores,
// then exact re-scoring of every item inside the band around each selection threshold
// (frontier top-ef, pool top-k, seeds top-kp, final top-k), so all decisions and all
// returned scores are the exact ones provided |approx - exact| < band / 2.
template <int MINB, int DH, int ZZ, int MODE>
__global__ void __launch_bounds__(GR_NT, MINB) hipanns_search_kernel(const SearchArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ CtaState st;
    __shared__ unsigned long long ph_acc[8];
    __shared__ unsigned bc[2];  // tensor-core band certificate (band_record)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const DevModel &M = a.M;
    // phase timing (thread 0, after the barrier that closes each phase)
    long long ph_t0 = 0;
    if (tid < 8) ph_acc[tid] = 0;
    if (tid < 2) bc[tid] = 0u;
#define GR_PH(i)                                                          \
    do {                                                                  \
        if (a.phase_cycles && tid == 0) {                                 \
            const long long now_ = clock64();                             \
            ph_acc[i] += (unsigned long long)(now_ - ph_t0);              \
            ph_t0 = now_;                                                 \
        }                                                                 \
    } while (0)
    const DevGraph &g = a.g;

    // ---- carve shared memory, load weights once per CTA
    float4 *sW0 = reinterpret_cast<float4 *>(smem + a.off_w0);
    const float4 *sWm[GR_MAX_MLP];
    const float *sbm[GR_MAX_MLP];
    const int O0 = M.dims[1], K0 = M.dims[0], nch0 = M.nch[0], pre = M.pre_ch;
    if constexpr (MODE == 0) {
        const int n0 = (nch0 - pre) * O0;
        for (int t = tid; t < n0; t += GR_NT) sW0[t] = M.W[0][pre * O0 + t];
        for (int m = 0; m < M.n_mlp; ++m) {
            float *sb = reinterpret_cast<float *>(smem + a.off_b[m]);
            for (int t = tid; t < M.dims[m + 1]; t += GR_NT) sb[t] = M.b[m][t];
            sbm[m] = sb;
            if (m >= 1) {
                float4 *sw = reinterpret_cast<float4 *>(smem + a.off_w[m]);
                const int nw = M.nch[m] * M.dims[m + 1];
                for (int t = tid; t < nw; t += GR_NT) sw[t] = M.W[m][t];
                sWm[m] = sw;
            } else {
                sWm[0] = sW0;
            }
        }
        float4 *sA = reinterpret_cast<float4 *>(smem + a.off_A);
        for (int t = tid; t < M.nch[M.n_mlp]; t += GR_NT) sA[t] = M.A[t];
    }
    const float4 *sA = reinterpret_cast<const float4 *>(smem + a.off_A);
    float4 *sAcc0 = reinterpret_cast<float4 *>(smem + a.off_acc0);
    TileSmem S;
    S.x0 = reinterpret_cast<float4 *>(smem + a.off_x0);
    S.ldx0 = a.ldx0;
    S.h[0] = reinterpret_cast<float4 *>(smem + a.off_h0);
    S.h[1] = reinterpret_cast<float4 *>(smem + a.off_h1);
    S.ldh = a.ldh;
    S.score = reinterpret_cast<float *>(smem + a.off_score);
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem + a.off_hist); // [GR_NW][256]
    uint64_t *sortk = reinterpret_cast<uint64_t *>(smem + a.off_sortk);
    int32_t *sortv = reinterpret_cast<int32_t *>(smem + a.off_sortv);
    int32_t *seg_cnt = reinterpret_cast<int32_t *>(smem + a.off_kp);
    int32_t *seg_off = seg_cnt + a.kp;
    int32_t *fn_off = seg_off + a.kp;
    const int x0_nch = nch0 - pre;
    if constexpr (MODE == 0) {
        // zero activation buffers once (padding lanes stay zero)
        for (int t = tid; t < GR_PT * a.ldx0; t += GR_NT) S.x0[t] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int t = tid; t < GR_PT * a.ldh; t += GR_NT) {
            S.h[0][t] = make_float4(0.f, 0.f, 0.f, 0.f);
            S.h[1][t] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    // ---- tensor-core mode: operands, TMEM, mbarrier
    uint32_t tmem = 0, phase = 0;
    using TC = TcMlp<(DH > 0 ? DH : 64), (ZZ > 0 ? ZZ : 2)>;
    using FX = FixedMlp<(DH > 0 ? DH : 64), (ZZ > 0 ? ZZ : 2)>;
    if constexpr (MODE == 1) {
        const uint4 *src = reinterpret_cast<const uint4 *>(M.tcB);
        uint4 *dst = reinterpret_cast<uint4 *>(smem + TC::OFF_B0H);
        for (int t = tid; t < (TC::OFF_AH - TC::OFF_B0H) / 16; t += GR_NT) dst[t] = src[t];
        float *b1 = reinterpret_cast<float *>(smem + TC::OFF_B1);
        for (int t = tid; t < 64; t += GR_NT) b1[t] = M.tcMisc[t];
        float *w2 = reinterpret_cast<float *>(smem + TC::OFF_W2);
        for (int t = tid; t < 64 * ZZ; t += GR_NT) w2[t] = M.tcMisc[64 + t];
        if (tid < 4) {
            reinterpret_cast<float *>(smem + TC::OFF_B2)[tid] = M.tcMisc[64 + 64 * ZZ + tid];
            reinterpret_cast<float *>(smem + TC::OFF_ATT)[tid] = M.tcMisc[68 + 64 * ZZ + tid];
        }
        uint32_t *tptr = reinterpret_cast<uint32_t *>(smem + TC::OFF_TMEM);
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             tc::smem_u32(tptr)), "r"(128));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        if (tid == 0) tc::mbar_init(reinterpret_cast<uint64_t *>(smem + TC::OFF_BAR), 1);
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        tmem = *tptr;
    }

    // ---- per-slot scratch
    const int64_t slot = blockIdx.x;
    uint32_t *tags = a.tags + slot * g.n;
    int32_t *fslot[2] = {a.f_slot + slot * 2 * a.capF, a.f_slot + slot * 2 * a.capF + a.capF};
    int32_t *fsrch[2] = {a.f_srch + slot * 2 * a.capF, a.f_srch + slot * 2 * a.capF + a.capF};
    int32_t *surv_v = a.surv_v + slot * a.capS, *surv_i = a.surv_i + slot * a.capS;
    int32_t *fr_v = a.fr_v + slot * a.capS, *fr_i = a.fr_i + slot * a.capS;
    uint64_t *fr_key = a.fr_key + slot * a.capS;
    int32_t *seg_v = a.seg_v + slot * a.capS;
    uint64_t *seg_key = a.seg_key + slot * a.capS;
    uint64_t *pkey[2] = {a.pool_key + slot * 2 * a.capP, a.pool_key + slot * 2 * a.capP + a.capP};
    int32_t *pslot[2] = {a.pool_slot + slot * 2 * a.capP, a.pool_slot + slot * 2 * a.capP + a.capP};
    int32_t *pmeta[2] = {nullptr, nullptr};
    if constexpr (MODE == 1) {
        pmeta[0] = a.pool_meta + slot * 2 * a.capP;
        pmeta[1] = pmeta[0] + a.capP;
    }
    int32_t *rq = surv_v;           // re-score request list (survivor buffer is free then)
    int32_t *seg_ex = fr_i;         // exact flags of seg entries (fr_i is dead after the scatter)
    auto band_of = [&](float T) { return a.band_rel * fabsf(T) + a.band_abs; };
    const int d_h = M.d_h;
    const bool fast_fill = (d_h % 16) == 0;
    const int top = g.n_layers - 1;
    const int nst = 5 + g.n_layers;

    for (;;) {
        __syncthreads();
        if (tid == 0) {
            st.q = atomicAdd(a.queue, 1);
            st.wrap = 0;
            if (st.q < a.Q) st.epoch = next_epoch(a.epochs, slot, tags, g.n, &st.wrap);
            st.nPool = 0; st.pool_cur = 0; st.f_cur = 0; st.poolT = 0ull;
            st.hopmax = 0ull; st.best = 0ull; st.besthop = -1;
            for (int l = 0; l < GR_MAX_LAYERS; ++l) st.per_layer[l] = 0;
            st.rows = 0; st.nbrs = 0;
        }
        __syncthreads();
        const int64_t q = st.q;
        if (q >= a.Q) break;
        if (st.wrap) {  // epoch wrapped: clear this slot's tags
            for (int64_t i = tid; i < g.n; i += GR_NT) tags[i] = 0u;
            __threadfence_block();
            __syncthreads();
        }
        if (tid == 0) ph_t0 = clock64();
        const uint32_t epoch = st.epoch;
        const float *hu = a.users + q * d_h;

        // ---- hoisted user-half accumulators of layer 0
        for (int o = tid; o < (MODE == 2 ? 0 : O0); o += GR_NT) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j = 0; j < pre; ++j) {
                const int c = chunk_perm(j, K0);
                const float4 x = make_float4(hu[4 * c], hu[4 * c + 1], hu[4 * c + 2], hu[4 * c + 3]);
                mac4(acc, x, M.W[0][j * O0 + o]);
            }
            sAcc0[o] = acc;
            if constexpr (MODE == 1)
                reinterpret_cast<float *>(smem + TC::OFF_U)[o] =
                    __fadd_rn(hsum4(acc), M.b[0][o]);
        }

        // ---- score fr_v[0..nFresh) (hop h, layer L): keys, pool append, hop max
        auto score_fresh = [&](int nFresh, int hop) {
            const int pc = st.pool_cur;
            const uint64_t poolT = st.poolT;
            if constexpr (MODE == 2) {
                // score-table lookup: key = dense rank of the fp64 score << 32 | ~id rank
                const uint32_t *crow = a.tab_code + q * a.tab_n;
                for (int i0 = 0; i0 < nFresh; i0 += GR_NT) {
                    const int i = i0 + tid;
                    uint64_t key = 0ull;
                    int32_t s = 0;
                    if (i < nFresh) {
                        s = fr_v[i];
                        key = ((uint64_t)__ldg(crow + g.ids[s]) << 32) | (uint64_t)(~slot_rank(g, s));
                        fr_key[i] = key;
                        if (key > poolT) {
                            const int idx = atomicAdd(&st.nPool, 1);
                            pkey[pc][idx] = key;
                            pslot[pc][idx] = s;
                        }
                    }
                    uint64_t mx = key;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const uint64_t y = __shfl_xor_sync(0xffffffffu, mx, o);
                        mx = y > mx ? y : mx;
                    }
                    if (lane == 0 && mx) atomicMax(reinterpret_cast<unsigned long long *>(&st.hopmax), mx);
                }
                __syncthreads();
                return;
            }
            if constexpr (MODE == 1) {
                // approximate scores on the tensor cores, 128 pairs per tile
                const float Ts = orderable_f32((uint32_t)(poolT >> 32));
                const float lo_cut = poolT ? Ts - band_of(Ts) : -INFINITY;
                const float *sc = reinterpret_cast<const float *>(smem + TC::OFF_SC);
                for (int base = 0; base < nFresh; base += TC::TM) {
                    const int nv = min(TC::TM, nFresh - base);
                    TC::tile(smem, tmem, phase, a.it, g, fr_v + base, nv);
                    if (tid < nv) {
                        const int32_t s = fr_v[base + tid];
                        const float v = sc[tid];
                        if (!isfinite(v)) atomicOr(a.nonfinite, 1);
                        const uint64_t key = make_key(v, slot_rank(g, s));
                        fr_key[base + tid] = key;
                        if (v >= lo_cut) { // relaxed pool filter: the exact score may be above poolT
                            const int idx = atomicAdd(&st.nPool, 1);
                            pkey[pc][idx] = key;
                            pslot[pc][idx] = s;
                            pmeta[pc][idx] = hop << 1;
                        }
                    }
                }
                if (tid == 0) atomicAdd(a.counters + 1, (unsigned long long)nFresh);
                __syncthreads();
                return;
            }
            for (int base = 0; base < nFresh; base += GR_PT) {
                const int nv = min(GR_PT, nFresh - base);
                // gather item rows into x0 (processing order)
                for (int pp = 0; pp < 4; ++pp) {
                    const int p = warp * 4 + pp;
                    float4 *xr = S.x0 + p * a.ldx0;
                    if (p < nv) {
                        const int32_t s = fr_v[base + p];
                        const float *hv = a.it.emb + slot_row(g, s) * a.it.ld;
                        if (fast_fill) {
                            for (int cc = lane; cc < d_h / 4; cc += 32) {
                                const float4 v = __ldg(reinterpret_cast<const float4 *>(hv) + cc);
                                xr[chunk_perm(d_h / 4 + cc, K0) - pre] = v;
                            }
                        } else {
                            for (int jj = lane; jj < x0_nch; jj += 32) {
                                const int c = chunk_perm(pre + jj, K0);
                                float e[4];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const int idx = 4 * c + u;
                                    e[u] = idx < d_h ? hu[idx] : (idx < 2 * d_h ? hv[idx - d_h] : 0.f);
                                }
                                xr[jj] = make_float4(e[0], e[1], e[2], e[3]);
                            }
                        }
                    } else {
                        for (int jj = lane; jj < x0_nch; jj += 32) xr[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
                __syncthreads();
                if constexpr (DH > 0)
                    FixedMlp<DH, ZZ>::tile(reinterpret_cast<float4 *>(smem), nv, a.nonfinite);
                else
                    mlp_tile(M, S, sWm, sbm, sA, sW0, x0_nch, pre > 0 ? sAcc0 : nullptr, nv,
                             a.nonfinite);
                __syncthreads();
                if (tid < 32) {  // nv <= GR_PT = 32: warp 0 holds the tile
                    const int32_t s = tid < nv ? fr_v[base + tid] : 0;
                    const uint64_t key = tid < nv ? make_key(S.score[tid], slot_rank(g, s)) : 0ull;
                    uint64_t mx = key;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const uint64_t y = __shfl_xor_sync(0xffffffffu, mx, o);
                        mx = y > mx ? y : mx;
                    }
                    if (tid == 0 && mx > st.hopmax) st.hopmax = mx;
                    if (tid < nv) {
                    fr_key[base + tid] = key;
                    if (key > poolT) {
                        const int idx = atomicAdd(&st.nPool, 1);
                        pkey[pc][idx] = key;
                        pslot[pc][idx] = s;
                    }
                    }
                }
            }
            __syncthreads();
        };

        // ---- exact re-scoring of rq[0..nrq) (indices into the pool (target 0) or seg arrays)
        auto rescore = [&](int nrq, int target) {
            if constexpr (MODE == 1) {
                const int pc = st.pool_cur;
                float4 *x0 = reinterpret_cast<float4 *>(smem + TC::OFF_EX_X0);
                const float *esc = reinterpret_cast<const float *>(smem + TC::OFF_EX_SC);
                for (int base = 0; base < nrq; base += GR_PT) {
                    const int nv = min(GR_PT, nrq - base);
                    for (int pp = 0; pp < 4; ++pp) {
                        const int p = warp * 4 + pp;
                        float4 *xr = x0 + p * FX::LDX0;
                        if (p < nv) {
                            const int idx = rq[base + p];
                            const int32_t s = target == 0 ? pslot[pc][idx] : seg_v[idx];
                            const float4 *hv = reinterpret_cast<const float4 *>(a.it.emb + slot_row(g, s) * a.it.ld);
                            for (int cc = lane; cc < DH / 4; cc += 32)
                                xr[chunk_perm(DH / 4 + cc, 2 * DH) - DH / 4] = __ldg(hv + cc);
                        } else {
                            for (int cc = lane; cc < DH / 4; cc += 32) xr[cc] = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                    }
                    __syncthreads();
                    FX::tile_p(M.W[0] + (DH / 4) * 64, M.W[1], M.W[2], M.A, M.b[0], M.b[1], M.b[2],
                               sAcc0, x0, reinterpret_cast<float4 *>(smem + TC::OFF_EX_H0),
                               reinterpret_cast<float4 *>(smem + TC::OFF_EX_H1),
                               reinterpret_cast<float *>(smem + TC::OFF_EX_Z),
                               reinterpret_cast<float *>(smem + TC::OFF_EX_SC), nv, a.nonfinite);
                    __syncthreads();
                    if (tid < nv) {
                        const int idx = rq[base + tid];
                        band_record(bc, target == 0 ? pkey[pc][idx] : seg_key[idx], esc[tid],
                                    a.band_rel, a.band_abs);
                        if (target == 0) {
                            pkey[pc][idx] = make_key(esc[tid], slot_rank(g, pslot[pc][idx]));
                            pmeta[pc][idx] |= 1;
                        } else {
                            seg_key[idx] = make_key(esc[tid], slot_rank(g, seg_v[idx]));
                            seg_ex[idx] = 1;
                        }
                    }
                    __syncthreads();
                }
                if (tid == 0 && nrq) atomicAdd(a.counters, (unsigned long long)nrq);
            }
        };
        // collect pool entries that are not exact and satisfy pred(score) into rq
        auto collect_pool = [&](auto pred) {
            const int pc = st.pool_cur, np = st.nPool;
            if (tid == 0) st.nS = 0;
            __syncthreads();
            for (int i0 = 0; i0 < np; i0 += GR_NT) {
                const int i = i0 + tid;
                bool ok = false;
                if (i < np && !(pmeta[pc][i] & 1))
                    ok = pred(orderable_f32((uint32_t)(pkey[pc][i] >> 32)));
                warp_append2(ok, i, 0, &st.nS, rq, surv_i);
            }
            __syncthreads();
            return st.nS;
        };

        // ---- after scoring: best tracking, per-layer count, pool compaction to top-k
        auto after_score = [&](int layer, int h, int nFresh) {
            if (tid == 0) {
                st.per_layer[layer] += nFresh;
                if (st.hopmax > st.best) { st.best = st.hopmax; st.besthop = h; }
                st.hopmax = 0ull;
            }
            __syncthreads();
            if (st.nPool > a.k) {
                const int pc = st.pool_cur;
                if constexpr (MODE == 1) {
                    const uint64_t Ta = cta_select_threshold(pkey[pc], st.nPool, a.k, hist, st.bcast);
                    const float Ts = orderable_f32((uint32_t)(Ta >> 32)), bd = band_of(Ts);
                    const int nrq = collect_pool([&](float v) { return fabsf(v - Ts) <= bd; });
                    rescore(nrq, 0);
                }
                const uint64_t T = cta_select_threshold(pkey[pc], st.nPool, a.k, hist, st.bcast);
                if (tid == 0) st.nPool2 = 0;
                __syncthreads();
                const int np = st.nPool;
                for (int i = tid; i < np; i += GR_NT) {
                    const uint64_t key = pkey[pc][i];
                    if (key >= T) {
                        const int idx = atomicAdd(&st.nPool2, 1);
                        pkey[pc ^ 1][idx] = key;
                        pslot[pc ^ 1][idx] = pslot[pc][i];
                        if constexpr (MODE == 1) pmeta[pc ^ 1][idx] = pmeta[pc][i];
                    }
                }
                __syncthreads();
                if (tid == 0) { st.pool_cur = pc ^ 1; st.nPool = st.nPool2; st.poolT = T; }
                __syncthreads();
            }
        };

        // ---- owner resolution: survivors whose tag still carries their code own the node
        auto resolve = [&](int nS, int fresh_base) {
            const uint32_t done = done_code(epoch);
            for (int t0 = 0; t0 < nS; t0 += GR_NT) {
                const int t = t0 + tid;
                bool ok = false;
                int32_t v = 0, i = 0;
                if (t < nS) {
                    v = surv_v[t];
                    i = surv_i[t];
                    // L2 read: the tag was last written by atomics (performed at L2)
                    if (__ldcg(tags + v) == claim_code(epoch, i))
                        ok = true;
                }
                __syncwarp();
                warp_append2(ok, v, i, &st.nFresh, fr_v, fr_i);
                (void)fresh_base;
            }
            __syncthreads();
            // owners mark done (after everyone compared against the claim codes)
            const int nF = st.nFresh;
            for (int t = tid; t < nF; t += GR_NT) tags[fr_v[t]] = done;
            __syncthreads();
        };

        // ================= init: entry + its top-layer neighbourhood (hop 0)
        if (tid == 0) {
            tags[g.entry] = done_code(epoch);
            fr_v[0] = g.entry;
            fr_i[0] = 0;
            st.nFresh = 1;
            st.nS = 0;
        }
        __syncthreads();
        if (warp == 0) {
            const int32_t *row = graph_row(g, top, g.entry);
            if (lane == 0) st.rows += 1;
            if (row) {
                const uint32_t code = claim_code(epoch, 0);
                for (int c0 = 0; c0 < g.deg[top]; c0 += 32) {
                    const int32_t v = (c0 + lane < g.deg[top]) ? __ldg(row + c0 + lane) : -1;
                    const unsigned nv = __popc(__ballot_sync(0xffffffffu, v >= 0));
                    if (lane == 0) st.nbrs += nv;
                    bool ok = false;
                    if (v >= 0) {
                        const uint32_t old = atomicMax(tags + v, code);
                        ok = old < code;
                    }
                    warp_append2(ok, v, 0, &st.nS, surv_v, surv_i);
                }
            }
        }
        __syncthreads();
        resolve(st.nS, 1);
        {
            const int nFresh = st.nFresh;
            score_fresh(nFresh, 0);
            after_score(top, 0, nFresh);
        }
        GR_PH(0);

        int h = 0;
        for (int layer = top; layer >= 0; --layer) {
            // ---- seeds: sorted pool, first min(kp, |pool|)
            {
                if constexpr (MODE == 1) {
                    // seeds (and their order) must be exact: re-score the top-kp region + band
                    const int np0 = st.nPool, pc0 = st.pool_cur;
                    int nrq;
                    if (np0 > a.kp) {
                        const uint64_t Ta = cta_select_threshold(pkey[pc0], np0, a.kp, hist, st.bcast);
                        const float Ts = orderable_f32((uint32_t)(Ta >> 32)), bd = band_of(Ts);
                        nrq = collect_pool([&](float v) { return v >= Ts - bd; });
                    } else {
                        nrq = collect_pool([&](float) { return true; });
                    }
                    rescore(nrq, 0);
                }
                const int np = st.nPool, pc = st.pool_cur;
                for (int i = tid; i < np; i += GR_NT) { sortk[i] = pkey[pc][i]; sortv[i] = pslot[pc][i]; }
                __syncthreads();
                cta_sort_desc(sortk, sortv, np, a.sortcap);
                const int ns = min(a.kp, np);
                for (int i = tid; i < ns; i += GR_NT) { fslot[0][i] = sortv[i]; fsrch[0][i] = i; }
                if (tid == 0) { st.nF = ns; st.f_cur = 0; }
                __syncthreads();
            }
            GR_PH(1);
            const int deg = g.deg[layer];
            for (int t = 0; t < a.hops; ++t) {
                ++h;
                const int nF = st.nF;
                if (nF == 0) { h += a.hops - 1 - t; break; }
                const int fc = st.f_cur;
                if (tid == 0) { st.nS = 0; st.nFresh = 0; }
                __syncthreads();
                // ---- expand + claim: 8 frontier rows per warp; row loads, then all claim
                // atomics back-to-back, then the ballots that consume them
                constexpr int R = 8;
                for (int e0 = warp * R; e0 < nF; e0 += GR_NW * R) {
                    int32_t s[R], srch[R];
                    const int32_t *row[R];
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const int e = e0 + u;
                        s[u] = e < nF ? fslot[fc][e] : -1;
                        srch[u] = e < nF ? fsrch[fc][e] : 0;
                    }
#pragma unroll
                    for (int u = 0; u < R; ++u) row[u] = s[u] >= 0 ? graph_row(g, layer, s[u]) : nullptr;
                    int nvalid = 0;
                    for (int c0 = 0; c0 < deg; c0 += 32) {
                        int32_t v[R];
                        uint32_t old[R];
#pragma unroll
                        for (int u = 0; u < R; ++u)
                            v[u] = (row[u] && c0 + lane < deg) ? __ldg(row[u] + c0 + lane) : -1;
#pragma unroll
                        for (int u = 0; u < R; ++u)
                            old[u] = v[u] >= 0 ? atomicMax(tags + v[u], claim_code(epoch, srch[u])) : 0xFFFFFFFFu;
#pragma unroll
                        for (int u = 0; u < R; ++u) {
                            nvalid += __popc(__ballot_sync(0xffffffffu, v[u] >= 0));
                            warp_append2(v[u] >= 0 && old[u] < claim_code(epoch, srch[u]), v[u], srch[u],
                                         &st.nS, surv_v, surv_i);
                        }
                    }
                    if (lane == 0) {
                        atomicAdd(reinterpret_cast<unsigned long long *>(&st.nbrs), (unsigned long long)nvalid);
                        atomicAdd(reinterpret_cast<unsigned long long *>(&st.rows),
                                  (unsigned long long)min(R, nF - e0));
                    }
                }
                __syncthreads();
                GR_PH(2);
                resolve(st.nS, 0);
                GR_PH(3);
                const int nFresh = st.nFresh;
                score_fresh(nFresh, h);
                GR_PH(4);
                after_score(layer, h, nFresh);
                GR_PH(5);
                if (t == a.hops - 1) break; // frontier after a layer's last hop is unused
                // ---- per-searcher top-ef of fresh claims -> next frontier
                const int nsr = a.kp;
                for (int i = tid; i < nsr; i += GR_NT) seg_cnt[i] = 0;
                __syncthreads();
                for (int t2 = tid; t2 < nFresh; t2 += GR_NT) atomicAdd(&seg_cnt[fr_i[t2]], 1);
                __syncthreads();
                if (tid == 0) {
                    int acc = 0, accf = 0;
                    for (int i = 0; i < nsr; ++i) {
                        seg_off[i] = acc;
                        fn_off[i] = accf;
                        acc += seg_cnt[i];
                        accf += min(seg_cnt[i], a.ef);
                        seg_cnt[i] = 0; // reused as scatter cursor
                    }
                    st.nFn = accf;
                }
                __syncthreads();
                for (int t2 = tid; t2 < nFresh; t2 += GR_NT) {
                    const int i = fr_i[t2];
                    const int pos = seg_off[i] + atomicAdd(&seg_cnt[i], 1);
                    seg_v[pos] = fr_v[t2];
                    seg_key[pos] = fr_key[t2];
                }
                __syncthreads();
                if constexpr (MODE == 1) {
                    // exact re-score of the band around each searcher's ef-th approximate key
                    for (int t2 = tid; t2 < nFresh; t2 += GR_NT) seg_ex[t2] = 0;
                    if (tid == 0) st.nS = 0;
                    __syncthreads();
                    for (int i = warp; i < nsr; i += GR_NW) {
                        const int ni = seg_cnt[i], off = seg_off[i];
                        if (ni <= a.ef) continue;
                        const uint64_t Ta = warp_select_threshold(seg_key + off, ni, a.ef, hist + warp * 256);
                        const float Ts = orderable_f32((uint32_t)(Ta >> 32)), bd = band_of(Ts);
                        for (int j0 = 0; j0 < ni; j0 += 32) {
                            const int j = j0 + lane;
                            const bool in = j < ni &&
                                fabsf(orderable_f32((uint32_t)(seg_key[off + j] >> 32)) - Ts) <= bd;
                            warp_append2(in, off + j, 0, &st.nS, rq, surv_i);
                        }
                    }
                    __syncthreads();
                    rescore(st.nS, 1);
                }
                const int fn = fc ^ 1;
                for (int i = warp; i < nsr; i += GR_NW) {
                    const int ni = seg_cnt[i], off = seg_off[i], fo = fn_off[i];
                    if (ni <= a.ef) {
                        for (int j = lane; j < ni; j += 32) { fslot[fn][fo + j] = seg_v[off + j]; fsrch[fn][fo + j] = i; }
                    } else {
                        const uint64_t T = warp_select_threshold(seg_key + off, ni, a.ef, hist + warp * 256);
                        int cnt = 0;
                        for (int j0 = 0; j0 < ni; j0 += 32) {
                            const int j = j0 + lane;
                            const bool keep = j < ni && seg_key[off + j] >= T;
                            const unsigned mask = __ballot_sync(0xffffffffu, keep);
                            if (keep) {
                                const int pos = fo + cnt + __popc(mask & ((1u << lane) - 1u));
                                fslot[fn][pos] = seg_v[off + j];
                                fsrch[fn][pos] = i;
                            }
                            cnt += __popc(mask);
                        }
                    }
                }
                __syncthreads();
                if (tid == 0) { st.nF = st.nFn; st.f_cur = fn; }
                __syncthreads();
                GR_PH(6);
            }
        }

        // ---- result: pool sorted (score desc, id asc), first min(k, |pool|)
        {
            if constexpr (MODE == 1) rescore(collect_pool([&](float) { return true; }), 0);
            const int np = st.nPool, pc = st.pool_cur;
            for (int i = tid; i < np; i += GR_NT) { sortk[i] = pkey[pc][i]; sortv[i] = pslot[pc][i]; }
            __syncthreads();
            cta_sort_desc(sortk, sortv, np, a.sortcap);
            const int nr = min(a.k, np);
            for (int j = tid; j < a.k; j += GR_NT) {
                if (j < nr) {
                    a.out_ids[q * a.k + j] = g.ids[sortv[j]];
                    if constexpr (MODE == 2)
                        a.out_scores[q * a.k + j] = a.tab_f64[q * a.tab_n + g.ids[sortv[j]]];
                    else
                        a.out_scores[q * a.k + j] = (double)orderable_f32((uint32_t)(sortk[j] >> 32));
                } else {
                    a.out_ids[q * a.k + j] = -1;
                    a.out_scores[q * a.k + j] = __longlong_as_double(0x7ff8000000000000ll);
                }
            }
            if constexpr (MODE == 1) {
                // hop at which the best item was scored (pool meta)
                for (int i = tid; i < np; i += GR_NT)
                    if (nr > 0 && pslot[pc][i] == sortv[0]) st.besthop = pmeta[pc][i] >> 1;
                __syncthreads();
            }
            if (tid == 0) {
                a.out_count[q] = nr;
                int64_t ev = 0;
                for (int l = 0; l < g.n_layers; ++l) { ev += st.per_layer[l]; a.out_stats[q * nst + 5 + l] = st.per_layer[l]; }
                a.out_stats[q * nst + 0] = ev;
                a.out_stats[q * nst + 1] = ev;
                a.out_stats[q * nst + 2] = nr > 0 ? st.besthop : -1;
                a.out_stats[q * nst + 3] = st.rows;
                a.out_stats[q * nst + 4] = st.nbrs;
            }
        }
        GR_PH(7);
    }
    if (a.phase_cycles && tid < 8) atomicAdd(a.phase_cycles + tid, ph_acc[tid]);
#undef GR_PH
    if constexpr (MODE == 1) {
        tc::fence_before();
        __syncthreads();
        if (tid == 0) band_flush(bc, a.counters, a.band_viol);
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
    }
}
