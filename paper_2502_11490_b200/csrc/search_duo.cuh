// Duo C-HiPANNS kernel: one 512-thread CTA per SM = TWO independent 256-thread units, each
// advancing its own G = 8 queries in lock-step (same layers, same hops; semantics of
// search_kernel.cuh / search_mq.cuh: hop-synchronous c_hipanns, search.py:194-286).  The
// units share only the read-only weight operands in shared memory and the TMEM allocation;
// they synchronise with their own named barrier (bar.sync 1 + unit, 256), so one unit's
// traversal phases (row gathers, claim atomics, selections) run while the other unit's
// tiles are on the TMA / tcgen05 / epilogue warps -- the overlap a single lock-step CTA
// cannot have (round-1 profile: expand 31% and score 40% of the launch, never concurrent).
//
// Visited state (claims) -- bounded by N/8 bytes per resident query, not 4N:
//   one bit per node per query slot: set by the node's first touch (every first touch is a
//   fresh claim, so "touched earlier this hop" and "claimed in an earlier hop" never need
//   to be told apart).
//   expand:  warp w of a unit owns query w and walks that query's frontier in list order
//            (searcher-ascending, search.py:261-265) in batches that never span two searchers;
//            a batch's claim atomics have all returned before the next batch issues its own.
//            old = atomicOr(word, bit): set -> claimed in an earlier hop, or touched earlier
//            this hop by the same or a LOWER searcher; clear -> first touch.  So the first
//            toucher is the lowest searcher listing the node -- the reference's lock-step
//            ownership (search.py:220-224) -- with no second resolution pass.
//   claim:   every first touch is fresh; the owning warp appends it to the survivors and to
//            its query's claim log; at query end the logged nodes' words are zeroed (or the
//            slot's whole bitset when the log overflowed).
// MODE 0: exact-fp32 scoring of every claim (32-pair tiles per unit, weights in shared memory).
// MODE 1: tcgen05 split-bf16 scoring of 128-pair tiles (tc_pipe2.cuh) + exact re-scoring of
//         the band around every selection threshold, with the run-time band certificate.
#pragma once
#include <cstdio>

#include "common.cuh"
#include "search_kernel.cuh"
#include "search_mq.cuh"
#include "select.cuh"
#include "tc_pipe2.cuh"
#include "tc_scorer.cuh"

// Exact fixed-shape MLP for one 256-thread unit (8 warps, 32-pair tiles): ExactQ's
// arithmetic (bit-exact einsum order) with unit-local thread indices and barrier.
template <int D_H, int Z>
struct ExactU {
    using EQ = ExactQ<D_H, Z, 8>;
    static constexpr int H = 64, NCH0 = EQ::NCH0, NCHH = EQ::NCHH, NCHZ = EQ::NCHZ;
    static constexpr int LDX0 = EQ::LDX0, LDH = EQ::LDH, LDZ = EQ::LDZ, PT = 32;
    static constexpr int OFF_X0 = EQ::OFF_X0, OFF_H0 = EQ::OFF_H0, OFF_H1 = EQ::OFF_H1,
                         OFF_Z = EQ::OFF_Z, OFF_SC = EQ::OFF_SC, OFF_PQ = EQ::OFF_PQ,
                         BUF_END = EQ::BUF_END, W_END = EQ::W_END;

    // PK: packed f32x2 products (mac4x2; measured faster for the tensor-core mode's sparse
    // re-scoring, slower for MODE 0's dense exact scoring, which keeps scalar mac4)
    template <int NCH, int LDX, bool HAS_INIT, bool PK>
    static __device__ __forceinline__ void big(int lt, const float4 *__restrict__ X, const float4 *__restrict__ W,
                                               const float *__restrict__ bias, const float4 *__restrict__ acc0,
                                               const int *__restrict__ pq, float *__restrict__ Y, float nz) {
        const int warp = lt >> 5, lane = lt & 31;
        float4 a[4][2];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
            if (HAS_INIT) {
                const int g = pq[warp * 4 + pp];
                a[pp][0] = acc0[g * H + lane];
                a[pp][1] = acc0[g * H + lane + 32];
            } else {
                a[pp][0] = make_float4(0.f, 0.f, 0.f, 0.f);
                a[pp][1] = a[pp][0];
            }
        }
        const float4 *xr = X + warp * 4 * LDX;
        const float4 *wr = W + lane;
#pragma unroll 8
        for (int j = 0; j < NCH; ++j) {
            const float4 w0 = wr[j * H], w1 = wr[j * H + 32];
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) {
                const float4 x = xr[pp * LDX + j];
                if constexpr (PK) {
                    mac4x2(a[pp][0], x, w0, nz);
                    mac4x2(a[pp][1], x, w1, nz);
                } else {
                    mac4(a[pp][0], x, w0);
                    mac4(a[pp][1], x, w1);
                }
            }
        }
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

    // W: weight block (ExactQ layout); buf: activation buffers; acc0: [G][64] float4
    template <bool PK, class Sync>
    static __device__ __forceinline__ void tile(int lt, const float4 *W, const float4 *W0, float4 *buf,
                                                const float4 *acc0, int n_valid, int *nonfinite, Sync sync,
                                                float nz) {
        const int *pq = reinterpret_cast<const int *>(buf + OFF_PQ);
        big<NCH0, LDX0, true, PK>(lt, buf + OFF_X0, W0, reinterpret_cast<const float *>(W + EQ::OFF_B0),
                              acc0, pq, reinterpret_cast<float *>(buf + OFF_H0), nz);
        sync();
        big<NCHH, LDH, false, PK>(lt, buf + OFF_H0, W + EQ::OFF_W1, reinterpret_cast<const float *>(W + EQ::OFF_B1),
                              nullptr, pq, reinterpret_cast<float *>(buf + OFF_H1), nz);
        sync();
        float *zb = reinterpret_cast<float *>(buf + OFF_Z);
        if (lt < PT * Z) {
            const int p = lt % PT, o = lt / PT;
            const float4 *hr = buf + OFF_H1 + p * LDH;
            const float4 *W2 = W + EQ::OFF_W2;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NCHH; ++j) mac4(acc, hr[j], W2[j * Z + o]);
            zb[p * LDZ * 4 + o] = __fadd_rn(hsum4(acc), reinterpret_cast<const float *>(W + EQ::OFF_B2)[o]);
        }
        sync();
        if (lt < PT) {
            const int p = lt;
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
                mac4(acc, make_float4(e[0], e[1], e[2], e[3]), W[EQ::OFF_A + j]);
            }
            reinterpret_cast<float *>(buf + OFF_SC)[p] = hsum4(acc);
            if (bad && p < n_valid) atomicOr(nonfinite, 1);
        }
        sync();
    }
};

// warp-aggregated append of v when ok
__device__ __forceinline__ void warp_append1(bool ok, int32_t v, int *counter, int32_t *dv) {
    const int lane = threadIdx.x & 31;
    const unsigned mask = __ballot_sync(0xffffffffu, ok);
    if (!mask) return;
    int base = 0;
    if (lane == 0) base = atomicAdd(counter, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (ok) dv[base + __popc(mask & ((1u << lane) - 1u))] = v;
}

// bounds checks for debugging builds (-DGR_DUO_DEBUG): report and trap
#ifdef GR_DUO_DEBUG
#define GR_DCHECK(cond, ...)                                  \
    do {                                                      \
        if (!(cond)) {                                        \
            printf("GR_DCHECK %s:%d: ", __FILE__, __LINE__);  \
            printf(__VA_ARGS__);                              \
            printf("\n");                                    \
            __trap();                                         \
        }                                                     \
    } while (0)
#else
#define GR_DCHECK(cond, ...) \
    do {                     \
    } while (0)
#endif

template <int DH, int ZZ, int MODE, int G>
__global__ void __launch_bounds__(512, 1) hipanns_duo_kernel(const __grid_constant__ SearchArgs a) {
    constexpr int NTH = 256, NW = 8, GT = NTH / G;
    static_assert(GT == 32 && NW == G, "one warp per query (pool sorts, expand)");
    using EX = ExactU<DH, ZZ>;
    using TP = TcPipe2<DH, ZZ>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // carve base aligned to 1024 bytes (SWIZZLE_128B stages); the host plan reserves the slack
    unsigned char *const smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ MqState<G> sts[2];
    __shared__ unsigned long long ph_acc[16];
    __shared__ unsigned bc[2];  // tensor-core band certificate (band_record)
    __shared__ int nlog_[2][G];
    const int tid = threadIdx.x, unit = tid >> 8, lt = tid & 255, warp = lt >> 5, lane = lt & 31;
    if (tid < 16) ph_acc[tid] = 0;
    if (tid < 2) bc[tid] = 0u;
    const DevModel &M = a.M;
    const DevGraph &g = a.g;
    auto usync = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + unit) : "memory"); };
    long long ph_t0 = 0;
#define GR_PH(i)                                                          \
    do {                                                                  \
        if (a.phase_cycles && tid == 0) {                                 \
            const long long now_ = clock64();                             \
            ph_acc[i] += (unsigned long long)(now_ - ph_t0);              \
            ph_t0 = now_;                                                 \
        }                                                                 \
    } while (0)
    // ---- shared weights: tcgen05 B operands (MODE 1) or the exact weight block (MODE 0)
    if constexpr (MODE == 1) {
        const uint4 *src = reinterpret_cast<const uint4 *>(M.tcB);
        uint4 *dst = reinterpret_cast<uint4 *>(smem + TP::OFF_B0H);
        for (int t = tid; t < TP::B_BYTES / 16; t += 512) dst[t] = src[t];
        // the exact re-scorer's layer-0 weights (item half, the bulk of its MACs) in shared
        // memory too: the rest of its block is read through L1 from M.exBlock
        const float4 *w0s = reinterpret_cast<const float4 *>(M.exBlock) + EX::EQ::OFF_W0;
        float4 *w0d = reinterpret_cast<float4 *>(smem + a.off_exw0);
        for (int t = tid; t < EX::NCH0 * 64; t += 512) w0d[t] = w0s[t];
    } else {
        const float4 *src = reinterpret_cast<const float4 *>(M.exBlock);
        float4 *dst = reinterpret_cast<float4 *>(smem);
        for (int t = tid; t < EX::W_END; t += 512) dst[t] = src[t];
    }
    unsigned char *const ub = smem + a.unit0 + unit * a.unit_stride;  // this unit's block
    const float4 *sW = MODE == 1 ? reinterpret_cast<const float4 *>(M.exBlock) : reinterpret_cast<const float4 *>(smem);
    float4 *sBuf = reinterpret_cast<float4 *>(ub + a.off_x0);
    // hoisted user halves: shared memory in MODE 0, global (per unit) in MODE 1
    float4 *sAcc0 = MODE == 1 ? a.acc0g + ((int64_t)blockIdx.x * 2 + unit) * G * 64
                              : reinterpret_cast<float4 *>(ub + a.off_acc0);
    const float4 *sW0 = MODE == 1 ? reinterpret_cast<const float4 *>(smem + a.off_exw0)
                                  : reinterpret_cast<const float4 *>(smem) + EX::EQ::OFF_W0;
    uint32_t *hist = reinterpret_cast<uint32_t *>(ub + a.off_hist);
    uint64_t *sortk = reinterpret_cast<uint64_t *>(ub + a.off_sortk);
    int32_t *sortv = reinterpret_cast<int32_t *>(ub + a.off_sortv);
    int32_t *seg_cnt = reinterpret_cast<int32_t *>(ub + a.off_kp);
    const int NSEG = G * a.kp;
    int32_t *seg_off = seg_cnt + NSEG;
    int32_t *fn_off = seg_off + NSEG;
    float *U = reinterpret_cast<float *>(ub + a.off_misc);            // [G][64] user half + b0
    float *sb1 = U + G * 64, *sW2 = sb1 + 64, *sb2 = sW2 + 64 * ZZ, *satt = sb2 + 4;
    uint32_t *tptr = reinterpret_cast<uint32_t *>(smem + a.off_tmemp);
    uint32_t tmem = 0, chunk_ctr = 0, tile_ctr = 0;
    if constexpr (MODE == 1) {
        for (int t = lt; t < 64; t += NTH) sb1[t] = M.tcMisc[t];
        for (int t = lt; t < 64 * ZZ; t += NTH) sW2[t] = M.tcMisc[64 + t];
        if (lt < 4) {
            sb2[lt] = M.tcMisc[64 + 64 * ZZ + lt];
            satt[lt] = M.tcMisc[68 + 64 * ZZ + lt];
        }
        if (warp == 0 && unit == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             tc::smem_u32(tptr)), "r"(2 * TP::COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        if (tc::smem_u32(ub) & 1023u) __trap();
        TP::init_barriers(ub, lt);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if constexpr (MODE == 1) {
        tmem = *tptr + unit * TP::COLS;
        // collapsed heads for the tensor-core epilogue: w_eff = sum_o att_o W2_o, c0 =
        // sum_o att_o b2_o, hlim = largest relu output for which no head can overflow
        float *weff = satt + 4;
        if (lt < 64) {
            float w = 0.f;
            for (int o = 0; o < ZZ; ++o) w = fmaf(satt[o], sW2[o * 64 + lt], w);
            weff[lt] = w;
        } else if (lt == 64) {
            float c0 = 0.f, hl = 3.0e38f;
            for (int o = 0; o < ZZ; ++o) {
                c0 = fmaf(satt[o], sb2[o], c0);
                float l1 = 0.f;
                for (int j = 0; j < 64; ++j) l1 += fabsf(sW2[o * 64 + j]);
                hl = fminf(hl, (1.0e37f - fabsf(sb2[o])) / fmaxf(l1, 1e-30f));
            }
            weff[64] = c0;
            weff[65] = hl;
        }
    }

    MqState<G> &st = sts[unit];
    int *nlog = nlog_[unit];
    // ---- scratch: unit-level flattened lists, per-query visited bitsets / logs / pools
    const int64_t ug = (int64_t)blockIdx.x * 2 + unit;  // global unit index
    const int64_t capF = a.capF, capS = a.capS, capP = a.capP;  // lists already x G
    // frontier lists c = 0/1 (pointer arithmetic, not a dynamically indexed local array)
    auto fslot = [&](int c) { return a.f_slot + (ug * 2 + c) * capF; };
    auto fsrch = [&](int c) { return a.f_srch + (ug * 2 + c) * capF; };
    int32_t *surv_v = a.surv_v + ug * capS, *surv_i = a.surv_i + ug * capS;
    int32_t *cont_v = a.cont_v + ug * capS, *cont_i = a.cont_i + ug * capS;
    // fresh claims ARE the survivors (unique per (query, node)); their searcher field is
    // lowered to the lowest toucher by the resolve pass before the frontier split reads it
    int32_t *fr_v = surv_v, *fr_i = surv_i;
    uint64_t *fr_key = a.fr_key + ug * capS;
    int32_t *seg_v = a.seg_v + ug * capS;
    uint64_t *seg_key = a.seg_key + ug * capS;
    int32_t *rq = cont_v;      // re-score requests (gq << 24 | index); contested lists are dead
    int32_t *seg_ex = cont_i;  // after resolve
    auto vis_of = [&](int gq) { return a.vis + (ug * G + gq) * a.vis_words; };
    auto log_of = [&](int gq) { return a.vlog + (ug * G + gq) * (int64_t)a.log_cap; };
    auto pkey = [&](int gq, int c) { return a.pool_key + ((ug * G + gq) * 2 + c) * capP; };
    auto pslot = [&](int gq, int c) { return a.pool_slot + ((ug * G + gq) * 2 + c) * capP; };
    auto pmeta = [&](int gq, int c) { return a.pool_meta + ((ug * G + gq) * 2 + c) * capP; };
    auto band_of = [&](float T) { return a.band_rel * fabsf(T) + a.band_abs; };
    const int top = g.n_layers - 1, nst = 5 + g.n_layers, d_h = DH;

    for (;;) {
        usync();
        if (lt == 0) st.base = atomicAdd(a.queue, G);
        usync();
        if (st.base >= a.Q) break;
        if (a.avail) {  // streamed call: wait until this batch's users have been copied in
            if (lt == 0) {
                const int need = (int)min((int64_t)st.base + G, a.Q);
                int got;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(got) : "l"(a.avail) : "memory");
                    if (got >= need) break;
                    __nanosleep(500);
                }
            }
            usync();
        }
        if (lt < G) {
            MqQuery &Q = st.qs[lt];
            Q.q = st.base + lt < a.Q ? st.base + lt : -1;
            Q.nPool = 0; Q.pool_cur = 0; Q.poolT = 0ull; Q.besthop = -1;
            for (int l = 0; l < GR_MAX_LAYERS; ++l) Q.per_layer[l] = 0;
            Q.rows = 0; Q.nbrs = 0;
            nlog[lt] = 0;
        }
        if (lt == 0) st.f_cur = 0;
        usync();
        if (tid == 0) ph_t0 = clock64();
        // ---- hoisted user halves (exact acc0; tensor-core U = user half + b0)
        for (int t = lt; t < G * 64; t += NTH) {
            const int gq = t >> 6, o = t & 63;
            const int q = st.qs[gq].q;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            if (q >= 0) {
                const float *hu = a.users + (int64_t)q * d_h;
                for (int j = 0; j < M.pre_ch; ++j) {
                    const int c = chunk_perm(j, 2 * d_h);
                    mac4(acc, make_float4(hu[4 * c], hu[4 * c + 1], hu[4 * c + 2], hu[4 * c + 3]),
                         M.W[0][j * 64 + o]);
                }
            }
            sAcc0[gq * 64 + o] = acc;
            if constexpr (MODE == 1) U[gq * 64 + o] = __fadd_rn(hsum4(acc), M.b[0][o]);
        }

        // ================= helpers
        auto score_fresh = [&](int n, int layer, int hop) {
            auto on_score = [&](int i, bool valid, float v, int gi, int32_t s, uint32_t rank) {
                const int gq = gi >> 16;  // evaluations are counted per query by expand
                if (valid && !isfinite(v)) atomicOr(a.nonfinite, 1);
                const uint64_t key = make_key(v, rank);
                if (valid) fr_key[i] = key;
                MqQuery &Q = st.qs[gq];
                bool app;
                if constexpr (MODE == 1) {
                    const float Ts = orderable_f32((uint32_t)(Q.poolT >> 32));
                    app = valid && (!Q.poolT || v >= Ts - band_of(Ts));
                } else {
                    app = valid && key > Q.poolT;
                }
                const int idx = warp_append(gq, app, [&](int q) { return &st.qs[q].nPool; });
                if (idx >= 0) {
                    pkey(gq, Q.pool_cur)[idx] = key;
                    pslot(gq, Q.pool_cur)[idx] = s;
                    pmeta(gq, Q.pool_cur)[idx] = (hop << 1) | (MODE == 1 ? 0 : 1);
                }
            };
            if constexpr (MODE == 1) {
                TP::run(smem, ub, U, sb1, sW2, sb2, satt, tmem, a.it, g, fr_v, fr_i, n, chunk_ctr, tile_ctr, lt,
                        on_score, usync, &a.hl_map,
                        a.phase_cycles && unit == 0 ? ph_acc + 8 : nullptr);
                if (lt == 0) atomicAdd(a.counters + 1, (unsigned long long)n);
            } else {
                int *pq = reinterpret_cast<int *>(sBuf + EX::OFF_PQ);
                const float *sc = reinterpret_cast<const float *>(sBuf + EX::OFF_SC);
                for (int base = 0; base < n; base += EX::PT) {
                    const int nv = min(EX::PT, n - base);
                    for (int pp = 0; pp < 4; ++pp) {
                        const int p = warp * 4 + pp;
                        float4 *xr = sBuf + EX::OFF_X0 + p * EX::LDX0;
                        if (p < nv) {
                            const float4 *hv = reinterpret_cast<const float4 *>(
                                a.it.emb + slot_row(g, fr_v[base + p]) * a.it.ld);
                            for (int cc = lane; cc < DH / 4; cc += 32)
                                xr[chunk_perm(DH / 4 + cc, 2 * DH) - DH / 4] = __ldg(hv + cc);
                        } else {
                            for (int cc = lane; cc < DH / 4; cc += 32) xr[cc] = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                        if (lane == 0) pq[p] = p < nv ? (fr_i[base + p] >> 16) : 0;
                    }
                    usync();
                    EX::template tile<false>(lt, sW, sW0, sBuf, sAcc0, nv, a.nonfinite, usync, a.negz);
                    if (lt < 32) {
                        const bool valid = lt < nv;
                        const int32_t es = valid ? fr_v[base + lt] : 0;
                        on_score(base + lt, valid, valid ? sc[lt] : 0.f, valid ? fr_i[base + lt] : 0, es,
                                 slot_rank(g, es));
                    }
                    usync();
                }
            }
        };
        // exact re-score of rq[0..n): entry = (gq << 24 | idx) into that query's current
        // pool (pool=1) or into the seg arrays (pool=0)
        auto rescore = [&](int n, bool pool) {
            if constexpr (MODE == 1) {
                int *pq = reinterpret_cast<int *>(sBuf + EX::OFF_PQ);
                const float *sc = reinterpret_cast<const float *>(sBuf + EX::OFF_SC);
                for (int base = 0; base < n; base += EX::PT) {
                    const int nv = min(EX::PT, n - base);
                    for (int pp = 0; pp < 4; ++pp) {
                        const int p = warp * 4 + pp;
                        float4 *xr = sBuf + EX::OFF_X0 + p * EX::LDX0;
                        if (p < nv) {
                            const int e = rq[base + p];
                            const int gq = e >> 24, idx = e & 0xFFFFFF;
                            const int32_t s = pool ? pslot(gq, st.qs[gq].pool_cur)[idx] : seg_v[idx];
                            const float4 *hv = reinterpret_cast<const float4 *>(a.it.emb + slot_row(g, s) * a.it.ld);
                            for (int cc = lane; cc < DH / 4; cc += 32)
                                xr[chunk_perm(DH / 4 + cc, 2 * DH) - DH / 4] = __ldg(hv + cc);
                            if (lane == 0) pq[p] = gq;
                        } else {
                            for (int cc = lane; cc < DH / 4; cc += 32) xr[cc] = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (lane == 0) pq[p] = 0;
                        }
                    }
                    usync();
                    EX::template tile<true>(lt, sW, sW0, sBuf, sAcc0, nv, a.nonfinite, usync, a.negz);
                    if (lt < nv) {
                        const int e = rq[base + lt];
                        const int gq = e >> 24, idx = e & 0xFFFFFF;
                        band_record(bc, pool ? pkey(gq, st.qs[gq].pool_cur)[idx] : seg_key[idx], sc[lt],
                                    a.band_rel, a.band_abs);
                        if (pool) {
                            const int c = st.qs[gq].pool_cur;
                            pkey(gq, c)[idx] = make_key(sc[lt], slot_rank(g, pslot(gq, c)[idx]));
                            pmeta(gq, c)[idx] |= 1;
                        } else {
                            seg_key[idx] = make_key(sc[lt], slot_rank(g, seg_v[idx]));
                            seg_ex[idx] = 1;
                        }
                    }
                    usync();
                }
                if (lt == 0 && n) atomicAdd(a.counters, (unsigned long long)n);
            }
        };
        auto collect_pool = [&](auto pred) {
            if (lt == 0) st.nRq = 0;
            usync();
            for (int gq = 0; gq < G; ++gq) {
                const MqQuery &Q = st.qs[gq];
                const int np = Q.nPool;
                const uint64_t *pk = pkey(gq, Q.pool_cur);
                const int32_t *pm = pmeta(gq, Q.pool_cur);
                for (int i0 = 0; i0 < np; i0 += NTH) {
                    const int i = i0 + lt;
                    bool ok = i < np && !(pm[i] & 1) && pred(gq, orderable_f32((uint32_t)(pk[i] >> 32)));
                    warp_append1(ok, (gq << 24) | i, &st.nRq, rq);
                }
            }
            usync();
            return st.nRq;
        };
        // per-query pool compaction to top-k (warp gq); tensor mode refines the band first
        auto compact_pools = [&]() {
            if constexpr (MODE == 1) {
                __shared__ float thr_[2][G];
                if (warp < G) {
                    const MqQuery &Q = st.qs[warp];
                    float Ts = INFINITY;
                    if (Q.nPool > a.k) {
                        const uint64_t Ta = warp_select_threshold(pkey(warp, Q.pool_cur), Q.nPool, a.k, hist + warp * 256);
                        Ts = orderable_f32((uint32_t)(Ta >> 32));
                    }
                    if (lane == 0) thr_[unit][warp] = Ts;
                }
                usync();
                const int n = collect_pool([&](int gq, float v) {
                    const float T = thr_[unit][gq];
                    return isfinite(T) && fabsf(v - T) <= band_of(T);
                });
                rescore(n, true);
            }
            if (warp < G) {
                MqQuery &Q = st.qs[warp];
                if (Q.nPool > a.k) {
                    const int c = Q.pool_cur, np = Q.nPool;
                    const uint64_t T = warp_select_threshold(pkey(warp, c), np, a.k, hist + warp * 256);
                    int cnt = 0;
                    for (int i0 = 0; i0 < np; i0 += 32) {
                        const int i = i0 + lane;
                        const bool keep = i < np && pkey(warp, c)[i] >= T;
                        const unsigned mask = __ballot_sync(0xffffffffu, keep);
                        if (keep) {
                            const int pos = cnt + __popc(mask & ((1u << lane) - 1u));
                            pkey(warp, c ^ 1)[pos] = pkey(warp, c)[i];
                            pslot(warp, c ^ 1)[pos] = pslot(warp, c)[i];
                            pmeta(warp, c ^ 1)[pos] = pmeta(warp, c)[i];
                        }
                        cnt += __popc(mask);
                    }
                    __syncwarp();
                    if (lane == 0) { Q.pool_cur = c ^ 1; Q.nPool = cnt; Q.poolT = T; }
                }
            }
            usync();
        };
        // this hop's first touches [0, nS) are the fresh claims (already in the visited bits and
        // in their query's claim log, written by the owning warp during expand)
        auto resolve = [&](int nS) {
            if (lt == 0) st.nFresh = nS;
            usync();
        };
        // append v (when ok) to query w's claim log; called by warp w (the only writer of nlog[w])
        auto log_push = [&](int w, bool ok, int32_t v) {
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            const int p = nlog[w] + __popc(m & ((1u << lane) - 1u));
            if (ok && p < a.log_cap) log_of(w)[p] = v;
            __syncwarp();
            if (lane == 0) nlog[w] += __popc(m);
            __syncwarp();
        };
        auto sort_pools = [&]() {
            const int gq = lt / GT, gt = lt % GT;
            const MqQuery &Q = st.qs[gq];
            uint64_t *sk = sortk + gq * a.sortcap;
            int32_t *sv = sortv + gq * a.sortcap;
            const int np = Q.nPool;
            for (int i = gt; i < np; i += GT) { sk[i] = pkey(gq, Q.pool_cur)[i]; sv[i] = i; }
            group_sort_desc<GT>(sk, sv, np, a.sortcap, gt, 0);
            usync();
        };

        // ================= init: entry + its top-layer neighbourhood (hop 0), as first
        // touches of searcher 0 (the entry's row never contains the entry)
        if (lt == 0) { st.nS = 0; st.nFresh = 0; }
        usync();
        if (lt < G && st.qs[lt].q >= 0) {
            const int idx = atomicAdd(&st.nS, 1);
            atomicOr(vis_of(lt) + (g.entry >> 5), 1u << (g.entry & 31));
            surv_v[idx] = g.entry;
            surv_i[idx] = lt << 16;
            log_of(lt)[0] = g.entry;
            nlog[lt] = 1;
        }
        usync();
        if (warp < G && st.qs[warp].q >= 0) {
            const int32_t *row = graph_row(g, top, g.entry);
            uint32_t *vb = vis_of(warp);
            if (lane == 0) st.qs[warp].rows += 1;
            if (row) {
                for (int c0 = 0; c0 < g.deg[top]; c0 += 32) {
                    const int32_t v = (c0 + lane < g.deg[top]) ? __ldg(row + c0 + lane) : -1;
                    const unsigned nv = __popc(__ballot_sync(0xffffffffu, v >= 0));
                    if (lane == 0) st.qs[warp].nbrs += nv;
                    uint32_t s2 = 1u;
                    if (v >= 0) s2 = (atomicOr(vb + (v >> 5), 1u << (v & 31)) >> (v & 31)) & 1u;
                    warp_append2(v >= 0 && s2 == 0u, v, warp << 16, &st.nS, surv_v, surv_i);
                    log_push(warp, v >= 0 && s2 == 0u, v);
                }
            }
            if (lane == 0) st.qs[warp].per_layer[top] = nlog[warp];  // entry + fresh neighbours
        }
        usync();
        resolve(st.nS);
        score_fresh(st.nFresh, top, 0);
        compact_pools();
        GR_PH(0);

        int h = 0;
        for (int layer = top; layer >= 0; --layer) {
            // ---- seeds: each query's pool sorted, first min(kp, |pool|) (exact in MODE 1)
            if constexpr (MODE == 1) {
                __shared__ float thr2_[2][G];
                if (warp < G) {
                    const MqQuery &Q = st.qs[warp];
                    float Ts = -INFINITY;  // all entries when |pool| <= kp
                    if (Q.nPool > a.kp) {
                        const uint64_t Ta = warp_select_threshold(pkey(warp, Q.pool_cur), Q.nPool, a.kp, hist + warp * 256);
                        Ts = orderable_f32((uint32_t)(Ta >> 32));
                        Ts = Ts - band_of(Ts);
                    }
                    if (lane == 0) thr2_[unit][warp] = Ts;
                }
                usync();
                rescore(collect_pool([&](int gq, float v) { return v >= thr2_[unit][gq]; }), true);
            }
            sort_pools();
            if (lt == 0) {
                int off = 0;
                for (int gq = 0; gq < G; ++gq) {
                    MqQuery &Q = st.qs[gq];
                    const int ns = Q.q >= 0 ? min(a.kp, Q.nPool) : 0;
                    Q.f_off = off;
                    Q.f_cnt = ns;
                    off += ns;
                }
                st.nF = off;
                st.f_cur = 0;
            }
            usync();
            for (int gq = 0; gq < G; ++gq) {
                const MqQuery &Q = st.qs[gq];
                for (int i = lt; i < Q.f_cnt; i += NTH) {
                    fslot(0)[Q.f_off + i] = pslot(gq, Q.pool_cur)[sortv[gq * a.sortcap + i]];
                    fsrch(0)[Q.f_off + i] = (gq << 16) | i;
                }
            }
            usync();
            GR_PH(1);
            for (int t = 0; t < a.hops; ++t) {
                ++h;
                const int nF = st.nF;
                if (nF == 0) { h += a.hops - 1 - t; break; }
                const int fc = st.f_cur;
                if (lt == 0) { st.nS = 0; st.nFresh = 0; }
                usync();
                // ---- expand + claim: warp w owns query w and walks its frontier in list order
                // (searcher-ascending) in batches of <= RW rows of ONE searcher; a batch's 16-byte
                // row pieces are spread over the lanes (<= 3 per lane), all row loads in flight,
                // then all claim atomics, then one survivor reservation.  Software-pipelined: the
                // next batch's frontier entries and rows are fetched under this batch's atomics,
                // whose results are consumed before the next batch issues its own.
                if (st.qs[warp].q >= 0) {
                    const int P = g.ld[layer] >> 2;
                    const int RW = min(32, 96 / P), NP = RW * P;
                    constexpr unsigned FULL = 0xffffffffu;
                    const int qend = st.qs[warp].f_off + st.qs[warp].f_cnt;
                    uint32_t *vb = vis_of(warp);
                    // the query's frontier entries stream through a two-window register buffer
                    // (lane i holds entry wbase + i of the current window, and of the next):
                    // batch boundaries come from shuffles, the list loads run a window ahead
                    int wbase = st.qs[warp].f_off;
                    int32_t cur_s = -1, cur_g = -1, nxt_s = -1, nxt_g = -1;
                    auto load_win = [&](int base, int32_t &ws, int32_t &wg) {
                        ws = -1;
                        wg = -1;
                        if (base + lane < qend) {
                            GR_DCHECK(base + lane < capF, "fslot index %d >= %lld", base + lane, (long long)capF);
                            ws = fslot(fc)[base + lane];
                            wg = fsrch(fc)[base + lane];
                            if (layer == 0) {  // rows of the next batches: L2 ahead of the piece loads
                                const char *rp = reinterpret_cast<const char *>(g.adj[0] + (int64_t)ws * g.ld[0]);
                                for (int o = 0; o < g.ld[0] * 4; o += 128)
                                    asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + o));
                            }
                            GR_DCHECK(ws >= 0 && ws < g.n && (wg >> 16) == warp, "frontier entry %d gi %x warp %d",
                                      ws, wg, warp);
                        }
                    };
                    load_win(wbase, cur_s, cur_g);
                    load_win(wbase + 32, nxt_s, nxt_g);
                    auto meta = [&](int e0, int32_t &ms, int &len) {
                        if (e0 >= wbase + 32) {  // advance the window (e0 < wbase + 64 always)
                            wbase += 32;
                            cur_s = nxt_s;
                            cur_g = nxt_g;
                            load_win(wbase + 32, nxt_s, nxt_g);
                        }
                        const int src = e0 - wbase + lane;  // < 64
                        const int32_t a_s = __shfl_sync(FULL, cur_s, src & 31), a_g = __shfl_sync(FULL, cur_g, src & 31);
                        const int32_t b_s = __shfl_sync(FULL, nxt_s, src & 31), b_g = __shfl_sync(FULL, nxt_g, src & 31);
                        const bool in = lane < RW && e0 + lane < qend;
                        ms = in ? (src < 32 ? a_s : b_s) : -1;
                        const int32_t mgi = in ? (src < 32 ? a_g : b_g) : 0;
                        const int32_t head = __shfl_sync(FULL, mgi, 0);  // every lane: no short circuit
                        const bool same = in && mgi == head;
                        len = __popc(__ballot_sync(FULL, same));  // a prefix: entries sorted by searcher
                        if (!same) ms = -1;
                        return head;
                    };
                    auto pieces = [&](int32_t ms, int4 (&pv)[3]) {
                        const int4 *mrow = ms >= 0 ? reinterpret_cast<const int4 *>(graph_row(g, layer, ms)) : nullptr;
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const int pc = lane + 32 * j, r = min(pc / P, 31), c = pc - r * P;
                            const int4 *rp = reinterpret_cast<const int4 *>(
                                __shfl_sync(FULL, reinterpret_cast<unsigned long long>(mrow), r));
                            pv[j] = (pc < NP && rp) ? __ldg(rp + c) : make_int4(-1, -1, -1, -1);
                        }
                    };
                    int32_t ms;
                    int len;
                    int4 pv[3];
                    int e0 = st.qs[warp].f_off;
                    int lbase = nlog[warp];  // this query's claim log (warp-private during expand)
                    int32_t *const lg = log_of(warp);
                    int32_t gi = meta(e0, ms, len);
                    pieces(ms, pv);
                    int nrows = 0, nnbr = 0;
                    while (len > 0) {
                        int32_t ms1;
                        int len1;
                        const int32_t gi1 = meta(e0 + len, ms1, len1);
                        uint32_t s2[3][4];  // visited bit before this touch
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const int vv[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                s2[j][u] = vv[u] >= 0 ? atomicOr(vb + (vv[u] >> 5), 1u << (vv[u] & 31)) : 1u;
                        }
                        int4 pv1[3];
                        pieces(ms1, pv1);
                        int cs = 0, nv = 0;
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const int vv[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                if (vv[u] >= 0) s2[j][u] = (s2[j][u] >> (vv[u] & 31)) & 1u;
                                nv += vv[u] >= 0;
                                cs += s2[j][u] == 0u;
                            }
                        }
                        int is = cs;  // one reservation per warp (inclusive scan of the lane counts)
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int ys = __shfl_up_sync(FULL, is, o);
                            if (lane >= o) is += ys;
                        }
                        int bs = 0;
                        if (lane == 31 && is) bs = atomicAdd(&st.nS, is);
                        bs = __shfl_sync(FULL, bs, 31) + is - cs;
                        int lp = lbase + is - cs;
                        lbase += __shfl_sync(FULL, is, 31);
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const int vv[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (vv[u] >= 0 && s2[j][u] == 0u) {
                                    GR_DCHECK(bs < capS && vv[u] < g.n, "survivor %d cap %lld v %d", bs, (long long)capS, vv[u]);
                                    surv_v[bs] = vv[u];
                                    surv_i[bs] = gi;
                                    ++bs;
                                    if (lp < a.log_cap) lg[lp] = vv[u];
                                    ++lp;
                                }
                        }
                        nrows += len;
                        nnbr += nv;
                        e0 += len;
                        ms = ms1;
                        len = len1;
                        gi = gi1;
#pragma unroll
                        for (int j = 0; j < 3; ++j) pv[j] = pv1[j];
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) nnbr += __shfl_xor_sync(FULL, nnbr, o);
                    if (lane == 0) {
                        st.qs[warp].rows += nrows;
                        st.qs[warp].nbrs += nnbr;
                        st.qs[warp].per_layer[layer] += lbase - nlog[warp];  // this hop's evaluations
                        nlog[warp] = lbase;
                    }
                }
                usync();
                GR_PH(2);
                resolve(st.nS);
                GR_PH(3);
                const int nFresh = st.nFresh;
                score_fresh(nFresh, layer, h);
                GR_PH(4);
                compact_pools();
                GR_PH(5);
                if (t == a.hops - 1) break;
                // ---- per-(query, searcher) top-ef of fresh claims -> next frontier
                for (int i = lt; i < NSEG; i += NTH) seg_cnt[i] = 0;
                usync();
                auto seg_of = [&](int gi) { return (gi >> 16) * a.kp + (gi & 0xFFFF); };
                for (int t0 = 0; t0 < nFresh; t0 += NTH) {
                    const int t2 = t0 + lt;
                    if (t0 + warp * 32 < nFresh) {
                        const int sg = t2 < nFresh ? seg_of(fr_i[t2]) : 0;
                        warp_count(&seg_cnt[sg], sg, 1, t2 < nFresh);
                    }
                }
                usync();
                if (warp == 0) {  // exclusive scans of counts and min(count, ef)
                    int acc = 0, accf = 0;
                    for (int i0 = 0; i0 < NSEG; i0 += 32) {
                        const int i = i0 + lane;
                        const int c = i < NSEG ? seg_cnt[i] : 0, cf = min(c, a.ef);
                        int x = c, xf = cf;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int y = __shfl_up_sync(0xffffffffu, x, o), yf = __shfl_up_sync(0xffffffffu, xf, o);
                            if (lane >= o) { x += y; xf += yf; }
                        }
                        if (i < NSEG) { seg_off[i] = acc + x - c; fn_off[i] = accf + xf - cf; seg_cnt[i] = 0; }
                        acc += __shfl_sync(0xffffffffu, x, 31);
                        accf += __shfl_sync(0xffffffffu, xf, 31);
                    }
                    __syncwarp();
                    if (lane == 0) st.nFn = accf;
                    if (lane < G) {  // each query's next frontier range (its segments are contiguous)
                        const int lo = fn_off[lane * a.kp], hi = lane + 1 < G ? fn_off[(lane + 1) * a.kp] : accf;
                        st.qs[lane].f_off = lo;
                        st.qs[lane].f_cnt = hi - lo;
                    }
                }
                usync();
                for (int t2 = lt; t2 < nFresh; t2 += NTH) {
                    const int sg = seg_of(fr_i[t2]);
                    const int pos = seg_off[sg] + atomicAdd(&seg_cnt[sg], 1);
                    seg_v[pos] = fr_v[t2];
                    seg_key[pos] = fr_key[t2];
                }
                usync();
                if constexpr (MODE == 1) {
                    for (int t2 = lt; t2 < nFresh; t2 += NTH) seg_ex[t2] = 0;
                    if (lt == 0) st.nRq = 0;
                    usync();
                    for (int sg = warp; sg < NSEG; sg += NW) {
                        const int ni = seg_cnt[sg], off = seg_off[sg], gq = sg / a.kp;
                        if (ni <= a.ef) continue;
                        const uint64_t Ta = warp_select_threshold(seg_key + off, ni, a.ef, hist + warp * 256);
                        const float Ts = orderable_f32((uint32_t)(Ta >> 32)), bd = band_of(Ts);
                        for (int j0 = 0; j0 < ni; j0 += 32) {
                            const int j = j0 + lane;
                            const bool in = j < ni &&
                                fabsf(orderable_f32((uint32_t)(seg_key[off + j] >> 32)) - Ts) <= bd;
                            warp_append1(in, (gq << 24) | (off + j), &st.nRq, rq);
                        }
                    }
                    usync();
                    rescore(st.nRq, false);
                }
                const int fn = fc ^ 1;
                for (int sg = warp; sg < NSEG; sg += NW) {
                    const int ni = seg_cnt[sg], off = seg_off[sg], fo = fn_off[sg];
                    const int gi = ((sg / a.kp) << 16) | (sg % a.kp);
                    if (ni <= a.ef) {
                        GR_DCHECK(fo + ni <= capF, "frontier write %d + %d > %lld", fo, ni, (long long)capF);
                        for (int j = lane; j < ni; j += 32) { fslot(fn)[fo + j] = seg_v[off + j]; fsrch(fn)[fo + j] = gi; }
                    } else {
                        const uint64_t T = warp_select_threshold(seg_key + off, ni, a.ef, hist + warp * 256);
                        int cnt = 0;
                        for (int j0 = 0; j0 < ni; j0 += 32) {
                            const int j = j0 + lane;
                            const bool keep = j < ni && seg_key[off + j] >= T;
                            const unsigned mask = __ballot_sync(0xffffffffu, keep);
                            if (keep) {
                                const int pos = fo + cnt + __popc(mask & ((1u << lane) - 1u));
                                fslot(fn)[pos] = seg_v[off + j];
                                fsrch(fn)[pos] = gi;
                            }
                            cnt += __popc(mask);
                        }
                    }
                }
                usync();
                if (lt == 0) { st.nF = st.nFn; st.f_cur = fn; }
                usync();
                GR_PH(6);
            }
        }

        // ---- results: every query's pool sorted, first min(k, |pool|), exact scores
        if constexpr (MODE == 1) rescore(collect_pool([&](int, float) { return true; }), true);
        sort_pools();
        for (int gq = 0; gq < G; ++gq) {
            MqQuery &Q = st.qs[gq];
            if (Q.q < 0) continue;
            const int64_t q = Q.q;
            const int np = Q.nPool, c = Q.pool_cur, nr = min(a.k, np);
            const int32_t *sv = sortv + gq * a.sortcap;
            for (int j = lt; j < a.k; j += NTH) {
                if (j < nr) {
                    const int idx = sv[j];
                    a.out_ids[q * a.k + j] = g.ids[pslot(gq, c)[idx]];
                    a.out_scores[q * a.k + j] = (double)orderable_f32((uint32_t)(pkey(gq, c)[idx] >> 32));
                } else {
                    a.out_ids[q * a.k + j] = -1;
                    a.out_scores[q * a.k + j] = __longlong_as_double(0x7ff8000000000000ll);
                }
            }
            if (lt == 0) {
                a.out_count[q] = nr;
                int64_t ev = 0;
                for (int l = 0; l < g.n_layers; ++l) { ev += Q.per_layer[l]; a.out_stats[q * nst + 5 + l] = Q.per_layer[l]; }
                a.out_stats[q * nst + 0] = ev;
                a.out_stats[q * nst + 1] = ev;
                a.out_stats[q * nst + 2] = nr > 0 ? (pmeta(gq, c)[sv[0]] >> 1) : -1;
                a.out_stats[q * nst + 3] = Q.rows;
                a.out_stats[q * nst + 4] = Q.nbrs;
            }
        }
        if (a.qdone) {  // streamed call: publish the finished queries of this batch
            __threadfence();
            usync();
            if (lt == 0) {
                int nq = 0;
                for (int gq = 0; gq < G; ++gq) nq += st.qs[gq].q >= 0;
                atomicAdd(a.qdone + st.base / a.chunk_q, nq);
            }
        }
        // ---- reset this unit's visited bitsets: zero the words of every claimed node (all
        // set bits belong to claimed nodes), or the whole bitset when the log overflowed
        for (int gq = 0; gq < G; ++gq) {
            const int nl = nlog[gq];
            uint32_t *vb = vis_of(gq);
            if (nl <= a.log_cap) {
                const int32_t *lg = log_of(gq);
                for (int j0 = 0; j0 < nl; j0 += 4 * NTH) {
                    int32_t v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = j0 + u * NTH + lt < nl ? lg[j0 + u * NTH + lt] : -1;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (v[u] >= 0) vb[v[u] >> 5] = 0u;
                }
            } else {
                for (int64_t w = lt; w < a.vis_words; w += NTH) vb[w] = 0u;
            }
        }
        GR_PH(7);
    }
    if (a.phase_cycles && tid < 16) atomicAdd(a.phase_cycles + tid, ph_acc[tid]);
#undef GR_PH
    tc::fence_before();
    __syncthreads();
    if constexpr (MODE == 1) {
        if (tid == 0) band_flush(bc, a.counters, a.band_viol);
        if (tid < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tptr), "r"(2 * TP::COLS));
    }
}
