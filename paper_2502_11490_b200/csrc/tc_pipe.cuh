// Warp-specialised tcgen05 scoring pipeline for one hop's fresh (query, item) pairs.
//
// Roles inside the 512-thread CTA:
//   warps 0-7  (E, two groups of 4 warps): epilogues.  Group e owns the tiles with
//              (global tile number & 1) == e; inside a group warp w reads TMEM lanes
//              32*(w&3).. (one pair row per thread).
//   warp 8     the tcgen05.mma issuer (converged warp, elect.sync picks the issuing lane)
//   warps 9-15 (L, 224 threads): loaders.  Items carry a pre-split bf16 hi/lo copy
//              (gr_items, [n][hi d | lo d]), so loading is pure cp.async: 16-byte pieces
//              straight into the UMMA K-major core-matrix layout, no registers, no conversion;
//              a cp.async.mbarrier arrival per thread completes the stage.
// Buffers: S = 4 stages of one 64-wide K chunk of the A operand (hi + lo, 32 KB each) in shared
// memory; in TMEM (512 columns): layer-0 accumulators D0[e] (64 cols each), layer-1
// accumulators D1[e], and the layer-1 A operand A1[e] (relu(layer 0) as bf16 hi/lo pairs,
// written by E with tcgen05.st and consumed by the ".ts" MMA form -- no shared memory).
// Hand-offs (mbarriers):
//   full[s]   loaders (cp.async arrivals, count NL) -> issuer   empty[s]  commit -> loaders
//   d0full[e] commit -> E        d0empty[e] E (128 arrivals) -> issuer
//   a1full[e] E (128 arrivals) -> issuer      d1full[e] commit -> E
// Parities come from kernel-lifetime chunk / tile counters, identical in every thread.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc_scorer.cuh"

template <int D_H, int Z, int G>
struct TcPipe {
    static constexpr int H = 64, TM = 128, KC = 64, NC = D_H / KC, S = 4;
    static constexpr int NT = 512, NE = 128, ISSUER_WARP = 8, L_WARP0 = 9, NL = NT - 32 * L_WARP0;
    static constexpr int NOPS = 2 * TM / 4;  // TMA gather4 ops per K chunk (hi + lo)
    // byte offsets
    static constexpr int OFF_B0H = 0;
    static constexpr int OFF_B0L = OFF_B0H + H * D_H * 2;
    static constexpr int OFF_B1H = OFF_B0L + H * D_H * 2;
    static constexpr int OFF_B1L = OFF_B1H + H * H * 2;
    static constexpr int OFF_A = OFF_B1L + H * H * 2;          // S chunk stages (hi, lo)
    static constexpr int CH_BYTES = TM * KC * 2;                // one hi or lo chunk: 16 KB
    static constexpr int A_REGION = S * 2 * CH_BYTES;           // 128 KB (aliased, outside run(), by the
                                                                // exact buffers, select histograms, pool sort)
    static constexpr int OFF_U = OFF_A + A_REGION;              // [G][64] user half + b0
    static constexpr int OFF_B1 = OFF_U + G * H * 4;
    static constexpr int OFF_W2 = OFF_B1 + H * 4;               // [Z][64]
    static constexpr int OFF_B2 = OFF_W2 + Z * H * 4;
    static constexpr int OFF_ATT = OFF_B2 + 16;
    static constexpr int OFF_BAR = (OFF_ATT + 16 + 15) & ~15;
    enum { FULL0 = 0, EMPTY0 = S, D0FULL0 = 2 * S, D0EMPTY0 = 2 * S + 2, A1FULL0 = 2 * S + 4,
           D1FULL0 = 2 * S + 6, NBAR = 2 * S + 8 };
    static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr int BYTES = (OFF_TMEM + 16 + 15) & ~15;
    static constexpr uint32_t IDESC = tc::idesc(TM, H);
    static constexpr uint32_t TMEM_COLS = 512;
    // TMEM columns ([e] at +64*e)
    // layer-0 accumulators are 128 columns wide: [0,64) = hi.W_hi + lo.W_hi, [64,128) = hi.W_lo
    // (one N=128 MMA reads A_hi once against [W_hi; W_lo], which are contiguous in smem)
    static constexpr uint32_t C_D0 = 0, C_D1 = 256, C_A1 = 384, D0W = 128;
    static constexpr uint32_t IDESC_N128 = tc::idesc(TM, 2 * H);

    static __device__ __forceinline__ uint64_t *bar(unsigned char *sm, int i) {
        return reinterpret_cast<uint64_t *>(sm + OFF_BAR) + i;
    }

    static __device__ void init_barriers(unsigned char *sm, bool tma = false) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < S; ++s) {
                tc::mbar_init(bar(sm, FULL0 + s), tma ? NOPS : NL);
                tc::mbar_init(bar(sm, EMPTY0 + s), 1);
            }
            for (int e = 0; e < 2; ++e) {
                tc::mbar_init(bar(sm, D0FULL0 + e), 1);
                tc::mbar_init(bar(sm, D0EMPTY0 + e), NE);
                tc::mbar_init(bar(sm, A1FULL0 + e), NE);
                tc::mbar_init(bar(sm, D1FULL0 + e), 1);
            }
        }
    }

    // Score pairs [0, n): item slot slots[i], pair tag gis[i] (query slot << 16 | searcher).
    // For every row E calls on_score(i, valid, score, gi, slot) with all 32 lanes of the warp.
    // it.hl must hold the bf16 hi/lo copy.  chunk_ctr / tile_ctr: kernel-lifetime counters.
    template <class OnScore>
    static __device__ __forceinline__ void run(unsigned char *sm, uint32_t tmem, const DevItems &it,
                                               const DevGraph &g, const int32_t *slots, const int32_t *gis,
                                               int n, uint32_t &chunk_ctr, uint32_t &tile_ctr,
                                               OnScore on_score, unsigned long long *sub = nullptr,
                                               const void *tmap = nullptr, bool pf = false) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        const int T = (n + TM - 1) / TM;
        if (T == 0) return;
        if (tmap) {
            // the A stages alias generic-proxy buffers outside run(); order those accesses
            // before the TMA (async-proxy) writes into them
            tc::fence_async_smem();
            __syncthreads();
        }
        // role timers (GMPGR_PHASE_TIMING): one writer thread per slot
        //   0 E layer-0 epilogue  1 E layer-1 epilogue  2 E d0full-wait  3 E d1full-wait  4 E total
        //   5 issuer idle (polling, nothing ready)  6 issuer busy issuing MMAs  7 loader empty-wait
        const long long t_run = sub ? clock64() : 0;
#define TP_WAIT(slot, expr)                                                   \
    do {                                                                      \
        const long long w0_ = sub ? clock64() : 0;                            \
        expr;                                                                 \
        if (sub) sub[slot] += (unsigned long long)(clock64() - w0_);          \
    } while (0)
        if (warp >= L_WARP0 && tmap) {
            // ================= TMA loaders: per K chunk, 64 tile::gather4 ops (32 four-row groups x
            // hi/lo halves, 128-byte swizzled rows = the SWIZZLE_128B K-major UMMA layout) spread
            // over the 7 loader warps (<= 10 issuing lanes each); every issuing lane arms the
            // stage's full barrier with its own 512 bytes (init count NOPS)
            const int lw = warp - L_WARP0, o = lane * (NL / 32) + lw;
            if (o < NOPS) {
                const int grp = o >> 1, half = o & 1;
                auto rows_of = [&](int t, int (&dst)[4]) {
                    const int base = t * TM, nv = t < T ? min(TM, n - base) : 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int r = 4 * grp + j;
                        const int32_t sl = r < nv ? slots[base + r] : -1;
                        dst[j] = sl < 0 ? 0 : (it.hl_by_slot ? (int)sl : (int)slot_row(g, sl));
                    }
                };
                int nx[4];
                rows_of(0, nx);
                for (int t = 0; t < T; ++t) {
                    int cur[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) cur[j] = nx[j];
                    if (t + 1 < T) {
                        rows_of(t + 1, nx);
                        // warm L2 with the next tile's rows while this tile's stages drain
                        if (pf)
#pragma unroll
                            for (int kc = 0; kc < NC; ++kc)
                                tc::tma_prefetch_gather4(tmap, half * D_H + kc * KC, nx[0], nx[1], nx[2], nx[3]);
                    }
#pragma unroll
                    for (int kc = 0; kc < NC; ++kc) {
                        const uint32_t qg = chunk_ctr + t * NC + kc, s = qg % S, u = qg / S;
                        if (u >= 1) {
                            if (sub && o == 0) TP_WAIT(7, tc::mbar_wait(bar(sm, EMPTY0 + s), (u - 1) & 1u));
                            else tc::mbar_wait(bar(sm, EMPTY0 + s), (u - 1) & 1u);
                        }
                        tc::mbar_arrive_expect_tx(bar(sm, FULL0 + s), 512);
                        tc::tma_gather4(tc::smem_u32(sm + OFF_A + s * 2 * CH_BYTES) + half * CH_BYTES + grp * 512, tmap,
                                        half * D_H + kc * KC, cur[0], cur[1], cur[2], cur[3], bar(sm, FULL0 + s));
                    }
                }
            }
        } else if (warp >= L_WARP0) {
            // ================= loaders: unit = 8 rows x 4 pieces of 16 B (conflict-free
            // core-matrix stores); pieces 0-7 = hi k 0..63 of the chunk, 8-15 = lo
            const int lt = tid - 32 * L_WARP0, lw = lt >> 5;
            constexpr int NLW = NL / 32, UPC = TM * 16 / 32, UPW = (UPC + NLW - 1) / NLW;
            const int rl = lane & 7, pl = lane >> 3;
            // slots of the rows of tiles t+1 and t+2: the slot loads are issued two tiles
            // before their rows are gathered, so their latency never gates the cp.async issue
            int32_t nx1[UPW], nx2[UPW];
            auto load_slots = [&](int t, int32_t (&dst)[UPW]) {
                const int base = t * TM, nv = t < T ? min(TM, n - base) : 0;
#pragma unroll
                for (int i = 0; i < UPW; ++i) {
                    const int un = lw + NLW * i, r = (un % (TM / 8)) * 8 + rl;
                    dst[i] = (un < UPC && r < nv) ? slots[base + r] : -1;
                }
            };
            load_slots(0, nx1);
            load_slots(1, nx2);
            for (int t = 0; t < T; ++t) {
                const uint16_t *rp[UPW];
#pragma unroll
                for (int i = 0; i < UPW; ++i)
                    rp[i] = nx1[i] >= 0 ? it.hl + (it.hl_by_slot ? (int64_t)nx1[i] : slot_row(g, nx1[i])) *
                                                      (2 * (int64_t)D_H)
                                        : nullptr;
#pragma unroll
                for (int i = 0; i < UPW; ++i) nx1[i] = nx2[i];
                load_slots(t + 2, nx2);
#pragma unroll
                for (int kc = 0; kc < NC; ++kc) {
                    const uint32_t qg = chunk_ctr + t * NC + kc, s = qg % S, u = qg / S;
                    if (u >= 1) {
                        if (sub && lt == 0) TP_WAIT(7, tc::mbar_wait(bar(sm, EMPTY0 + s), (u - 1) & 1u));
                        else tc::mbar_wait(bar(sm, EMPTY0 + s), (u - 1) & 1u);
                    }
                    const uint32_t Ah = tc::smem_u32(sm + OFF_A + s * 2 * CH_BYTES);
#pragma unroll
                    for (int i = 0; i < UPW; ++i) {
                        if (!rp[i]) continue;
                        const int un = lw + NLW * i, r = (un % (TM / 8)) * 8 + rl;
                        const int p = (un / (TM / 8)) * 4 + pl;  // 0..15
                        const int hl = p >> 3, k8 = p & 7;
                        tc::cp_async16(Ah + hl * CH_BYTES + tc::kmaj_off(r, k8 * 8, KC),
                                       rp[i] + hl * D_H + kc * KC + k8 * 8);
                    }
                    tc::cp_async_arrive(bar(sm, FULL0 + s));
                }
            }
        } else if (warp == ISSUER_WARP) {
            // ================= MMA issuer (one warp, converged; elect.sync issues): polls the
            // barriers and issues whatever is ready -- layer 1 of an earlier tile as soon as
            // its A1 operand is in TMEM, else the next layer-0 K chunk.  Barrier probes are
            // made warp-uniform (lane 0's answer) so control flow never diverges.
            {
                constexpr unsigned FULLM = 0xffffffffu;
                const uint32_t bH0 = tc::smem_u32(sm + OFF_B0H);
                const uint32_t bH1 = tc::smem_u32(sm + OFF_B1H), bL1 = tc::smem_u32(sm + OFF_B1L);
                auto ready = [&](int b, uint32_t par) {
                    return __shfl_sync(FULLM, lane == 0 ? (int)tc::mbar_test(bar(sm, b), par) : 0, 0) != 0;
                };
                int l0t = 0, l0k = 0, l1t = 0;
                long long idle0 = 0;
                const bool tim = sub && lane == 0;
                while (l1t < T) {
                    if (l1t < l0t) {
                        const uint32_t tg = tile_ctr + l1t, e = tg & 1u, v = tg >> 1;
                        if (ready(A1FULL0 + e, v & 1u)) {
                            const long long ti0 = tim ? clock64() : 0;
                            tc::fence_after();
                            const uint32_t a1 = tmem + C_A1 + 64 * e, d1 = tmem + C_D1 + 64 * e;
#pragma unroll
                            for (int k = 0; k < H / 16; ++k) {
                                const uint64_t bh = tc::desc(bH1 + k * 256, H), bl = tc::desc(bL1 + k * 256, H);
                                tc::mma_ts_w(d1, a1 + k * 8, bh, IDESC, k ? 1u : 0u);  // hi . hi
                                tc::mma_ts_w(d1, a1 + k * 8, bl, IDESC, 1u);           // hi . lo
                                tc::mma_ts_w(d1, a1 + 32 + k * 8, bh, IDESC, 1u);      // lo . hi
                            }
                            tc::commit_w(bar(sm, D1FULL0 + e));
                            if (tim) sub[6] += (unsigned long long)(clock64() - ti0);
                            ++l1t;
                            idle0 = 0;
                            continue;
                        }
                    }
                    bool issued = false;
                    if (l0t < T) {
                        const uint32_t tg = tile_ctr + l0t, e = tg & 1u, v = tg >> 1;
                        const uint32_t qg = chunk_ctr + l0t * NC + l0k, s = qg % S, u = qg / S;
                        if ((l0k != 0 || v == 0 || ready(D0EMPTY0 + e, (v - 1) & 1u)) && ready(FULL0 + s, u & 1u)) {
                            const long long ti0 = tim ? clock64() : 0;
                            tc::fence_async_smem();
                            tc::fence_after();
                            const uint32_t d0 = tmem + C_D0 + D0W * e;
                            const uint32_t aH = tc::smem_u32(sm + OFF_A + s * 2 * CH_BYTES), aL = aH + CH_BYTES;
#pragma unroll
                            for (int k = 0; k < KC / 16; ++k) {
                                const uint64_t ah = tmap ? tc::desc_sw128(aH + k * 32) : tc::desc(aH + k * 256, KC);
                                const uint64_t al = tmap ? tc::desc_sw128(aL + k * 32) : tc::desc(aL + k * 256, KC);
                                const uint32_t kb = (l0k * (KC / 16) + k) * 256;
                                const uint64_t bh = tc::desc(bH0 + kb, D_H);
                                tc::mma_w(d0, ah, bh, IDESC_N128, (l0k | k) ? 1u : 0u);  // hi . [W_hi; W_lo]
                                tc::mma_w(d0, al, bh, IDESC, 1u);                          // lo . W_hi
                            }
                            tc::commit_w(bar(sm, EMPTY0 + s));
                            if (tim) sub[6] += (unsigned long long)(clock64() - ti0);
                            if (++l0k == NC) {
                                tc::commit_w(bar(sm, D0FULL0 + e));
                                l0k = 0;
                                ++l0t;
                            }
                            issued = true;
                        }
                    }
                    if (tim) {  // issuer idle time (no barrier ready)
                        const long long now = clock64();
                        if (!issued && idle0) sub[5] += (unsigned long long)(now - idle0);
                        idle0 = issued ? 0 : now;
                    }
                }
            }
            __syncwarp();
        } else {
            // ================= epilogue groups: row = TMEM lane
            const int e = warp >> 2, q4 = warp & 3, row = q4 * 32 + lane;
            const uint32_t lanebase = (uint32_t)(q4 * 32) << 16;
            const float *Uall = reinterpret_cast<const float *>(sm + OFF_U);
            const float *b1 = reinterpret_cast<const float *>(sm + OFF_B1);
            const float *W2 = reinterpret_cast<const float *>(sm + OFF_W2);
            const float *b2 = reinterpret_cast<const float *>(sm + OFF_B2);
            const float *att = reinterpret_cast<const float *>(sm + OFF_ATT);
            const bool timer = sub && e == 0 && row == 0;
            for (int t = 0; t < T; ++t) {
                const uint32_t tg = tile_ctr + t, v = tg >> 1;
                if ((tg & 1u) != (uint32_t)e) continue;
                const int base = t * TM, nv = min(TM, n - base);
                // the row's pair (issued before the wait so the L2 latency hides behind it)
                const int gi = row < nv ? gis[base + row] : 0, gq = gi >> 16;
                const int32_t my_s = row < nv ? slots[base + row] : 0;
                const float *u = Uall + gq * H;
                if (timer) TP_WAIT(2, tc::mbar_wait(bar(sm, D0FULL0 + e), v & 1u));
                else tc::mbar_wait(bar(sm, D0FULL0 + e), v & 1u);
                tc::fence_after();
                const long long te0 = timer ? clock64() : 0;
                float h[64];
                {
                    const uint32_t d0 = tmem + lanebase + C_D0 + D0W * e;
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        float va[32], vb[32];
                        tc::tmem_ld32(d0 + 32 * half, va);
                        tc::tmem_ld32(d0 + 64 + 32 * half, vb);
#pragma unroll
                        for (int j = 0; j < 32; ++j) h[32 * half + j] = va[j] + vb[j];
                    }
                }
                tc::fence_before();
                tc::mbar_arrive(bar(sm, D0EMPTY0 + e));
                // relu(layer 0) -> bf16 hi/lo pairs -> A1[e] (TMEM cols hi 0..31, lo 32..63)
                const uint32_t a1 = tmem + lanebase + C_A1 + 64 * e;
#pragma unroll
                for (int o = 0; o < 64; o += 16) {
                    uint32_t hi[8], lo[8];
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        const float4 uo = *reinterpret_cast<const float4 *>(u + o + j);
                        const float y0 = fmaxf(h[o + j] + uo.x, 0.f), y1 = fmaxf(h[o + j + 1] + uo.y, 0.f);
                        const float y2 = fmaxf(h[o + j + 2] + uo.z, 0.f), y3 = fmaxf(h[o + j + 3] + uo.w, 0.f);
                        uint2 hh, ll;
                        tc::split4(make_float4(y0, y1, y2, y3), hh, ll);
                        hi[j / 2] = hh.x; hi[j / 2 + 1] = hh.y;
                        lo[j / 2] = ll.x; lo[j / 2 + 1] = ll.y;
                    }
                    tc::tmem_st8(a1 + o / 2, hi);
                    tc::tmem_st8(a1 + 32 + o / 2, lo);
                }
                tc::tmem_wait_st();
                tc::fence_before();
                tc::mbar_arrive(bar(sm, A1FULL0 + e));
                if (timer) sub[0] += (unsigned long long)(clock64() - te0);
                if (timer) TP_WAIT(3, tc::mbar_wait(bar(sm, D1FULL0 + e), v & 1u));
                else tc::mbar_wait(bar(sm, D1FULL0 + e), v & 1u);
                tc::fence_after();
                const long long te1 = timer ? clock64() : 0;
                {
                    float va[32], vb[32];
                    tc::tmem_ld32(tmem + lanebase + C_D1 + 64 * e, va);
                    tc::tmem_ld32(tmem + lanebase + C_D1 + 64 * e + 32, vb);
#pragma unroll
                    for (int j = 0; j < 32; ++j) { h[j] = fmaxf(va[j] + b1[j], 0.f); h[32 + j] = fmaxf(vb[j] + b1[32 + j], 0.f); }
                }
                tc::fence_before();
                // approximate path: reassociated (4 partial sums per output) -- the exact
                // refinement re-scores everything near a threshold, so only the error bound matters
                float s = 0.f;
                bool bad = false;
                const float4 *W2v = reinterpret_cast<const float4 *>(W2);
                float zp[Z][4];
#pragma unroll
                for (int o = 0; o < Z; ++o) zp[o][0] = zp[o][1] = zp[o][2] = zp[o][3] = 0.f;
#pragma unroll
                for (int j = 0; j < 64; j += 4) {
#pragma unroll
                    for (int o = 0; o < Z; ++o) {
                        const float4 w = W2v[o * (H / 4) + j / 4];
                        zp[o][0] = fmaf(h[j], w.x, zp[o][0]);
                        zp[o][1] = fmaf(h[j + 1], w.y, zp[o][1]);
                        zp[o][2] = fmaf(h[j + 2], w.z, zp[o][2]);
                        zp[o][3] = fmaf(h[j + 3], w.w, zp[o][3]);
                    }
                }
#pragma unroll
                for (int o = 0; o < Z; ++o) {
                    const float z = b2[o] + ((zp[o][0] + zp[o][1]) + (zp[o][2] + zp[o][3]));
                    bad |= !isfinite(z);
                    s = fmaf(z, att[o], s);
                }
                if (timer) sub[1] += (unsigned long long)(clock64() - te1);
                on_score(base + row, row < nv, bad ? __int_as_float(0x7fc00000) : s, gi, my_s);
            }
            if (timer) sub[4] += (unsigned long long)(clock64() - t_run);
        }
        chunk_ctr += T * NC;
        tile_ctr += T;
        __syncthreads();
#undef TP_WAIT
    }
};
