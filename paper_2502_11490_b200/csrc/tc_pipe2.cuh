// Warp-specialised tcgen05 scoring pipeline for ONE 256-thread unit of the duo kernel
// (search_duo.cuh: a 512-thread CTA runs two independent units, each with its own queries,
// barriers and pipeline, sharing the weight operands in shared memory and one TMEM
// allocation).  Same arithmetic as tc_pipe.cuh (split-bf16 "bf16x3": hi.[W_hi; W_lo] as one
// N=128 MMA + lo.W_hi per k-step, layer-1 A operand in TMEM via the ".ts" form), with the
// roles of a unit:
//   warps 0-3  epilogue (one group; warp w reads TMEM lanes 32*(w&3)..: one pair row per thread)
//   warp 4     tcgen05.mma issuer (converged warp, elect.sync issues)
//   warps 5-7  TMA loaders: per 64-wide K chunk of a 128-pair tile, 64 tile::gather4 ops
//              (32 four-row groups x hi/lo halves, 128-byte swizzled rows) over 96 lanes
// Buffers per unit: S = 2 stages of one K chunk of the A operand (hi + lo, 32 KB each) in
// shared memory; TMEM window of 256 columns: D0 double-buffered [0,64) / [64,128) (layer 0:
// hi.W_hi + hi.W_lo + lo.W_hi accumulated in one fp32 accumulator), D1 [128,192) (layer 1),
// A1 [192,256) (relu(layer 0) as bf16 hi|lo pairs).  With two D0 buffers the issuer runs
// layer 0 of tile t+1 while the epilogue still works on tile t, so a stage is released as
// soon as its MMAs retire and the next gathers start one epilogue earlier.
// Hand-offs (mbarriers): full[s] (TMA tx) -> issuer, empty[s] commit -> loaders,
// d0full[b] commit -> E, d0empty[b] E -> issuer, a1full E -> issuer, d1full commit -> E.
// The single epilogue group serialises A1 / D1 reuse by program order.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc_scorer.cuh"

template <int D_H, int Z>
struct TcPipe2 {
    static constexpr int H = 64, TM = 128, KC = 64, NC = D_H / KC, S = 2;
    static constexpr int NT = 256, NE = 128, ISSUER_WARP = 4, L_WARP0 = 5, NLW = 3;
    static constexpr int NOPS = 2 * TM / 4;  // TMA gather4 ops per K chunk (hi + lo)
    // shared (both units) weight operands, at the CTA carve base
    static constexpr int OFF_B0H = 0;
    static constexpr int OFF_B0L = OFF_B0H + H * D_H * 2;
    static constexpr int OFF_B1H = OFF_B0L + H * D_H * 2;
    static constexpr int OFF_B1L = OFF_B1H + H * H * 2;
    static constexpr int B_BYTES = OFF_B1L + H * H * 2;
    // per-unit block (1024-aligned: SWIZZLE_128B stages)
    static constexpr int CH_BYTES = TM * KC * 2;                // one hi or lo chunk: 16 KB
    static constexpr int OFF_A = 0;                             // S chunk stages (hi, lo)
    static constexpr int A_REGION = S * 2 * CH_BYTES;           // 64 KB, aliased outside run()
    static constexpr int OFF_BAR = OFF_A + A_REGION;
    enum { FULL0 = 0, EMPTY0 = S, D0FULL = 2 * S, D0EMPTY = 2 * S + 2, A1FULL = 2 * S + 4, D1FULL, NBAR };
    static constexpr int UNIT_BYTES = ((OFF_BAR + NBAR * 8 + 1023) / 1024) * 1024;
    static constexpr uint32_t IDESC = tc::idesc(TM, H);
    static constexpr uint32_t C_D0 = 0, C_D1 = 128, C_A1 = 192, COLS = 256;  // D0 buffer b at 64 b

    static __device__ __forceinline__ uint64_t *bar(unsigned char *u, int i) {
        return reinterpret_cast<uint64_t *>(u + OFF_BAR) + i;
    }

    // lt: thread index inside the unit
    static __device__ void init_barriers(unsigned char *u, int lt) {
        if (lt == 0) {
            for (int s = 0; s < S; ++s) {
                tc::mbar_init(bar(u, FULL0 + s), NOPS);
                tc::mbar_init(bar(u, EMPTY0 + s), 1);
            }
            for (int b = 0; b < 2; ++b) {
                tc::mbar_init(bar(u, D0FULL + b), 1);
                tc::mbar_init(bar(u, D0EMPTY + b), NE);
            }
            tc::mbar_init(bar(u, A1FULL), NE);
            tc::mbar_init(bar(u, D1FULL), 1);
        }
    }

    // Score pairs [0, n) of this unit: item slot slots[i], pair tag gis[i] (query << 16 |
    // searcher).  Every epilogue thread calls on_score(i, valid, score, gi, slot, rank) per row
    // (all 32 lanes of its warp together).  sm: CTA carve base (weights); u: this unit's
    // block; misc: U [G][64] (user half + b0), b1[64], W2[Z][64], b2[4], att[4], w_eff[64],
    // c0, hlim (shared memory); tmem: this unit's TMEM window; chunk_ctr / tile_ctr: unit-lifetime counters;
    // sync(): the unit's barrier.
    template <class OnScore, class Sync>
    static __device__ __forceinline__ void run(unsigned char *sm, unsigned char *u, const float *U,
                                               const float *b1, const float *W2, const float *b2,
                                               const float *att, uint32_t tmem, const DevItems &it,
                                               const DevGraph &g, const int32_t *slots, const int32_t *gis,
                                               int n, uint32_t &chunk_ctr, uint32_t &tile_ctr, int lt,
                                               OnScore on_score, Sync sync, const void *tmap,
                                               unsigned long long *tmr = nullptr) {
        // tmr (GMPGR_PHASE_TIMING, unit 0): [0] epilogue layer-0 work, [1] layer-1 work,
        // [2] D0FULL wait, [3] D1FULL wait, [4] epilogue total, [5] issuer idle polls,
        // [6] issuer issuing, [7] loader EMPTY wait (cycles of one thread per role)
        const int warp = lt >> 5, lane = lt & 31;
#ifdef GMPGR_PIPE_TIMERS
        const bool timed = tmr && lane == 0;
#else
        constexpr bool timed = false;  // role timers compiled out (registers): -DGMPGR_PIPE_TIMERS
        (void)tmr;
#endif
        auto clk = [&]() { return timed ? clock64() : 0ll; };
        const int T = (n + TM - 1) / TM;
        if (T == 0) return;
        // the A stages alias generic-proxy buffers outside run(): order those accesses before
        // the TMA (async-proxy) writes into them
        tc::fence_async_smem();
        sync();
        if (warp >= L_WARP0) {
            const int lw = warp - L_WARP0, o = lane * NLW + lw;
            if (o < NOPS) {
                const int grp = o >> 1, half = o & 1;
                auto rows_of = [&](int t, int (&dst)[4]) {
                    const int base = t * TM, nv = t < T ? min(TM, n - base) : 0;
                    int32_t sl[4];
                    if (4 * grp + 3 < nv) {  // whole group: one 16-byte load (lists are 16-byte aligned)
                        const int4 v = *reinterpret_cast<const int4 *>(slots + base + 4 * grp);
                        sl[0] = v.x; sl[1] = v.y; sl[2] = v.z; sl[3] = v.w;
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) sl[j] = 4 * grp + j < nv ? slots[base + 4 * grp + j] : -1;
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        dst[j] = sl[j] < 0 ? 0 : (it.hl_by_slot ? (int)sl[j] : (int)slot_row(g, sl[j]));
                    // the tile after: its slot ids into L2 now (the list may have left L2 since expand)
                    if (t + 1 < T && (grp & 7) == 0 && half == 0)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(slots + base + TM + 4 * grp));
                };
                int nx[4];
                rows_of(0, nx);
                for (int t = 0; t < T; ++t) {
                    int cur[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) cur[j] = nx[j];
                    if (t + 1 < T) rows_of(t + 1, nx);
#pragma unroll
                    for (int kc = 0; kc < NC; ++kc) {
                        const uint32_t qg = chunk_ctr + t * NC + kc, s = qg % S, r = qg / S;
                        if (r >= 1) {
                            const long long c0 = clk();
                            // suspended, not spinning: the epilogue warps share these SMSPs
                            // poll with a back-off: the loaders' spinning would take issue slots
                            // from the epilogue warps on the same SMSPs
                            while (!tc::mbar_test(bar(u, EMPTY0 + s), (r - 1) & 1u)) __nanosleep(64);
                            if (timed && lw == 0) tmr[7] += clk() - c0;
                        }
                        tc::mbar_arrive_expect_tx(bar(u, FULL0 + s), 512);
                        tc::tma_gather4(tc::smem_u32(u + OFF_A + s * 2 * CH_BYTES) + half * CH_BYTES + grp * 512,
                                        tmap, half * D_H + kc * KC, cur[0], cur[1], cur[2], cur[3],
                                        bar(u, FULL0 + s));
                    }
                }
            }
        } else if (warp == ISSUER_WARP) {
            constexpr unsigned FULLM = 0xffffffffu;
            const uint32_t bH0 = tc::smem_u32(sm + OFF_B0H), bL0 = tc::smem_u32(sm + OFF_B0L);
            const uint32_t bH1 = tc::smem_u32(sm + OFF_B1H), bL1 = tc::smem_u32(sm + OFF_B1L);
            auto ready = [&](int b, uint32_t par) {
                return __shfl_sync(FULLM, lane == 0 ? (int)tc::mbar_test(bar(u, b), par) : 0, 0) != 0;
            };
            int l0t = 0, l0k = 0, l1t = 0;
            long long c_last = clk();
            auto acct = [&](int slot) {
                if (timed) { const long long c = clock64(); tmr[slot] += c - c_last; c_last = c; }
            };
            while (l1t < T) {
                if (l1t < l0t) {  // layer 1 of an earlier tile as soon as its A1 is in TMEM
                    const uint32_t tg = tile_ctr + l1t;
                    if (ready(A1FULL, tg & 1u)) {
                        tc::fence_after();
                        const uint32_t a1 = tmem + C_A1, d1 = tmem + C_D1;
#pragma unroll
                        for (int k = 0; k < H / 16; ++k) {
                            const uint64_t bh = tc::desc(bH1 + k * 256, H), bl = tc::desc(bL1 + k * 256, H);
                            tc::mma_ts_w(d1, a1 + k * 8, bh, IDESC, k ? 1u : 0u);       // hi . hi
                            tc::mma_ts_w(d1, a1 + k * 8, bl, IDESC, 1u);                // hi . lo
                            tc::mma_ts_w(d1, a1 + 32 + k * 8, bh, IDESC, 1u);           // lo . hi
                        }
                        tc::commit_w(bar(u, D1FULL));
                        ++l1t;
                        acct(6);
                        continue;
                    }
                }
                // a pending layer 1 goes first: the next tile's layer 0 starts only once every
                // earlier layer 1 is issued, so the epilogue's layer-1 round trip never queues
                // behind 24 layer-0 MMAs (those then run under the epilogue's layer-1 work)
                if (l0t < T && !(l1t < l0t && l0k == 0)) {
                    const uint32_t tg = tile_ctr + l0t, b = tg & 1u, use = tg >> 1;
                    const uint32_t qg = chunk_ctr + l0t * NC + l0k, s = qg % S, r = qg / S;
                    // D0 buffer b must have been read by the epilogue (two tiles back)
                    if ((l0k != 0 || use == 0 || ready(D0EMPTY + b, (use - 1) & 1u)) && ready(FULL0 + s, r & 1u)) {
                        tc::fence_async_smem();
                        tc::fence_after();
                        const uint32_t d0 = tmem + C_D0 + 64 * b;
                        const uint32_t aH = tc::smem_u32(u + OFF_A + s * 2 * CH_BYTES), aL = aH + CH_BYTES;
#pragma unroll
                        for (int k = 0; k < KC / 16; ++k) {
                            const uint64_t ah = tc::desc_sw128(aH + k * 32), al = tc::desc_sw128(aL + k * 32);
                            const uint32_t kb = (l0k * (KC / 16) + k) * 256;
                            const uint64_t bh = tc::desc(bH0 + kb, D_H), bl = tc::desc(bL0 + kb, D_H);
                            tc::mma_w(d0, ah, bh, IDESC, (l0k | k) ? 1u : 0u);  // hi . W_hi
                            tc::mma_w(d0, ah, bl, IDESC, 1u);                // hi . W_lo
                            tc::mma_w(d0, al, bh, IDESC, 1u);                // lo . W_hi
                        }
                        tc::commit_w(bar(u, EMPTY0 + s));
                        if (++l0k == NC) {
                            tc::commit_w(bar(u, D0FULL + b));
                            l0k = 0;
                            ++l0t;
                        }
                        acct(6);
                        continue;
                    }
                }
                __nanosleep(100);  // nothing ready: yield the SMSP to the epilogue warps
                acct(5);
            }
            __syncwarp();
        } else {
            // ================= epilogue: row = TMEM lane
            const int q4 = warp & 3, row = q4 * 32 + lane;
            const uint32_t lanebase = (uint32_t)(q4 * 32) << 16;
            const bool et = timed && warp == 0;  // folds to false unless GMPGR_PIPE_TIMERS
            const long long e_start = et ? clock64() : 0;
            for (int t = 0; t < T; ++t) {
                const uint32_t tg = tile_ctr + t;
                const int base = t * TM, nv = min(TM, n - base);
                const int gi = row < nv ? gis[base + row] : 0, gq = gi >> 16;
                const int32_t my_s = row < nv ? slots[base + row] : 0;
                // the tie-break rank is loaded here, under the tile's MMA waits, not after the heads
                const uint32_t my_rank = slot_rank(g, my_s);
                const float *uq = U + gq * H;
                const uint32_t b = tg & 1u;
                long long c0 = et ? clock64() : 0;
                tc::mbar_wait(bar(u, D0FULL + b), (tg >> 1) & 1u);
                if (et) { const long long c = clock64(); tmr[2] += c - c0; c0 = c; }
                tc::fence_after();
                float h[64];
                {
                    tc::tmem_ld64(tmem + lanebase + C_D0 + 64 * b, h);
                }
                tc::fence_before();
                tc::mbar_arrive(bar(u, D0EMPTY + b));
                const uint32_t a1 = tmem + lanebase + C_A1;
#pragma unroll
                for (int o = 0; o < 64; o += 16) {
                    uint32_t hi[8], lo[8];
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        const float4 uo = *reinterpret_cast<const float4 *>(uq + o + j);
                        float y0, y1, y2, y3;
                        tc::add2(y0, y1, h[o + j], h[o + j + 1], uo.x, uo.y);
                        tc::add2(y2, y3, h[o + j + 2], h[o + j + 3], uo.z, uo.w);
                        y0 = fmaxf(y0, 0.f); y1 = fmaxf(y1, 0.f); y2 = fmaxf(y2, 0.f); y3 = fmaxf(y3, 0.f);
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
                tc::mbar_arrive(bar(u, A1FULL));
                if (et) { const long long c = clock64(); tmr[0] += c - c0; c0 = c; }
                tc::mbar_wait(bar(u, D1FULL), tg & 1u);
                if (et) { const long long c = clock64(); tmr[3] += c - c0; c0 = c; }
                tc::fence_after();
                int hmax_bits;
                {
                    tc::tmem_ld64(tmem + lanebase + C_D1, h);
                    // relu; the integer max of the pre-activation bit patterns is the largest
                    // relu output (negative values have the sign bit set) and catches NaN / +inf
                    int hbits = 0;
#pragma unroll
                    for (int j = 0; j < 64; j += 2) {
                        float x0, x1;
                        tc::add2(x0, x1, h[j], h[j + 1], b1[j], b1[j + 1]);
                        hbits = max(hbits, max(__float_as_int(x0), __float_as_int(x1)));
                        h[j] = fmaxf(x0, 0.f);
                        h[j + 1] = fmaxf(x1, 0.f);
                    }
                    hmax_bits = hbits;
                }
                tc::fence_before();
                // approximate path (reassociated): the exact refinement re-scores every item
                // near a threshold, and the band certificate checks the error at run time.
                // Heads + attention are linear: score = c0 + h . w_eff (w_eff = sum_o att_o W2_o,
                // c0 = sum_o att_o b2_o) whenever no head can overflow (max h < hlim); otherwise
                // the heads are evaluated one by one for the reference's non-finite check.
                float s = 0.f;
                bool bad = false;
                const float *weff = att + 4;  // [64] w_eff, then c0, hlim
                if (hmax_bits < __float_as_int(weff[65])) {
                    const float4 *wv = reinterpret_cast<const float4 *>(weff);
                    float sp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < 64; j += 4) {
                        const float4 w = wv[j / 4];
                        tc::fma2(sp[0], sp[1], h[j], h[j + 1], w.x, w.y);
                        tc::fma2(sp[2], sp[3], h[j + 2], h[j + 3], w.z, w.w);
                    }
                    s = weff[64] + ((sp[0] + sp[1]) + (sp[2] + sp[3]));
                } else {
                    const float4 *W2v = reinterpret_cast<const float4 *>(W2);
                    for (int o = 0; o < Z; ++o) {
                        float zp[4] = {0.f, 0.f, 0.f, 0.f};
                        for (int j = 0; j < 64; j += 4) {
                            const float4 w = W2v[o * (H / 4) + j / 4];
                            zp[0] = fmaf(h[j], w.x, zp[0]);
                            zp[1] = fmaf(h[j + 1], w.y, zp[1]);
                            zp[2] = fmaf(h[j + 2], w.z, zp[2]);
                            zp[3] = fmaf(h[j + 3], w.w, zp[3]);
                        }
                        const float z = b2[o] + ((zp[0] + zp[1]) + (zp[2] + zp[3]));
                        bad |= !isfinite(z) || hmax_bits >= 0x7f800000;
                        s = fmaf(z, att[o], s);
                    }
                }
                on_score(base + row, row < nv, bad ? __int_as_float(0x7fc00000) : s, gi, my_s, my_rank);
                if (et) tmr[1] += clock64() - c0;
            }
            if (et) tmr[4] += clock64() - e_start;
        }
        chunk_ctr += T * NC;
        tile_ctr += T;
        sync();
    }
};
