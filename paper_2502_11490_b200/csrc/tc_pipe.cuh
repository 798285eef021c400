// Warp-specialised tcgen05 scoring pipeline for one hop's fresh (query, item) pairs.
//
// Roles inside a 512-thread CTA:
//   warps 0-3  (E, 128 threads = the 128 TMEM lanes = one pair row each): epilogues
//   warp 4     (lane 0): the single tcgen05.mma issuer
//   warps 5-15 (L, 352 threads): loaders — gather fp32 item rows, split to bf16 hi/lo and
//              write 64-wide K chunks of the A operand (UMMA K-major core-matrix layout)
// Buffers: two A chunk buffers (the loaders fill chunk q+1 while the tensor core reads
// chunk q), two layer-0 accumulators in TMEM (the MMAs of tile t+1 run while E drains tile
// t), one layer-1 operand + accumulator.  Producer/consumer hand-offs are mbarriers:
//   full[b]   loaders -> issuer       empty[b]  tcgen05.commit -> loaders
//   d0full[b] commit -> E             d0empty[b] E (128 arrivals) -> issuer
//   a1full    E -> issuer             d1full    commit -> E
// Phase parities come from kernel-lifetime chunk/tile counters, identical in all threads.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc_scorer.cuh"

template <int D_H, int Z, int G>
struct TcPipe {
    static constexpr int H = 64, TM = 128, KC = 64, NC = D_H / KC;
    static constexpr int NT = 512, NE = 128, ISSUER_WARP = 4, L_WARP0 = 5, NL = NT - 32 * L_WARP0;
    // byte offsets
    static constexpr int OFF_B0H = 0;
    static constexpr int OFF_B0L = OFF_B0H + H * D_H * 2;
    static constexpr int OFF_B1H = OFF_B0L + H * D_H * 2;
    static constexpr int OFF_B1L = OFF_B1H + H * H * 2;
    static constexpr int OFF_A = OFF_B1L + H * H * 2;          // 2 chunk buffers (hi, lo) + A1
    static constexpr int CH_BYTES = TM * KC * 2;                // one hi or lo chunk: 16 KB
    static constexpr int OFF_A1H = OFF_A + 4 * CH_BYTES;
    static constexpr int OFF_A1L = OFF_A1H + TM * H * 2;
    static constexpr int A_REGION = 4 * CH_BYTES + 2 * TM * H * 2; // 96 KB (aliased by exact buffers)
    static constexpr int OFF_U = OFF_A + A_REGION;              // [G][64] user half + b0
    static constexpr int OFF_B1 = OFF_U + G * H * 4;
    static constexpr int OFF_W2 = OFF_B1 + H * 4;               // [Z][64]
    static constexpr int OFF_B2 = OFF_W2 + Z * H * 4;
    static constexpr int OFF_ATT = OFF_B2 + 16;
    static constexpr int OFF_BAR = (OFF_ATT + 16 + 15) & ~15;   // 10 mbarriers
    static constexpr int OFF_TMEM = OFF_BAR + 10 * 8;
    static constexpr int BYTES = (OFF_TMEM + 16 + 15) & ~15;
    static constexpr uint32_t IDESC = tc::idesc(TM, H);
    static constexpr uint32_t TMEM_COLS = 256;                  // D0[0], D0[1], D1

    static __device__ __forceinline__ uint64_t *bar(unsigned char *sm, int i) {
        return reinterpret_cast<uint64_t *>(sm + OFF_BAR) + i;
    }
    // barrier indices
    enum { FULL0 = 0, EMPTY0 = 2, D0FULL0 = 4, D0EMPTY0 = 6, A1FULL = 8, D1FULL = 9 };

    static __device__ void init_barriers(unsigned char *sm) {
        if (threadIdx.x == 0) {
            for (int b = 0; b < 2; ++b) {
                tc::mbar_init(bar(sm, FULL0 + b), 1);
                tc::mbar_init(bar(sm, EMPTY0 + b), 1);
                tc::mbar_init(bar(sm, D0FULL0 + b), 1);
                tc::mbar_init(bar(sm, D0EMPTY0 + b), NE);
            }
            tc::mbar_init(bar(sm, A1FULL), 1);
            tc::mbar_init(bar(sm, D1FULL), 1);
        }
    }
    static __device__ __forceinline__ void arrive(uint64_t *b) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(b)) : "memory");
    }

    // Score pairs [0, n) (item slot slots[i], query slot gq_of(i)); for every valid row E
    // calls on_score(i, score).  chunk_ctr / tile_ctr: kernel-lifetime counters (all threads).
    template <class OnScore>
    static __device__ __forceinline__ void run(unsigned char *sm, uint32_t tmem, const DevItems &it,
                                               const DevGraph &g, const int32_t *slots, const int32_t *gis, int n,
                                               uint32_t &chunk_ctr, uint32_t &tile_ctr,
                                               OnScore on_score, unsigned long long *sub = nullptr) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        // role timers (GMPGR_PHASE_TIMING): one writer thread per slot
        //   0 E layer-0 epilogue  1 E layer-1 epilogue  2 E d0full-wait  3 E d1full-wait  4 E total
        //   5 issuer full-wait   6 issuer a1full-wait  7 issuer d0empty-wait
        const long long t_run = sub ? clock64() : 0;
#define TP_WAIT(slot, expr)                                                   \
    do {                                                                      \
        const long long w0_ = sub ? clock64() : 0;                            \
        expr;                                                                 \
        if (sub) sub[slot] += (unsigned long long)(clock64() - w0_);          \
    } while (0)
        const int T = (n + TM - 1) / TM;
        if (T == 0) return;
        if (warp >= L_WARP0) {
            // ================= loaders
            const int lt = tid - 32 * L_WARP0, lw = lt >> 5;
            constexpr int NLW = NL / 32;
            // Each warp owns units un = lw + NLW*i (8 rows x 4 float4, conflict-free
            // core-matrix stores).  All of a tile's loads (every K chunk) are issued before the
            // first empty-wait, so the HBM latency overlaps the tensor core draining the
            // previous tile instead of being paid once per unit.
            constexpr int UPC = TM * 16 / 32, UPW = (UPC + NLW - 1) / NLW;
            for (int t = 0; t < T; ++t) {
                const int base = t * TM, nv = min(TM, n - base);
                const float4 *rp[UPW];
#pragma unroll
                for (int i = 0; i < UPW; ++i) {
                    const int un = lw + NLW * i, r = (un % (TM / 8)) * 8 + (lane & 7);
                    rp[i] = nullptr;
                    if (un < UPC && r < nv)
                        rp[i] = reinterpret_cast<const float4 *>(it.emb + slot_row(g, slots[base + r]) * it.ld) +
                                (un / (TM / 8)) * 4 + (lane >> 3);
                }
                float4 x[NC][UPW];
#pragma unroll
                for (int kc = 0; kc < NC; ++kc)
#pragma unroll
                    for (int i = 0; i < UPW; ++i)
                        if (rp[i]) x[kc][i] = __ldg(rp[i] + kc * 16);
#pragma unroll
                for (int kc = 0; kc < NC; ++kc) {
                    const uint32_t qg = chunk_ctr + t * NC + kc, b = qg & 1u, u = qg >> 1;
                    if (u >= 1) {
                        tc::mbar_wait(bar(sm, EMPTY0 + b), (u - 1) & 1u);
                    }
                    unsigned char *Ah = sm + OFF_A + b * 2 * CH_BYTES, *Al = Ah + CH_BYTES;
#pragma unroll
                    for (int i = 0; i < UPW; ++i) {
                        if (!rp[i]) continue;
                        const int un = lw + NLW * i, r = (un % (TM / 8)) * 8 + (lane & 7),
                                  c = (un / (TM / 8)) * 4 + (lane >> 3);
                        uint2 hi, lo;
                        tc::split4(x[kc][i], hi, lo);
                        const uint32_t off = tc::kmaj_off(r, 4 * c, KC);
                        *reinterpret_cast<uint2 *>(Ah + off) = hi;
                        *reinterpret_cast<uint2 *>(Al + off) = lo;
                    }
                    tc::fence_async_smem();
                    asm volatile("bar.sync 14, %0;" ::"r"(NL) : "memory");
                    if (lt == 0) arrive(bar(sm, FULL0 + b));
                }
            }
        } else if (warp == ISSUER_WARP) {
            // ================= MMA issuer (one thread)
            if (lane == 0) {
                const uint32_t bH0 = tc::smem_u32(sm + OFF_B0H), bL0 = tc::smem_u32(sm + OFF_B0L);
                const uint32_t bH1 = tc::smem_u32(sm + OFF_B1H), bL1 = tc::smem_u32(sm + OFF_B1L);
                const uint32_t a1H = tc::smem_u32(sm + OFF_A1H), a1L = tc::smem_u32(sm + OFF_A1L);
                auto layer1 = [&](int t) {
                    const uint32_t tg = tile_ctr + t;
                    TP_WAIT(6, tc::mbar_wait(bar(sm, A1FULL), tg & 1u));
                    tc::fence_after();
#pragma unroll
                    for (int k = 0; k < H / 16; ++k) {
                        const uint64_t ah = tc::desc(a1H + k * 256, H), al = tc::desc(a1L + k * 256, H);
                        const uint64_t bh = tc::desc(bH1 + k * 256, H), bl = tc::desc(bL1 + k * 256, H);
                        tc::mma(tmem + 128, ah, bh, IDESC, k ? 1u : 0u);
                        tc::mma(tmem + 128, ah, bl, IDESC, 1u);
                        tc::mma(tmem + 128, al, bh, IDESC, 1u);
                    }
                    tc::commit(bar(sm, D1FULL));
                };
                for (int t = 0; t <= T; ++t) {
                    if (t < T) {
                        const uint32_t tg = tile_ctr + t, db = tg & 1u, v = tg >> 1;
                        if (v >= 1) TP_WAIT(7, tc::mbar_wait(bar(sm, D0EMPTY0 + db), (v - 1) & 1u));
                        const uint32_t d0 = tmem + db * 64;
                        for (int kc = 0; kc < NC; ++kc) {
                            const uint32_t qg = chunk_ctr + t * NC + kc, b = qg & 1u, u = qg >> 1;
                            TP_WAIT(5, tc::mbar_wait(bar(sm, FULL0 + b), u & 1u));
                            tc::fence_after();
                            const uint32_t aH = tc::smem_u32(sm + OFF_A + b * 2 * CH_BYTES), aL = aH + CH_BYTES;
#pragma unroll
                            for (int k = 0; k < KC / 16; ++k) {
                                const uint64_t ah = tc::desc(aH + k * 256, KC), al = tc::desc(aL + k * 256, KC);
                                const uint32_t kb = (kc * (KC / 16) + k) * 256;
                                const uint64_t bh = tc::desc(bH0 + kb, D_H), bl = tc::desc(bL0 + kb, D_H);
                                tc::mma(d0, ah, bh, IDESC, (kc | k) ? 1u : 0u);
                                tc::mma(d0, ah, bl, IDESC, 1u);
                                tc::mma(d0, al, bh, IDESC, 1u);
                            }
                            tc::commit(bar(sm, EMPTY0 + b));
                        }
                        tc::commit(bar(sm, D0FULL0 + db));
                    }
                    if (t >= 1) layer1(t - 1);
                }
            }
            __syncwarp();
        } else {
            // ================= epilogue warps: row = TMEM lane
            const int row = tid;  // warps 0..3 -> lanes 0..127
            const uint32_t lanebase = (uint32_t)(warp * 32) << 16;
            const float *Uall = reinterpret_cast<const float *>(sm + OFF_U);
            const float *b1 = reinterpret_cast<const float *>(sm + OFF_B1);
            const float *W2 = reinterpret_cast<const float *>(sm + OFF_W2);
            const float *b2 = reinterpret_cast<const float *>(sm + OFF_B2);
            const float *att = reinterpret_cast<const float *>(sm + OFF_ATT);
            unsigned char *A1h = sm + OFF_A1H, *A1l = sm + OFF_A1L;
            for (int t = 0; t < T; ++t) {
                const uint32_t tg = tile_ctr + t, db = tg & 1u, v = tg >> 1;
                const int base = t * TM, nv = min(TM, n - base);
                // the row's pair (issued before the wait so the L2 latency hides behind it)
                const int gi = row < nv ? gis[base + row] : 0, gq = gi >> 16;
                const int32_t my_s = row < nv ? slots[base + row] : 0;
                const float *u = Uall + gq * H;
                if (row == 0) TP_WAIT(2, tc::mbar_wait(bar(sm, D0FULL0 + db), v & 1u));
                else tc::mbar_wait(bar(sm, D0FULL0 + db), v & 1u);
                tc::fence_after();
                const long long te0 = (sub && row == 0) ? clock64() : 0;
                float h[64];
                {
                    float va[32], vb[32];
                    tc::tmem_ld32(tmem + lanebase + db * 64, va);
                    tc::tmem_ld32(tmem + lanebase + db * 64 + 32, vb);
#pragma unroll
                    for (int j = 0; j < 32; ++j) { h[j] = va[j]; h[32 + j] = vb[j]; }
                }
                tc::fence_before();
                arrive(bar(sm, D0EMPTY0 + db));
#pragma unroll
                for (int o = 0; o < 64; o += 4) {
                    const float4 uo = *reinterpret_cast<const float4 *>(u + o);
                    float4 y = make_float4(fmaxf(h[o] + uo.x, 0.f), fmaxf(h[o + 1] + uo.y, 0.f),
                                           fmaxf(h[o + 2] + uo.z, 0.f), fmaxf(h[o + 3] + uo.w, 0.f));
                    uint2 hi, lo;
                    tc::split4(y, hi, lo);
                    const uint32_t off = tc::kmaj_off(row, o, H);
                    *reinterpret_cast<uint2 *>(A1h + off) = hi;
                    *reinterpret_cast<uint2 *>(A1l + off) = lo;
                }
                tc::fence_async_smem();
                asm volatile("bar.sync 15, %0;" ::"r"(NE) : "memory");
                if (row == 0) arrive(bar(sm, A1FULL));
                if (sub && row == 0) sub[0] += (unsigned long long)(clock64() - te0);
                if (row == 0) TP_WAIT(3, tc::mbar_wait(bar(sm, D1FULL), tg & 1u));
                else tc::mbar_wait(bar(sm, D1FULL), tg & 1u);
                tc::fence_after();
                const long long te1 = (sub && row == 0) ? clock64() : 0;
                {
                    float va[32], vb[32];
                    tc::tmem_ld32(tmem + lanebase + 128, va);
                    tc::tmem_ld32(tmem + lanebase + 128 + 32, vb);
#pragma unroll
                    for (int j = 0; j < 32; ++j) { h[j] = fmaxf(va[j] + b1[j], 0.f); h[32 + j] = fmaxf(vb[j] + b1[32 + j], 0.f); }
                }
                tc::fence_before();
                // approximate path: reassociated (4 partial sums per output) — the exact
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
                if (sub && row == 0) sub[1] += (unsigned long long)(clock64() - te1);
                on_score(base + row, row < nv, bad ? __int_as_float(0x7fc00000) : s, gi, my_s);
            }
            if (sub && row == 0) sub[4] += (unsigned long long)(clock64() - t_run);
        }
        chunk_ctr += T * NC;
        tile_ctr += T;
        __syncthreads();
#undef TP_WAIT
    }
};
