// Multi-query persistent C-HiPANNS kernel: one 512-thread CTA per SM advances G = 4
// queries in lock-step (same layers, same hops), so every phase works on 4 queries'
// frontiers / claims / fresh sets at once — more independent memory traffic in flight,
// fuller scoring tiles, one copy of the weights per SM.  Semantics are exactly those of
// search_kernel.cuh (hop-synchronous c_hipanns, search.py:194-286): each query owns its
// own epoch-stamped tag array, pool and frontier; flattened work lists carry the query
// slot g in the high half of the searcher field (g << 16 | searcher).
//
// MODE 0: exact-fp32 scoring of every claim (64-pair tiles, weights in shared memory).
// MODE 1: tcgen05 split-bf16 scoring of 128-pair tiles + exact re-scoring of the band
//         around every selection threshold (see search_kernel.cuh for the argument).
#pragma once
#include "common.cuh"
#include "mlp_exact.cuh"
#include "search_kernel.cuh"
#include "select.cuh"
#include "tc_scorer.cuh"
#include "tc_pipe.cuh"

// launch shapes: (NT threads, G queries per CTA).  512x4: one CTA per SM with every
// weight resident; 256x2: two CTAs per SM (tensor-core mode), exact weights read through L1.

// Exact fixed-shape MLP on 64-pair tiles whose pairs may belong to different queries
// (per-pair hoisted user half acc0[g]).  Same arithmetic as FixedMlp (bit-exact order).
template <int D_H, int Z, int NW>
struct ExactQ {
    static constexpr int H = 64, NCH0 = D_H / 4, NCHH = H / 4, NCHZ = (Z + 3) / 4;
    static constexpr int LDX0 = NCH0 | 1, LDH = NCHH | 1, LDZ = NCHZ | 1, PT = 4 * NW;
    // float4 offsets of the weight block (same layout as FixedMlp) ...
    static constexpr int OFF_W0 = 0;
    static constexpr int OFF_W1 = OFF_W0 + NCH0 * H;
    static constexpr int OFF_W2 = OFF_W1 + NCHH * H;
    static constexpr int OFF_A = OFF_W2 + NCHH * Z;
    static constexpr int OFF_B0 = OFF_A + NCHZ;
    static constexpr int OFF_B1 = OFF_B0 + H / 4;
    static constexpr int OFF_B2 = OFF_B1 + H / 4;
    static constexpr int W_END = OFF_B2 + NCHZ;
    // ... and of the activation buffers (relative to their own base)
    static constexpr int OFF_X0 = 0;
    static constexpr int OFF_H0 = OFF_X0 + PT * LDX0;
    static constexpr int OFF_H1 = OFF_H0 + PT * LDH;
    static constexpr int OFF_Z = OFF_H1 + PT * LDH;
    static constexpr int OFF_SC = OFF_Z + PT * LDZ;
    static constexpr int OFF_PQ = OFF_SC + PT / 4;
    static constexpr int BUF_END = OFF_PQ + PT / 4;

    template <int NCH, int LDX, bool HAS_INIT>
    static __device__ __forceinline__ void big(const float4 *__restrict__ X,
                                               const float4 *__restrict__ W,
                                               const float *__restrict__ bias,
                                               const float4 *__restrict__ acc0,
                                               const int *__restrict__ pq, float *__restrict__ Y) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
                mac4(a[pp][0], x, w0);
                mac4(a[pp][1], x, w1);
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

    // W: weight block (smem); buf: activation buffers (smem); acc0: [G][64] float4
    static __device__ __forceinline__ void tile(const float4 *W, float4 *buf, const float4 *acc0,
                                                int n_valid, int *nonfinite) {
        const int *pq = reinterpret_cast<const int *>(buf + OFF_PQ);
        big<NCH0, LDX0, true>(buf + OFF_X0, W + OFF_W0, reinterpret_cast<const float *>(W + OFF_B0),
                              acc0, pq, reinterpret_cast<float *>(buf + OFF_H0));
        __syncthreads();
        big<NCHH, LDH, false>(buf + OFF_H0, W + OFF_W1, reinterpret_cast<const float *>(W + OFF_B1),
                              nullptr, pq, reinterpret_cast<float *>(buf + OFF_H1));
        __syncthreads();
        float *zb = reinterpret_cast<float *>(buf + OFF_Z);
        if (threadIdx.x < PT * Z) {
            const int p = threadIdx.x % PT, o = threadIdx.x / PT;
            const float4 *hr = buf + OFF_H1 + p * LDH;
            const float4 *W2 = W + OFF_W2;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NCHH; ++j) mac4(acc, hr[j], W2[j * Z + o]);
            zb[p * LDZ * 4 + o] =
                __fadd_rn(hsum4(acc), reinterpret_cast<const float *>(W + OFF_B2)[o]);
        }
        __syncthreads();
        if (threadIdx.x < PT) {
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
                mac4(acc, make_float4(e[0], e[1], e[2], e[3]), W[OFF_A + j]);
            }
            reinterpret_cast<float *>(buf + OFF_SC)[p] = hsum4(acc);
            if (bad && p < n_valid) atomicOr(nonfinite, 1);
        }
        __syncthreads();
    }
};

// tcgen05 scorer for 512-thread CTAs: 128-pair tiles, per-pair query user half.
template <int D_H, int Z, int NT, int G, int KC_ = D_H>
struct TcQ {
    // layer 0 in D_H / KC K-chunks (KC = D_H: one chunk, A = 128 x D_H hi/lo = 64 KB at
    // d_h 128 -> two MMA round trips per tile; KC = 64 halves the A buffer)
    static constexpr int H = 64, TM = 128, KC = KC_, NKC0 = D_H / KC_;
    static constexpr int NW = NT / 32, CQ = NW / 4, CW = H / CQ; // column groups / width
    static constexpr int OFF_B0H = 0;
    static constexpr int OFF_B0L = OFF_B0H + H * D_H * 2;
    static constexpr int OFF_B1H = OFF_B0L + H * D_H * 2;
    static constexpr int OFF_B1L = OFF_B1H + H * H * 2;
    static constexpr int A_BYTES = 2 * TM * KC * 2;       // A operand (hi, lo): caller-provided
    static constexpr int OFF_U = OFF_B1L + H * H * 2;     // [G][64] f32 user half + b0
    static constexpr int OFF_B1 = OFF_U + G * H * 4;
    static constexpr int OFF_W2 = OFF_B1 + H * 4;         // [Z][64]
    static constexpr int OFF_B2 = OFF_W2 + Z * H * 4;
    static constexpr int OFF_ATT = OFF_B2 + 16;
    static constexpr int OFF_ZP = OFF_ATT + 16;           // [128][CQ][Z]
    static constexpr int OFF_SC = OFF_ZP + TM * CQ * Z * 4;
    static constexpr int OFF_PQ = OFF_SC + TM * 4;        // [128] query slot per row
    static constexpr int OFF_BAR = (OFF_PQ + TM * 4 + 15) & ~15;
    static constexpr int OFF_TMEM = OFF_BAR + 16;
    static constexpr int BYTES = OFF_TMEM + 16;
    static constexpr uint32_t IDESC = tc::idesc(TM, H);

    static __device__ __forceinline__ void tmem_ldw(uint32_t addr, float (&v)[32]) {
        tc::tmem_ld32(addr, v);
    }
    static __device__ __forceinline__ void tmem_ldw(uint32_t addr, float (&v)[16]) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
    }

    // rows: slots[0..nv), query slot per row in PQ (written by the caller)
    static __device__ __forceinline__ void tile(unsigned char *sm, unsigned char *abuf, uint32_t tmem,
                                                uint32_t &phase, const DevItems &it,
                                                const DevGraph &g, const int32_t *slots, int nv,
                                                unsigned long long *sub = nullptr,
                                                const int32_t *next_slots = nullptr, int next_nv = 0) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        long long t_sub = (sub && tid == 0) ? clock64() : 0;
        auto SUB = [&](int i) {
            if (sub && tid == 0) { const long long n_ = clock64(); sub[i] += n_ - t_sub; t_sub = n_; }
        };
        unsigned char *Ah = abuf, *Al = abuf + TM * KC * 2;
        uint64_t *bar = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
        const uint32_t aH = tc::smem_u32(Ah), aL = tc::smem_u32(Al);
        for (int kc = 0; kc < NKC0; ++kc) {
            constexpr int CPR = KC / 4; // float4 per row chunk
            // warp unit = 8 rows x 4 float4: the 8-byte hi/lo stores of a warp then cover
            // two whole 128-byte core-matrix rows -> conflict-free (row-major mapping would
            // put 16 lanes on one bank group); global reads stay 64-byte row segments
            for (int t = tid; t < TM * CPR; t += NT) {
                const int u = t >> 5, l = t & 31;
                const int r = (u % (TM / 8)) * 8 + (l & 7), c = (u / (TM / 8)) * 4 + (l >> 3);
                if (r < nv) {
                    const float4 x = __ldg(reinterpret_cast<const float4 *>(
                                               it.emb + slot_row(g, slots[r]) * it.ld) + kc * CPR + c);
                    uint2 hi, lo;
                    tc::split4(x, hi, lo);
                    const uint32_t off = tc::kmaj_off(r, 4 * c, KC);
                    *reinterpret_cast<uint2 *>(Ah + off) = hi;
                    *reinterpret_cast<uint2 *>(Al + off) = lo;
                }
            }
            tc::fence_async_smem();
            tc::fence_before();
            __syncthreads();
            SUB(0);
            if (tid == 0) {
                tc::fence_after();
                const uint32_t bH = tc::smem_u32(sm + OFF_B0H), bL = tc::smem_u32(sm + OFF_B0L);
#pragma unroll
                for (int k = 0; k < KC / 16; ++k) {
                    const uint64_t ah = tc::desc(aH + k * 256, KC), al = tc::desc(aL + k * 256, KC);
                    const uint32_t kb = (kc * (KC / 16) + k) * 256;
                    const uint64_t bh = tc::desc(bH + kb, D_H), bl = tc::desc(bL + kb, D_H);
                    tc::mma(tmem, ah, bh, IDESC, (kc | k) ? 1u : 0u);
                    tc::mma(tmem, ah, bl, IDESC, 1u);
                    tc::mma(tmem, al, bh, IDESC, 1u);
                }
                tc::commit(bar);
            }
            // while the tensor core works: pull the next tile's rows toward L2
            if (kc == NKC0 - 1 && next_slots) {
                constexpr int LPR = D_H / 32; // 128-byte lines per row
                for (int t = tid; t < next_nv * LPR; t += NT) {
                    const float *rp = it.emb + slot_row(g, next_slots[t / LPR]) * it.ld + (t % LPR) * 32;
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(rp));
                }
            }
            tc::mbar_wait(bar, phase);
            phase ^= 1u;
            tc::fence_after();
            SUB(1);
        }
        const int q4 = warp & 3, cq = warp >> 2, row = q4 * 32 + lane;
        const int gq = reinterpret_cast<const int *>(sm + OFF_PQ)[row];
        const float *u = reinterpret_cast<const float *>(sm + OFF_U) + gq * H;
        {
            float v[CW];
            tmem_ldw(tmem + ((uint32_t)(q4 * 32) << 16) + cq * CW, v);
#pragma unroll
            for (int j = 0; j < CW; j += 4) {
                const int o = cq * CW + j;
                float4 y = make_float4(fmaxf(v[j] + u[o], 0.f), fmaxf(v[j + 1] + u[o + 1], 0.f),
                                       fmaxf(v[j + 2] + u[o + 2], 0.f), fmaxf(v[j + 3] + u[o + 3], 0.f));
                uint2 hi, lo;
                tc::split4(y, hi, lo);
                const uint32_t off = tc::kmaj_off(row, o, H);
                *reinterpret_cast<uint2 *>(Ah + off) = hi;
                *reinterpret_cast<uint2 *>(Al + off) = lo;
            }
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncthreads();
        SUB(2);
        if (tid == 0) {
            tc::fence_after();
            const uint32_t bH = tc::smem_u32(sm + OFF_B1H), bL = tc::smem_u32(sm + OFF_B1L);
#pragma unroll
            for (int k = 0; k < H / 16; ++k) {
                const uint64_t ah = tc::desc(aH + k * 256, H), al = tc::desc(aL + k * 256, H);
                const uint64_t bh = tc::desc(bH + k * 256, H), bl = tc::desc(bL + k * 256, H);
                tc::mma(tmem + 64, ah, bh, IDESC, k ? 1u : 0u);
                tc::mma(tmem + 64, ah, bl, IDESC, 1u);
                tc::mma(tmem + 64, al, bh, IDESC, 1u);
            }
            tc::commit(bar);
        }
        tc::mbar_wait(bar, phase);
        phase ^= 1u;
        tc::fence_after();
        SUB(3);
        {
            float v[CW];
            tmem_ldw(tmem + ((uint32_t)(q4 * 32) << 16) + 64 + cq * CW, v);
            const float *b1 = reinterpret_cast<const float *>(sm + OFF_B1);
            const float *W2 = reinterpret_cast<const float *>(sm + OFF_W2);
            float zp[Z];
#pragma unroll
            for (int o = 0; o < Z; ++o) zp[o] = 0.f;
#pragma unroll
            for (int j = 0; j < CW; ++j) {
                const float h = fmaxf(v[j] + b1[cq * CW + j], 0.f);
#pragma unroll
                for (int o = 0; o < Z; ++o) zp[o] = fmaf(h, W2[o * H + cq * CW + j], zp[o]);
            }
            float *ZP = reinterpret_cast<float *>(sm + OFF_ZP);
#pragma unroll
            for (int o = 0; o < Z; ++o) ZP[(row * CQ + cq) * Z + o] = zp[o];
        }
        tc::fence_before();
        __syncthreads();
        if (tid < TM) {
            const float *ZP = reinterpret_cast<const float *>(sm + OFF_ZP);
            const float *b2 = reinterpret_cast<const float *>(sm + OFF_B2);
            const float *att = reinterpret_cast<const float *>(sm + OFF_ATT);
            float s = 0.f;
#pragma unroll
            for (int o = 0; o < Z; ++o) {
                float z = b2[o];
#pragma unroll
                for (int c = 0; c < CQ; ++c) z += ZP[(tid * CQ + c) * Z + o];
                s = fmaf(z, att[o], s);
            }
            reinterpret_cast<float *>(sm + OFF_SC)[tid] = s;
        }
        __syncthreads();
        SUB(4);
    }
};

template <int G>
struct MqState;

struct MqQuery {
    int q;             // global query index, -1 if this slot is idle
    uint32_t epoch;
    int nPool, nPool2, pool_cur, f_off, f_cnt;
    uint64_t poolT;
    int besthop;
    // 32-bit counters: shared-memory 32-bit atomics are native (64-bit ones would CAS-loop
    // under the 128-way contention of a tile epilogue)
    int per_layer[GR_MAX_LAYERS];
    int rows, nbrs;
};

// one atomic per group of lanes sharing the same query slot (whole warp must call)
__device__ __forceinline__ void warp_count(int *addr, int gq, int inc, bool active) {
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    const unsigned peers = __match_any_sync(act, gq);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(addr, inc * __popc(peers));
}

// Warp-aggregated slot reservation: lanes with the same gq share one shared-memory atomic
// (per-lane atomics on one query's pool counter serialise).  All 32 lanes must call.
// Returns the lane's index, or -1 when !active.
template <class CtrOf>
__device__ __forceinline__ int warp_append(int gq, bool active, CtrOf ctr_of) {
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (!active) return -1;
    const int lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(act, gq);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(ctr_of(gq), __popc(peers));
    base = __shfl_sync(peers, base, leader);
    return base + __popc(peers & ((1u << lane) - 1u));
}

template <int G>
struct MqState {
    MqQuery qs[G];
    int nF, nS, nFresh, nFn, nRq, f_cur, base, wrap[G];
    uint32_t bcast[4];
};

// Shared-memory plan (host computes the same offsets): [model block][exact buffers]
// [hist NW x 256][sort G x sortcap keys+vals][seg cnt/off/fn: 3 x G*kp][acc0 G x 64 float4]
template <int DH, int ZZ, int MODE, int NT, int G, int KC, bool PIPE>
__global__ void __launch_bounds__(NT, (NT >= 512 ? 1 : 2)) hipanns_mq_kernel(const __grid_constant__ SearchArgs a) {
    constexpr int NW = NT / 32, GT = NT / G;
    // exact weight block in smem, else the global image (the pipelined scorer needs the room)
    constexpr bool W_SMEM = (NT >= 512) && !(MODE == 1 && PIPE);
    using EX = ExactQ<DH, ZZ, NW>;
    using TC = TcQ<DH, ZZ, NT, G, KC>;
    using TP = TcPipe<DH, ZZ, G>;
    constexpr int OFF_U = PIPE ? TP::OFF_U : TC::OFF_U;
    constexpr int OFF_B1 = PIPE ? TP::OFF_B1 : TC::OFF_B1;
    constexpr int OFF_W2 = PIPE ? TP::OFF_W2 : TC::OFF_W2;
    constexpr int OFF_B2 = PIPE ? TP::OFF_B2 : TC::OFF_B2;
    constexpr int OFF_ATT = PIPE ? TP::OFF_ATT : TC::OFF_ATT;
    constexpr int OFF_TMEMP = PIPE ? TP::OFF_TMEM : TC::OFF_TMEM;
    constexpr uint32_t TMEM_COLS = PIPE ? TP::TMEM_COLS : 128;
    uint32_t chunk_ctr = 0, tile_ctr = 0;  // pipelined scorer barrier phases
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // the pipelined scorer's SWIZZLE_128B A stages need 1024-byte aligned shared addresses; the
    // dynamic window is not 1024-aligned next to the static state, so the host plan reserves
    // 1024 bytes of slack (plan_mq) and the carve starts at the next 1024-byte boundary
    unsigned char *const smem = PIPE ? smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u) : smem_raw;
    __shared__ MqState<G> st;
    __shared__ unsigned long long ph_acc[16];
    __shared__ unsigned bc[2];  // tensor-core band certificate (band_record)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    long long ph_t0 = 0;
    if (tid < 16) ph_acc[tid] = 0;
    if (tid < 2) bc[tid] = 0u;
#define GR_PH(i)                                                          \
    do {                                                                  \
        if (a.phase_cycles && tid == 0) {                                 \
            const long long now_ = clock64();                             \
            ph_acc[i] += (unsigned long long)(now_ - ph_t0);              \
            ph_t0 = now_;                                                 \
        }                                                                 \
    } while (0)
    const DevModel &M = a.M;
    const DevGraph &g = a.g;
    // ---- shared memory carve (offsets from the host plan)
    const float4 *sW = W_SMEM ? reinterpret_cast<const float4 *>(smem + a.off_w0)
                              : reinterpret_cast<const float4 *>(M.exBlock); // exact weights
    float4 *sBuf = reinterpret_cast<float4 *>(smem + a.off_x0);    // exact activation buffers
    float4 *sAcc0 = reinterpret_cast<float4 *>(smem + a.off_acc0); // [G][64]
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem + a.off_hist);
    uint64_t *sortk = reinterpret_cast<uint64_t *>(smem + a.off_sortk); // [G][sortcap]
    int32_t *sortv = reinterpret_cast<int32_t *>(smem + a.off_sortv);
    int32_t *seg_cnt = reinterpret_cast<int32_t *>(smem + a.off_kp);    // [G*kp]
    const int NSEG = G * a.kp;
    int32_t *seg_off = seg_cnt + NSEG;
    int32_t *fn_off = seg_off + NSEG;
    // ---- exact weights (both modes: the tensor-core mode re-scores near thresholds)
    if constexpr (W_SMEM) {
        float4 *sWm = reinterpret_cast<float4 *>(smem + a.off_w0);
        const float4 *src = reinterpret_cast<const float4 *>(M.exBlock);
        for (int t = tid; t < EX::W_END; t += NT) sWm[t] = src[t];
    }
    uint32_t tmem = 0, tphase = 0;
    unsigned char *tcs = smem + a.off_A; // tensor-core block (MODE 1)
    if constexpr (MODE == 1) {
        const uint4 *src = reinterpret_cast<const uint4 *>(M.tcB);
        uint4 *dst = reinterpret_cast<uint4 *>(tcs + TC::OFF_B0H);  // same B layout in TC and TP
        for (int t = tid; t < (TC::OFF_U - TC::OFF_B0H) / 16; t += NT) dst[t] = src[t];
        float *b1 = reinterpret_cast<float *>(tcs + OFF_B1);
        for (int t = tid; t < 64; t += NT) b1[t] = M.tcMisc[t];
        float *w2 = reinterpret_cast<float *>(tcs + OFF_W2);
        for (int t = tid; t < 64 * ZZ; t += NT) w2[t] = M.tcMisc[64 + t];
        if (tid < 4) {
            reinterpret_cast<float *>(tcs + OFF_B2)[tid] = M.tcMisc[64 + 64 * ZZ + tid];
            reinterpret_cast<float *>(tcs + OFF_ATT)[tid] = M.tcMisc[68 + 64 * ZZ + tid];
        }
        uint32_t *tptr = reinterpret_cast<uint32_t *>(tcs + OFF_TMEMP);
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             tc::smem_u32(tptr)), "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        if constexpr (PIPE) {
            // SWIZZLE_128B stages need 1024-byte aligned shared addresses
            if (a.tma && (tc::smem_u32(tcs + TP::OFF_A) & 1023u)) __trap();
            TP::init_barriers(tcs, a.tma != 0);
        }
        else if (tid == 0) tc::mbar_init(reinterpret_cast<uint64_t *>(tcs + TC::OFF_BAR), 1);
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        tmem = *tptr;
    }
    // ---- scratch: CTA-level flattened lists (capacities x G), per-query tags and pools
    const int64_t cta = blockIdx.x;
    const int64_t capF = a.capF, capS = a.capS, capP = a.capP; // already multiplied by G for lists
    int32_t *fslot[2] = {a.f_slot + cta * 2 * capF, a.f_slot + cta * 2 * capF + capF};
    int32_t *fsrch[2] = {a.f_srch + cta * 2 * capF, a.f_srch + cta * 2 * capF + capF};
    int32_t *surv_v = a.surv_v + cta * capS, *surv_i = a.surv_i + cta * capS;
    int32_t *fr_v = a.fr_v + cta * capS, *fr_i = a.fr_i + cta * capS;
    uint64_t *fr_key = a.fr_key + cta * capS;
    int32_t *seg_v = a.seg_v + cta * capS;
    uint64_t *seg_key = a.seg_key + cta * capS;
    int32_t *rq = surv_v;     // re-score requests (index | target bit 31)
    int32_t *seg_ex = fr_i;   // after the scatter
    auto tags_of = [&](int gq) { return a.tags + (cta * G + gq) * g.n; };
    auto pkey = [&](int gq, int c) { return a.pool_key + ((cta * G + gq) * 2 + c) * capP; };
    auto pslot = [&](int gq, int c) { return a.pool_slot + ((cta * G + gq) * 2 + c) * capP; };
    auto pmeta = [&](int gq, int c) { return a.pool_meta + ((cta * G + gq) * 2 + c) * capP; };
    auto band_of = [&](float T) { return a.band_rel * fabsf(T) + a.band_abs; };
    const int top = g.n_layers - 1, nst = 5 + g.n_layers, d_h = DH;

    for (;;) {
        __syncthreads();
        if (tid == 0) st.base = atomicAdd(a.queue, G);
        __syncthreads();
        if (st.base >= a.Q) break;
        if (tid < G) {
            MqQuery &Q = st.qs[tid];
            Q.q = st.base + tid < a.Q ? st.base + tid : -1;
            st.wrap[tid] = 0;
            if (Q.q >= 0) Q.epoch = next_epoch(a.epochs, cta * G + tid, tags_of(tid), g.n, &st.wrap[tid]);
            Q.nPool = 0; Q.pool_cur = 0; Q.poolT = 0ull; Q.besthop = -1;
            for (int l = 0; l < GR_MAX_LAYERS; ++l) Q.per_layer[l] = 0;
            Q.rows = 0; Q.nbrs = 0;
        }
        if (tid == 0) { st.f_cur = 0; }
        __syncthreads();
        for (int gq = 0; gq < G; ++gq)
            if (st.wrap[gq]) {  // epoch wrapped: clear that slot's tags
                uint32_t *tg = tags_of(gq);
                for (int64_t i = tid; i < g.n; i += NT) tg[i] = 0u;
                __syncthreads();
            }
        if (tid == 0) ph_t0 = clock64();
        // ---- hoisted user halves (exact acc0; tensor-core u = user half + b0)
        for (int t = tid; t < G * 64; t += NT) {
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
            if constexpr (MODE == 1)
                reinterpret_cast<float *>(tcs + OFF_U)[gq * 64 + o] = __fadd_rn(hsum4(acc), M.b[0][o]);
        }

        // ================= helpers
        // score fresh (fr_v, fr_i) [0, n): keys; per-query per-layer counts; pool append
        auto score_fresh = [&](int n, int layer, int hop) {
            if constexpr (MODE == 1 && PIPE) {
                TP::run(tcs, tmem, a.it, g, fr_v, fr_i, n, chunk_ctr, tile_ctr,
                        [&](int i, bool valid, float v, int gi, int32_t s) {
                            const int gq = gi >> 16;
                            warp_count(&st.qs[gq].per_layer[layer], gq, 1, valid);
                            if (valid && !isfinite(v)) atomicOr(a.nonfinite, 1);
                            const uint64_t key = make_key(v, slot_rank(g, s));
                            if (valid) fr_key[i] = key;
                            MqQuery &Q = st.qs[gq];
                            const float Ts = orderable_f32((uint32_t)(Q.poolT >> 32));
                            const int idx = warp_append(gq, valid && (!Q.poolT || v >= Ts - band_of(Ts)),
                                                        [&](int q) { return &st.qs[q].nPool; });
                            if (idx >= 0) {
                                pkey(gq, Q.pool_cur)[idx] = key;
                                pslot(gq, Q.pool_cur)[idx] = s;
                                pmeta(gq, Q.pool_cur)[idx] = hop << 1;
                            }
                        }, a.phase_cycles ? ph_acc + 8 : nullptr, a.tma ? &a.hl_map : nullptr, a.tma == 2);
                if (tid == 0) atomicAdd(a.counters + 1, (unsigned long long)n);
                __syncthreads();
            } else if constexpr (MODE == 1) {
                const float *sc = reinterpret_cast<const float *>(tcs + TC::OFF_SC);
                int *pq = reinterpret_cast<int *>(tcs + TC::OFF_PQ);
                for (int base = 0; base < n; base += TC::TM) {
                    const int nv = min(TC::TM, n - base);
                    int32_t my_s = 0;
                    int my_gi = 0;
                    if (tid < nv) { my_s = fr_v[base + tid]; my_gi = fr_i[base + tid]; }
                    if (tid < TC::TM) pq[tid] = my_gi >> 16;  // read after the tile's first barrier
                    const int nb = base + TC::TM;
                    TC::tile(tcs, reinterpret_cast<unsigned char *>(sBuf), tmem, tphase, a.it, g,
                             fr_v + base, nv, a.phase_cycles ? ph_acc + 8 : nullptr,
                             nb < n ? fr_v + nb : nullptr, nb < n ? min(TC::TM, n - nb) : 0);
                    if (tid < 32 * ((nv + 31) / 32)) {
                        const bool valid = tid < nv;
                        const int gq = my_gi >> 16;
                        warp_count(&st.qs[gq].per_layer[layer], gq, 1, valid);
                        const int32_t s = my_s;
                        const float v = valid ? sc[tid] : 0.f;
                        if (valid && !isfinite(v)) atomicOr(a.nonfinite, 1);
                        const uint64_t key = make_key(v, slot_rank(g, s));
                        if (valid) fr_key[base + tid] = key;
                        MqQuery &Q = st.qs[gq];
                        const float Ts = orderable_f32((uint32_t)(Q.poolT >> 32));
                        const int idx = warp_append(gq, valid && (!Q.poolT || v >= Ts - band_of(Ts)),
                                                    [&](int q) { return &st.qs[q].nPool; });
                        if (idx >= 0) {
                            pkey(gq, Q.pool_cur)[idx] = key;
                            pslot(gq, Q.pool_cur)[idx] = s;
                            pmeta(gq, Q.pool_cur)[idx] = hop << 1;
                        }
                    }
                    __syncthreads();
                }
                if (tid == 0) atomicAdd(a.counters + 1, (unsigned long long)n);
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
                    __syncthreads();
                    EX::tile(sW, sBuf, sAcc0, nv, a.nonfinite);
                    if (tid < 32 * ((nv + 31) / 32)) {
                        const bool valid = tid < nv;
                        const int gq = valid ? (fr_i[base + tid] >> 16) : 0;
                        warp_count(&st.qs[gq].per_layer[layer], gq, 1, valid);
                        const int32_t s = valid ? fr_v[base + tid] : 0;
                        const uint64_t key = make_key(valid ? sc[tid] : 0.f, slot_rank(g, s));
                        if (valid) fr_key[base + tid] = key;
                        MqQuery &Q = st.qs[gq];
                        const int idx = warp_append(gq, valid && key > Q.poolT,
                                                    [&](int q) { return &st.qs[q].nPool; });
                        if (idx >= 0) {
                            pkey(gq, Q.pool_cur)[idx] = key;
                            pslot(gq, Q.pool_cur)[idx] = s;
                            pmeta(gq, Q.pool_cur)[idx] = (hop << 1) | 1;
                        }
                    }
                    __syncthreads();
                }
            }
        };
        // exact re-score of rq[0..n): entry = (gq << 24 | idx) with idx into that query's
        // current pool (pool=1) or into the seg arrays (pool=0, gq from the seg entry)
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
                    __syncthreads();
                    EX::tile(sW, sBuf, sAcc0, nv, a.nonfinite);
                    if (tid < nv) {
                        const int e = rq[base + tid];
                        const int gq = e >> 24, idx = e & 0xFFFFFF;
                        band_record(bc, pool ? pkey(gq, st.qs[gq].pool_cur)[idx] : seg_key[idx], sc[tid],
                                    a.band_rel, a.band_abs);
                        if (pool) {
                            const int c = st.qs[gq].pool_cur;
                            pkey(gq, c)[idx] = make_key(sc[tid], slot_rank(g, pslot(gq, c)[idx]));
                            pmeta(gq, c)[idx] |= 1;
                        } else {
                            seg_key[idx] = make_key(sc[tid], slot_rank(g, seg_v[idx]));
                            seg_ex[idx] = 1;
                        }
                    }
                    __syncthreads();
                }
                if (tid == 0 && n) atomicAdd(a.counters, (unsigned long long)n);
            }
        };
        // collect non-exact pool entries of every query with pred(gq, score) into rq
        auto collect_pool = [&](auto pred) {
            if (tid == 0) st.nRq = 0;
            __syncthreads();
            for (int gq = 0; gq < G; ++gq) {
                const MqQuery &Q = st.qs[gq];
                const int np = Q.nPool;
                const uint64_t *pk = pkey(gq, Q.pool_cur);
                const int32_t *pm = pmeta(gq, Q.pool_cur);
                for (int i0 = 0; i0 < np; i0 += NT) {
                    const int i = i0 + tid;
                    bool ok = i < np && !(pm[i] & 1) && pred(gq, orderable_f32((uint32_t)(pk[i] >> 32)));
                    warp_append2(ok, (gq << 24) | i, 0, &st.nRq, rq, surv_i);
                }
            }
            __syncthreads();
            return st.nRq;
        };
        // per-query pool compaction to top-k (warp gq), tensor mode refines the band first
        auto compact_pools = [&]() {
            if constexpr (MODE == 1) {
                __shared__ float thr[G];
                if (warp < G) {
                    const MqQuery &Q = st.qs[warp];
                    float Ts = INFINITY;
                    if (Q.nPool > a.k) {
                        const uint64_t Ta = warp_select_threshold(pkey(warp, Q.pool_cur), Q.nPool, a.k, hist + warp * 256);
                        Ts = orderable_f32((uint32_t)(Ta >> 32));
                    }
                    if (lane == 0) thr[warp] = Ts;
                }
                __syncthreads();
                const int n = collect_pool([&](int gq, float v) {
                    return isfinite(thr[gq]) && fabsf(v - thr[gq]) <= band_of(thr[gq]);
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
            __syncthreads();
        };
        // owner resolution: survivors whose tag still carries their code own the node
        auto resolve = [&](int nS) {
            for (int t0 = 0; t0 < nS; t0 += NT) {
                const int t = t0 + tid;
                bool ok = false;
                int32_t v = 0, gi = 0;
                if (t < nS) {
                    v = surv_v[t];
                    gi = surv_i[t];
                    const int gq = gi >> 16;
                    if (__ldcg(tags_of(gq) + v) == claim_code(st.qs[gq].epoch, gi & 0xFFFF))
                        ok = true;
                }
                warp_append2(ok, v, gi, &st.nFresh, fr_v, fr_i);
            }
            __syncthreads();
            const int nF = st.nFresh;
            for (int t = tid; t < nF; t += NT) {
                const int gq = fr_i[t] >> 16;
                tags_of(gq)[fr_v[t]] = done_code(st.qs[gq].epoch);
            }
            __syncthreads();
        };
        // sort each query's pool (group of GT threads per query, named barrier 1 + gq)
        auto sort_pools = [&]() {
            const int gq = tid / GT, gt = tid % GT;
            const MqQuery &Q = st.qs[gq];
            uint64_t *sk = sortk + gq * a.sortcap;
            int32_t *sv = sortv + gq * a.sortcap;
            const int np = Q.nPool;
            for (int i = gt; i < np; i += GT) { sk[i] = pkey(gq, Q.pool_cur)[i]; sv[i] = i; }
            group_sort_desc<GT>(sk, sv, np, a.sortcap, gt, 1 + gq);
            __syncthreads();
        };

        // ================= init: entry + its top-layer neighbourhood (hop 0)
        if (tid == 0) { st.nS = 0; st.nFresh = 0; }
        __syncthreads();
        if (tid < G && st.qs[tid].q >= 0) {
            const int idx = atomicAdd(&st.nFresh, 1);
            tags_of(tid)[g.entry] = done_code(st.qs[tid].epoch);
            fr_v[idx] = g.entry;
            fr_i[idx] = tid << 16;
        }
        if (warp < G && st.qs[warp].q >= 0) {
            const int32_t *row = graph_row(g, top, g.entry);
            uint32_t *tg = tags_of(warp);
            if (lane == 0) st.qs[warp].rows += 1;
            if (row) {
                const uint32_t code = claim_code(st.qs[warp].epoch, 0);
                for (int c0 = 0; c0 < g.deg[top]; c0 += 32) {
                    const int32_t v = (c0 + lane < g.deg[top]) ? __ldg(row + c0 + lane) : -1;
                    const unsigned nv = __popc(__ballot_sync(0xffffffffu, v >= 0));
                    if (lane == 0) st.qs[warp].nbrs += nv;
                    bool ok = false;
                    if (v >= 0) {
                        const uint32_t old = atomicMax(tg + v, code);
                        ok = old < code;
                    }
                    warp_append2(ok, v, warp << 16, &st.nS, surv_v, surv_i);
                }
            }
        }
        __syncthreads();
        resolve(st.nS);
        score_fresh(st.nFresh, top, 0);
        compact_pools();
        GR_PH(0);

        int h = 0;
        for (int layer = top; layer >= 0; --layer) {
            // ---- seeds: each query's pool sorted, first min(kp, |pool|) (exact in MODE 1)
            if constexpr (MODE == 1) {
                __shared__ float thr2[G];
                if (warp < G) {
                    const MqQuery &Q = st.qs[warp];
                    float Ts = -INFINITY;  // all entries when |pool| <= kp
                    if (Q.nPool > a.kp) {
                        const uint64_t Ta = warp_select_threshold(pkey(warp, Q.pool_cur), Q.nPool, a.kp, hist + warp * 256);
                        Ts = orderable_f32((uint32_t)(Ta >> 32));
                        Ts = Ts - band_of(Ts);
                    }
                    if (lane == 0) thr2[warp] = Ts;
                }
                __syncthreads();
                rescore(collect_pool([&](int gq, float v) { return v >= thr2[gq]; }), true);
            }
            sort_pools();
            if (tid == 0) {
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
            __syncthreads();
            for (int gq = 0; gq < G; ++gq) {
                const MqQuery &Q = st.qs[gq];
                for (int i = tid; i < Q.f_cnt; i += NT) {
                    fslot[0][Q.f_off + i] = pslot(gq, Q.pool_cur)[sortv[gq * a.sortcap + i]];
                    fsrch[0][Q.f_off + i] = (gq << 16) | i;
                }
            }
            __syncthreads();
            GR_PH(1);
            const int deg = g.deg[layer];
            for (int t = 0; t < a.hops; ++t) {
                ++h;
                const int nF = st.nF;
                if (nF == 0) { h += a.hops - 1 - t; break; }
                const int fc = st.f_cur;
                if (tid == 0) { st.nS = 0; st.nFresh = 0; }
                __syncthreads();
                // ---- expand + claim.  A warp takes RW frontier rows and spreads their 16-byte
                // pieces over the lanes (<= 3 per lane): every row load is in flight at once,
                // then every claim atomic, then ONE aggregated survivor append per warp.
                // Software-pipelined: the next batch's frontier entries and row pieces are
                // fetched while this batch's claim atomics are in flight.
                {
                    const int P = g.ld[layer] >> 2;           // int4 pieces per row
                    const int RW = min(32, 96 / P), NP = RW * P;
                    constexpr unsigned FULL = 0xffffffffu;
                    auto meta = [&](int e0, int32_t &ms, int32_t &mgi) {
                        ms = -1;
                        mgi = 0;
                        if (lane < RW && e0 + lane < nF) { ms = fslot[fc][e0 + lane]; mgi = fsrch[fc][e0 + lane]; }
                    };
                    auto pieces = [&](int32_t ms, int32_t mgi, int4 (&pv)[3], int (&pgi)[3]) {
                        const int4 *mrow = ms >= 0 ? reinterpret_cast<const int4 *>(graph_row(g, layer, ms)) : nullptr;
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const int pc = lane + 32 * j, r = min(pc / P, 31), c = pc - r * P;
                            const int4 *rp = reinterpret_cast<const int4 *>(
                                __shfl_sync(FULL, reinterpret_cast<unsigned long long>(mrow), r));
                            pgi[j] = __shfl_sync(FULL, mgi, r);
                            pv[j] = (pc < NP && rp) ? __ldg(rp + c) : make_int4(-1, -1, -1, -1);
                        }
                    };
                    int32_t ms, mgi;
                    int4 pv[3];
                    int pgi[3];
                    int e0 = warp * RW;
                    meta(e0, ms, mgi);
                    pieces(ms, mgi, pv, pgi);
                    for (; e0 < nF; e0 += NW * RW) {
                        int32_t ms1, mgi1;
                        meta(e0 + NW * RW, ms1, mgi1);
                        uint32_t old[3][4];
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const int gq = pgi[j] >> 16;
                            const uint32_t code = claim_code(st.qs[gq].epoch, pgi[j] & 0xFFFF);
                            uint32_t *tg = tags_of(gq);
                            const int vv[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) old[j][u] = vv[u] >= 0 ? atomicMax(tg + vv[u], code) : 0xFFFFFFFFu;
                        }
                        int4 pv1[3];
                        int pgi1[3];
                        pieces(ms1, mgi1, pv1, pgi1);
                        int cnt = 0, nv = 0;
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const uint32_t code = claim_code(st.qs[pgi[j] >> 16].epoch, pgi[j] & 0xFFFF);
                            const int vv[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                nv += vv[u] >= 0;
                                cnt += (vv[u] >= 0 && old[j][u] < code);
                            }
                        }
                        // one survivor reservation per warp (inclusive scan of the lane counts)
                        int incl = cnt;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int y = __shfl_up_sync(FULL, incl, o);
                            if (lane >= o) incl += y;
                        }
                        int base = 0;
                        if (lane == 31 && incl) base = atomicAdd(&st.nS, incl);
                        base = __shfl_sync(FULL, base, 31) + incl - cnt;
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const uint32_t code = claim_code(st.qs[pgi[j] >> 16].epoch, pgi[j] & 0xFFFF);
                            const int vv[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (vv[u] >= 0 && old[j][u] < code) {
                                    surv_v[base] = vv[u];
                                    surv_i[base] = pgi[j];
                                    ++base;
                                }
                        }
                        // stats: rows expanded / neighbour ids read per query (usually one
                        // query per warp iteration: one reduction + one atomic)
                        const int gq0 = __shfl_sync(FULL, mgi, 0) >> 16;
                        if (__all_sync(FULL, ms < 0 || (mgi >> 16) == gq0)) {
                            int nrow = __popc(__ballot_sync(FULL, ms >= 0)), tot = nv;
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
                            if (lane == 0) { atomicAdd(&st.qs[gq0].rows, nrow); atomicAdd(&st.qs[gq0].nbrs, tot); }
                        } else {
                            if (ms >= 0) atomicAdd(&st.qs[mgi >> 16].rows, 1);
#pragma unroll
                            for (int j = 0; j < 3; ++j) {
                                const int n4 = (pv[j].x >= 0) + (pv[j].y >= 0) + (pv[j].z >= 0) + (pv[j].w >= 0);
                                if (n4) atomicAdd(&st.qs[pgi[j] >> 16].nbrs, n4);
                            }
                        }
                        ms = ms1;
                        mgi = mgi1;
#pragma unroll
                        for (int j = 0; j < 3; ++j) { pv[j] = pv1[j]; pgi[j] = pgi1[j]; }
                    }
                }
                __syncthreads();
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
                for (int i = tid; i < NSEG; i += NT) seg_cnt[i] = 0;
                __syncthreads();
                auto seg_of = [&](int gi) { return (gi >> 16) * a.kp + (gi & 0xFFFF); };
                for (int t0 = 0; t0 < nFresh; t0 += NT) {
                    const int t2 = t0 + tid;
                    if (t0 + warp * 32 < nFresh) {
                        const int sg = t2 < nFresh ? seg_of(fr_i[t2]) : 0;
                        warp_count(&seg_cnt[sg], sg, 1, t2 < nFresh);
                    }
                }
                __syncthreads();
                if (warp == 0) { // exclusive scans of counts and min(count, ef)
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
                    if (lane == 0) st.nFn = accf;
                }
                __syncthreads();
                for (int t2 = tid; t2 < nFresh; t2 += NT) {
                    const int sg = seg_of(fr_i[t2]);
                    const int pos = seg_off[sg] + atomicAdd(&seg_cnt[sg], 1);
                    seg_v[pos] = fr_v[t2];
                    seg_key[pos] = fr_key[t2];
                }
                __syncthreads();
                if constexpr (MODE == 1) {
                    for (int t2 = tid; t2 < nFresh; t2 += NT) seg_ex[t2] = 0;
                    if (tid == 0) st.nRq = 0;
                    __syncthreads();
                    for (int sg = warp; sg < NSEG; sg += NW) {
                        const int ni = seg_cnt[sg], off = seg_off[sg], gq = sg / a.kp;
                        if (ni <= a.ef) continue;
                        const uint64_t Ta = warp_select_threshold(seg_key + off, ni, a.ef, hist + warp * 256);
                        const float Ts = orderable_f32((uint32_t)(Ta >> 32)), bd = band_of(Ts);
                        for (int j0 = 0; j0 < ni; j0 += 32) {
                            const int j = j0 + lane;
                            const bool in = j < ni &&
                                fabsf(orderable_f32((uint32_t)(seg_key[off + j] >> 32)) - Ts) <= bd;
                            warp_append2(in, (gq << 24) | (off + j), 0, &st.nRq, rq, surv_i);
                        }
                    }
                    __syncthreads();
                    rescore(st.nRq, false);
                }
                const int fn = fc ^ 1;
                for (int sg = warp; sg < NSEG; sg += NW) {
                    const int ni = seg_cnt[sg], off = seg_off[sg], fo = fn_off[sg];
                    const int gi = ((sg / a.kp) << 16) | (sg % a.kp);
                    if (ni <= a.ef) {
                        for (int j = lane; j < ni; j += 32) { fslot[fn][fo + j] = seg_v[off + j]; fsrch[fn][fo + j] = gi; }
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
                                fsrch[fn][pos] = gi;
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

        // ---- results: every query's pool sorted, first min(k, |pool|), exact scores
        if constexpr (MODE == 1) rescore(collect_pool([&](int, float) { return true; }), true);
        sort_pools();
        for (int gq = 0; gq < G; ++gq) {
            MqQuery &Q = st.qs[gq];
            if (Q.q < 0) continue;
            const int64_t q = Q.q;
            const int np = Q.nPool, c = Q.pool_cur, nr = min(a.k, np);
            const int32_t *sv = sortv + gq * a.sortcap;
            for (int j = tid; j < a.k; j += NT) {
                if (j < nr) {
                    const int idx = sv[j];
                    a.out_ids[q * a.k + j] = g.ids[pslot(gq, c)[idx]];
                    a.out_scores[q * a.k + j] = (double)orderable_f32((uint32_t)(pkey(gq, c)[idx] >> 32));
                } else {
                    a.out_ids[q * a.k + j] = -1;
                    a.out_scores[q * a.k + j] = __longlong_as_double(0x7ff8000000000000ll);
                }
            }
            if (tid == 0) {
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
        GR_PH(7);
    }
    if (a.phase_cycles && tid < 16) atomicAdd(a.phase_cycles + tid, ph_acc[tid]);
#undef GR_PH
    if constexpr (MODE == 1) {
        tc::fence_before();
        __syncthreads();
        if (tid == 0) band_flush(bc, a.counters, a.band_viol);
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}
