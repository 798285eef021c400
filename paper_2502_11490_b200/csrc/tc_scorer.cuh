// tcgen05 (5th-gen tensor core) metric scorer: split-bf16 ("bf16x3") MLP on 128-pair tiles.
//
// Layer 0 (item half) and layer 1 are UMMA contractions D[128 pairs x 64] += A . B^T with
// A = activations, B = weights, both bf16 hi/lo splits of the fp32 values
// (x = hi + lo + O(2^-16 x)); three MMAs per k-step (hi.hi + hi.lo + lo.hi), fp32
// accumulators in TMEM.  One elected thread issues tcgen05.mma; completion is signalled
// with tcgen05.commit on an mbarrier; the epilogue warps read the accumulators with
// tcgen05.ld (32 lanes x 32 columns per warp), add the hoisted user half + bias, ReLU,
// split again to bf16 hi/lo for the next layer, and run the Z-head + attention on CUDA cores.
//
// Operands use the SWIZZLE_NONE K-major canonical layout: 8-row x 16-byte core matrices,
// K-adjacent cores 128 B apart (LBO), 8-row groups K*2*8 bytes apart (SBO)
// (cute UMMA::make_umma_desc<Major::K> INTERLEAVE form; validated by tools/tc_probe.cu).
//
// These scores are approximations (|err| ~1e-5 relative); the search kernel re-scores
// every item whose selection could depend on the difference with the exact scorer.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "mlp_exact.cuh"

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__host__ __device__ __forceinline__ uint32_t kmaj_off(int r, int k, int K) {
    return (uint32_t)((r >> 3) * (K * 16) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t K) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128u >> 4) & 0x3FFF) << 16;         // LBO: next core along K
    d |= (uint64_t)(((K * 16u) >> 4) & 0x3FFF) << 32;    // SBO: next 8-row group
    d |= (uint64_t)1 << 46;                               // descriptor version (sm_100)
    return d;
}
// bf16 x bf16 -> f32, K-major A/B, M x N
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t id,
                                    uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}
// wait with a suspend-time hint (ns): the warp may be descheduled until the phase completes
// (or the hint elapses) instead of re-issuing the probe
__device__ __forceinline__ void mbar_wait_hint(uint64_t *bar, uint32_t phase, uint32_t ns) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
            "selp.b32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase), "r"(ns)
            : "memory");
    }
}
// non-blocking probe of a phase (the issuer polls several barriers)
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;"); }

__device__ __forceinline__ void tmem_ld32(uint32_t addr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}
// two 32-column loads under one wait::ld
__device__ __forceinline__ void tmem_ld64(uint32_t addr, float (&v)[64]) {
    uint32_t r[64];
#define GR_LD32(OFF, R)                                                                              \
    asm volatile(                                                                                    \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"      \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"            \
        : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]),        \
          "=r"(R[7]), "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]), "=r"(R[13]),    \
          "=r"(R[14]), "=r"(R[15]), "=r"(R[16]), "=r"(R[17]), "=r"(R[18]), "=r"(R[19]),             \
          "=r"(R[20]), "=r"(R[21]), "=r"(R[22]), "=r"(R[23]), "=r"(R[24]), "=r"(R[25]),             \
          "=r"(R[26]), "=r"(R[27]), "=r"(R[28]), "=r"(R[29]), "=r"(R[30]), "=r"(R[31])              \
        : "r"(addr + OFF));
    GR_LD32(0, r);
    GR_LD32(32, (r + 32));
#undef GR_LD32
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = __uint_as_float(r[j]);
}

// A operand from tensor memory (".ts" form): lane = row, column c = bf16 pair (k = 2c, 2c+1)
__device__ __forceinline__ void mma_ts(uint32_t dtmem, uint32_t atmem, uint64_t db, uint32_t id,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "r"(atmem), "l"(db), "r"(id), "r"(acc));
}
// Whole-warp (converged) forms: every lane executes the asm with warp-uniform operands and
// elect.sync picks the issuing lane, so the descriptors stay in uniform registers (no
// per-MMA R2UR broadcast loop as when a single divergent lane issues).
__device__ __forceinline__ void mma_w(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t id,
                                      uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts_w(uint32_t dtmem, uint32_t atmem, uint64_t db, uint32_t id,
                                         uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "r"(atmem), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_w(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 16-byte global -> shared asynchronous copy (L1 bypass) and the mbarrier arrival that fires
// when every earlier cp.async of this thread has landed (.noinc: counted in the init count)
__device__ __forceinline__ void cp_async16(uint32_t sdst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// TMA row gather: 4 rows x 64 bf16 (the tensor map's 128-byte box) of a 2-D [rows][cols] table
// into 512 contiguous bytes of shared memory, 128-byte swizzled; completion counted in bytes
// on the mbarrier (the issuer armed it with arrive.expect_tx)
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t sdst, const void *tmap, int col, int r0, int r1, int r2,
                                            int r3, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sdst),
        "l"(tmap), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_gather4(const void *tmap, int col, int r0, int r1, int r2, int r3) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile::gather4 [%0, {%1, %2, %3, %4, %5}];" ::"l"(tmap),
                 "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                 : "memory");
}
// K-major SWIZZLE_128B operand: 128-byte rows (64 bf16 of K), 8-row atoms 1024 B apart (SBO);
// the K step inside the atom advances the start address by 32 B per 16 elements
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                               // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024u >> 4) << 32;                    // SBO: next 8-row atom
    d |= (uint64_t)1 << 46;                               // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                               // layout: SWIZZLE_128B
    return d;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t *>(&h);
}

// packed f32x2 helpers for the approximate epilogue (any rounding order is fine there)
__device__ __forceinline__ unsigned long long f2pk(float lo, float hi) {
    return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ void add2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a0, a1)), "l"(f2pk(b0, b1)));
    r0 = __uint_as_float((uint32_t)r);
    r1 = __uint_as_float((uint32_t)(r >> 32));
}
__device__ __forceinline__ void fma2(float &c0, float &c1, float a0, float a1, float b0, float b1) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2pk(a0, a1)), "l"(f2pk(b0, b1)), "l"(f2pk(c0, c1)));
    c0 = __uint_as_float((uint32_t)r);
    c1 = __uint_as_float((uint32_t)(r >> 32));
}
// split 4 fp32 into bf16 hi/lo pairs packed as 2 x u32 each
__device__ __forceinline__ void split4(float4 x, uint2 &hi, uint2 &lo) {
    // hi = bf16(x), lo = bf16(x - hi); cvt.rn.bf16x2.f32 packs two lanes per instruction
    const __nv_bfloat162 h01 = __floats2bfloat162_rn(x.x, x.y), h23 = __floats2bfloat162_rn(x.z, x.w);
    const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
    const __nv_bfloat162 l01 = __floats2bfloat162_rn(x.x - f01.x, x.y - f01.y),
                         l23 = __floats2bfloat162_rn(x.z - f23.x, x.w - f23.y);
    hi.x = *reinterpret_cast<const uint32_t *>(&h01);
    hi.y = *reinterpret_cast<const uint32_t *>(&h23);
    lo.x = *reinterpret_cast<const uint32_t *>(&l01);
    lo.y = *reinterpret_cast<const uint32_t *>(&l23);
}

} // namespace tc

// Shared-memory block of the tensor-core scorer for d_h = D_H, hidden (64, 64), Z heads.
template <int D_H, int Z>
struct TcMlp {
    static_assert(D_H % 64 == 0, "layer-0 item half is processed in 64-wide K chunks");
    static constexpr int H = 64, TM = 128, KC = 64;
    static constexpr int NKC0 = D_H / KC; // layer-0 K chunks
    // byte offsets
    static constexpr int OFF_B0H = 0;
    static constexpr int OFF_B0L = OFF_B0H + H * D_H * 2;
    static constexpr int OFF_B1H = OFF_B0L + H * D_H * 2;
    static constexpr int OFF_B1L = OFF_B1H + H * H * 2;
    static constexpr int OFF_AH = OFF_B1L + H * H * 2;     // A operand hi [128 x 64] bf16
    static constexpr int OFF_AL = OFF_AH + TM * KC * 2;    // A operand lo
    static constexpr int A_BYTES = 2 * TM * KC * 2;       // 32 KB
    // exact re-scoring buffers (FixedMlp x0/h0/h1/z/score) alias the A operand region
    using FX = FixedMlp<D_H, Z>;
    static constexpr int EX_BYTES = 16 * (GR_PT * FX::LDX0 + 2 * GR_PT * FX::LDH + GR_PT * FX::LDZ + GR_PT / 4);
    static constexpr int A_REGION = A_BYTES > EX_BYTES ? A_BYTES : EX_BYTES;
    static constexpr int OFF_EX_X0 = OFF_AH;
    static constexpr int OFF_EX_H0 = OFF_EX_X0 + 16 * GR_PT * FX::LDX0;
    static constexpr int OFF_EX_H1 = OFF_EX_H0 + 16 * GR_PT * FX::LDH;
    static constexpr int OFF_EX_Z = OFF_EX_H1 + 16 * GR_PT * FX::LDH;
    static constexpr int OFF_EX_SC = OFF_EX_Z + 16 * GR_PT * FX::LDZ;
    static constexpr int OFF_U = OFF_AH + A_REGION;       // user half + b0 per output [64] f32
    static constexpr int OFF_B1 = OFF_U + H * 4;
    static constexpr int OFF_W2 = OFF_B1 + H * 4;         // fp32 [Z][64]
    static constexpr int OFF_B2 = OFF_W2 + Z * H * 4;
    static constexpr int OFF_ATT = OFF_B2 + 16;
    static constexpr int OFF_ZP = OFF_ATT + 16;           // partial heads [128][2][Z] f32
    static constexpr int OFF_SC = OFF_ZP + TM * 2 * Z * 4; // approx scores [128]
    static constexpr int OFF_BAR = (OFF_SC + TM * 4 + 15) & ~15;
    static constexpr int OFF_TMEM = OFF_BAR + 16;
    static constexpr int OFF_ACC0 = OFF_TMEM + 16;        // exact hoisted user half [64] float4
    static constexpr int BYTES = OFF_ACC0 + H * 16;
    static constexpr uint32_t IDESC = tc::idesc(TM, H);

    // Approximate scores of up to 128 pairs (rows = item rows gathered by slot).
    // tmem: allocated base (>= 128 columns: D0 = cols 0..63, D1 = cols 64..127).
    static __device__ __forceinline__ void tile(unsigned char *sm, uint32_t tmem, uint32_t &phase,
                                                const DevItems &it, const DevGraph &g,
                                                const int32_t *slots, int nv) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        unsigned char *Ah = sm + OFF_AH, *Al = sm + OFF_AL;
        uint64_t *bar = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
        const uint32_t aH = tc::smem_u32(Ah), aL = tc::smem_u32(Al);
        // ---- layer 0: D0 = x_item . W0_item^T over NKC0 chunks of 64
        for (int kc = 0; kc < NKC0; ++kc) {
            for (int t = tid; t < TM * 16; t += GR_NT) {
                // 8 rows x 4 float4 per warp: conflict-free core-matrix stores
                const int u = t >> 5, l = t & 31;
                const int r = (u % (TM / 8)) * 8 + (l & 7), c = (u / (TM / 8)) * 4 + (l >> 3);
                if (r < nv) {
                    const int32_t s = slots[r];
                    const float4 x = __ldg(reinterpret_cast<const float4 *>(it.emb + slot_row(g, s) * it.ld) + kc * 16 + c);
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
            tc::mbar_wait(bar, phase);
            phase ^= 1u;
            tc::fence_after();
        }
        // ---- epilogue 0: + (user half + b0), ReLU, split -> A (layer-1 operand, K = 64)
        const int q4 = warp & 3, half = warp >> 2, row = q4 * 32 + lane;
        const float *u = reinterpret_cast<const float *>(sm + OFF_U);
        {
            float v[32];
            tc::tmem_ld32(tmem + ((uint32_t)(q4 * 32) << 16) + half * 32, v);
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const int o = half * 32 + j;
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
        // ---- layer 1: D1 = h0 . W1^T
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
        // ---- epilogue 1: ReLU(+b1), Z heads (fp32), attention
        {
            float v[32];
            tc::tmem_ld32(tmem + ((uint32_t)(q4 * 32) << 16) + 64 + half * 32, v);
            const float *b1 = reinterpret_cast<const float *>(sm + OFF_B1);
            const float *W2 = reinterpret_cast<const float *>(sm + OFF_W2);
            float zp[Z];
#pragma unroll
            for (int o = 0; o < Z; ++o) zp[o] = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float h = fmaxf(v[j] + b1[half * 32 + j], 0.f);
#pragma unroll
                for (int o = 0; o < Z; ++o) zp[o] = fmaf(h, W2[o * H + half * 32 + j], zp[o]);
            }
            float *ZP = reinterpret_cast<float *>(sm + OFF_ZP);
#pragma unroll
            for (int o = 0; o < Z; ++o) ZP[(row * 2 + half) * Z + o] = zp[o];
        }
        tc::fence_before();
        __syncthreads();
        if (tid < TM) {
            const float *ZP = reinterpret_cast<const float *>(sm + OFF_ZP);
            const float *b2 = reinterpret_cast<const float *>(sm + OFF_B2);
            const float *att = reinterpret_cast<const float *>(sm + OFF_ATT);
            float s = 0.f;
#pragma unroll
            for (int o = 0; o < Z; ++o)
                s = fmaf(ZP[(tid * 2) * Z + o] + ZP[(tid * 2 + 1) * Z + o] + b2[o], att[o], s);
            reinterpret_cast<float *>(sm + OFF_SC)[tid] = s;
        }
        __syncthreads();
    }
};

