// tcgen05 probe: D[128 x N] (fp32, TMEM) = A[128 x K] . B[N x K]^T with bf16 operands in
// shared memory (K-major, no-swizzle core-matrix layout), single elected thread issues
// tcgen05.mma, tcgen05.commit -> mbarrier, epilogue tcgen05.ld 32x32b.  Also bf16x3
// (hi*hi + hi*lo + lo*hi) on fp32 inputs.  Validates descriptors before the search kernel
// uses them.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tc_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int M = 128, N = 64, K = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// core-matrix (8 rows x 16 bytes) K-major layout: byte offset of element (r, k) in a
// [rows x K] bf16 operand: cores ordered K-fastest (LBO = 128 B), row-groups at SBO = K*16 B
__host__ __device__ __forceinline__ uint32_t kmaj_off(int r, int k, int Kdim) {
    return (uint32_t)((r >> 3) * (Kdim * 16) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46; // version = 1 (Blackwell)
    // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
    return d;
}
// instruction descriptor: bf16 x bf16 -> f32, K-major A and B, M x N
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
    return (1u << 4)            // c_format F32
         | (1u << 7)            // a_format BF16
         | (1u << 10)           // b_format BF16
         | (0u << 15) | (0u << 16) // K-major
         | ((uint32_t)(n >> 3) << 17)
         | ((uint32_t)(m >> 4) << 24);
}

__global__ void probe(const float *A, const float *B, float *D1, float *D3, float *DT, int mode) {
    extern __shared__ __align__(1024) unsigned char sm[];
    // layout: Ahi, Alo (M*K*2 each), Bhi, Blo (N*K*2 each), mbarrier, tmem addr
    unsigned char *sAh = sm, *sAl = sm + M * K * 2, *sBh = sAl + M * K * 2, *sBl = sBh + N * K * 2;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sBl + N * K * 2);
    uint32_t *tptr = reinterpret_cast<uint32_t *>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < M * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        float x = A[i];
        __nv_bfloat16 h = __float2bfloat16_rn(x);
        __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
        *reinterpret_cast<__nv_bfloat16 *>(sAh + kmaj_off(r, k, K)) = h;
        *reinterpret_cast<__nv_bfloat16 *>(sAl + kmaj_off(r, k, K)) = l;
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        float x = B[i];
        __nv_bfloat16 h = __float2bfloat16_rn(x);
        __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
        *reinterpret_cast<__nv_bfloat16 *>(sBh + kmaj_off(r, k, K)) = h;
        *reinterpret_cast<__nv_bfloat16 *>(sBl + kmaj_off(r, k, K)) = l;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tptr)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tptr;
    const uint32_t idesc = make_idesc(M, N);
    // A (bf16 hi) into TMEM cols 192..255 for the TS variant: lane = row, column c holds
    // the bf16 pair (k = 2c, 2c+1), low half = even k
    if (warp < 4) {
        const int row = warp * 32 + lane;
        for (int c0 = 0; c0 < K / 2; c0 += 8) {
            uint32_t v[8];
            for (int j = 0; j < 8; ++j) {
                const int k = 2 * (c0 + j);
                __nv_bfloat162 h = __floats2bfloat162_rn(A[row * K + k], A[row * K + k + 1]);
                v[j] = *reinterpret_cast<uint32_t *>(&h);
            }
            const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + 192 + c0;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                         :: "r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                            "r"(v[6]), "r"(v[7]) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
        // pass 1: D[cols 0..63] = Ahi . Bhi ; pass 2: D[cols 64..127] = hi.hi + hi.lo + lo.hi
        for (int pass = 0; pass < 2; ++pass) {
            const uint32_t dcol = tmem + pass * 64;
            int nterm = pass == 0 ? 1 : 3;
            bool acc = false;
            for (int t = 0; t < nterm; ++t) {
                unsigned char *a = (t == 2) ? sAl : sAh;
                unsigned char *b = (t == 1) ? sBl : sBh;
                for (int kk = 0; kk < K / 16; ++kk) {
                    uint64_t da = make_desc(smem_u32(a) + kk * 256, 128, K * 16);
                    uint64_t db = make_desc(smem_u32(b) + kk * 256, 128, K * 16);
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                        :: "r"(dcol), "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)acc));
                    acc = true;
                }
            }
        }
        // pass 3 (TS): D[cols 128..191] = A(TMEM) . Bhi   (mode 0: skipped)
        for (int kk = 0; kk < (mode ? K / 16 : 0); ++kk) {
            uint64_t db = make_desc(smem_u32(sBh) + kk * 256, 128, K * 16);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                :: "r"(tmem + 128), "r"(tmem + 192 + kk * 8), "l"(db), "r"(idesc), "r"((uint32_t)(kk > 0)));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(smem_u32(bar)) : "memory");
    }
    // wait phase 0
    {
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                         "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(0) : "memory");
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        const int row = warp * 32 + lane;
        for (int pass = 0; pass < 3; ++pass) {
            for (int c0 = 0; c0 < N; c0 += 8) {
                uint32_t v[8];
                const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + pass * 64 + c0;
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                               "=r"(v[6]), "=r"(v[7]) : "r"(addr));
                asm volatile("tcgen05.wait::ld.sync.aligned;");
                float *D = pass == 0 ? D1 : pass == 1 ? D3 : DT;
                for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(256));
}

static float bf(float x) { // round-to-nearest-even to bf16, back to float
    uint32_t u; memcpy(&u, &x, 4);
    u += 0x7FFF + ((u >> 16) & 1);
    u &= 0xFFFF0000u;
    float r; memcpy(&r, &u, 4);
    return r;
}

int main(int argc, char **argv) {
    float *hA = (float *)malloc(M * K * 4), *hB = (float *)malloc(N * K * 4);
    srand(1);
    for (int i = 0; i < M * K; ++i) hA[i] = (rand() / (float)RAND_MAX - 0.5f) * 4.f;
    for (int i = 0; i < N * K; ++i) hB[i] = (rand() / (float)RAND_MAX - 0.5f) * 0.3f;
    float *dA, *dB, *dD1, *dD3, *dDT;
    CK(cudaMalloc(&dDT, M * N * 4));
    CK(cudaMalloc(&dA, M * K * 4)); CK(cudaMalloc(&dB, N * K * 4));
    CK(cudaMalloc(&dD1, M * N * 4)); CK(cudaMalloc(&dD3, M * N * 4));
    CK(cudaMemcpy(dA, hA, M * K * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB, N * K * 4, cudaMemcpyHostToDevice));
    int smem = 2 * M * K * 2 + 2 * N * K * 2 + 64;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int mode = argc > 1 ? atoi(argv[1]) : 1;
    printf("mode %d\n", mode);
    probe<<<1, 256, smem>>>(dA, dB, dD1, dD3, dDT, mode);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    float *D1 = (float *)malloc(M * N * 4), *D3 = (float *)malloc(M * N * 4);
    CK(cudaMemcpy(D1, dD1, M * N * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(D3, dD3, M * N * 4, cudaMemcpyDeviceToHost));
    float *DT = (float *)malloc(M * N * 4);
    CK(cudaMemcpy(DT, dDT, M * N * 4, cudaMemcpyDeviceToHost));
    int ts_bad = 0;
    for (int i = 0; i < M * N; ++i) ts_bad += DT[i] != D1[i];
    printf("TS (A in TMEM) vs SS bf16: %d / %d differ\n", ts_bad, M * N);
    double e1 = 0, e3 = 0, e3rel = 0;
    for (int r = 0; r < M; ++r)
        for (int c = 0; c < N; ++c) {
            double ref1 = 0, ref = 0, mag = 0;
            for (int k = 0; k < K; ++k) {
                ref1 += (double)bf(hA[r * K + k]) * bf(hB[c * K + k]);
                ref += (double)hA[r * K + k] * hB[c * K + k];
                mag += fabs((double)hA[r * K + k] * hB[c * K + k]);
            }
            e1 = fmax(e1, fabs(D1[r * N + c] - ref1) / mag);
            e3 = fmax(e3, fabs(D3[r * N + c] - ref) / mag);
            e3rel = fmax(e3rel, fabs(D3[r * N + c] - ref) / fmax(fabs(ref), 1e-6));
        }
    printf("bf16 MMA vs fp64 of bf16 inputs: max err / sum|ab| = %.3e\n", e1);
    printf("bf16x3 vs fp64 of fp32 inputs:    max err / sum|ab| = %.3e (rel %.3e)\n", e3, e3rel);
    printf("%s\n", (e1 < 1e-5 && e3 < 1e-4 && ts_bad == 0) ? "PROBE OK" : "PROBE MISMATCH");
    printf("D1[0..3] = %f %f %f %f\n", D1[0], D1[1], D1[2], D1[3]);
    return 0;
}
