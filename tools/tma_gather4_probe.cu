// Probe: TMA tile::gather4 of bf16 rows into 128-byte-swizzled shared memory (sm_100a).
// Checks (1) dynamic smem alignment next to static smem, (2) gather4 lands rows where the
// SWIZZLE_128B K-major UMMA layout expects them: row r chunk c at r*128 + ((c ^ (r & 7)) * 16).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_2502_11490_b200/csrc/tc_scorer.cuh"

__global__ void probe(const __grid_constant__ CUtensorMap map, const int *rows, int col, uint16_t *out,
                      unsigned *info) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ int st[37];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) st[0] = 1;
    if (threadIdx.x == 0) { info[0] = tc::smem_u32(sm); info[1] = tc::smem_u32(st); }
    if (threadIdx.x == 0) tc::mbar_init(&bar, 1);
    __syncthreads();
    const int lane = threadIdx.x;
    if (lane == 0) tc::mbar_arrive_expect_tx(&bar, 128 * 128);
    __syncwarp();
    const int *r = rows + 4 * lane;
    tc::tma_gather4(tc::smem_u32(sm) + lane * 512, &map, col, r[0], r[1], r[2], r[3], &bar);
    tc::mbar_wait(&bar, 0);
    for (int i = lane; i < 128 * 64; i += 32) out[i] = reinterpret_cast<uint16_t *>(sm)[i];
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    const int n = 1000, W = 256;  // [n][256] bf16 rows (hi 128 | lo 128)
    std::vector<uint16_t> h((size_t)n * W);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < W; ++j) h[(size_t)i * W + j] = (uint16_t)((i * 7 + j) & 0xFFFF);
    uint16_t *d; cudaMalloc(&d, h.size() * 2); cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    std::vector<int> rows(128);
    for (int i = 0; i < 128; ++i) rows[i] = (i * 37 + 11) % n;
    int *drows; cudaMalloc(&drows, 512); cudaMemcpy(drows, rows.data(), 512, cudaMemcpyHostToDevice);
    uint16_t *dout; cudaMalloc(&dout, 128 * 64 * 2);
    unsigned *dinfo; cudaMalloc(&dinfo, 8);
    void *p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)n}, strides[1] = {(cuuint64_t)W * 2};
    const cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = ((EncodeTiledFn)p)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    for (int col : {0, 128 + 64}) {
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        probe<<<1, 32, 64 * 1024>>>(map, drows, col, dout, dinfo);
        cudaError_t e = cudaDeviceSynchronize();
        printf("col %d launch: %s\n", col, cudaGetErrorString(e));
        if (e) return 1;
        std::vector<uint16_t> o(128 * 64); unsigned info[2];
        cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
        cudaMemcpy(info, dinfo, 8, cudaMemcpyDeviceToHost);
        printf("dynamic smem base 0x%x (mod 1024 = %u), static 0x%x\n", info[0], info[0] % 1024, info[1]);
        int bad = 0, bad_plain = 0;
        for (int rr = 0; rr < 128; ++rr)
            for (int c = 0; c < 8; ++c)
                for (int e2 = 0; e2 < 8; ++e2) {
                    const uint16_t want = h[(size_t)rows[rr] * W + col + c * 8 + e2];
                    const int sw = rr * 64 + ((c ^ (rr & 7)) * 8) + e2, pl = rr * 64 + c * 8 + e2;
                    bad += o[sw] != want;
                    bad_plain += o[pl] != want;
                }
        printf("col %d: swizzled-layout mismatches %d, plain-layout mismatches %d (of %d)\n", col, bad, bad_plain,
               128 * 64);
    }
    return 0;
}
