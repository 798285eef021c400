// Pair scorer (ScoreFn / BatchEngine), exact brute force, and shard top-k merge.
#pragma once
#include "common.cuh"
#include "mlp_exact.cuh"
#include "select.cuh"

// ---------------------------------------------------------------------------
// gr_score_pairs: relevance_batch over arbitrary (user, item) pairs
// (metric.py:150-154 via RelevanceModel.score 222-226 / BatchEngine.evaluate).
// Grid-stride over tiles of GR_PT pairs; no hoisting (users differ per pair).
// ---------------------------------------------------------------------------
struct PairArgs {
    DevModel M;
    DevItems it;
    const float *users;
    int64_t n_users;
    const int32_t *user_index; // nullable -> users[0]
    const int64_t *item_ids;
    int64_t n;
    double *out;
    int *nonfinite;
    int *bad_index;
    int off_w[GR_MAX_MLP], off_b[GR_MAX_MLP], off_A, off_x0, off_h0, off_h1, off_score;
    int ldx0, ldh;
};

__device__ __forceinline__ void load_weights_full(const DevModel &M, unsigned char *smem,
                                                  const int *off_w, const int *off_b, int off_A,
                                                  const float4 **sWm, const float **sbm) {
    for (int m = 0; m < M.n_mlp; ++m) {
        float4 *sw = reinterpret_cast<float4 *>(smem + off_w[m]);
        const int nw = M.nch[m] * M.dims[m + 1];
        for (int t = threadIdx.x; t < nw; t += GR_NT) sw[t] = M.W[m][t];
        float *sb = reinterpret_cast<float *>(smem + off_b[m]);
        for (int t = threadIdx.x; t < M.dims[m + 1]; t += GR_NT) sb[t] = M.b[m][t];
        sWm[m] = sw;
        sbm[m] = sb;
    }
    float4 *sA = reinterpret_cast<float4 *>(smem + off_A);
    for (int t = threadIdx.x; t < M.nch[M.n_mlp]; t += GR_NT) sA[t] = M.A[t];
}

// fill x0 row (processing order over K0 = 2 d_h) from hu | hv
__device__ __forceinline__ void fill_pair_row(float4 *xr, int nch0, int K0, int d_h,
                                              const float *hu, const float *hv, int lane) {
    for (int j = lane; j < nch0; j += 32) {
        const int c = chunk_perm(j, K0);
        float e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int idx = 4 * c + u;
            e[u] = idx < d_h ? hu[idx] : (idx < K0 ? hv[idx - d_h] : 0.f);
        }
        xr[j] = make_float4(e[0], e[1], e[2], e[3]);
    }
}

__global__ void __launch_bounds__(GR_NT) score_pairs_kernel(const PairArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DevModel &M = a.M;
    const float4 *sWm[GR_MAX_MLP];
    const float *sbm[GR_MAX_MLP];
    load_weights_full(M, smem, a.off_w, a.off_b, a.off_A, sWm, sbm);
    const float4 *sA = reinterpret_cast<const float4 *>(smem + a.off_A);
    TileSmem S;
    S.x0 = reinterpret_cast<float4 *>(smem + a.off_x0);
    S.ldx0 = a.ldx0;
    S.h[0] = reinterpret_cast<float4 *>(smem + a.off_h0);
    S.h[1] = reinterpret_cast<float4 *>(smem + a.off_h1);
    S.ldh = a.ldh;
    S.score = reinterpret_cast<float *>(smem + a.off_score);
    for (int t = threadIdx.x; t < GR_PT * a.ldh; t += GR_NT) {
        S.h[0][t] = make_float4(0.f, 0.f, 0.f, 0.f);
        S.h[1][t] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d_h = M.d_h, K0 = M.dims[0], nch0 = M.nch[0];
    __syncthreads();
    for (int64_t base = (int64_t)blockIdx.x * GR_PT; base < a.n; base += (int64_t)gridDim.x * GR_PT) {
        const int nv = (int)min((int64_t)GR_PT, a.n - base);
        for (int pp = 0; pp < 4; ++pp) {
            const int p = warp * 4 + pp;
            float4 *xr = S.x0 + p * a.ldx0;
            if (p < nv) {
                const int64_t i = base + p;
                int64_t u = a.user_index ? (int64_t)a.user_index[i] : 0;
                int64_t row = a.item_ids[i];
                if (u < 0 || u >= a.n_users || row < 0 || row >= a.it.n) {
                    if (lane == 0) atomicOr(a.bad_index, 1);
                    u = 0;
                    row = 0;
                }
                fill_pair_row(xr, nch0, K0, d_h, a.users + u * d_h, a.it.emb + row * a.it.ld, lane);
            } else {
                for (int j = lane; j < nch0; j += 32) xr[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncthreads();
        mlp_tile(M, S, sWm, sbm, sA, sWm[0], nch0, nullptr, nv, a.nonfinite);
        __syncthreads();
        if (threadIdx.x < nv) a.out[base + threadIdx.x] = (double)S.score[threadIdx.x];
    }
}

// ---------------------------------------------------------------------------
// gr_brute_force: exact top-k over all items for each query (search.py:93-108).
// Phase 1: grid (P partitions x B queries); each CTA scores its item range with
// the hoisted user half and keeps a running top-k (threshold + compaction).
// Phase 2: one CTA per query merges the P local lists (select + sort).
// ---------------------------------------------------------------------------
struct BruteArgs {
    DevModel M;
    DevItems it;
    const float *users; // [B][d_h] for this batch
    int B, P, k;
    int64_t cap;        // per-CTA candidate buffer (>= k + items per round)
    uint64_t *cand_key; // [B][P][2][cap]
    int32_t *cand_row;
    uint64_t *loc_key;  // [B][P][k]
    int32_t *loc_row;
    int32_t *loc_n;     // [B][P]
    int *nonfinite;
    int off_w0, off_w[GR_MAX_MLP], off_b[GR_MAX_MLP], off_A, off_acc0, off_x0, off_h0, off_h1,
        off_score, off_hist;
    int ldx0, ldh;
};

struct BruteState {
    int n, n2, cur;
    uint64_t T;
    uint32_t bcast[4];
};

__global__ void __launch_bounds__(GR_NT) brute_partial_kernel(const BruteArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ BruteState st;
    const DevModel &M = a.M;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int O0 = M.dims[1], K0 = M.dims[0], nch0 = M.nch[0], pre = M.pre_ch, d_h = M.d_h;
    const int x0_nch = nch0 - pre;
    float4 *sW0 = reinterpret_cast<float4 *>(smem + a.off_w0);
    for (int t = tid; t < x0_nch * O0; t += GR_NT) sW0[t] = M.W[0][pre * O0 + t];
    const float4 *sWm[GR_MAX_MLP];
    const float *sbm[GR_MAX_MLP];
    for (int m = 0; m < M.n_mlp; ++m) {
        float *sb = reinterpret_cast<float *>(smem + a.off_b[m]);
        for (int t = tid; t < M.dims[m + 1]; t += GR_NT) sb[t] = M.b[m][t];
        sbm[m] = sb;
        if (m >= 1) {
            float4 *sw = reinterpret_cast<float4 *>(smem + a.off_w[m]);
            for (int t = tid; t < M.nch[m] * M.dims[m + 1]; t += GR_NT) sw[t] = M.W[m][t];
            sWm[m] = sw;
        } else {
            sWm[0] = sW0;
        }
    }
    float4 *sA = reinterpret_cast<float4 *>(smem + a.off_A);
    for (int t = tid; t < M.nch[M.n_mlp]; t += GR_NT) sA[t] = M.A[t];
    TileSmem S;
    S.x0 = reinterpret_cast<float4 *>(smem + a.off_x0);
    S.ldx0 = a.ldx0;
    S.h[0] = reinterpret_cast<float4 *>(smem + a.off_h0);
    S.h[1] = reinterpret_cast<float4 *>(smem + a.off_h1);
    S.ldh = a.ldh;
    S.score = reinterpret_cast<float *>(smem + a.off_score);
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem + a.off_hist);
    float4 *sAcc0 = reinterpret_cast<float4 *>(smem + a.off_acc0);
    for (int t = tid; t < GR_PT * a.ldx0; t += GR_NT) S.x0[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int t = tid; t < GR_PT * a.ldh; t += GR_NT) {
        S.h[0][t] = make_float4(0.f, 0.f, 0.f, 0.f);
        S.h[1][t] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int b = blockIdx.y, part = blockIdx.x;
    const float *hu = a.users + (int64_t)b * d_h;
    for (int o = tid; o < O0; o += GR_NT) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = 0; j < pre; ++j) {
            const int c = chunk_perm(j, K0);
            mac4(acc, make_float4(hu[4 * c], hu[4 * c + 1], hu[4 * c + 2], hu[4 * c + 3]),
                 M.W[0][j * O0 + o]);
        }
        sAcc0[o] = acc;
    }
    if (tid == 0) { st.n = 0; st.cur = 0; st.T = 0ull; }
    const int64_t per = (a.it.n + a.P - 1) / a.P;
    const int64_t lo = (int64_t)part * per, hi = min(a.it.n, lo + per);
    const int64_t cb = ((int64_t)b * a.P + part) * 2 * a.cap;
    uint64_t *ck[2] = {a.cand_key + cb, a.cand_key + cb + a.cap};
    int32_t *cr[2] = {a.cand_row + cb, a.cand_row + cb + a.cap};
    const bool fast_fill = (d_h % 16) == 0;
    __syncthreads();
    for (int64_t base = lo; base < hi; base += GR_PT) {
        const int nv = (int)min((int64_t)GR_PT, hi - base);
        for (int pp = 0; pp < 4; ++pp) {
            const int p = warp * 4 + pp;
            float4 *xr = S.x0 + p * a.ldx0;
            if (p < nv) {
                const float *hv = a.it.emb + (base + p) * a.it.ld;
                if (fast_fill) {
                    for (int cc = lane; cc < d_h / 4; cc += 32)
                        xr[chunk_perm(d_h / 4 + cc, K0) - pre] = __ldg(reinterpret_cast<const float4 *>(hv) + cc);
                } else {
                    for (int jj = lane; jj < x0_nch; jj += 32) {
                        const int c = chunk_perm(pre + jj, K0);
                        float e[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int idx = 4 * c + u;
                            e[u] = idx < d_h ? hu[idx] : (idx < K0 ? hv[idx - d_h] : 0.f);
                        }
                        xr[jj] = make_float4(e[0], e[1], e[2], e[3]);
                    }
                }
            } else {
                for (int jj = lane; jj < x0_nch; jj += 32) xr[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncthreads();
        mlp_tile(M, S, sWm, sbm, sA, sW0, x0_nch, pre > 0 ? sAcc0 : nullptr, nv, a.nonfinite);
        __syncthreads();
        if (tid < nv) {
            const uint64_t key = make_key(S.score[tid], (uint32_t)(base + tid));
            if (key > st.T) {
                const int idx = atomicAdd(&st.n, 1);
                ck[st.cur][idx] = key;
                cr[st.cur][idx] = (int32_t)(base + tid);
            }
        }
        __syncthreads();
        if (st.n > a.cap - GR_PT) { // compact to top-k
            const int c = st.cur;
            const uint64_t T = cta_select_threshold(ck[c], st.n, a.k, hist, st.bcast);
            if (tid == 0) st.n2 = 0;
            __syncthreads();
            for (int i = tid; i < st.n; i += GR_NT) {
                if (ck[c][i] >= T) {
                    const int idx = atomicAdd(&st.n2, 1);
                    ck[c ^ 1][idx] = ck[c][i];
                    cr[c ^ 1][idx] = cr[c][i];
                }
            }
            __syncthreads();
            if (tid == 0) { st.cur = c ^ 1; st.n = st.n2; st.T = T; }
            __syncthreads();
        }
    }
    // final local top-k
    __syncthreads();
    const int c = st.cur;
    uint64_t T = 0ull;
    if (st.n > a.k) T = cta_select_threshold(ck[c], st.n, a.k, hist, st.bcast);
    if (tid == 0) st.n2 = 0;
    __syncthreads();
    const int64_t lb = ((int64_t)b * a.P + part) * a.k;
    for (int i = tid; i < st.n; i += GR_NT) {
        if (ck[c][i] >= T) {
            const int idx = atomicAdd(&st.n2, 1);
            a.loc_key[lb + idx] = ck[c][i];
            a.loc_row[lb + idx] = cr[c][i];
        }
    }
    __syncthreads();
    if (tid == 0) a.loc_n[(int64_t)b * a.P + part] = st.n2;
}

// one CTA per query: concatenate P local lists, sort desc, emit top-k
__global__ void __launch_bounds__(GR_NT) brute_merge_kernel(const uint64_t *loc_key,
                                                            const int32_t *loc_row,
                                                            const int32_t *loc_n, int P, int k,
                                                            int sortcap, int64_t *out_ids,
                                                            double *out_scores) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *sk = reinterpret_cast<uint64_t *>(smem);
    int32_t *sv = reinterpret_cast<int32_t *>(smem + sizeof(uint64_t) * sortcap);
    __shared__ int total;
    const int b = blockIdx.x;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    for (int p = 0; p < P; ++p) {
        const int n = loc_n[(int64_t)b * P + p];
        const int base = total;
        for (int i = threadIdx.x; i < n; i += GR_NT) {
            sk[base + i] = loc_key[((int64_t)b * P + p) * k + i];
            sv[base + i] = loc_row[((int64_t)b * P + p) * k + i];
        }
        __syncthreads();
        if (threadIdx.x == 0) total = base + n;
        __syncthreads();
    }
    cta_sort_desc(sk, sv, total, sortcap);
    for (int j = threadIdx.x; j < k; j += GR_NT) {
        if (j < total) {
            out_ids[(int64_t)b * k + j] = sv[j];
            out_scores[(int64_t)b * k + j] = (double)orderable_f32((uint32_t)(sk[j] >> 32));
        } else {
            out_ids[(int64_t)b * k + j] = -1;
            out_scores[(int64_t)b * k + j] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
}

// ---------------------------------------------------------------------------
// gr_merge_topk: R lists per query -> one top-k by (score desc, id asc).
// Keys: orderable(fp32 score) << 32 | ~id (ids < 2^32).  One CTA per query.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(GR_NT) merge_topk_kernel(const int64_t *in_ids,
                                                           const double *in_scores, int R,
                                                           int64_t Q, int kin, int k, int sortcap,
                                                           int64_t *out_ids, double *out_scores,
                                                           int32_t *out_count) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *sk = reinterpret_cast<uint64_t *>(smem);
    int32_t *sv = reinterpret_cast<int32_t *>(smem + sizeof(uint64_t) * sortcap);
    __shared__ int total;
    const int64_t q = blockIdx.x;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < R * kin; t += GR_NT) {
        const int r = t / kin, j = t % kin;
        const int64_t id = in_ids[((int64_t)r * Q + q) * kin + j];
        if (id >= 0) {
            const float s = (float)in_scores[((int64_t)r * Q + q) * kin + j];
            const int pos = atomicAdd(&total, 1);
            sk[pos] = ((uint64_t)f32_orderable(s) << 32) | (uint64_t)(~(uint32_t)id);
            sv[pos] = t;
        }
    }
    __syncthreads();
    const int n = total;
    cta_sort_desc(sk, sv, n, sortcap);
    const int nr = min(n, k);
    for (int j = threadIdx.x; j < k; j += GR_NT) {
        if (j < nr) {
            const int t = sv[j];
            const int r = t / kin, jj = t % kin;
            out_ids[q * k + j] = in_ids[((int64_t)r * Q + q) * kin + jj];
            out_scores[q * k + j] = in_scores[((int64_t)r * Q + q) * kin + jj];
        } else {
            out_ids[q * k + j] = -1;
            out_scores[q * k + j] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    if (threadIdx.x == 0) out_count[q] = nr;
}

// ---------------------------------------------------------------------------
// Shard-merge wire format (8 bytes per entry, one all-gather): orderable(fp32 score) << 32 |
// id (0 <= id < 2^32); 0 = empty slot.  The returned scores are exact fp32 values widened to
// fp64 (search.py:88), so the fp32 field is lossless.
// ---------------------------------------------------------------------------
__global__ void pack_topk_kernel(const int64_t *ids, const double *scores, int64_t n, uint64_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t id = ids[i];
        out[i] = id < 0 ? 0ull : (((uint64_t)f32_orderable((float)scores[i]) << 32) | (uint64_t)(uint32_t)id);
    }
}

// R packed lists per query -> one top-k by (score desc, id asc); one CTA per query
__global__ void __launch_bounds__(GR_NT) merge_packed_kernel(const uint64_t *in, int R, int64_t Q, int kin,
                                                             int k, int sortcap, int64_t *out_ids,
                                                             double *out_scores, int32_t *out_count) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *sk = reinterpret_cast<uint64_t *>(smem);
    int32_t *sv = reinterpret_cast<int32_t *>(smem + sizeof(uint64_t) * sortcap);
    __shared__ int total;
    const int64_t q = blockIdx.x;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < R * kin; t += GR_NT) {
        const int r = t / kin, j = t % kin;
        const uint64_t e = in[((int64_t)r * Q + q) * kin + j];
        if (e) {
            const int pos = atomicAdd(&total, 1);
            sk[pos] = (e & 0xFFFFFFFF00000000ull) | (uint64_t)(~(uint32_t)e);
            sv[pos] = (int32_t)(uint32_t)e;
        }
    }
    __syncthreads();
    const int n = total;
    cta_sort_desc(sk, sv, n, sortcap);
    const int nr = min(n, k);
    for (int j = threadIdx.x; j < k; j += GR_NT) {
        if (j < nr) {
            out_ids[q * k + j] = (int64_t)(uint32_t)sv[j];
            out_scores[q * k + j] = (double)orderable_f32((uint32_t)(sk[j] >> 32));
        } else {
            out_ids[q * k + j] = -1;
            out_scores[q * k + j] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    if (threadIdx.x == 0) out_count[q] = nr;
}
