// libgmpgr.so — C ABI (include/gmpgr.h) over the sm_100a HiPANNS kernels.
//
// Host side: handle construction (processing-order weight packing, compact
// device graph layout, padded item rows), scratch management and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/gmpgr.h"
#include "aux_kernels.cuh"
#include "common.cuh"
#include "search_kernel.cuh"
#include "search_mq.cuh"
#include "search_duo.cuh"
#include "kernels.h"
#include "scores.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define GR_CUDA(call)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess) {                                                            \
            return fail(e_ == cudaErrorMemoryAllocation ? GR_ENOMEM : GR_ECUDA,             \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                \
        }                                                                                   \
    } while (0)

int round4(int x) { return (x + 3) & ~3; }

uint16_t bf16_rne(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
float bf16_to_f(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
// hi/lo bf16 images of a [rows x K] fp32 operand in the UMMA K-major core-matrix layout
void pack_kmajor(const float *src, int rows, int K, int ld, int col0, uint8_t *hi, uint8_t *lo) {
    for (int r = 0; r < rows; ++r)
        for (int k = 0; k < K; ++k) {
            const float x = src[(size_t)r * ld + col0 + k];
            const uint16_t h = bf16_rne(x);
            const uint16_t l = bf16_rne(x - bf16_to_f(h));
            const uint32_t off = tc::kmaj_off(r, k, K);
            std::memcpy(hi + off, &h, 2);
            std::memcpy(lo + off, &l, 2);
        }
}
int odd(int x) { return x | 1; }
int pow2ceil(int x) {
    int p = 32;
    while (p < x) p <<= 1;
    return p;
}

template <class T>
int dmalloc(T **p, size_t count) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(GR_ENOMEM, std::string("cudaMalloc ") + std::to_string(count * sizeof(T)) +
                                   " bytes: " + cudaGetErrorString(e));
    }
    return GR_OK;
}

struct DevBuf {
    void *p = nullptr;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
    }
};

int num_sms(int device) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n > 0 ? n : 1;
}

} // namespace

// ------------------------------------------------------------------ handles
struct gr_model {
    int device;
    DevModel dm;
    void *dbuf;
    void *tcbuf[3] = {nullptr, nullptr, nullptr};
    std::vector<int> dims;
};

struct gr_graph {
    int device;
    DevGraph dg;
    std::vector<void *> bufs;
    int max_deg;
    int64_t max_row = 0;  // largest embedding row any slot reads (checked against the items)
    // bf16 hi/lo item rows in device-slot order for one items handle (built on first use),
    // so the scorer's gathers follow the graph's locality and need no row indirection.
    // hl_mu is held from the (re)build check until the search using it is enqueued, so a
    // rebuild for another items handle (which synchronises the device first) never
    // overwrites rows a queued search still reads.
    std::mutex hl_mu;
    uint64_t hl_serial = 0;
    int64_t hl_n = 0;
    int hl_d = 0;
    uint16_t *hl_slot = nullptr;
};

struct gr_items {
    int device;
    DevItems di;
    void *dbuf;
    void *hbuf = nullptr;
    uint64_t serial = 0;
};
static std::atomic<uint64_t> g_items_serial{0};

__global__ void gather_hl_kernel(const uint16_t *hl, const int32_t *rows, int64_t n, int d,
                                 uint16_t *out) {
    // one 16-byte piece per thread: row s of out = row rows[s] of hl ([n][2d] bf16)
    const int per = 2 * d / 8;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * per;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / per;
        const int c = (int)(i % per);
        reinterpret_cast<uint4 *>(out + s * 2 * d)[c] =
            reinterpret_cast<const uint4 *>(hl + (int64_t)rows[s] * 2 * d)[c];
    }
}

__global__ void split_items_kernel(const float *emb, int64_t n, int d, int ld, uint16_t *hl) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * d;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / d;
        const int c = (int)(i % d);
        const float x = emb[r * ld + c];
        const __nv_bfloat16 h = __float2bfloat16_rn(x);
        const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
        hl[r * 2 * d + c] = __bfloat16_as_ushort(h);
        hl[r * 2 * d + d + c] = __bfloat16_as_ushort(l);
    }
}

struct gr_scores {
    int device;
    int64_t Q = 0, n = 0;
    double *tab = nullptr;   // [Q][n] fp64 scores by item id
    uint32_t *code = nullptr; // [Q][n] per-query dense rank + 1 (scores.cuh)
};

struct gr_searcher {
    int device;
    // one search at a time per searcher: staging buffers, scratch and the status flags are
    // per searcher (ctypes releases the GIL, so Python threads can share one)
    std::mutex mu;
    // scratch reuse across streams: every launch waits for the previous one on this event
    cudaEvent_t done = nullptr;
    int64_t band_reruns = 0;
    int64_t slots = 0, n = 0, capF = 0, capS = 0, capP = 0;
    uint32_t *tags = nullptr;
    uint32_t *epochs = nullptr;
    int32_t *f_slot = nullptr, *f_srch = nullptr, *surv_v = nullptr, *surv_i = nullptr,
            *fr_v = nullptr, *fr_i = nullptr, *seg_v = nullptr, *pool_slot = nullptr;
    uint64_t *fr_key = nullptr, *seg_key = nullptr, *pool_key = nullptr;
    int32_t *pool_meta = nullptr;
    unsigned long long *counters = nullptr; // [4]: see SearchArgs::counters
    unsigned long long *phase = nullptr; // [8] when GMPGR_PHASE_TIMING=1
    int *flags = nullptr; // [0] queue, [1] nonfinite, [2] bad index, [3] band violations
    int64_t launches = 0;
    // duo-kernel scratch (search_duo.cuh): per unit lists, per query-slot bitsets/logs/pools
    struct Duo {
        int64_t units = 0, G = 0, capF = 0, capS = 0, capP = 0, hcap = 0, vwords = 0, logcap = 0;
        int32_t *f_slot = nullptr, *f_srch = nullptr, *surv_v = nullptr, *surv_i = nullptr,
                *cont_v = nullptr, *cont_i = nullptr, *fr_v = nullptr, *fr_i = nullptr,
                *seg_v = nullptr, *pool_slot = nullptr, *pool_meta = nullptr, *vlog = nullptr;
        uint64_t *fr_key = nullptr, *seg_key = nullptr, *pool_key = nullptr, *hash = nullptr;
        uint32_t *vis = nullptr;
        float4 *acc0 = nullptr;  // [units][G][64] hoisted user halves (tensor-core mode)
        size_t bytes = 0;
        void free_all() {
            void *ps[] = {f_slot, f_srch, surv_v, surv_i, cont_v, cont_i, fr_v, fr_i, seg_v, pool_slot,
                          pool_meta, vlog, fr_key, seg_key, pool_key, hash, vis, acc0};
            for (void *p : ps)
                if (p) cudaFree(p);
            *this = Duo();
        }
    } duo;
    int64_t duo_units_last = 0;  // resident units of the last duo launch (bench / tests)
    // streamed host calls (gr_search with host buffers): copy-in / copy-out streams that run
    // beside the kernel, chunk flags (avail, qdone[]) and their events
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_reset = nullptr, ev_out = nullptr;
    int *sflags = nullptr;  // [0] avail, [1 + c] queries finished in chunk c
    // staging for host-pointer calls
    DevBuf st_users, st_ids, st_scores, st_count, st_stats;
    size_t st_users_n = 0, st_out_n = 0, st_stats_n = 0;
    void free_scratch() {
        void *ps[] = {tags, epochs, f_slot, f_srch, surv_v, surv_i, fr_v, fr_i, seg_v, pool_slot,
                      fr_key, seg_key, pool_key, pool_meta};
        for (void *p : ps)
            if (p) cudaFree(p);
        tags = nullptr; epochs = nullptr; f_slot = f_srch = surv_v = surv_i = fr_v = fr_i = seg_v =
            pool_slot = nullptr;
        fr_key = seg_key = pool_key = nullptr;
        pool_meta = nullptr;
        slots = n = capF = capS = capP = 0;
    }
};

extern "C" {

const char *gr_last_error(void) { return g_err.c_str(); }
int gr_abi_version(void) { return GR_ABI_VERSION; }
int gr_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// ------------------------------------------------------------------ model
int gr_model_create(int device, int n_mlp, const int32_t *dims, const float *const *W,
                    const float *const *b, const float *attention, int relu, gr_model **out) {
    if (!out || !dims || !W || !b || !attention) return fail(GR_EINVAL, "null argument");
    if (n_mlp < 1 || n_mlp > GR_MAX_MLP) return fail(GR_EINVAL, "n_mlp out of range [1, 6]");
    if (dims[0] < 2 || dims[0] % 2) return fail(GR_EINVAL, "dims[0] must be 2*d_h");
    for (int m = 0; m <= n_mlp; ++m)
        if (dims[m] < 1 || dims[m] > 2048) return fail(GR_EINVAL, "layer width out of range");
    GR_CUDA(cudaSetDevice(device));
    // processing-order packing (common.cuh)
    std::vector<float> host;
    std::vector<size_t> offW(n_mlp), offb(n_mlp);
    for (int m = 0; m < n_mlp; ++m) {
        const int K = dims[m], O = dims[m + 1], nch = n_chunks(K);
        offW[m] = host.size();
        host.resize(host.size() + (size_t)nch * O * 4, 0.f);
        float *dst = host.data() + offW[m];
        for (int j = 0; j < nch; ++j) {
            const int c = chunk_perm(j, K);
            for (int o = 0; o < O; ++o)
                for (int u = 0; u < 4; ++u) {
                    const int kk = 4 * c + u;
                    dst[((size_t)j * O + o) * 4 + u] = kk < K ? W[m][(size_t)o * K + kk] : 0.f;
                }
        }
        offb[m] = host.size();
        host.resize(host.size() + round4(O), 0.f);
        std::memcpy(host.data() + offb[m], b[m], sizeof(float) * O);
    }
    const int Z = dims[n_mlp], nchA = n_chunks(Z);
    const size_t offA = host.size();
    host.resize(host.size() + (size_t)nchA * 4, 0.f);
    for (int j = 0; j < nchA; ++j) {
        const int c = chunk_perm(j, Z);
        for (int u = 0; u < 4; ++u) {
            const int kk = 4 * c + u;
            host[offA + (size_t)j * 4 + u] = kk < Z ? attention[kk] : 0.f;
        }
    }
    gr_model *M = new gr_model();
    M->device = device;
    M->dims.assign(dims, dims + n_mlp + 1);
    float *d = nullptr;
    int rc = dmalloc(&d, host.size());
    if (rc) { delete M; return rc; }
    cudaError_t e = cudaMemcpy(d, host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(d); delete M; return fail(GR_ECUDA, cudaGetErrorString(e)); }
    M->dbuf = d;
    DevModel &dm = M->dm;
    std::memset(&dm, 0, sizeof(dm));
    // tensor-core operand images (TcMlp shape: 3 layers, hidden 64/64, d_h in {64,128}, Z 2..3)
    const int dh = dims[0] / 2;
    if (n_mlp == 3 && relu && dims[1] == 64 && dims[2] == 64 && (dh == 64 || dh == 128) &&
        (Z == 2 || Z == 3)) {
        const size_t b0 = (size_t)64 * dh * 2, b1 = (size_t)64 * 64 * 2;
        std::vector<uint8_t> img(2 * b0 + 2 * b1, 0);
        pack_kmajor(W[0], 64, dh, 2 * dh, dh, img.data(), img.data() + b0);
        pack_kmajor(W[1], 64, 64, 64, 0, img.data() + 2 * b0, img.data() + 2 * b0 + b1);
        std::vector<float> misc(64 + 64 * Z + 8, 0.f);
        std::memcpy(misc.data(), b[1], 64 * 4);
        std::memcpy(misc.data() + 64, W[2], (size_t)64 * Z * 4);
        std::memcpy(misc.data() + 64 + 64 * Z, b[2], (size_t)Z * 4);
        std::memcpy(misc.data() + 68 + 64 * Z, attention, (size_t)Z * 4);
        uint8_t *dimg = nullptr;
        float *dmisc = nullptr;
        if (dmalloc(&dimg, img.size()) || dmalloc(&dmisc, misc.size())) {
            cudaFree(d); delete M; return GR_ENOMEM;
        }
        cudaMemcpy(dimg, img.data(), img.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dmisc, misc.data(), misc.size() * 4, cudaMemcpyHostToDevice);
        M->tcbuf[0] = dimg;
        M->tcbuf[1] = dmisc;
        dm.tcB = dimg;
        dm.tcMisc = dmisc;
        dm.tc_ok = 1;
        // exact weight block (FixedMlp / ExactQ layout): W0 item half, W1, W2, A, b0, b1, b2
        const int pre = 4 * (dh / 16), nch0 = n_chunks(2 * dh), nchz = n_chunks(Z);
        std::vector<float> ex;
        auto put4 = [&](const float *src, size_t nf4) { ex.insert(ex.end(), src, src + nf4 * 4); };
        put4(host.data() + offW[0] + (size_t)pre * 64 * 4, (size_t)(nch0 - pre) * 64);
        put4(host.data() + offW[1], (size_t)16 * 64);
        put4(host.data() + offW[2], (size_t)16 * Z);
        put4(host.data() + offA, (size_t)nchz);
        put4(host.data() + offb[0], 16);
        put4(host.data() + offb[1], 16);
        put4(host.data() + offb[2], (size_t)nchz);
        float *dex = nullptr;
        if (dmalloc(&dex, ex.size())) { cudaFree(d); delete M; return GR_ENOMEM; }
        cudaMemcpy(dex, ex.data(), ex.size() * 4, cudaMemcpyHostToDevice);
        M->tcbuf[2] = dex;
        dm.exBlock = dex;
    }
    dm.n_mlp = n_mlp;
    dm.relu = relu ? 1 : 0;
    dm.d_h = dims[0] / 2;
    dm.Z = Z;
    for (int m = 0; m <= n_mlp; ++m) { dm.dims[m] = dims[m]; dm.nch[m] = n_chunks(dims[m]); }
    for (int m = 0; m < n_mlp; ++m) {
        dm.W[m] = reinterpret_cast<const float4 *>(d + offW[m]);
        dm.b[m] = d + offb[m];
    }
    dm.A = reinterpret_cast<const float4 *>(d + offA);
    dm.pre_ch = 4 * (dm.d_h / 16);
    *out = M;
    return GR_OK;
}

int gr_model_destroy(gr_model *m) {
    if (!m) return GR_OK;
    cudaSetDevice(m->device);
    cudaFree(m->dbuf);
    if (m->tcbuf[0]) cudaFree(m->tcbuf[0]);
    if (m->tcbuf[1]) cudaFree(m->tcbuf[1]);
    if (m->tcbuf[2]) cudaFree(m->tcbuf[2]);
    delete m;
    return GR_OK;
}

// ------------------------------------------------------------------ graph
int gr_graph_create(int device, int n_layers, int64_t n, const int32_t *const *nbrs,
                    const int64_t *row_stride, const int32_t *const *cnts, const int32_t *levels,
                    int32_t entry_slot, const int64_t *ids, const int32_t *rows, gr_graph **out) {
    return gr_graph_create_ordered(device, n_layers, n, nbrs, row_stride, cnts, levels, entry_slot, ids, rows,
                                   nullptr, out);
}

int gr_graph_create_ordered(int device, int n_layers, int64_t n, const int32_t *const *nbrs,
                            const int64_t *row_stride, const int32_t *const *cnts, const int32_t *levels,
                            int32_t entry_slot, const int64_t *ids, const int32_t *rows, const int64_t *order,
                            gr_graph **out) {
    if (!out || !nbrs || !row_stride || !cnts || !ids) return fail(GR_EINVAL, "null argument");
    if (n < 1) return fail(GR_EINVAL, "index is empty");
    if (n > 0x7ffffff0LL) return fail(GR_EINVAL, "more than 2^31 slots");
    if (n_layers < 1 || n_layers > GR_MAX_LAYERS) return fail(GR_EINVAL, "n_layers out of range [1, 8]");
    if (entry_slot < 0 || entry_slot >= n) return fail(GR_EINVAL, "entry_slot out of range");
    GR_CUDA(cudaSetDevice(device));
    gr_graph *G = new gr_graph();
    G->device = device;
    DevGraph &dg = G->dg;
    std::memset(&dg, 0, sizeof(dg));
    dg.n_layers = n_layers;
    dg.n = n;
    dg.entry = entry_slot;
    G->max_deg = 0;
    auto cleanup = [&](int rc) {
        for (void *p : G->bufs) cudaFree(p);
        delete G;
        return rc;
    };
    for (int l = 0; l < n_layers; ++l)
        if (row_stride[l] < 0 || row_stride[l] > 4096) return cleanup(fail(GR_EINVAL, "row stride out of range"));
    // Device slot order: breadth-first from the entry over layer 0 (GMPGR_REORDER=0 keeps the
    // caller's order).  Graph neighbours get nearby device slots, so the per-query visited
    // tags and adjacency rows they touch share L2 lines.  Invisible to callers: results are
    // reported by id and every tie-break uses the id rank, never the slot.
    std::vector<int64_t> perm;  // device slot -> caller slot (empty = identity)
    std::vector<int32_t> inv;   // caller slot -> device slot
    if (order) {  // caller-provided locality order (a permutation of the slots)
        perm.assign(order, order + n);
        inv.assign(n, -1);
        for (int64_t s = 0; s < n; ++s) {
            const int64_t o = perm[s];
            if (o < 0 || o >= n || inv[o] >= 0) return cleanup(fail(GR_EINVAL, "order is not a permutation of the slots"));
            inv[o] = (int32_t)s;
        }
    } else {
        const char *renv = getenv("GMPGR_REORDER");
        if (!(renv && std::strcmp(renv, "0") == 0) && n > 1) {
            perm.reserve(n);
            inv.assign(n, -1);
            const int64_t st0 = row_stride[0];
            auto visit_from = [&](int64_t root) {
                size_t head = perm.size();
                inv[root] = (int32_t)perm.size();
                perm.push_back(root);
                while (head < perm.size()) {
                    const int64_t o = perm[head++];
                    const int32_t c = cnts[0][o];
                    if (c <= 0 || c > st0) continue;
                    const int32_t *src = nbrs[0] + o * st0;
                    for (int j = 0; j < c; ++j) {
                        const int32_t v = src[j];
                        if (v >= 0 && v < n && inv[v] < 0) {
                            inv[v] = (int32_t)perm.size();
                            perm.push_back(v);
                        }
                    }
                }
            };
            visit_from(entry_slot);
            for (int64_t o = 0; o < n; ++o)
                if (inv[o] < 0) visit_from(o);
        }
    }
    const bool re = !perm.empty();
    auto old_of = [&](int64_t s) { return re ? perm[s] : s; };
    auto new_of = [&](int32_t o) { return re ? inv[o] : o; };
    dg.entry = new_of(entry_slot);
    // upper-layer membership: level >= 1 (index.py:77, nesting); fall back to "has edges"
    std::vector<int32_t> up_row(n, -1);
    int64_t n_up = 0;
    if (n_layers > 1) {
        for (int64_t s = 0; s < n; ++s) {
            const int64_t o = old_of(s);
            bool member = levels ? levels[o] >= 1 : false;
            if (!levels)
                for (int l = 1; l < n_layers; ++l) member |= cnts[l][o] > 0;
            if (member) up_row[s] = (int32_t)n_up++;
        }
    }
    for (int l = 0; l < n_layers; ++l) {
        const int64_t stride = row_stride[l];
        const int deg = (int)std::max<int64_t>(stride, 1);
        const int ld = round4(deg);
        const int64_t nrows = l == 0 ? n : std::max<int64_t>(n_up, 1);
        std::vector<int32_t> h((size_t)nrows * ld, -1);
        for (int64_t s = 0; s < n; ++s) {
            const int64_t o = old_of(s);
            const int32_t c = cnts[l][o];
            if (c == 0) continue;
            if (c < 0 || c > stride)
                return cleanup(fail(GR_EINVAL, "layer " + std::to_string(l) + " slot " +
                                                   std::to_string(o) + ": bad neighbour count"));
            int64_t r = l == 0 ? s : up_row[s];
            if (r < 0) continue; // not a member of this layer: never expanded
            const int32_t *src = nbrs[l] + o * stride;
            for (int j = 0; j < c; ++j) {
                if (src[j] < 0 || src[j] >= n)
                    return cleanup(fail(GR_EINVAL, "neighbour slot out of range"));
                h[(size_t)r * ld + j] = new_of(src[j]);
            }
        }
        int32_t *d = nullptr;
        if (int rc = dmalloc(&d, h.size())) return cleanup(rc);
        G->bufs.push_back(d);
        if (cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
            return cleanup(fail(GR_ECUDA, "graph upload failed"));
        dg.adj[l] = d;
        dg.ld[l] = ld;
        dg.deg[l] = deg;
        G->max_deg = std::max(G->max_deg, deg);
    }
    {
        int32_t *d = nullptr;
        if (int rc = dmalloc(&d, n)) return cleanup(rc);
        G->bufs.push_back(d);
        cudaMemcpy(d, up_row.data(), n * 4, cudaMemcpyHostToDevice);
        dg.up_row = d;
    }
    {
        int64_t *d = nullptr;
        if (int rc = dmalloc(&d, n)) return cleanup(rc);
        G->bufs.push_back(d);
        if (re) {
            std::vector<int64_t> ids_dev(n);
            for (int64_t s = 0; s < n; ++s) ids_dev[s] = ids[perm[s]];
            cudaMemcpy(d, ids_dev.data(), n * 8, cudaMemcpyHostToDevice);
        } else {
            cudaMemcpy(d, ids, n * 8, cudaMemcpyHostToDevice);
        }
        dg.ids = d;
    }
    // embedding rows: explicit, else ids (model_scorer convention); identity -> nullptr
    {
        std::vector<int32_t> r(n);
        bool ident = true;
        for (int64_t s = 0; s < n; ++s) {
            const int64_t o = old_of(s);
            const int64_t v = rows ? (int64_t)rows[o] : ids[o];
            if (v < 0 || v > 0x7fffffffLL)
                return cleanup(fail(GR_EINVAL, "item ids must be row indexes >= 0 (search.py:84-90)"));
            r[s] = (int32_t)v;
            ident &= (v == s);
            G->max_row = std::max<int64_t>(G->max_row, v);
        }
        if (!ident) {
            int32_t *d = nullptr;
            if (int rc = dmalloc(&d, n)) return cleanup(rc);
            G->bufs.push_back(d);
            cudaMemcpy(d, r.data(), n * 4, cudaMemcpyHostToDevice);
            dg.rows = d;
        }
    }
    // tie-break rank: slot when ids ascend, else rank of id
    {
        auto id_of = [&](int64_t s) { return ids[old_of(s)]; };
        bool mono = true;
        for (int64_t s = 1; s < n && mono; ++s) mono = id_of(s) > id_of(s - 1);
        if (!mono) {
            std::vector<int64_t> order(n);
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(),
                             [&](int64_t a, int64_t b) {
                                 const int64_t ia = id_of(a), ib = id_of(b);
                                 return ia < ib || (ia == ib && old_of(a) < old_of(b));
                             });
            std::vector<uint32_t> rank(n);
            for (int64_t i = 0; i < n; ++i) rank[order[i]] = (uint32_t)i;
            uint32_t *d = nullptr;
            if (int rc = dmalloc(&d, n)) return cleanup(rc);
            G->bufs.push_back(d);
            cudaMemcpy(d, rank.data(), n * 4, cudaMemcpyHostToDevice);
            dg.rank = d;
        }
    }
    GR_CUDA(cudaDeviceSynchronize());
    *out = G;
    return GR_OK;
}

int gr_graph_destroy(gr_graph *g) {
    if (!g) return GR_OK;
    cudaSetDevice(g->device);
    for (void *p : g->bufs) cudaFree(p);
    if (g->hl_slot) cudaFree(g->hl_slot);
    delete g;
    return GR_OK;
}

// ------------------------------------------------------------------ items
int gr_items_create(int device, const float *emb, int64_t n, int32_t d, int emb_on_device,
                    gr_items **out) {
    if (!out || !emb) return fail(GR_EINVAL, "null argument");
    if (n < 1 || d < 1) return fail(GR_EINVAL, "empty item embeddings");
    GR_CUDA(cudaSetDevice(device));
    const int ld = round4(d);
    float *p = nullptr;
    if (int rc = dmalloc(&p, (size_t)n * ld)) return rc;
    if (ld != d) cudaMemset(p, 0, (size_t)n * ld * 4);
    cudaError_t e = cudaMemcpy2D(p, (size_t)ld * 4, emb, (size_t)d * 4, (size_t)d * 4, n,
                                 emb_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(p); return fail(GR_ECUDA, cudaGetErrorString(e)); }
    // bf16 hi/lo copy for the pipelined tensor-core scorer (cp.async-able, no conversion
    // on the search path); items are immutable for the handle's lifetime
    uint16_t *hl = nullptr;
    if (d % 64 == 0 && d <= 128) {
        if (int rc = dmalloc(&hl, (size_t)n * 2 * d)) { cudaFree(p); return rc; }
        const int64_t total = n * d;
        split_items_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 64), 256>>>(p, n, d, ld, hl);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { cudaFree(p); cudaFree(hl); return fail(GR_ECUDA, cudaGetErrorString(e)); }
    }
    gr_items *I = new gr_items();
    I->device = device;
    I->di.emb = p;
    I->di.n = n;
    I->di.d = d;
    I->di.ld = ld;
    I->di.hl = hl;
    I->dbuf = p;
    I->hbuf = hl;
    I->serial = ++g_items_serial;
    *out = I;
    return GR_OK;
}

int gr_items_destroy(gr_items *it) {
    if (!it) return GR_OK;
    cudaSetDevice(it->device);
    cudaFree(it->dbuf);
    if (it->hbuf) cudaFree(it->hbuf);
    delete it;
    return GR_OK;
}

} // extern "C"

// ------------------------------------------------------------------ layouts
namespace {

struct SmemPlan {
    int bytes = 0;
    int alloc(int nbytes) {
        int off = bytes;
        bytes += (nbytes + 15) & ~15;
        return off;
    }
};

// weights for layers >= 1 + biases + attention (shared by all kernels)
void plan_weights(const DevModel &M, SmemPlan &P, int *off_w, int *off_b, int *off_A) {
    for (int m = 0; m < M.n_mlp; ++m) {
        off_w[m] = m >= 1 ? P.alloc(M.nch[m] * M.dims[m + 1] * 16) : 0;
        off_b[m] = P.alloc(round4(M.dims[m + 1]) * 4);
    }
    *off_A = P.alloc(M.nch[M.n_mlp] * 16);
}

int hidden_ld(const DevModel &M) {
    int mx = 1;
    for (int m = 1; m <= M.n_mlp; ++m) mx = std::max(mx, M.nch[m]);
    return odd(mx);
}

// which compile-time scorer fits this model (0: generic)
int fixed_shape(const DevModel &M) {
    if (M.n_mlp != 3 || !M.relu || M.dims[1] != 64 || M.dims[2] != 64) return 0;
    const int dh = M.d_h, z = M.Z;
    if ((dh == 128 || dh == 64) && (z == 2 || z == 3)) return dh * 10 + z;
    return 0;
}

template <int DH, int ZZ>
void plan_fixed(SearchArgs &a) {
    using F = FixedMlp<DH, ZZ>;
    a.off_w0 = F::OFF_W0 * 16;
    a.off_w[0] = 0;
    a.off_w[1] = F::OFF_W1 * 16;
    a.off_w[2] = F::OFF_W2 * 16;
    a.off_b[0] = F::OFF_B0 * 16;
    a.off_b[1] = F::OFF_B1 * 16;
    a.off_b[2] = F::OFF_B2 * 16;
    a.off_A = F::OFF_A * 16;
    a.off_acc0 = F::OFF_ACC0 * 16;
    a.off_x0 = F::OFF_X0 * 16;
    a.ldx0 = F::LDX0;
    a.off_h0 = F::OFF_H0 * 16;
    a.off_h1 = F::OFF_H1 * 16;
    a.ldh = F::LDH;
    a.off_score = F::OFF_SCORE * 16;
}

template <int DH, int ZZ>
void plan_tc(SearchArgs &a, SmemPlan &P) {
    using T = TcMlp<DH, ZZ>;
    a.off_acc0 = T::OFF_ACC0;
    P.bytes = T::BYTES;
}

int plan_search(const DevModel &M, int k, int kp, SearchArgs &a, int shape, int mode) {
    SmemPlan P;
    if (mode == GR_MODE_TC) {
        switch (shape) {
        case 1283: plan_tc<128, 3>(a, P); break;
        case 1282: plan_tc<128, 2>(a, P); break;
        case 643: plan_tc<64, 3>(a, P); break;
        default: plan_tc<64, 2>(a, P); break;
        }
    } else if (shape) {
        switch (shape) {
        case 1283: plan_fixed<128, 3>(a); P.bytes = FixedMlp<128, 3>::TOTAL * 16; break;
        case 1282: plan_fixed<128, 2>(a); P.bytes = FixedMlp<128, 2>::TOTAL * 16; break;
        case 643: plan_fixed<64, 3>(a); P.bytes = FixedMlp<64, 3>::TOTAL * 16; break;
        default: plan_fixed<64, 2>(a); P.bytes = FixedMlp<64, 2>::TOTAL * 16; break;
        }
    } else {
        const int x0_nch = M.nch[0] - M.pre_ch;
        a.off_w0 = P.alloc(x0_nch * M.dims[1] * 16);
        plan_weights(M, P, a.off_w, a.off_b, &a.off_A);
        a.off_acc0 = P.alloc(M.dims[1] * 16);
        a.ldx0 = odd(x0_nch);
        a.off_x0 = P.alloc(GR_PT * a.ldx0 * 16);
        a.ldh = hidden_ld(M);
        a.off_h0 = P.alloc(GR_PT * a.ldh * 16);
        a.off_h1 = P.alloc(GR_PT * a.ldh * 16);
        a.off_score = P.alloc(GR_PT * 4);
    }
    a.off_hist = P.alloc(GR_NW * 256 * 4);
    a.sortcap = pow2ceil(std::max(k, kp));
    a.off_sortk = P.alloc(a.sortcap * 8);
    a.off_sortv = P.alloc(a.sortcap * 4);
    a.off_kp = P.alloc(3 * kp * 4);
    return P.bytes;
}

int plan_pairs(const DevModel &M, PairArgs &a) {
    SmemPlan P;
    for (int m = 0; m < M.n_mlp; ++m) {
        a.off_w[m] = P.alloc(M.nch[m] * M.dims[m + 1] * 16);
        a.off_b[m] = P.alloc(round4(M.dims[m + 1]) * 4);
    }
    a.off_A = P.alloc(M.nch[M.n_mlp] * 16);
    a.ldx0 = odd(M.nch[0]);
    a.off_x0 = P.alloc(GR_PT * a.ldx0 * 16);
    a.ldh = hidden_ld(M);
    a.off_h0 = P.alloc(GR_PT * a.ldh * 16);
    a.off_h1 = P.alloc(GR_PT * a.ldh * 16);
    a.off_score = P.alloc(GR_PT * 4);
    return P.bytes;
}

int plan_brute(const DevModel &M, BruteArgs &a) {
    SmemPlan P;
    const int x0_nch = M.nch[0] - M.pre_ch;
    a.off_w0 = P.alloc(x0_nch * M.dims[1] * 16);
    plan_weights(M, P, a.off_w, a.off_b, &a.off_A);
    a.off_acc0 = P.alloc(M.dims[1] * 16);
    a.ldx0 = odd(x0_nch);
    a.off_x0 = P.alloc(GR_PT * a.ldx0 * 16);
    a.ldh = hidden_ld(M);
    a.off_h0 = P.alloc(GR_PT * a.ldh * 16);
    a.off_h1 = P.alloc(GR_PT * a.ldh * 16);
    a.off_score = P.alloc(GR_PT * 4);
    a.off_hist = P.alloc(256 * 4);
    return P.bytes;
}

const int kMaxSmem = 227 * 1024;

template <class K>
int set_smem(K kernel, int bytes) {
    if (bytes > kMaxSmem) return fail(GR_EINVAL, "model too large for shared memory");
    GR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    // prefer the largest shared-memory carveout so two ~100 KB CTAs co-reside per SM
    GR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    return GR_OK;
}

// staging helper for host-pointer calls
template <class T>
int stage(DevBuf &buf, size_t &cap, size_t count) {
    if (count <= cap && buf.p) return GR_OK;
    buf.release();
    T *p = nullptr;
    if (int rc = dmalloc(&p, count)) return rc;
    buf.p = p;
    cap = count;
    return GR_OK;
}

int ensure_search_scratch(gr_searcher *S, const gr_graph *G, int64_t slots, int64_t capF,
                          int64_t capS, int64_t capP) {
    const int64_t n = G->dg.n;
    if (S->slots >= slots && S->n == n && S->capF >= capF && S->capS >= capS && S->capP >= capP)
        return GR_OK;
    slots = std::max(slots, S->slots);
    capF = std::max(capF, S->capF);
    capS = std::max(capS, S->capS);
    capP = std::max(capP, S->capP);
    S->free_scratch();
    int rc = GR_OK;
    if ((rc = dmalloc(&S->tags, (size_t)slots * n))) return rc;
    if ((rc = dmalloc(&S->epochs, (size_t)slots))) return rc;
    if ((rc = dmalloc(&S->f_slot, (size_t)slots * 2 * capF))) return rc;
    if ((rc = dmalloc(&S->f_srch, (size_t)slots * 2 * capF))) return rc;
    if ((rc = dmalloc(&S->surv_v, (size_t)slots * capS))) return rc;
    if ((rc = dmalloc(&S->surv_i, (size_t)slots * capS))) return rc;
    if ((rc = dmalloc(&S->fr_v, (size_t)slots * capS))) return rc;
    if ((rc = dmalloc(&S->fr_i, (size_t)slots * capS))) return rc;
    if ((rc = dmalloc(&S->fr_key, (size_t)slots * capS))) return rc;
    if ((rc = dmalloc(&S->seg_v, (size_t)slots * capS))) return rc;
    if ((rc = dmalloc(&S->seg_key, (size_t)slots * capS))) return rc;
    if ((rc = dmalloc(&S->pool_key, (size_t)slots * 2 * capP))) return rc;
    if ((rc = dmalloc(&S->pool_slot, (size_t)slots * 2 * capP))) return rc;
    if ((rc = dmalloc(&S->pool_meta, (size_t)slots * 2 * capP))) return rc;
    GR_CUDA(cudaMemset(S->tags, 0, (size_t)slots * n * 4));
    GR_CUDA(cudaMemset(S->epochs, 0, (size_t)slots * 4));
    S->slots = slots;
    S->n = n;
    S->capF = capF;
    S->capS = capS;
    S->capP = capP;
    return GR_OK;
}

int check_params(const gr_search_params *p) {
    if (!p) return fail(GR_EINVAL, "null params");
    if (p->k < 1 || p->k_parallel < 1 || p->hops < 1)
        return fail(GR_EINVAL, "k, k_parallel, and hops must be >= 1");
    if (p->k_parallel > p->k) return fail(GR_EINVAL, "k_parallel must not exceed k");
    if (p->ef < 1) return fail(GR_EINVAL, "ef must be >= 1");
    if (p->k > 8192) return fail(GR_EINVAL, "k > 8192 not supported on the device path");
    if (p->mode != GR_MODE_EXACT && p->mode != GR_MODE_TC) return fail(GR_EINVAL, "unknown mode");
    if (p->k_parallel > 4094) return fail(GR_EINVAL, "k_parallel > 4094 not supported (claim tag width)");
    return GR_OK;
}

template <int DH, int ZZ, int MODE, int NT, int G, int KC, bool PIPE = false>
int plan_mq(int k, int kp, SearchArgs &a) {
    using EX = ExactQ<DH, ZZ, NT / 32>;
    using TC = TcQ<DH, ZZ, NT, G, KC>;
    using TP = TcPipe<DH, ZZ, G>;
    SmemPlan P;
    a.sortcap = pow2ceil(std::max(k, kp));
    const int hist_b = (NT / 32) * 256 * 4, sortk_b = G * a.sortcap * 8, sortv_b = G * a.sortcap * 4;
    if (MODE == 1 && PIPE) {
        static_assert(TP::A_REGION >= EX::BUF_END * 16 || !PIPE, "exact buffers must fit the A region");
        a.off_w0 = 0;
        a.off_A = P.alloc(TP::BYTES);
        // the A-operand stages are dead outside the scoring pipeline: the exact re-scoring
        // buffers, the radix-select histograms and the pool sort alias them when they fit
        a.off_x0 = a.off_A + TP::OFF_A;
        const int h = a.off_x0 + ((EX::BUF_END * 16 + 15) & ~15);
        const int sk = h + hist_b, sv = sk + sortk_b;
        if (sv + sortv_b <= a.off_A + TP::OFF_A + TP::A_REGION) {
            a.off_hist = h;
            a.off_sortk = sk;
            a.off_sortv = sv;
        } else {
            a.off_hist = P.alloc(hist_b);
            a.off_sortk = P.alloc(sortk_b);
            a.off_sortv = P.alloc(sortv_b);
        }
        a.off_acc0 = P.alloc(G * 64 * 16);
        a.off_kp = P.alloc(3 * G * kp * 4);
        return P.bytes + 1024;  // slack for the kernel's 1024-byte alignment of the carve
    }
    a.off_w0 = NT >= 512 ? P.alloc(EX::W_END * 16) : 0;
    a.off_x0 = P.alloc(std::max(EX::BUF_END * 16, MODE == 1 ? TC::A_BYTES : 0));
    a.off_A = MODE == 1 ? P.alloc(TC::BYTES) : 0;
    a.off_acc0 = P.alloc(G * 64 * 16);
    a.off_hist = P.alloc(hist_b);
    a.off_sortk = P.alloc(sortk_b);
    a.off_sortv = P.alloc(sortv_b);
    a.off_kp = P.alloc(3 * G * kp * 4);
    return P.bytes;
}

// Caller holds G->hl_mu until its search is enqueued.
int ensure_slot_hl(gr_graph *G, const gr_items *I, cudaStream_t stream) {
    if (G->hl_slot && G->hl_serial == I->serial) return GR_OK;
    if (G->max_row >= I->di.n) return fail(GR_EINVAL, "items table smaller than the graph");
    // searches queued on any stream may still read the current copy
    GR_CUDA(cudaDeviceSynchronize());
    if (G->hl_slot && (G->hl_n != G->dg.n || G->hl_d != I->di.d)) {
        cudaFree(G->hl_slot);
        G->hl_slot = nullptr;
    }
    if (!G->hl_slot) {
        if (int rc = dmalloc(&G->hl_slot, (size_t)G->dg.n * 2 * I->di.d)) return rc;
        G->hl_n = G->dg.n;
        G->hl_d = I->di.d;
    }
    const int64_t work = G->dg.n * (2 * I->di.d / 8);
    gather_hl_kernel<<<(unsigned)std::min<int64_t>((work + 255) / 256, 148 * 64), 256, 0, stream>>>(
        I->di.hl, G->dg.rows, G->dg.n, I->di.d, G->hl_slot);
    GR_CUDA(cudaGetLastError());
    G->hl_serial = I->serial;
    return GR_OK;
}

// Tensor map over a bf16 hi/lo item table [rows][2d] for the TMA gather4 loader: 64-element
// (128-byte) boxes of one row, 128-byte swizzle.  cuTensorMapEncodeTiled comes from the driver
// through the runtime's entry-point query (no -lcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int make_hl_map(CUtensorMap *map, const uint16_t *hl, int64_t rows, int d) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        GR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) return fail(GR_ECUDA, "cuTensorMapEncodeTiled not available");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)(2 * d), (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(2 * d) * 2};
    const cuuint32_t box[2] = {64, 1}, estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t *>(hl), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(GR_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return GR_OK;
}

bool env_flag(const char *name, bool dflt) {
    const char *v = std::getenv(name);
    if (!v || !*v) return dflt;
    return v[0] != '0';
}

// multi-query kernel for the fixed model shapes (search_mq.cuh); returns -1 if not applicable
int launch_mq(gr_searcher *S, const gr_graph *G, const gr_model *M, const gr_items *I,
              const float *users, int64_t Q, const gr_search_params *p, int64_t *ids,
              double *scores, int32_t *count, int64_t *stats, cudaStream_t stream, int shape) {
    SearchArgs a;
    std::memset(&a, 0, sizeof(a));
    const int mode = p->mode;
    // One 512-thread CTA per SM, 16 (tc) or 8 (exact) queries in lock-step.  Tensor-core mode runs the
    // warp-specialised tcgen05 scoring pipeline (tc_pipe.cuh) and needs the bf16 hi/lo item
    // copy; without it the per-query kernel (search_kernel.cuh) runs.  Measured on cfg3
    // (65,536 queries, tc): 2x256-thread CTAs x 2 queries 854 ms, 1x512 x 4 queries 590 ms,
    // 8 queries +6%, lock-step tile scorer 374 ms -> pipelined scorer 273 ms -> + BFS slot
    // order 237 ms (those variants were retired from the build).
    if (mode == GR_MODE_TC && I->di.hl == nullptr) return -1;
    const bool pipe = mode == GR_MODE_TC;
    // tensor-core mode advances 16 queries per CTA (cfg3: 234.6 -> 221.5 ms vs 8) once the
    // batch fills every SM twice over; smaller batches use 8 (more CTAs busy); exact mode 8
    // re-score requests pack (query slot << 24 | index) with index < capS * G (CTA-level
    // segment arrays) or < capP (per-query pools): larger budgets take the per-query kernel
    const int64_t capS_q = std::max<int64_t>(std::min<int64_t>((int64_t)p->k_parallel * p->ef * G->max_deg,
                                                               (int64_t)p->k_parallel * G->dg.n),
                                             G->max_deg + 1) + 64;
    const int64_t capP_q = p->k + capS_q;
    if (capS_q * 8 >= (1 << 24) || capP_q >= (1 << 24)) return -1;
    const bool g16 = pipe && Q >= 2 * 16 * (int64_t)num_sms(G->device) && capS_q * 16 < (1 << 24);
    int smem = 0, nthreads = 512, gq = g16 ? 16 : 8;
    void (*kern)(const SearchArgs) = nullptr;
#define GR_MQ_CASE(CODE, DH, ZZ)                                                                   \
    case CODE:                                                                                     \
        if (g16) {                                                                                 \
            smem = plan_mq<DH, ZZ, 1, 512, 16, DH, true>(p->k, p->k_parallel, a);                  \
            kern = mq_kernel<DH, ZZ, 1, 512, 16, DH, true>();                                \
        } else if (pipe) {                                                                         \
            smem = plan_mq<DH, ZZ, 1, 512, 8, DH, true>(p->k, p->k_parallel, a);                   \
            kern = mq_kernel<DH, ZZ, 1, 512, 8, DH, true>();                                 \
        } else {                                                                                   \
            smem = plan_mq<DH, ZZ, 0, 512, 8, DH>(p->k, p->k_parallel, a);                         \
            kern = mq_kernel<DH, ZZ, 0, 512, 8, DH, false>();                                \
        }                                                                                          \
        break;
    switch (shape) {
        GR_MQ_CASE(1283, 128, 3)
        GR_MQ_CASE(1282, 128, 2)
        GR_MQ_CASE(643, 64, 3)
        GR_MQ_CASE(642, 64, 2)
    default: return -1;
    }
#undef GR_MQ_CASE
    const int G_ = gq;
    if (smem > kMaxSmem) return -1;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 0;
    GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthreads, smem));
    if (per_sm < 1) return -1;
    const int64_t blocks = std::min<int64_t>((Q + G_ - 1) / G_, (int64_t)per_sm * num_sms(G->device));
    const int64_t capF = (int64_t)p->k_parallel * p->ef;
    const int64_t capS = capS_q, capP = capP_q;
    if (int rc = ensure_search_scratch(S, G, blocks * G_, capF, capS, capP)) return rc;
    a.g = G->dg;
    a.M = M->dm;
    a.it = I->di;
    std::unique_lock<std::mutex> hl_lock;
    if (pipe && mode == GR_MODE_TC && G->dg.rows) {
        hl_lock = std::unique_lock<std::mutex>(const_cast<gr_graph *>(G)->hl_mu);
        if (int rc = ensure_slot_hl(const_cast<gr_graph *>(G), I, stream)) return rc;
        a.it.hl = G->hl_slot;
        a.it.hl_by_slot = 1;
    }
    if (pipe && env_flag("GMPGR_TMA", true)) {  // GMPGR_TMA=0: cp.async loaders
        const int64_t rows = a.it.hl_by_slot ? G->dg.n : I->di.n;
        if (int rc = make_hl_map(&a.hl_map, a.it.hl, rows, I->di.d)) return rc;
        a.tma = env_flag("GMPGR_TMA_PF", false) ? 2 : 1;  // 2: + L2 prefetch of the next tile's rows
    }
    a.users = users;
    a.Q = Q;
    a.k = p->k;
    a.kp = p->k_parallel;
    a.hops = p->hops;
    a.ef = p->ef;
    a.out_ids = ids;
    a.out_scores = scores;
    a.out_count = count;
    a.out_stats = stats;
    a.tags = S->tags;
    a.epochs = S->epochs;
    a.f_slot = S->f_slot;
    a.f_srch = S->f_srch;
    a.surv_v = S->surv_v;
    a.surv_i = S->surv_i;
    a.fr_v = S->fr_v;
    a.fr_i = S->fr_i;
    a.fr_key = S->fr_key;
    a.seg_v = S->seg_v;
    a.seg_key = S->seg_key;
    a.pool_key = S->pool_key;
    a.pool_slot = S->pool_slot;
    a.pool_meta = S->pool_meta;
    a.counters = S->counters;
    a.phase_cycles = S->phase;
    a.band_rel = p->band_rel > 0.f ? p->band_rel : 1e-3f;
    a.band_abs = p->band_abs > 0.f ? p->band_abs : 1e-3f;
    a.capF = S->capF * G_;  // CTA-level flattened lists
    a.capS = S->capS * G_;
    a.capP = S->capP;          // per-query pools
    a.queue = S->flags;
    a.nonfinite = S->flags + 1;
    a.band_viol = S->flags + 3;
    GR_CUDA(cudaMemsetAsync(S->flags, 0, sizeof(int), stream));
    kern<<<(int)blocks, nthreads, smem, stream>>>(a);
    GR_CUDA(cudaGetLastError());
    S->launches += 1;
    return GR_OK;
}

// ------------------------------------------------------------------ duo kernel
// bytes of duo scratch per unit (lists x G queries, hash, per-query pools / bitsets / logs)
size_t duo_unit_bytes(int64_t G, int64_t capF, int64_t capS, int64_t capP, int64_t hcap, int64_t vwords,
                      int64_t logcap) {
    const int64_t lF = capF * G, lS = capS * G;
    return (size_t)(2 * 2 * lF * 4 + 5 * lS * 4 + 2 * lS * 8 + hcap * 8 + G * 2 * capP * 16 + G * vwords * 4 +
                    G * logcap * 4 + G * 64 * 16);
}

int ensure_duo_scratch(gr_searcher *S, int64_t units, int64_t G, int64_t capF, int64_t capS, int64_t capP,
                       int64_t hcap, int64_t vwords, int64_t logcap) {
    gr_searcher::Duo &D = S->duo;
    if (D.units >= units && D.G == G && D.capF >= capF && D.capS >= capS && D.capP >= capP && D.hcap >= hcap &&
        D.vwords == vwords && D.logcap == logcap)
        return GR_OK;
    D.free_all();
    const int64_t lF = capF * G, lS = capS * G, slots = units * G;
    int rc = GR_OK;
    if ((rc = dmalloc(&D.f_slot, (size_t)units * 2 * lF))) return rc;
    if ((rc = dmalloc(&D.f_srch, (size_t)units * 2 * lF))) return rc;
    int32_t **lists[] = {&D.surv_v, &D.surv_i, &D.cont_v, &D.cont_i, &D.seg_v};
    for (int32_t **l : lists)
        if ((rc = dmalloc(l, (size_t)units * lS))) return rc;
    if ((rc = dmalloc(&D.fr_key, (size_t)units * lS))) return rc;
    if ((rc = dmalloc(&D.seg_key, (size_t)units * lS))) return rc;
    if (hcap && (rc = dmalloc(&D.hash, (size_t)units * hcap))) return rc;
    if ((rc = dmalloc(&D.pool_key, (size_t)slots * 2 * capP))) return rc;
    if ((rc = dmalloc(&D.pool_slot, (size_t)slots * 2 * capP))) return rc;
    if ((rc = dmalloc(&D.pool_meta, (size_t)slots * 2 * capP))) return rc;
    if ((rc = dmalloc(&D.vis, (size_t)slots * vwords))) return rc;
    if ((rc = dmalloc(&D.vlog, (size_t)slots * logcap))) return rc;
    if ((rc = dmalloc(&D.acc0, (size_t)slots * 64))) return rc;
    if (hcap) GR_CUDA(cudaMemset(D.hash, 0xFF, (size_t)units * hcap * 8));
    GR_CUDA(cudaMemset(D.vis, 0, (size_t)slots * vwords * 4));
    D.units = units;
    D.G = G;
    D.capF = capF;
    D.capS = capS;
    D.capP = capP;
    D.hcap = hcap;
    D.vwords = vwords;
    D.logcap = logcap;
    D.bytes = duo_unit_bytes(G, capF, capS, capP, hcap, vwords, logcap) * units;
    return GR_OK;
}

template <int DH, int ZZ, int MODE, int G>
int plan_duo(int k, int kp, SearchArgs &a) {
    using EX = ExactU<DH, ZZ>;
    using TP = TcPipe2<DH, ZZ>;
    a.sortcap = pow2ceil(std::max(k, kp));
    const int hist_b = 8 * 256 * 4, sortk_b = G * a.sortcap * 8, sortv_b = G * a.sortcap * 4;
    int shared_b = MODE == 1 ? TP::B_BYTES : EX::W_END * 16;
    auto up = [](int x, int al) { return (x + al - 1) / al * al; };
    if (MODE == 1) {  // + the exact re-scorer's layer-0 weights (item half)
        a.off_exw0 = up(shared_b, 16);
        shared_b = a.off_exw0 + EX::NCH0 * 64 * 16;
    }
    a.unit0 = up(shared_b, 1024);
    SmemPlan U;  // unit-relative
    int alias_end = 0;
    if (MODE == 1) {
        U.alloc(TP::UNIT_BYTES);  // A stages + barriers
        alias_end = TP::A_REGION;
    }
    // exact buffers, histograms and pool sort live in the A stages when they fit (dead
    // outside the scoring pipeline), else after them
    int off = 0;
    auto place = [&](int bytes) {
        if (MODE == 1 && off + bytes <= alias_end) {
            const int o = off;
            off += (bytes + 15) & ~15;
            return o;
        }
        return U.alloc(bytes);
    };
    a.off_x0 = place(EX::BUF_END * 16);
    a.off_hist = place(hist_b);
    a.off_sortk = place(sortk_b);
    a.off_sortv = place(sortv_b);
    a.off_misc = U.alloc((G * 64 + 64 + 64 * ZZ + 8 + 64 + 4) * 4);  // + w_eff, c0, hlim
    if (MODE == 0) a.off_acc0 = U.alloc(G * 64 * 16);  // MODE 1: global (SearchArgs::acc0g)
    a.off_kp = U.alloc(3 * G * kp * 4);
    a.unit_stride = up(U.bytes, 1024);
    a.off_tmemp = a.unit0 + 2 * a.unit_stride;
    return a.off_tmemp + 16 + 1024;  // + slack for the kernel's 1024-byte alignment of the carve
}

// Duo kernel for the fixed model shapes; returns -1 if not applicable
int launch_duo(gr_searcher *S, const gr_graph *G, const gr_model *M, const gr_items *I, const float *users,
               int64_t Q, const gr_search_params *p, int64_t *ids, double *scores, int32_t *count,
               int64_t *stats, cudaStream_t stream, int shape, const int *avail = nullptr,
               int *qdone = nullptr, int chunk_q = 0) {
    SearchArgs a;
    std::memset(&a, 0, sizeof(a));
    const int mode = p->mode;
    if (mode == GR_MODE_TC && I->di.hl == nullptr) return -1;
    constexpr int GQ = 8;
    int smem = 0;
    void (*kern)(const SearchArgs) = nullptr;
#define GR_DUO_CASE(CODE, DH, ZZ)                                            \
    case CODE:                                                               \
        if (mode == GR_MODE_TC) {                                            \
            smem = plan_duo<DH, ZZ, 1, GQ>(p->k, p->k_parallel, a);          \
            kern = duo_kernel<DH, ZZ, 1, GQ>();                        \
        } else {                                                             \
            smem = plan_duo<DH, ZZ, 0, GQ>(p->k, p->k_parallel, a);          \
            kern = duo_kernel<DH, ZZ, 0, GQ>();                        \
        }                                                                    \
        break;
    switch (shape) {
        GR_DUO_CASE(1283, 128, 3)
        GR_DUO_CASE(1282, 128, 2)
        GR_DUO_CASE(643, 64, 3)
        GR_DUO_CASE(642, 64, 2)
    default: return -1;
    }
#undef GR_DUO_CASE
    if (smem > kMaxSmem) return -1;
    // lists: re-score requests pack (query << 24 | index) with index < capS * G or < capP
    const int64_t capF = (int64_t)p->k_parallel * p->ef;
    const int64_t capS = std::max<int64_t>(std::min<int64_t>(capF * G->max_deg, (int64_t)p->k_parallel * G->dg.n),
                                           G->max_deg + 1) + 64;
    const int64_t capP = p->k + capS;
    if (capS * GQ >= (1 << 24) || capP >= (1 << 24)) return -1;
    const int64_t hcap = 0;  // (query, node) hash: not needed (the first toucher is the owner)
    const int64_t vwords = (G->dg.n + 31) / 32;  // one visited bit per node
    const int64_t logcap = std::min<int64_t>(G->dg.n + 1, 1 << 16);
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 0;
    GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 512, smem));
    if (per_sm < 1) return -1;
    // resident units: enough for the batch, at most one CTA per SM, and within the scratch
    // memory budget (free device memory + what this searcher already holds, times
    // GMPGR_SCRATCH_FRAC (default 0.8), or GMPGR_SCRATCH_GB)
    int64_t units = std::min<int64_t>((Q + GQ - 1) / GQ, 2LL * per_sm * num_sms(G->device));
    units = (units + 1) & ~1LL;
    const size_t per_unit = duo_unit_bytes(GQ, capF, capS, capP, hcap, vwords, logcap);
    size_t budget = 0;
    if (const char *gb = getenv("GMPGR_SCRATCH_GB")) {
        budget = (size_t)(atof(gb) * 1e9);
    } else {
        size_t fr = 0, tot = 0;
        GR_CUDA(cudaMemGetInfo(&fr, &tot));
        double frac = 0.8;
        if (const char *f = getenv("GMPGR_SCRATCH_FRAC")) frac = atof(f);
        budget = (size_t)((double)(fr + S->duo.bytes) * frac);
    }
    units = std::min<int64_t>(units, (int64_t)(budget / per_unit) & ~1LL);
    if (units < 2)
        return fail(GR_ENOMEM, "search scratch for one CTA (" + std::to_string(2 * per_unit) +
                                   " bytes) exceeds the device memory budget");
    if (int rc = ensure_duo_scratch(S, units, GQ, capF, capS, capP, hcap, vwords, logcap)) return rc;
    S->duo_units_last = units;
    const gr_searcher::Duo &D = S->duo;
    a.g = G->dg;
    a.M = M->dm;
    a.it = I->di;
    std::unique_lock<std::mutex> hl_lock;
    if (mode == GR_MODE_TC) {
        int64_t rows = I->di.n;
        if (G->dg.rows) {  // slot-ordered copy (the graph's BFS order) when slots != rows
            hl_lock = std::unique_lock<std::mutex>(const_cast<gr_graph *>(G)->hl_mu);
            if (int rc = ensure_slot_hl(const_cast<gr_graph *>(G), I, stream)) return rc;
            a.it.hl = G->hl_slot;
            a.it.hl_by_slot = 1;
            rows = G->dg.n;
        }
        if (int rc = make_hl_map(&a.hl_map, a.it.hl, rows, I->di.d)) return rc;
        a.tma = 1;
    }
    a.users = users;
    a.Q = Q;
    a.k = p->k;
    a.kp = p->k_parallel;
    a.hops = p->hops;
    a.ef = p->ef;
    a.out_ids = ids;
    a.out_scores = scores;
    a.out_count = count;
    a.out_stats = stats;
    a.f_slot = D.f_slot;
    a.f_srch = D.f_srch;
    a.surv_v = D.surv_v;
    a.surv_i = D.surv_i;
    a.cont_v = D.cont_v;
    a.cont_i = D.cont_i;
    a.fr_key = D.fr_key;
    a.seg_v = D.seg_v;
    a.seg_key = D.seg_key;
    a.pool_key = D.pool_key;
    a.pool_slot = D.pool_slot;
    a.pool_meta = D.pool_meta;
    a.hash = D.hash;
    a.hash_cap = D.hcap;
    a.vis = D.vis;
    a.vis_words = D.vwords;
    a.vlog = D.vlog;
    a.acc0g = D.acc0;
    a.log_cap = (int)D.logcap;
    a.counters = S->counters;
    a.phase_cycles = S->phase;
    a.band_rel = p->band_rel > 0.f ? p->band_rel : 1e-3f;
    a.band_abs = p->band_abs > 0.f ? p->band_abs : 1e-3f;
    a.capF = D.capF * GQ;  // unit-level flattened lists
    a.capS = D.capS * GQ;
    a.capP = D.capP;       // per-query pools
    a.queue = S->flags;
    a.nonfinite = S->flags + 1;
    a.band_viol = S->flags + 3;
    a.avail = avail;
    a.qdone = qdone;
    a.chunk_q = chunk_q;
    a.negz = -0.0f;
    GR_CUDA(cudaMemsetAsync(S->flags, 0, sizeof(int), stream));
    kern<<<(int)(units / 2), 512, smem, stream>>>(a);
    GR_CUDA(cudaGetLastError());
    S->launches += 1;
    return GR_OK;
}

// ------------------------------------------------------------------ streamed host calls
// Stream memory operations (driver API, through the runtime's entry-point query).
typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
    StreamValueFn wait = nullptr, write = nullptr;
    bool ok = false;
};
const MemOps &mem_ops() {
    static MemOps m = [] {
        MemOps r;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess && p &&
            q == cudaDriverEntryPointSuccess)
            r.wait = reinterpret_cast<StreamValueFn>(p);
        p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess && p &&
            q == cudaDriverEntryPointSuccess)
            r.write = reinterpret_cast<StreamValueFn>(p);
        cudaGetLastError();
        r.ok = r.wait && r.write;
        return r;
    }();
    return m;
}

// gr_search with host buffers, overlapped: users are copied in chunk by chunk on s_in while
// the (single, persistent) duo kernel already runs -- each unit waits for its batch's chunk
// (avail) -- and each chunk's results are copied out on s_out as soon as the kernel has
// finished its queries (qdone[c], cuStreamWaitValue32).  So the e2e time is the kernel time
// plus the first chunk's copy-in and the last chunk's copy-out.  Returns -1 when not
// applicable (other kernels, small batches, no stream memory operations).
int launch_streamed(gr_searcher *S, const gr_graph *G, const gr_model *M, const gr_items *I, const float *h_users,
                    float *d_users, int64_t Q, const gr_search_params *p, int64_t *h_ids, double *h_scores,
                    int32_t *h_count, int64_t *h_stats, int64_t *d_ids, double *d_scores, int32_t *d_count,
                    int64_t *d_stats, int nst, cudaStream_t st) {
    // opt-in (GMPGR_STREAM=1): measured slower end to end at cfg3 (383k vs 404k QPS) and cfg2
    // -- the stream waits on the chunk counters add more latency than the copies they hide
    const char *kenv = getenv("GMPGR_KERNEL");
    const char *senv = getenv("GMPGR_STREAM");
    if ((kenv && *kenv) || !(senv && senv[0] == '1') || Q < 4096) return -1;
    const int shape = fixed_shape(M->dm);
    if (!shape || (p->mode == GR_MODE_TC && !M->dm.tc_ok)) return -1;
    const MemOps &mo = mem_ops();
    if (!mo.ok) return -1;
    constexpr int kChunks = 8;
    if (!S->s_in) {
        GR_CUDA(cudaStreamCreateWithFlags(&S->s_in, cudaStreamNonBlocking));
        GR_CUDA(cudaStreamCreateWithFlags(&S->s_out, cudaStreamNonBlocking));
        GR_CUDA(cudaEventCreateWithFlags(&S->ev_reset, cudaEventDisableTiming));
        GR_CUDA(cudaEventCreateWithFlags(&S->ev_out, cudaEventDisableTiming));
        if (int rc = dmalloc(&S->sflags, 1 + kChunks)) return rc;
    }
    const int d = M->dm.d_h, k = p->k;
    const int chunk_q = (int)((((Q + kChunks - 1) / kChunks) + 7) / 8 * 8);
    const int nchunks = (int)((Q + chunk_q - 1) / chunk_q);
    GR_CUDA(cudaMemsetAsync(S->sflags, 0, (1 + kChunks) * sizeof(int), st));
    GR_CUDA(cudaEventRecord(S->ev_reset, st));
    // copy-in stream: chunk c's users, then avail = end of chunk c
    GR_CUDA(cudaStreamWaitEvent(S->s_in, S->ev_reset, 0));
    for (int c = 0; c < nchunks; ++c) {
        const int64_t q0 = (int64_t)c * chunk_q, q1 = std::min<int64_t>(Q, q0 + chunk_q);
        GR_CUDA(cudaMemcpyAsync(d_users + q0 * d, h_users + q0 * d, (size_t)(q1 - q0) * d * 4,
                                cudaMemcpyHostToDevice, S->s_in));
        if (mo.write((CUstream)S->s_in, (CUdeviceptr)S->sflags, (cuuint32_t)q1, 0) != CUDA_SUCCESS)
            return fail(GR_ECUDA, "cuStreamWriteValue32 failed");
    }
    const int rc = launch_duo(S, G, M, I, d_users, Q, p, d_ids, d_scores, d_count, d_stats, st, shape,
                              S->sflags, S->sflags + 1, chunk_q);
    if (rc == -1) {  // the duo kernel does not take this call: drain the copy-in, plain path
        GR_CUDA(cudaStreamSynchronize(S->s_in));
        return -1;
    }
    if (rc) return rc;
    // copy-out stream: each chunk as soon as its queries are finished
    GR_CUDA(cudaStreamWaitEvent(S->s_out, S->ev_reset, 0));
    for (int c = 0; c < nchunks; ++c) {
        const int64_t q0 = (int64_t)c * chunk_q, q1 = std::min<int64_t>(Q, q0 + chunk_q), nq = q1 - q0;
        if (mo.wait((CUstream)S->s_out, (CUdeviceptr)(S->sflags + 1 + c), (cuuint32_t)nq, 0 /*GEQ*/) != CUDA_SUCCESS)
            return fail(GR_ECUDA, "cuStreamWaitValue32 failed");
        GR_CUDA(cudaMemcpyAsync(h_ids + q0 * k, d_ids + q0 * k, (size_t)nq * k * 8, cudaMemcpyDeviceToHost, S->s_out));
        GR_CUDA(cudaMemcpyAsync(h_scores + q0 * k, d_scores + q0 * k, (size_t)nq * k * 8, cudaMemcpyDeviceToHost,
                                S->s_out));
        GR_CUDA(cudaMemcpyAsync(h_count + q0, d_count + q0, (size_t)nq * 4, cudaMemcpyDeviceToHost, S->s_out));
        GR_CUDA(cudaMemcpyAsync(h_stats + q0 * nst, d_stats + q0 * nst, (size_t)nq * nst * 8,
                                cudaMemcpyDeviceToHost, S->s_out));
    }
    GR_CUDA(cudaEventRecord(S->ev_out, S->s_out));
    GR_CUDA(cudaStreamWaitEvent(st, S->ev_out, 0));
    return GR_OK;
}

// approximate (first-pass) tensor-core scores of one user against item rows: error studies
template <int DH, int ZZ>
__global__ void __launch_bounds__(GR_NT, 1) tc_pairs_kernel(DevModel M, DevItems it, const float *user,
                                                            const int32_t *rows, int64_t n, double *out) {
    using T = TcMlp<DH, ZZ>;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint4 *src = reinterpret_cast<const uint4 *>(M.tcB);
    uint4 *dst = reinterpret_cast<uint4 *>(smem + T::OFF_B0H);
    for (int t = tid; t < (T::OFF_AH - T::OFF_B0H) / 16; t += GR_NT) dst[t] = src[t];
    float *b1 = reinterpret_cast<float *>(smem + T::OFF_B1);
    for (int t = tid; t < 64; t += GR_NT) b1[t] = M.tcMisc[t];
    float *w2 = reinterpret_cast<float *>(smem + T::OFF_W2);
    for (int t = tid; t < 64 * ZZ; t += GR_NT) w2[t] = M.tcMisc[64 + t];
    if (tid < 4) {
        reinterpret_cast<float *>(smem + T::OFF_B2)[tid] = M.tcMisc[64 + 64 * ZZ + tid];
        reinterpret_cast<float *>(smem + T::OFF_ATT)[tid] = M.tcMisc[68 + 64 * ZZ + tid];
    }
    for (int o = tid; o < 64; o += GR_NT) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = 0; j < M.pre_ch; ++j) {
            const int c = chunk_perm(j, 2 * DH);
            mac4(acc, make_float4(user[4 * c], user[4 * c + 1], user[4 * c + 2], user[4 * c + 3]),
                 M.W[0][j * 64 + o]);
        }
        reinterpret_cast<float *>(smem + T::OFF_U)[o] = __fadd_rn(hsum4(acc), M.b[0][o]);
    }
    uint32_t *tptr = reinterpret_cast<uint32_t *>(smem + T::OFF_TMEM);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tc::smem_u32(tptr)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) tc::mbar_init(reinterpret_cast<uint64_t *>(smem + T::OFF_BAR), 1);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tptr;
    uint32_t phase = 0;
    DevGraph g;
    memset(&g, 0, sizeof(g));
    for (int64_t base = (int64_t)blockIdx.x * T::TM; base < n; base += (int64_t)gridDim.x * T::TM) {
        const int nv = (int)min((int64_t)T::TM, n - base);
        T::tile(smem, tmem, phase, it, g, rows + base, nv);
        if (tid < nv) out[base + tid] = (double)reinterpret_cast<const float *>(smem + T::OFF_SC)[tid];
        __syncthreads();
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

int launch_search(gr_searcher *S, const gr_graph *G, const gr_model *M, const gr_items *I,
                  const float *users, int64_t Q, const gr_search_params *p, int64_t *ids,
                  double *scores, int32_t *count, int64_t *stats, cudaStream_t stream) {
    if (M->dm.d_h != I->di.d) return fail(GR_EINVAL, "item embedding dim != model d_h");
    if (G->max_row >= I->di.n)
        return fail(GR_EINVAL, "graph reads embedding row " + std::to_string(G->max_row) + " but the items table has " +
                                   std::to_string(I->di.n) + " rows (item_embeddings[ids], search.py:88)");
    SearchArgs a;
    std::memset(&a, 0, sizeof(a));
    const int shape = fixed_shape(M->dm);
    const int mode = p->mode;
    if (mode == GR_MODE_TC && (!shape || !M->dm.tc_ok))
        return fail(GR_EINVAL, "tensor-core mode needs the (d_h in {64,128}, hidden (64,64), Z in {2,3}) model shape");
    // fixed shapes run the duo kernel (two 256-thread units per CTA, bitset visited state);
    // GMPGR_KERNEL=mq selects the round-1 lock-step multi-query kernel (per-slot N-wide claim
    // tags), GMPGR_KERNEL=cta the per-query kernel
    const char *kenv = getenv("GMPGR_KERNEL");
    const bool k_cta = kenv && std::strcmp(kenv, "cta") == 0, k_mq = kenv && std::strcmp(kenv, "mq") == 0;
    if (shape && !k_cta && !k_mq) {
        const int rc = launch_duo(S, G, M, I, users, Q, p, ids, scores, count, stats, stream, shape);
        if (rc != -1) return rc;
    }
    if (shape && !k_cta) {
        const int rc = launch_mq(S, G, M, I, users, Q, p, ids, scores, count, stats, stream, shape);
        if (rc != -1) return rc;
    }
    const int smem = plan_search(M->dm, p->k, p->k_parallel, a, shape, mode);
    void (*kern)(const SearchArgs) = nullptr;
    if (mode == GR_MODE_TC) {
        switch (shape) {
        case 1283: kern = search_kernel<2, 128, 3, 1>(); break;
        case 1282: kern = search_kernel<2, 128, 2, 1>(); break;
        case 643: kern = search_kernel<2, 64, 3, 1>(); break;
        default: kern = search_kernel<2, 64, 2, 1>(); break;
        }
    } else {
        switch (shape) {
        case 1283: kern = search_kernel<2, 128, 3, 0>(); break;
        case 1282: kern = search_kernel<2, 128, 2, 0>(); break;
        case 643: kern = search_kernel<2, 64, 3, 0>(); break;
        case 642: kern = search_kernel<2, 64, 2, 0>(); break;
        default:
            kern = smem <= 110 * 1024 ? search_kernel<2, 0, 0, 0>()
                                      : search_kernel<1, 0, 0, 0>();
        }
    }
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 0;
    GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, GR_NT, smem));
    if (per_sm < 1) return fail(GR_EINVAL, "search kernel does not fit on an SM");
    int64_t slots = std::min<int64_t>(Q, (int64_t)per_sm * num_sms(G->device));
    const int64_t capF = (int64_t)p->k_parallel * p->ef;
    int64_t capS = std::min<int64_t>(capF * G->max_deg, (int64_t)p->k_parallel * G->dg.n);
    capS = std::max<int64_t>(capS, G->max_deg + 1) + 64;
    const int64_t capP = p->k + capS;
    if (int rc = ensure_search_scratch(S, G, slots, capF, capS, capP)) return rc;
    a.g = G->dg;
    a.M = M->dm;
    a.it = I->di;
    a.users = users;
    a.Q = Q;
    a.k = p->k;
    a.kp = p->k_parallel;
    a.hops = p->hops;
    a.ef = p->ef;
    a.out_ids = ids;
    a.out_scores = scores;
    a.out_count = count;
    a.out_stats = stats;
    a.tags = S->tags;
    a.epochs = S->epochs;
    a.f_slot = S->f_slot;
    a.f_srch = S->f_srch;
    a.surv_v = S->surv_v;
    a.surv_i = S->surv_i;
    a.fr_v = S->fr_v;
    a.fr_i = S->fr_i;
    a.fr_key = S->fr_key;
    a.seg_v = S->seg_v;
    a.seg_key = S->seg_key;
    a.pool_key = S->pool_key;
    a.pool_slot = S->pool_slot;
    a.pool_meta = S->pool_meta;
    a.counters = S->counters;
    a.phase_cycles = S->phase;
    a.band_rel = p->band_rel > 0.f ? p->band_rel : 1e-3f;
    a.band_abs = p->band_abs > 0.f ? p->band_abs : 1e-3f;
    a.capF = S->capF;
    a.capS = S->capS;
    a.capP = S->capP;
    a.queue = S->flags;
    a.nonfinite = S->flags + 1;
    a.band_viol = S->flags + 3;
    GR_CUDA(cudaMemsetAsync(S->flags, 0, sizeof(int), stream));
    kern<<<(int)slots, GR_NT, smem, stream>>>(a);
    GR_CUDA(cudaGetLastError());
    S->launches += 1;
    return GR_OK;
}

// traversal-only score-table search (MODE 2 of hipanns_search_kernel, scores.cuh)
int launch_search_scores(gr_searcher *S, const gr_graph *G, const gr_scores *T,
                         const gr_search_params *p, int64_t *ids, double *scores, int32_t *count,
                         int64_t *stats, cudaStream_t stream) {
    SearchArgs a;
    std::memset(&a, 0, sizeof(a));
    SmemPlan P;
    a.off_hist = P.alloc(GR_NW * 256 * 4);
    a.sortcap = pow2ceil(std::max(p->k, p->k_parallel));
    a.off_sortk = P.alloc(a.sortcap * 8);
    a.off_sortv = P.alloc(a.sortcap * 4);
    a.off_kp = P.alloc(3 * p->k_parallel * 4);
    const int smem = P.bytes;
    auto kern = smem <= 110 * 1024 ? search_kernel<2, 0, 0, 2>() : search_kernel<1, 0, 0, 2>();
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 0;
    GR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, GR_NT, smem));
    if (per_sm < 1) return fail(GR_EINVAL, "search kernel does not fit on an SM");
    const int64_t Q = T->Q;
    int64_t slots = std::min<int64_t>(Q, (int64_t)per_sm * num_sms(G->device));
    const int64_t capF = (int64_t)p->k_parallel * p->ef;
    int64_t capS = std::min<int64_t>(capF * G->max_deg, (int64_t)p->k_parallel * G->dg.n);
    capS = std::max<int64_t>(capS, G->max_deg + 1) + 64;
    const int64_t capP = p->k + capS;
    if (int rc = ensure_search_scratch(S, G, slots, capF, capS, capP)) return rc;
    a.g = G->dg;
    a.Q = Q;
    a.k = p->k;
    a.kp = p->k_parallel;
    a.hops = p->hops;
    a.ef = p->ef;
    a.out_ids = ids;
    a.out_scores = scores;
    a.out_count = count;
    a.out_stats = stats;
    a.tags = S->tags;
    a.epochs = S->epochs;
    a.f_slot = S->f_slot;
    a.f_srch = S->f_srch;
    a.surv_v = S->surv_v;
    a.surv_i = S->surv_i;
    a.fr_v = S->fr_v;
    a.fr_i = S->fr_i;
    a.fr_key = S->fr_key;
    a.seg_v = S->seg_v;
    a.seg_key = S->seg_key;
    a.pool_key = S->pool_key;
    a.pool_slot = S->pool_slot;
    a.pool_meta = S->pool_meta;
    a.counters = S->counters;
    a.phase_cycles = S->phase;
    a.capF = S->capF;
    a.capS = S->capS;
    a.capP = S->capP;
    a.queue = S->flags;
    a.nonfinite = S->flags + 1;
    a.tab_code = T->code;
    a.tab_f64 = T->tab;
    a.tab_n = T->n;
    GR_CUDA(cudaMemsetAsync(S->flags, 0, sizeof(int), stream));
    kern<<<(int)slots, GR_NT, smem, stream>>>(a);
    GR_CUDA(cudaGetLastError());
    S->launches += 1;
    return GR_OK;
}

} // namespace


extern "C" {

int gr_searcher_create(int device, gr_searcher **out) {
    if (!out) return fail(GR_EINVAL, "null argument");
    GR_CUDA(cudaSetDevice(device));
    gr_searcher *S = new gr_searcher();
    S->device = device;
    if (int rc = dmalloc(&S->flags, 4)) { delete S; return rc; }
    cudaMemset(S->flags, 0, 16);
    if (int rc = dmalloc(&S->counters, 4)) { cudaFree(S->flags); delete S; return rc; }
    cudaMemset(S->counters, 0, 32);
    if (cudaEventCreateWithFlags(&S->done, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(S->flags);
        cudaFree(S->counters);
        delete S;
        return fail(GR_ECUDA, "cudaEventCreate failed");
    }
    const char *pt = getenv("GMPGR_PHASE_TIMING");
    if (pt && pt[0] == '1') {
        if (dmalloc(&S->phase, 16) == GR_OK) cudaMemset(S->phase, 0, 128);
    }
    *out = S;
    return GR_OK;
}

int gr_searcher_destroy(gr_searcher *s) {
    if (!s) return GR_OK;
    cudaSetDevice(s->device);
    {
        std::lock_guard<std::mutex> lk(s->mu);
        cudaDeviceSynchronize();
    }
    s->free_scratch();
    s->duo.free_all();
    if (s->s_in) cudaStreamDestroy(s->s_in);
    if (s->s_out) cudaStreamDestroy(s->s_out);
    if (s->ev_reset) cudaEventDestroy(s->ev_reset);
    if (s->ev_out) cudaEventDestroy(s->ev_out);
    if (s->sflags) cudaFree(s->sflags);
    cudaFree(s->flags);
    cudaFree(s->counters);
    if (s->done) cudaEventDestroy(s->done);
    if (s->phase) cudaFree(s->phase);
    s->st_users.release();
    s->st_ids.release();
    s->st_scores.release();
    s->st_count.release();
    s->st_stats.release();
    delete s;
    return GR_OK;
}

int64_t gr_searcher_launches(const gr_searcher *s) { return s ? s->launches : 0; }

int gr_searcher_counters(gr_searcher *s, int64_t *out) {
    if (!s || !out) return fail(GR_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(s->mu);
    GR_CUDA(cudaSetDevice(s->device));
    GR_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < 22; ++i) out[i] = 0;
    uint64_t c[4];
    GR_CUDA(cudaMemcpy(c, s->counters, 32, cudaMemcpyDeviceToHost));
    out[0] = (int64_t)c[0];
    out[1] = (int64_t)c[1];
    if (s->phase) GR_CUDA(cudaMemcpy(out + 2, s->phase, 128, cudaMemcpyDeviceToHost));
    out[18] = (int64_t)c[2];
    out[19] = (int64_t)c[3];
    out[20] = s->band_reruns;
    out[21] = s->duo_units_last;
    return GR_OK;
}

int gr_search_async(gr_searcher *s, const gr_graph *g, const gr_model *m, const gr_items *it,
                    const float *users, int64_t Q, const gr_search_params *p, int64_t *out_ids,
                    double *out_scores, int32_t *out_count, int64_t *out_stats, void *stream) {
    if (!s || !g || !m || !it || !users || !out_ids || !out_scores || !out_count || !out_stats)
        return fail(GR_EINVAL, "null argument");
    if (int rc = check_params(p)) return rc;
    if (Q <= 0) return GR_OK;
    std::lock_guard<std::mutex> lk(s->mu);
    GR_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = (cudaStream_t)stream;
    GR_CUDA(cudaStreamWaitEvent(st, s->done, 0));
    const int rc = launch_search(s, g, m, it, users, Q, p, out_ids, out_scores, out_count, out_stats, st);
    GR_CUDA(cudaEventRecord(s->done, st));
    return rc;
}

namespace {
// flags[1] (non-finite) and flags[3] (tensor-core band violations) since the last read
int read_status(gr_searcher *s, cudaStream_t st, int *nonfinite, int *band) {
    GR_CUDA(cudaStreamWaitEvent(st, s->done, 0));
    int f[4] = {0, 0, 0, 0};
    GR_CUDA(cudaMemcpyAsync(f, s->flags, sizeof(f), cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    if (f[1]) GR_CUDA(cudaMemsetAsync(s->flags + 1, 0, sizeof(int), st));
    if (f[3]) GR_CUDA(cudaMemsetAsync(s->flags + 3, 0, sizeof(int), st));
    *nonfinite = f[1];
    *band = f[3];
    return GR_OK;
}
}  // namespace

int gr_searcher_status(gr_searcher *s, void *stream) {
    if (!s) return fail(GR_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(s->mu);
    GR_CUDA(cudaSetDevice(s->device));
    int nonfinite = 0, band = 0;
    if (int rc = read_status(s, (cudaStream_t)stream, &nonfinite, &band)) return rc;
    if (nonfinite) return fail(GR_ENUMERIC, "non-finite value in metric forward pass");
    if (band)
        return fail(GR_EBAND, std::to_string(band) + " tensor-core scores were farther than half the "
                              "refinement band from their exact value: re-run in exact mode");
    return GR_OK;
}

int gr_search(gr_searcher *s, const gr_graph *g, const gr_model *m, const gr_items *it,
              const float *users, int64_t Q, const gr_search_params *p, int64_t *out_ids,
              double *out_scores, int32_t *out_count, int64_t *out_stats, int on_device,
              void *stream) {
    if (!s || !g || !m || !it || !users || !out_ids || !out_scores || !out_count || !out_stats)
        return fail(GR_EINVAL, "null argument");
    if (int rc = check_params(p)) return rc;
    if (Q <= 0) return GR_OK;
    std::lock_guard<std::mutex> lk(s->mu);
    GR_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = (cudaStream_t)stream;
    GR_CUDA(cudaStreamWaitEvent(st, s->done, 0));
    GR_CUDA(cudaMemsetAsync(s->flags + 1, 0, 3 * sizeof(int), st));
    const int nst = 5 + g->dg.n_layers;
    gr_search_params pe = *p;
    for (int attempt = 0;; ++attempt) {
    if (on_device) {
        if (int rc = launch_search(s, g, m, it, users, Q, &pe, out_ids, out_scores, out_count,
                                   out_stats, st))
            return rc;
    } else {
        const size_t nu = (size_t)Q * m->dm.d_h, no = (size_t)Q * p->k, ns = (size_t)Q * nst;
        size_t cap_u = s->st_users_n, cap_s = s->st_stats_n;
        if (int rc = stage<float>(s->st_users, cap_u, nu)) return rc;
        s->st_users_n = cap_u;
        size_t c1 = s->st_out_n, c2 = s->st_out_n, c3 = s->st_out_n;
        if (no > s->st_out_n || !s->st_ids.p) {
            s->st_ids.release(); s->st_scores.release(); s->st_count.release();
            c1 = c2 = c3 = 0;
            if (int rc = stage<int64_t>(s->st_ids, c1, no)) return rc;
            if (int rc = stage<double>(s->st_scores, c2, no)) return rc;
            if (int rc = stage<int32_t>(s->st_count, c3, std::max<size_t>(no, (size_t)Q))) return rc;
            s->st_out_n = no;
        }
        if (int rc = stage<int64_t>(s->st_stats, cap_s, ns)) return rc;
        s->st_stats_n = cap_s;
        float *du = (float *)s->st_users.p;
        if (attempt == 0) {
            if (m->dm.d_h != it->di.d) return fail(GR_EINVAL, "item embedding dim != model d_h");
            if (g->max_row >= it->di.n) return fail(GR_EINVAL, "items table smaller than the graph");
            const int rs = launch_streamed(s, g, m, it, users, du, Q, &pe, out_ids, out_scores, out_count,
                                           out_stats, (int64_t *)s->st_ids.p, (double *)s->st_scores.p,
                                           (int32_t *)s->st_count.p, (int64_t *)s->st_stats.p, nst, st);
            if (rs != -1) {
                if (rs) return rs;
                goto launched;
            }
            GR_CUDA(cudaMemcpyAsync(du, users, nu * 4, cudaMemcpyHostToDevice, st));
        }
        if (int rc = launch_search(s, g, m, it, du, Q, &pe, (int64_t *)s->st_ids.p,
                                   (double *)s->st_scores.p, (int32_t *)s->st_count.p,
                                   (int64_t *)s->st_stats.p, st))
            return rc;
        GR_CUDA(cudaMemcpyAsync(out_ids, s->st_ids.p, no * 8, cudaMemcpyDeviceToHost, st));
        GR_CUDA(cudaMemcpyAsync(out_scores, s->st_scores.p, no * 8, cudaMemcpyDeviceToHost, st));
        GR_CUDA(cudaMemcpyAsync(out_count, s->st_count.p, (size_t)Q * 4, cudaMemcpyDeviceToHost, st));
        GR_CUDA(cudaMemcpyAsync(out_stats, s->st_stats.p, ns * 8, cudaMemcpyDeviceToHost, st));
    }
launched:
    GR_CUDA(cudaEventRecord(s->done, st));
    int nonfinite = 0, band = 0;
    if (int rc = read_status(s, st, &nonfinite, &band)) return rc;
    if (nonfinite) return fail(GR_ENUMERIC, "non-finite value in metric forward pass");
    // tensor-core certificate failed somewhere in the batch: the whole batch is searched
    // again with exact scoring (results are then exact by construction)
    if (band && pe.mode == GR_MODE_TC && attempt == 0) {
        pe.mode = GR_MODE_EXACT;
        s->band_reruns += 1;
        continue;
    }
    return GR_OK;
    }
}

// ------------------------------------------------------------------ score tables
namespace {
int scores_finish(gr_scores *T, int *bad, cudaStream_t st, gr_scores **out) {
    cudaError_t e = build_score_codes(T->tab, T->Q, T->n, T->code, bad, st);
    int hbad = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost);
    cudaFree(bad);
    if (e != cudaSuccess) {
        gr_scores_destroy(T);
        return fail(GR_ECUDA, std::string("score table: ") + cudaGetErrorString(e));
    }
    if (hbad) {
        gr_scores_destroy(T);
        return fail(GR_ENUMERIC, "NaN in score table");
    }
    *out = T;
    return GR_OK;
}
int scores_alloc(int device, int64_t Q, int64_t n, gr_scores **T, int **bad) {
    if (Q < 1 || n < 1) return fail(GR_EINVAL, "empty score table");
    if (n >= (int64_t)1 << 31) return fail(GR_EINVAL, "score table wider than 2^31 items");
    GR_CUDA(cudaSetDevice(device));
    gr_scores *t = new gr_scores();
    t->device = device;
    t->Q = Q;
    t->n = n;
    int rc = dmalloc(&t->tab, (size_t)(Q * n));
    if (!rc) rc = dmalloc(&t->code, (size_t)(Q * n));
    if (!rc) rc = dmalloc(bad, 1);
    if (rc) { gr_scores_destroy(t); return rc; }
    cudaMemset(*bad, 0, 4);
    *T = t;
    return GR_OK;
}
} // namespace

int gr_scores_create(int device, const double *table, int64_t Q, int64_t n_items, int on_device,
                     gr_scores **out) {
    if (!table || !out) return fail(GR_EINVAL, "null argument");
    gr_scores *T = nullptr;
    int *bad = nullptr;
    if (int rc = scores_alloc(device, Q, n_items, &T, &bad)) return rc;
    const cudaError_t e = cudaMemcpy(T->tab, table, (size_t)(Q * n_items) * 8,
                                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(bad); gr_scores_destroy(T); return fail(GR_ECUDA, cudaGetErrorString(e)); }
    return scores_finish(T, bad, 0, out);
}

int gr_scores_euclid(int device, const double *vectors, int64_t n_items, int32_t dim,
                     const double *queries, int64_t Q, gr_scores **out) {
    if (!vectors || !queries || !out) return fail(GR_EINVAL, "null argument");
    if (dim < 1) return fail(GR_EINVAL, "dim must be >= 1");
    gr_scores *T = nullptr;
    int *bad = nullptr;
    if (int rc = scores_alloc(device, Q, n_items, &T, &bad)) return rc;
    double *dv = nullptr, *dq = nullptr;
    int rc = dmalloc(&dv, (size_t)(n_items * dim));
    if (!rc) rc = dmalloc(&dq, (size_t)(Q * dim));
    if (rc) { cudaFree(dv); cudaFree(bad); gr_scores_destroy(T); return rc; }
    cudaMemcpy(dv, vectors, (size_t)(n_items * dim) * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, queries, (size_t)(Q * dim) * 8, cudaMemcpyHostToDevice);
    const int64_t total = Q * n_items;
    euclid_table_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256>>>(
        dv, n_items, dim, dq, Q, T->tab, bad);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaFree(dv);
    cudaFree(dq);
    if (e != cudaSuccess) { cudaFree(bad); gr_scores_destroy(T); return fail(GR_ECUDA, cudaGetErrorString(e)); }
    return scores_finish(T, bad, 0, out);
}

int gr_scores_destroy(gr_scores *t) {
    if (!t) return GR_OK;
    cudaSetDevice(t->device);
    cudaFree(t->tab);
    cudaFree(t->code);
    delete t;
    return GR_OK;
}

int gr_scores_read(const gr_scores *t, double *out) {
    if (!t || !out) return fail(GR_EINVAL, "null argument");
    GR_CUDA(cudaSetDevice(t->device));
    GR_CUDA(cudaMemcpy(out, t->tab, (size_t)(t->Q * t->n) * 8, cudaMemcpyDeviceToHost));
    return GR_OK;
}

int gr_search_scores(gr_searcher *s, const gr_graph *g, const gr_scores *t,
                     const gr_search_params *p, int64_t *out_ids, double *out_scores,
                     int32_t *out_count, int64_t *out_stats, int on_device, void *stream) {
    if (!s || !g || !t || !out_ids || !out_scores || !out_count || !out_stats)
        return fail(GR_EINVAL, "null argument");
    if (int rc = check_params(p)) return rc;
    if (p->mode != GR_MODE_EXACT) return fail(GR_EINVAL, "score tables are exact-mode only");
    if (t->device != s->device || g->device != s->device) return fail(GR_EINVAL, "handles on different devices");
    std::lock_guard<std::mutex> lk(s->mu);
    GR_CUDA(cudaSetDevice(s->device));
    {   // every item id must index the table (ids = score-table columns, search.py:79)
        std::vector<int64_t> hid(g->dg.n);
        GR_CUDA(cudaMemcpy(hid.data(), g->dg.ids, g->dg.n * 8, cudaMemcpyDeviceToHost));
        for (int64_t v : hid)
            if (v < 0 || v >= t->n) return fail(GR_EINVAL, "graph item id outside the score table");
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t Q = t->Q, no = Q * p->k, ns = Q * (5 + g->dg.n_layers);
    GR_CUDA(cudaStreamWaitEvent(st, s->done, 0));
    if (on_device) {
        const int rc = launch_search_scores(s, g, t, p, out_ids, out_scores, out_count, out_stats, st);
        GR_CUDA(cudaEventRecord(s->done, st));
        return rc;
    }
    int64_t *di = nullptr, *dst = nullptr;
    double *ds = nullptr;
    int32_t *dc = nullptr;
    int rc = dmalloc(&di, (size_t)no);
    if (!rc) rc = dmalloc(&ds, (size_t)no);
    if (!rc) rc = dmalloc(&dc, (size_t)Q);
    if (!rc) rc = dmalloc(&dst, (size_t)ns);
    if (!rc) rc = launch_search_scores(s, g, t, p, di, ds, dc, dst, st);
    cudaEventRecord(s->done, st);
    if (!rc) {
        cudaMemcpyAsync(out_ids, di, no * 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(out_scores, ds, no * 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(out_count, dc, Q * 4, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(out_stats, dst, ns * 8, cudaMemcpyDeviceToHost, st);
        const cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = fail(GR_ECUDA, cudaGetErrorString(e));
    }
    cudaFree(di); cudaFree(ds); cudaFree(dc); cudaFree(dst);
    return rc;
}

// ------------------------------------------------------------------ pairs
int gr_score_pairs(const gr_model *m, const gr_items *it, const float *users, int64_t n_users,
                   const int32_t *user_index, const int64_t *item_ids, int64_t n,
                   double *out_scores, int on_device, void *stream) {
    if (!m || !it || !users || !item_ids || !out_scores) return fail(GR_EINVAL, "null argument");
    if (m->dm.d_h != it->di.d) return fail(GR_EINVAL, "item embedding dim != model d_h");
    if (n_users < 1) return fail(GR_EINVAL, "no user embeddings");
    if (n <= 0) return GR_OK;
    GR_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    const float *du = users;
    const int32_t *dui = user_index;
    const int64_t *dids = item_ids;
    double *dout = out_scores;
    std::vector<void *> tmp;
    auto cleanup = [&](int rc) {
        for (void *p : tmp) cudaFree(p);
        return rc;
    };
    if (!on_device) {
        float *a = nullptr;
        int64_t *b = nullptr;
        double *c = nullptr;
        int32_t *u = nullptr;
        if (int rc = dmalloc(&a, (size_t)n_users * m->dm.d_h)) return cleanup(rc);
        tmp.push_back(a);
        if (int rc = dmalloc(&b, (size_t)n)) return cleanup(rc);
        tmp.push_back(b);
        if (int rc = dmalloc(&c, (size_t)n)) return cleanup(rc);
        tmp.push_back(c);
        cudaMemcpyAsync(a, users, (size_t)n_users * m->dm.d_h * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(b, item_ids, (size_t)n * 8, cudaMemcpyHostToDevice, st);
        if (user_index) {
            if (int rc = dmalloc(&u, (size_t)n)) return cleanup(rc);
            tmp.push_back(u);
            cudaMemcpyAsync(u, user_index, (size_t)n * 4, cudaMemcpyHostToDevice, st);
        }
        du = a;
        dids = b;
        dout = c;
        dui = u;
    }
    int *flags = nullptr;
    if (int rc = dmalloc(&flags, 2)) return cleanup(rc);
    tmp.push_back(flags);
    cudaMemsetAsync(flags, 0, 8, st);
    PairArgs a;
    std::memset(&a, 0, sizeof(a));
    const int smem = plan_pairs(m->dm, a);
    if (int rc = set_smem(score_pairs_kernel, smem)) return cleanup(rc);
    a.M = m->dm;
    a.it = it->di;
    a.users = du;
    a.n_users = n_users;
    a.user_index = dui;
    a.item_ids = dids;
    a.n = n;
    a.out = dout;
    a.nonfinite = flags;
    a.bad_index = flags + 1;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, score_pairs_kernel, GR_NT, smem);
    const int64_t tiles = (n + GR_PT - 1) / GR_PT;
    const int grid = (int)std::min<int64_t>(tiles, (int64_t)std::max(per_sm, 1) * num_sms(m->device));
    score_pairs_kernel<<<grid, GR_NT, smem, st>>>(a);
    if (cudaGetLastError() != cudaSuccess) return cleanup(fail(GR_ECUDA, "score_pairs launch failed"));
    int hflags[2] = {0, 0};
    cudaMemcpyAsync(hflags, flags, 8, cudaMemcpyDeviceToHost, st);
    if (!on_device) cudaMemcpyAsync(out_scores, dout, (size_t)n * 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cleanup(fail(GR_ECUDA, cudaGetErrorString(e)));
    cleanup(GR_OK);
    if (hflags[1]) return fail(GR_EINVAL, "user index or item id out of range");
    if (hflags[0]) return fail(GR_ENUMERIC, "non-finite value in metric forward pass");
    return GR_OK;
}

// ------------------------------------------------------------------ approximate pairs
int gr_score_items_approx(const gr_model *m, const gr_items *it, const float *user,
                          const int64_t *item_ids, int64_t n, double *out_scores) {
    if (!m || !it || !user || !item_ids || !out_scores) return fail(GR_EINVAL, "null argument");
    const int shape = fixed_shape(m->dm);
    if (!shape || !m->dm.tc_ok) return fail(GR_EINVAL, "model shape has no tensor-core scorer");
    if (m->dm.d_h != it->di.d) return fail(GR_EINVAL, "item embedding dim != model d_h");
    if (n <= 0) return GR_OK;
    GR_CUDA(cudaSetDevice(m->device));
    std::vector<int32_t> rows(n);
    for (int64_t i = 0; i < n; ++i) {
        if (item_ids[i] < 0 || item_ids[i] >= it->di.n) return fail(GR_EINVAL, "item id out of range");
        rows[i] = (int32_t)item_ids[i];
    }
    float *du = nullptr;
    int32_t *dr = nullptr;
    double *dout = nullptr;
    if (int rc = dmalloc(&du, (size_t)m->dm.d_h)) return rc;
    if (int rc = dmalloc(&dr, (size_t)n)) { cudaFree(du); return rc; }
    if (int rc = dmalloc(&dout, (size_t)n)) { cudaFree(du); cudaFree(dr); return rc; }
    cudaMemcpy(du, user, m->dm.d_h * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dr, rows.data(), n * 4, cudaMemcpyHostToDevice);
    void (*kern)(DevModel, DevItems, const float *, const int32_t *, int64_t, double *) = nullptr;
    int smem = 0;
    switch (shape) {
    case 1283: kern = tc_pairs_kernel<128, 3>; smem = TcMlp<128, 3>::BYTES; break;
    case 1282: kern = tc_pairs_kernel<128, 2>; smem = TcMlp<128, 2>::BYTES; break;
    case 643: kern = tc_pairs_kernel<64, 3>; smem = TcMlp<64, 3>::BYTES; break;
    default: kern = tc_pairs_kernel<64, 2>; smem = TcMlp<64, 2>::BYTES; break;
    }
    int rc = set_smem(kern, smem);
    if (rc == GR_OK) {
        const int grid = (int)std::min<int64_t>((n + 127) / 128, num_sms(m->device));
        kern<<<grid, GR_NT, smem>>>(m->dm, it->di, du, dr, n, dout);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) rc = fail(GR_ECUDA, cudaGetErrorString(e));
        else cudaMemcpy(out_scores, dout, n * 8, cudaMemcpyDeviceToHost);
    }
    cudaFree(du); cudaFree(dr); cudaFree(dout);
    return rc;
}

// ------------------------------------------------------------------ brute force
int gr_brute_force(const gr_model *m, const gr_items *it, const float *users, int64_t Q,
                   int32_t k, int64_t *out_ids, double *out_scores, int on_device, void *stream) {
    if (!m || !it || !users || !out_ids || !out_scores) return fail(GR_EINVAL, "null argument");
    if (m->dm.d_h != it->di.d) return fail(GR_EINVAL, "item embedding dim != model d_h");
    if (k < 1 || k > it->di.n) return fail(GR_EINVAL, "k exceeds item count");
    if (k > 4096) return fail(GR_EINVAL, "k > 4096 not supported");
    if (Q <= 0) return GR_OK;
    GR_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    BruteArgs a;
    std::memset(&a, 0, sizeof(a));
    const int smem = plan_brute(m->dm, a);
    if (int rc = set_smem(brute_partial_kernel, smem)) return rc;
    const int sms = num_sms(m->device);
    const int B = (int)std::min<int64_t>(Q, 16);
    // partitions per query: fill ~2 CTAs/SM, but keep the merge list (P*k) within 8192 keys
    const int P = std::max(1, std::min((2 * sms + B - 1) / B, std::max(1, 8192 / k)));
    a.B = B;
    a.P = P;
    a.k = k;
    a.cap = std::max<int64_t>(4 * k, k + 4096);
    a.M = m->dm;
    a.it = it->di;
    std::vector<void *> tmp;
    auto cleanup = [&](int rc) {
        for (void *p : tmp) cudaFree(p);
        return rc;
    };
    float *du = nullptr;
    int64_t *dids = nullptr;
    double *dsc = nullptr;
    if (int rc = dmalloc(&a.cand_key, (size_t)B * P * 2 * a.cap)) return cleanup(rc);
    tmp.push_back(a.cand_key);
    if (int rc = dmalloc(&a.cand_row, (size_t)B * P * 2 * a.cap)) return cleanup(rc);
    tmp.push_back(a.cand_row);
    if (int rc = dmalloc(&a.loc_key, (size_t)B * P * k)) return cleanup(rc);
    tmp.push_back(a.loc_key);
    if (int rc = dmalloc(&a.loc_row, (size_t)B * P * k)) return cleanup(rc);
    tmp.push_back(a.loc_row);
    if (int rc = dmalloc(&a.loc_n, (size_t)B * P)) return cleanup(rc);
    tmp.push_back(a.loc_n);
    if (int rc = dmalloc(&a.nonfinite, 1)) return cleanup(rc);
    tmp.push_back(a.nonfinite);
    cudaMemsetAsync(a.nonfinite, 0, 4, st);
    if (!on_device) {
        if (int rc = dmalloc(&du, (size_t)Q * m->dm.d_h)) return cleanup(rc);
        tmp.push_back(du);
        if (int rc = dmalloc(&dids, (size_t)Q * k)) return cleanup(rc);
        tmp.push_back(dids);
        if (int rc = dmalloc(&dsc, (size_t)Q * k)) return cleanup(rc);
        tmp.push_back(dsc);
        cudaMemcpyAsync(du, users, (size_t)Q * m->dm.d_h * 4, cudaMemcpyHostToDevice, st);
    } else {
        du = const_cast<float *>(users);
        dids = out_ids;
        dsc = out_scores;
    }
    const int sortcap = pow2ceil(P * k);
    const int msmem = sortcap * 12;
    if (int rc = set_smem(brute_merge_kernel, msmem)) return cleanup(rc);
    for (int64_t q0 = 0; q0 < Q; q0 += B) {
        const int nb = (int)std::min<int64_t>(B, Q - q0);
        a.users = du + q0 * m->dm.d_h;
        a.B = nb;
        brute_partial_kernel<<<dim3(P, nb), GR_NT, smem, st>>>(a);
        brute_merge_kernel<<<nb, GR_NT, msmem, st>>>(a.loc_key, a.loc_row, a.loc_n, P, k, sortcap,
                                                    dids + q0 * k, dsc + q0 * k);
    }
    if (cudaGetLastError() != cudaSuccess) return cleanup(fail(GR_ECUDA, "brute force launch failed"));
    int flag = 0;
    cudaMemcpyAsync(&flag, a.nonfinite, 4, cudaMemcpyDeviceToHost, st);
    if (!on_device) {
        cudaMemcpyAsync(out_ids, dids, (size_t)Q * k * 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(out_scores, dsc, (size_t)Q * k * 8, cudaMemcpyDeviceToHost, st);
    }
    cudaError_t e = cudaStreamSynchronize(st);
    cleanup(GR_OK);
    if (e != cudaSuccess) return fail(GR_ECUDA, cudaGetErrorString(e));
    if (flag) return fail(GR_ENUMERIC, "non-finite value in metric forward pass");
    return GR_OK;
}

// ------------------------------------------------------------------ shard merge
int gr_merge_topk(int device, const int64_t *in_ids, const double *in_scores, int32_t R, int64_t Q,
                  int32_t k_in, int32_t k, int64_t *out_ids, double *out_scores,
                  int32_t *out_count, void *stream) {
    if (!in_ids || !in_scores || !out_ids || !out_scores || !out_count)
        return fail(GR_EINVAL, "null argument");
    if (R < 1 || k_in < 1 || k < 1) return fail(GR_EINVAL, "R, k_in, k must be >= 1");
    if ((int64_t)R * k_in > 16384) return fail(GR_EINVAL, "R * k_in > 16384 not supported");
    if (Q <= 0) return GR_OK;
    GR_CUDA(cudaSetDevice(device));
    const int sortcap = pow2ceil(R * k_in);
    const int smem = sortcap * 12;
    if (int rc = set_smem(merge_topk_kernel, smem)) return rc;
    merge_topk_kernel<<<(unsigned)Q, GR_NT, smem, (cudaStream_t)stream>>>(
        in_ids, in_scores, R, Q, k_in, k, sortcap, out_ids, out_scores, out_count);
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

int gr_pack_topk(int device, const int64_t *ids, const double *scores, int64_t n, uint64_t *out,
                 void *stream) {
    if (!ids || !scores || !out) return fail(GR_EINVAL, "null argument");
    if (n <= 0) return GR_OK;
    GR_CUDA(cudaSetDevice(device));
    pack_topk_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
        ids, scores, n, out);
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

int gr_merge_topk_packed(int device, const uint64_t *in, int32_t R, int64_t Q, int32_t k_in, int32_t k,
                         int64_t *out_ids, double *out_scores, int32_t *out_count, void *stream) {
    if (!in || !out_ids || !out_scores || !out_count) return fail(GR_EINVAL, "null argument");
    if (R < 1 || k_in < 1 || k < 1) return fail(GR_EINVAL, "R, k_in, k must be >= 1");
    if ((int64_t)R * k_in > 16384) return fail(GR_EINVAL, "R * k_in > 16384 not supported");
    if (Q <= 0) return GR_OK;
    GR_CUDA(cudaSetDevice(device));
    const int sortcap = pow2ceil(R * k_in);
    const int smem = sortcap * 12;
    if (int rc = set_smem(merge_packed_kernel, smem)) return rc;
    merge_packed_kernel<<<(unsigned)Q, GR_NT, smem, (cudaStream_t)stream>>>(in, R, Q, k_in, k, sortcap, out_ids,
                                                                         out_scores, out_count);
    GR_CUDA(cudaGetLastError());
    return GR_OK;
}

} // extern "C"
