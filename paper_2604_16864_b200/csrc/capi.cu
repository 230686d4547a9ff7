// C-ABI entry points (include/hierasparse_b200.h): argument validation with the
// reference's error taxonomy, pool sizing, TMA descriptor encoding, per-stream
// workspaces and kernel launches.  No host synchronisation on the hot entry
// points (hs_prune_compress, hs_decode*, hs_prefill).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>

#include <cmath>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/hierasparse_b200.h"
#include "kernels.h"


namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launch_count{0};

hs_status fail(hs_status code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define HS_CHECK_CONFIG(ok, ...) \
    do {                         \
        if (!(ok)) return fail(HS_ERR_CONFIG, __VA_ARGS__); \
    } while (0)

hs_status cuda_fail(cudaError_t e, const char* where) {
    return fail(HS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// ------------------------------------------------------------ TMA encode ---
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// A small always-valid device buffer backing descriptors of empty pools.
void* dummy_buffer() {
    static void* p = nullptr;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (!p) {
        if (cudaMalloc(&p, 1 << 16) != cudaSuccess) p = nullptr;
        else cudaMemset(p, 0, 1 << 16);
    }
    return p;
}

bool make_map_halves(CUtensorMap* m, const void* ptr, uint64_t outer, uint32_t box_outer);

// 2-D tile map over a row-major [outer][inner] 16-bit array.  Encoded maps are
// cached by (pointer, geometry, swizzle) so steady-state calls skip the driver.
bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
              uint32_t box_outer, CUtensorMapSwizzle sw) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    if (ptr == nullptr || outer == 0) {
        ptr = dummy_buffer();
        outer = box_outer;
        if (!ptr) return false;
    }
    using Key = std::tuple<const void*, uint64_t, uint64_t, uint32_t, uint32_t, int>;
    static std::mutex mu;
    static std::map<Key, CUtensorMap> cache;
    const Key key{ptr, inner, outer, box_inner, box_outer, static_cast<int>(sw)};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *m = it->second;
            return true;
        }
    }
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    const bool ok = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    if (ok) {
        std::lock_guard<std::mutex> lk(mu);
        if (cache.size() > 4096) cache.clear();
        cache[key] = *m;
    }
    return ok;
}

// 3-D view of a row-major [outer][128] 16-bit array as [2 halves][outer][64]
// (half stride 128 B): one box {64, box_outer, 2} lands as the two SW128
// column-half tiles [half][row][64] a K-major UMMA operand of K = 128 expects.
// 4-D view of the queries [unit*gqa + head][n_q][128] as [half][head][query][64]:
// one box {64, qt, hg, 2} is the SW128 K-major B operand of a GEMM1 over hg
// stacked heads (hg * qt = 128 rows); queries past n_q are zero-filled.
bool make_map_q(CUtensorMap* m, const void* ptr, uint64_t n_q, uint64_t heads, uint32_t qt, uint32_t hg) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {64, n_q, heads, 2};
    cuuint64_t strides[3] = {256, 256 * n_q, 128};
    cuuint32_t box[4] = {64, qt, hg, 2};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map_halves(CUtensorMap* m, const void* ptr, uint64_t outer, uint32_t box_outer) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    if (ptr == nullptr || outer == 0) {
        ptr = dummy_buffer();
        outer = box_outer;
        if (!ptr) return false;
    }
    using Key = std::tuple<const void*, uint64_t, uint32_t>;
    static std::mutex mu;
    static std::map<Key, CUtensorMap> cache;
    const Key key{ptr, outer, box_outer};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *m = it->second;
            return true;
        }
    }
    cuuint64_t dims[3] = {64, outer, 2};
    cuuint64_t strides[2] = {256, 128};
    cuuint32_t box[3] = {64, box_outer, 2};
    cuuint32_t es[3] = {1, 1, 1};
    const bool ok = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    if (ok) {
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = *m;
    }
    return ok;
}

// ------------------------------------------------------------ workspaces ---
struct Workspace {
    void* ptr = nullptr;
    size_t bytes = 0;
};
std::mutex g_ws_mu;
std::map<std::tuple<int, cudaStream_t, int>, Workspace> g_ws;

enum WsKind { kWsCompress = 0, kWsDecode = 1, kWsMisc = 2, kWsPrefill = 3, kWsMailbox = 4 };

std::vector<void*> g_ws_retired;  // outgrown workspaces: never freed (a captured graph may still use them)

// Per (device, stream, purpose) scratch; grows on demand and is zeroed on
// (re)allocation (the decode arrival counters rely on that and self-reset).
// An outgrown buffer is retired, not freed: a CUDA graph captured earlier on
// this stream handle keeps pointing at it.  Graphs that must not share state
// with other work on a recycled stream handle pass their own workspace
// (hs_decode_ws).
void* workspace(cudaStream_t s, size_t bytes, int kind, hs_status* st) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace& w = g_ws[std::make_tuple(dev, s, kind)];
    if (w.bytes < bytes) {
        if (w.ptr) g_ws_retired.push_back(w.ptr);
        w.ptr = nullptr;
        w.bytes = 0;
        const size_t nb = bytes + (bytes >> 2) + 4096;
        cudaError_t e = cudaMalloc(&w.ptr, nb);
        if (e != cudaSuccess) {
            *st = cuda_fail(e, "workspace allocation");
            return nullptr;
        }
        w.bytes = nb;
        e = cudaMemsetAsync(w.ptr, 0, nb, s);
        if (e != cudaSuccess) {
            *st = cuda_fail(e, "workspace clear");
            return nullptr;
        }
    }
    *st = HS_OK;
    return w.ptr;
}

// -------------------------------------------------------------- geometry ---
hs_status pool_counts(uint64_t rows, const hs_sparsity_config* cfg, double s, uint32_t* nb_out,
                      uint32_t* dense, uint32_t* sparse, uint32_t* prefix_out, uint32_t* suffix_out,
                      uint32_t* quota_out) {
    HS_CHECK_CONFIG(cfg != nullptr, "SparsityConfig: null");
    HS_CHECK_CONFIG(cfg->s_key >= 0.0 && cfg->s_key <= 1.0, "SparsityConfig: s_key outside [0, 1]");
    HS_CHECK_CONFIG(cfg->s_value >= 0.0 && cfg->s_value <= 1.0, "SparsityConfig: s_value outside [0, 1]");
    HS_CHECK_CONFIG(s >= 0.0 && s <= 1.0, "select_blocks: sparsity outside [0, 1]");
    HS_CHECK_CONFIG(cfg->block_size > 0 && cfg->block_size % 4 == 0,
                    "SparsityConfig: block_size must be a positive multiple of m_group");
    HS_CHECK_CONFIG(rows % cfg->block_size == 0,
                    "prune_cache: sequence length not divisible by block_size");
    const uint64_t nb = rows / cfg->block_size;
    // masks.hpp:93-98 rounding, pruner.hpp:130-131 clamping.
    uint64_t p = (cfg->sink_tokens + cfg->block_size - 1) / cfg->block_size;
    uint64_t q = (cfg->local_window + cfg->block_size - 1) / cfg->block_size;
    if (p > nb) p = nb;
    if (q > nb - p) q = nb - p;
    const uint64_t prunable = nb - p - q;
    const uint64_t quota = static_cast<uint64_t>(floor(s * static_cast<double>(prunable)));
    HS_CHECK_CONFIG(nb - quota <= 32767, "compress: dense pool exceeds int16 index capacity");
    HS_CHECK_CONFIG(quota <= 32767, "compress: sparse pool exceeds int16 index capacity");
    if (nb_out) *nb_out = static_cast<uint32_t>(nb);
    if (dense) *dense = static_cast<uint32_t>(nb - quota);
    if (sparse) *sparse = static_cast<uint32_t>(quota);
    if (prefix_out) *prefix_out = static_cast<uint32_t>(p);
    if (suffix_out) *suffix_out = static_cast<uint32_t>(q);
    if (quota_out) *quota_out = static_cast<uint32_t>(quota);
    return HS_OK;
}

hs_status check_device_cache(const hs_device_cache* c, const char* what) {
    HS_CHECK_CONFIG(c != nullptr, "%s: null cache", what);
    HS_CHECK_CONFIG(c->dtype == HS_DTYPE_BF16 || c->dtype == HS_DTYPE_F16, "%s: unsupported dtype", what);
    // masks.hpp:87 (block_size a positive multiple of m_group); pruner.hpp:172-173 /
    // compressed_cache.hpp:123-126 (the channel grouping axis divisible by m_group)
    HS_CHECK_CONFIG(c->block_size >= 4 && c->block_size % 4 == 0,
                    "%s: block_size must be a positive multiple of m_group", what);
    HS_CHECK_CONFIG(c->head_dim >= 4 && c->head_dim % 4 == 0, "%s: head dimension not divisible by m_group", what);
    HS_CHECK_CONFIG(c->n_units >= 1, "%s: n_units must be positive", what);
    // dense_count / sparse_count are the pool slots per unit: exactly the block
    // count for caches from hs_prune_compress, possibly more for pooled caches
    // whose units differ in their dense counts (sequence-split shards).
    HS_CHECK_CONFIG(c->dense_count + c->sparse_count >= c->logical_blocks,
                    "%s: pool counts do not cover the block map", what);
    HS_CHECK_CONFIG(c->dense_count <= 32767 && c->sparse_count <= 32767,
                    "%s: pool exceeds int16 index capacity", what);
    HS_CHECK_CONFIG(c->logical_blocks == 0 || c->index_map != nullptr, "%s: null index map", what);
    HS_CHECK_CONFIG(c->dense_count == 0 || c->dense_pool != nullptr, "%s: null dense pool", what);
    HS_CHECK_CONFIG(c->sparse_count == 0 || (c->nnz_pool && c->meta_pool), "%s: null sparse pools", what);
    return HS_OK;
}

hs_status check_pair(const hs_device_cache* k, const hs_device_cache* v) {
    hs_status st;
    if ((st = check_device_cache(k, "key cache"))) return st;
    if ((st = check_device_cache(v, "value cache"))) return st;
    HS_CHECK_CONFIG(k->axis == HS_AXIS_CHANNEL, "attention: key cache must be channel-grouped");
    HS_CHECK_CONFIG(v->axis == HS_AXIS_SEQUENCE, "attention: value cache must be sequence-grouped");
    HS_CHECK_CONFIG(k->logical_blocks == v->logical_blocks, "attention: key/value block counts differ");
    HS_CHECK_CONFIG(k->block_size == v->block_size, "attention: key/value block sizes differ");
    HS_CHECK_CONFIG(k->head_dim == v->head_dim, "attention: key/value head dims differ");
    HS_CHECK_CONFIG(k->n_units == v->n_units, "attention: key/value unit counts differ");
    HS_CHECK_CONFIG(k->dtype == v->dtype, "attention: key/value dtypes differ");
    return HS_OK;
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Split count: fill the machine (decode_ctas_per_sm CTAs per SM) with balanced ranges.
int choose_splits(int n_units, int nb) {
    const int slots = hs::decode_ctas_per_sm() * sm_count();
    int best = 1;
    double best_cost = 1e30;
    for (int s = 1; s <= nb && s <= 1024; ++s) {
        const int ctas = n_units * s;
        const int waves = (ctas + slots - 1) / slots;
        const double per_cta = std::ceil(static_cast<double>(nb) / s);  // blocks per CTA
        // wave-quantised time + per-CTA fixed overhead (~3 blocks) + combine cost
        const double cost = waves * (per_cta + 3.0) + 0.02 * s;
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = s;
        }
    }
    return best;
}

hs_status fill_decode_maps(hs::DecodeLaunch& L, const hs_device_cache* k, const hs_device_cache* v) {
    const uint64_t U = k->n_units;
    bool ok = true;
    ok &= make_map(&L.tm_knnz, k->nnz_pool, 64, U * k->sparse_count * 64, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B);
    ok &= make_map(&L.tm_kden, k->dense_pool, 128, U * k->dense_count * 64, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B);
    ok &= make_map(&L.tm_vnnz, v->nnz_pool, 32, U * v->sparse_count * 128, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B);
    ok &= make_map(&L.tm_vden, v->dense_pool, 64, U * v->dense_count * 128, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!ok) return fail(HS_ERR_CUDA, "cuTensorMapEncodeTiled failed (driver entry point unavailable?)");
    return HS_OK;
}

void count_launch(int n = 1) { g_launch_count.fetch_add(n); }

}  // namespace

extern "C" {

HS_API const char* hs_last_error(void) { return g_err.c_str(); }
HS_API int hs_version(void) { return 1; }
HS_API uint64_t hs_kernel_launches(void) { return g_launch_count.load(); }

HS_API hs_status hs_pool_counts(uint64_t rows, const hs_sparsity_config* cfg, double sparsity,
                                uint32_t* logical_blocks, uint32_t* dense_count,
                                uint32_t* sparse_count, uint32_t* prefix_blocks,
                                uint32_t* suffix_blocks) {
    return pool_counts(rows, cfg, sparsity, logical_blocks, dense_count, sparse_count, prefix_blocks,
                       suffix_blocks, nullptr);
}

HS_API hs_status hs_cache_bytes(const hs_device_cache* c, uint64_t* index_bytes, uint64_t* dense_bytes,
                                uint64_t* nnz_bytes, uint64_t* meta_bytes, uint64_t* slot_block_bytes) {
    HS_CHECK_CONFIG(c != nullptr, "hs_cache_bytes: null cache");
    const uint64_t U = c->n_units, be = static_cast<uint64_t>(c->block_size) * c->head_dim;
    if (index_bytes) *index_bytes = U * c->logical_blocks * 2;
    if (dense_bytes) *dense_bytes = U * c->dense_count * be * 2;
    if (nnz_bytes) *nnz_bytes = U * c->sparse_count * be;
    if (meta_bytes) *meta_bytes = U * c->sparse_count * be / 8;
    if (slot_block_bytes) *slot_block_bytes = U * c->logical_blocks * 4;
    return HS_OK;
}

static hs_status prune_compress_common(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                       const hs_sparsity_config* cfg, double sparsity,
                                       hs_device_cache* out, double* losses, uint8_t* flags,
                                       uint64_t* status, void* stream, const hs_device_cache* in) {
    HS_CHECK_CONFIG(out != nullptr && (src != nullptr || in != nullptr), "prune_cache: null argument");
    uint32_t nb, dc, sc, pre, suf, quota;
    hs_status st = pool_counts(rows, cfg, sparsity, &nb, &dc, &sc, &pre, &suf, &quota);
    if (st) return st;
    HS_CHECK_CONFIG(out->head_dim % 4 == 0, "prune_cache: head dimension not divisible by m_group");
    HS_CHECK_CONFIG(out->block_size == cfg->block_size, "prune_cache: cache block size mismatch");
    HS_CHECK_CONFIG(out->logical_blocks == nb, "prune_cache: cache block count %u != %u", out->logical_blocks, nb);
    HS_CHECK_CONFIG(out->dense_count == dc && out->sparse_count == sc,
                    "prune_cache: pool counts (%u, %u) do not match the selection (%u, %u)",
                    out->dense_count, out->sparse_count, dc, sc);
    if ((st = check_device_cache(out, "prune_cache"))) return st;
    HS_CHECK_CONFIG(in != nullptr || out->n_units == 1 || src_unit_stride >= rows * out->head_dim,
                    "prune_cache: unit stride too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool static_sel = quota == 0 || quota == nb - pre - suf;
    hs::CompressLaunch L{};
    L.bf16 = out->dtype == HS_DTYPE_BF16;
    L.axis = out->axis;
    L.block_size = static_cast<int>(out->block_size);
    L.head_dim = static_cast<int>(out->head_dim);
    L.n_units = out->n_units;
    L.nb = nb;
    L.dense_count = dc;
    L.sparse_count = sc;
    L.prefix = pre;
    L.suffix = suf;
    L.quota = quota;
    L.static_selection = static_sel;
    L.all_sparse = quota > 0;
    L.src = src;
    L.src_unit_stride = src_unit_stride;
    L.flags_out = flags;
    L.losses = losses;
    L.index_map = out->index_map;
    L.slot_block = out->slot_block;
    L.dense_pool = out->dense_pool;
    L.nnz_pool = out->nnz_pool;
    L.meta_pool = out->meta_pool;
    if (nb == 0) return HS_OK;
    if (!static_sel) {
        const size_t need_l = losses ? 0 : static_cast<size_t>(out->n_units) * nb * sizeof(double);
        const size_t need = need_l + static_cast<size_t>(out->n_units) * nb + 256;
        uint8_t* ws = static_cast<uint8_t*>(workspace(s, need, kWsCompress, &st));
        if (st) return st;
        if (!losses) L.losses = reinterpret_cast<double*>(ws);
        L.flags_tmp = ws + need_l;
    }
    if (in) {
        L.in_index = in->index_map;
        L.in_nb = static_cast<int>(in->logical_blocks);
        L.in_dense_count = static_cast<int>(in->dense_count);
        L.in_sparse_count = static_cast<int>(in->sparse_count);
        L.in_dense = in->dense_pool;
        L.in_nnz = in->nnz_pool;
        L.in_meta = in->meta_pool;
        // decompress's DataErrors on a corrupt input cache go to the status word
        L.status = reinterpret_cast<unsigned long long*>(status);
    }
    cudaError_t e = hs::launch_prune_compress(L, s);
    count_launch(static_sel ? 2 : 4);
    if (e != cudaSuccess) return cuda_fail(e, "prune_compress launch");
    return HS_OK;
}

HS_API hs_status hs_prune_compress(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                   const hs_sparsity_config* cfg, double sparsity,
                                   hs_device_cache* out, double* losses, uint8_t* flags,
                                   void* stream) {
    HS_CHECK_CONFIG(src != nullptr, "prune_cache: null argument");
    return prune_compress_common(src, src_unit_stride, rows, cfg, sparsity, out, losses, flags, nullptr, stream,
                                 nullptr);
}

static hs_status recompress_common(const hs_device_cache* in, const void* tail, uint64_t tail_unit_stride,
                                   uint64_t tail_rows, const hs_sparsity_config* cfg, double sparsity,
                                   hs_device_cache* out, double* losses, uint8_t* flags, uint64_t* status,
                                   void* stream, const char* what) {
    HS_CHECK_CONFIG(in != nullptr && out != nullptr, "%s: null argument", what);
    hs_status st = check_device_cache(in, what);
    if (st) return st;
    HS_CHECK_CONFIG(in != out && in->index_map != out->index_map, "%s: output aliases the input cache", what);
    HS_CHECK_CONFIG(in->axis == out->axis && in->dtype == out->dtype && in->n_units == out->n_units &&
                        in->head_dim == out->head_dim && in->block_size == out->block_size,
                    "%s: input and output caches differ in axis, dtype, units or shape", what);
    HS_CHECK_CONFIG(tail_rows % in->block_size == 0, "%s: tail rows %llu are not whole blocks", what,
                    static_cast<unsigned long long>(tail_rows));
    HS_CHECK_CONFIG(tail_rows == 0 || tail != nullptr, "%s: null tail", what);
    HS_CHECK_CONFIG(tail_rows == 0 || in->n_units == 1 || tail_unit_stride >= tail_rows * in->head_dim,
                    "%s: tail unit stride too small", what);
    return prune_compress_common(tail, tail_unit_stride,
                                 static_cast<uint64_t>(in->logical_blocks) * in->block_size + tail_rows, cfg,
                                 sparsity, out, losses, flags, status, stream, in);
}

HS_API hs_status hs_recompress(const hs_device_cache* in, const hs_sparsity_config* cfg, double sparsity,
                               hs_device_cache* out, double* losses, uint8_t* flags, uint64_t* status,
                               void* stream) {
    return recompress_common(in, nullptr, 0, 0, cfg, sparsity, out, losses, flags, status, stream, "recompress");
}

HS_API hs_status hs_absorb_tail(const hs_device_cache* in, const void* tail, uint64_t tail_unit_stride,
                                uint64_t tail_rows, const hs_sparsity_config* cfg, double sparsity,
                                hs_device_cache* out, double* losses, uint8_t* flags, uint64_t* status,
                                void* stream) {
    return recompress_common(in, tail, tail_unit_stride, tail_rows, cfg, sparsity, out, losses, flags, status,
                             stream, "absorb_tail");
}

static hs_status compress_flags_common(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                       const uint8_t* flags, const uint8_t* element_mask,
                                       uint64_t mask_unit_stride, hs_device_cache* out, uint64_t* status,
                                       void* stream, const char* what) {
    HS_CHECK_CONFIG(out != nullptr && src != nullptr && flags != nullptr, "%s: null argument", what);
    HS_CHECK_CONFIG(rows % out->block_size == 0, "compress: sequence length not divisible by block_size");
    const uint32_t nb = static_cast<uint32_t>(rows / out->block_size);
    HS_CHECK_CONFIG(out->logical_blocks == nb, "compress: block mask does not cover the sequence");
    hs_status st = check_device_cache(out, what);
    if (st) return st;
    HS_CHECK_CONFIG(out->n_units == 1 || src_unit_stride >= rows * out->head_dim, "%s: unit stride too small", what);
    HS_CHECK_CONFIG(element_mask == nullptr || out->n_units == 1 || mask_unit_stride >= rows * out->head_dim,
                    "%s: element mask unit stride too small", what);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // The BlockMask's dense count per unit must equal out->dense_count: checked on
    // the device (status word, ConfigError) with no host round trip.
    hs::CompressLaunch L{};
    L.bf16 = out->dtype == HS_DTYPE_BF16;
    L.axis = out->axis;
    L.block_size = static_cast<int>(out->block_size);
    L.head_dim = static_cast<int>(out->head_dim);
    L.n_units = out->n_units;
    L.nb = nb;
    L.dense_count = out->dense_count;
    L.sparse_count = out->sparse_count;
    L.src = src;
    L.src_unit_stride = src_unit_stride;
    L.flags_in = flags;
    L.element_mask = element_mask;
    L.mask_unit_stride = mask_unit_stride ? mask_unit_stride : rows * out->head_dim;
    L.status = reinterpret_cast<unsigned long long*>(status);
    L.index_map = out->index_map;
    L.slot_block = out->slot_block;
    L.dense_pool = out->dense_pool;
    L.nnz_pool = out->nnz_pool;
    L.meta_pool = out->meta_pool;
    if (nb == 0) return HS_OK;
    cudaError_t e = hs::launch_prune_compress(L, s);
    count_launch(2);
    if (e != cudaSuccess) return cuda_fail(e, "compress launch");
    return HS_OK;
}

HS_API hs_status hs_compress_with_flags(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                        const uint8_t* flags, hs_device_cache* out, uint64_t* status,
                                        void* stream) {
    return compress_flags_common(src, src_unit_stride, rows, flags, nullptr, 0, out, status, stream,
                                 "fused_magnitude_compress");
}

HS_API hs_status hs_compress_with_mask(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                       const uint8_t* element_mask, uint64_t mask_unit_stride,
                                       const uint8_t* flags, hs_device_cache* out, uint64_t* status,
                                       void* stream) {
    HS_CHECK_CONFIG(element_mask != nullptr, "compress: null element mask");
    return compress_flags_common(src, src_unit_stride, rows, flags, element_mask, mask_unit_stride, out, status,
                                 stream, "compress");
}

HS_API hs_status hs_decompress(const hs_device_cache* c, void* dst, uint64_t* status, void* stream) {
    hs_status st = check_device_cache(c, "decompress");
    if (st) return st;
    HS_CHECK_CONFIG(dst != nullptr, "decompress: null destination");
    if (c->logical_blocks == 0) return HS_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    hs::DecompressLaunch L{c->axis, static_cast<int>(c->n_units), static_cast<int>(c->logical_blocks),
                           static_cast<int>(c->dense_count), static_cast<int>(c->sparse_count),
                           c->index_map, c->dense_pool, c->nnz_pool, c->meta_pool, dst,
                           reinterpret_cast<unsigned long long*>(status), static_cast<int>(c->block_size),
                           static_cast<int>(c->head_dim)};
    cudaError_t e = hs::launch_decompress(L, s);
    count_launch();
    if (e != cudaSuccess) return cuda_fail(e, "decompress launch");
    return HS_OK;
}

HS_API hs_status hs_block_losses(const void* src, uint64_t src_unit_stride, uint64_t rows,
                                 const hs_device_cache* geometry, double* losses, void* stream) {
    HS_CHECK_CONFIG(src != nullptr && geometry != nullptr && losses != nullptr, "block_loss: null argument");
    const hs_device_cache* g = geometry;
    HS_CHECK_CONFIG(g->dtype == HS_DTYPE_BF16 || g->dtype == HS_DTYPE_F16, "block_loss: unsupported dtype");
    HS_CHECK_CONFIG(g->block_size >= 4 && g->block_size % 4 == 0,
                    "SparsityConfig: block_size must be a positive multiple of m_group");
    HS_CHECK_CONFIG(g->head_dim >= 4 && g->head_dim % 4 == 0, "prune_cache: head dimension not divisible by m_group");
    HS_CHECK_CONFIG(rows % g->block_size == 0, "prune_cache: sequence length not divisible by block_size");
    HS_CHECK_CONFIG(g->n_units == 1 || src_unit_stride >= rows * g->head_dim, "block_loss: unit stride too small");
    hs::CompressLaunch L{};
    L.bf16 = g->dtype == HS_DTYPE_BF16;
    L.axis = g->axis;
    L.block_size = static_cast<int>(g->block_size);
    L.head_dim = static_cast<int>(g->head_dim);
    L.n_units = static_cast<int>(g->n_units);
    L.nb = static_cast<int>(rows / g->block_size);
    L.src = src;
    L.src_unit_stride = src_unit_stride;
    L.losses = losses;
    if (L.nb == 0) return HS_OK;
    cudaError_t e = hs::launch_block_losses(L, static_cast<cudaStream_t>(stream));
    count_launch();
    if (e != cudaSuccess) return cuda_fail(e, "block_loss launch");
    return HS_OK;
}

HS_API hs_status hs_select_blocks(const double* losses, uint32_t n_units, uint32_t logical_blocks,
                                  const hs_sparsity_config* cfg, double sparsity, uint8_t* flags, void* stream) {
    HS_CHECK_CONFIG(losses != nullptr && flags != nullptr, "select_blocks: null argument");
    uint32_t nb, dc, sc, pre, suf, quota;
    hs_status st = pool_counts(static_cast<uint64_t>(logical_blocks) * (cfg ? cfg->block_size : 0), cfg, sparsity,
                               &nb, &dc, &sc, &pre, &suf, &quota);
    if (st) return st;
    if (nb == 0 || n_units == 0) return HS_OK;
    cudaError_t e = hs::launch_select_blocks(losses, static_cast<int>(n_units), static_cast<int>(nb),
                                             static_cast<int>(pre), static_cast<int>(suf), static_cast<int>(quota),
                                             flags, static_cast<cudaStream_t>(stream));
    count_launch();
    if (e != cudaSuccess) return cuda_fail(e, "select_blocks launch");
    return HS_OK;
}

HS_API hs_status hs_status_word_decode(uint64_t word) {
    if (word == 0) return HS_OK;
    switch (static_cast<uint32_t>(word & 0xFFu)) {
        case hs::kReasonZeroEntry: return fail(HS_ERR_DATA, "decompress: index map holds a zero entry");
        case hs::kReasonDanglingDense: return fail(HS_ERR_DATA, "decompress: dangling dense offset");
        case hs::kReasonDanglingSparse: return fail(HS_ERR_DATA, "decompress: dangling sparse offset");
        case hs::kReasonCodesOrder:
            return fail(HS_ERR_DATA, "unpack_metadata: corrupt metadata, codes not increasing");
        case hs::kReasonKeepsMore: return fail(HS_ERR_DATA, "compress: group keeps more than n_keep elements");
        case hs::kReasonKeepsFewer: return fail(HS_ERR_DATA, "compress: group keeps fewer than n_keep elements");
        case hs::kReasonMaskCount:
            return fail(HS_ERR_CONFIG, "compress: block mask dense count does not fit the cache's pools");
        default: return fail(HS_ERR_DATA, "device status word 0x%llx", static_cast<unsigned long long>(word));
    }
}

constexpr int kDynamicMaxBlocks = 256;  // blocks per split up to which decode claims blocks dynamically

static size_t decode_plain_bytes(uint32_t n_units, int ns, uint32_t gqa) {
    return ((static_cast<size_t>(n_units) * ns * gqa * (hs::kHeadDim + 2) * sizeof(float) + 255) / 256) * 256;
}
static size_t decode_mailbox_bytes(uint32_t n_units, int ns, uint32_t gqa) {
    return static_cast<size_t>(n_units) * ns * gqa * hs::kHeadDim * 2 * sizeof(unsigned long long);
}

// Split count and workspace bytes of a decode launch (counters + split partials).
static void decode_geometry(uint32_t n_units, uint32_t span, uint32_t gqa, uint32_t splits, int* ns_out,
                            size_t* cnt_bytes, size_t* part_bytes) {
    int ns = splits ? static_cast<int>(splits) : choose_splits(static_cast<int>(n_units), static_cast<int>(span));
    if (ns > static_cast<int>(span)) ns = static_cast<int>(span);  // attention.hpp:373-374 clamp
    if (ns < 1) ns = 1;
    *ns_out = ns;
    // split partials [u][ns][gqa][d+2] f32, then the coop combine's tagged
    // mailbox [u][ns][gqa][d] x 16 B (decode.cu)
    *part_bytes = decode_plain_bytes(n_units, ns, gqa) + decode_mailbox_bytes(n_units, ns, gqa);
    *cnt_bytes = ((3 * static_cast<size_t>(n_units) * sizeof(int) + 255) / 256) * 256;
}

// Fast kernels cover block_size 64 x head_dim 128 (the reference default B and
// Llama-3.1-8B's d); other shapes run the generic CUDA-core attention.
static bool specialised(const hs_device_cache* k) {
    return k->block_size == static_cast<uint32_t>(hs::kBlock) && k->head_dim == static_cast<uint32_t>(hs::kHeadDim);
}

static hs_status generic_attention(const void* q, uint32_t n_q, uint32_t gqa, const hs_device_cache* k,
                                   const hs_device_cache* v, const void* k_tail, const void* v_tail, uint32_t tail,
                                   int causal, float scale, uint32_t block_begin, uint32_t block_end,
                                   int include_tail, float* out, int out_mode, cudaStream_t s) {
    HS_CHECK_CONFIG(k->head_dim <= static_cast<uint32_t>(hs::kGenericMaxHeadDim),
                    "attention: head_dim %u above the generic kernel's %d", k->head_dim, hs::kGenericMaxHeadDim);
    hs::GenericAttnLaunch G{};
    G.bf16 = k->dtype == HS_DTYPE_BF16;
    G.n_units = static_cast<int>(k->n_units);
    G.nb = static_cast<int>(k->logical_blocks);
    G.B = static_cast<int>(k->block_size);
    G.d = static_cast<int>(k->head_dim);
    G.gqa = static_cast<int>(gqa);
    G.n_q = static_cast<int>(n_q);
    G.tail = static_cast<int>(tail);
    G.causal = causal;
    G.scale = scale;
    G.q = q;
    G.k_index = k->index_map;
    G.v_index = v->index_map;
    G.k_dense_count = static_cast<int>(k->dense_count);
    G.k_sparse_count = static_cast<int>(k->sparse_count);
    G.v_dense_count = static_cast<int>(v->dense_count);
    G.v_sparse_count = static_cast<int>(v->sparse_count);
    G.k_dense = k->dense_pool;
    G.k_nnz = k->nnz_pool;
    G.k_meta = k->meta_pool;
    G.v_dense = v->dense_pool;
    G.v_nnz = v->nnz_pool;
    G.v_meta = v->meta_pool;
    G.k_tail = k_tail;
    G.v_tail = v_tail;
    G.block_begin = static_cast<int>(block_begin);
    G.block_end = static_cast<int>(block_end);
    G.include_tail = include_tail;
    G.out = out;
    G.out_mode = out_mode;
    cudaError_t e = hs::launch_generic_attention(G, s);
    count_launch();
    if (e != cudaSuccess) return cuda_fail(e, "generic attention launch");
    return HS_OK;
}

static hs_status decode_common_rows(const void* q, const hs_device_cache* k, const hs_device_cache* v,
                                    const void* k_tail, const void* v_tail, uint32_t tail, uint32_t gqa,
                                    uint32_t q_rows, uint32_t row0, float scale, uint32_t splits,
                                    uint32_t block_begin, uint32_t block_end, int include_tail, float* out,
                                    int out_mode, void* user_ws, uint64_t user_ws_bytes, cudaStream_t s);

static hs_status decode_common(const void* q, const hs_device_cache* k, const hs_device_cache* v,
                               const void* k_tail, const void* v_tail, uint32_t tail, uint32_t gqa,
                               float scale, uint32_t splits, uint32_t block_begin, uint32_t block_end,
                               int include_tail, float* out, int out_mode, void* user_ws,
                               uint64_t user_ws_bytes, void* stream) {
    hs_status st = check_pair(k, v);
    if (st) return st;
    HS_CHECK_CONFIG(q != nullptr && out != nullptr, "decode_attention: null argument");
    HS_CHECK_CONFIG(gqa >= 1, "decode_attention: no query rows");
    HS_CHECK_CONFIG(tail == 0 || (k_tail && v_tail), "decode_attention: null dense tail");
    HS_CHECK_CONFIG(static_cast<uint64_t>(k->logical_blocks) * k->block_size + tail > 0,
                    "decode_attention: empty cache");
    HS_CHECK_CONFIG(block_begin <= block_end && block_end <= k->logical_blocks,
                    "attend_range: block range out of bounds");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!specialised(k))
        return generic_attention(q, 1, gqa, k, v, k_tail, v_tail, tail, 0, scale, block_begin, block_end, include_tail,
                                 out, out_mode, s);
    if (gqa > 8) {
        // The mma.sp decode stacks up to 8 query rows on N: larger GQA groups run
        // as chunks of 8 rows (q / out strides stay the group's).
        for (uint32_t r0 = 0; r0 < gqa; r0 += 8) {
            const uint32_t n = gqa - r0 < 8 ? gqa - r0 : 8;
            hs_status st2 = decode_common_rows(q, k, v, k_tail, v_tail, tail, n, gqa, r0, scale, splits, block_begin,
                                               block_end, include_tail, out, out_mode, user_ws, user_ws_bytes, s);
            if (st2) return st2;
        }
        return HS_OK;
    }
    return decode_common_rows(q, k, v, k_tail, v_tail, tail, gqa, gqa, 0, scale, splits, block_begin, block_end,
                              include_tail, out, out_mode, user_ws, user_ws_bytes, s);
}

static hs_status decode_common_rows(const void* q, const hs_device_cache* k, const hs_device_cache* v,
                                    const void* k_tail, const void* v_tail, uint32_t tail, uint32_t gqa,
                                    uint32_t q_rows, uint32_t row0, float scale, uint32_t splits,
                                    uint32_t block_begin, uint32_t block_end, int include_tail, float* out,
                                    int out_mode, void* user_ws, uint64_t user_ws_bytes, cudaStream_t s) {
    hs_status st = HS_OK;
    q = static_cast<const uint16_t*>(q) + static_cast<size_t>(row0) * hs::kHeadDim;
    out += static_cast<size_t>(row0) * (out_mode == 0 ? hs::kHeadDim : hs::kHeadDim + 2);
    hs::DecodeLaunch L{};
    L.bf16 = k->dtype == HS_DTYPE_BF16;
    L.n_units = k->n_units;
    L.nb = k->logical_blocks;
    L.gqa = gqa;
    L.q_rows = q_rows;
    L.tail = tail;
    L.k_dense_count = k->dense_count;
    L.k_sparse_count = k->sparse_count;
    L.v_dense_count = v->dense_count;
    L.v_sparse_count = v->sparse_count;
    L.scale_log2 = scale * 1.4426950408889634f;
    L.q = q;
    L.k_index = k->index_map;
    L.v_index = v->index_map;
    L.k_meta = k->meta_pool;
    L.v_meta = v->meta_pool;
    L.k_nnz = k->nnz_pool;
    L.v_nnz = v->nnz_pool;
    L.k_dense = k->dense_pool;
    L.v_dense = v->dense_pool;
    L.prefetch_distance = 0;  // measured: L2 prefetch ahead of the TMA ring costs 3% (tools/tune_decode.py)
    if (const char* env = getenv("HS_DECODE_PF")) L.prefetch_distance = atoi(env);
    if (const char* env = getenv("HS_DECODE_DEBUG_STREAM_ONLY")) L.debug_stream_only = atoi(env);
    if (const char* env = getenv("HS_DECODE_XP_TAIL")) L.debug_tail = atoi(env);
    L.k_tail = k_tail;
    L.v_tail = v_tail;
    L.block_begin = block_begin;
    L.block_end = block_end;
    L.include_tail = include_tail;
    const int span = static_cast<int>(block_end - block_begin);
    int ns;
    size_t cnt_bytes, part_bytes;
    decode_geometry(L.n_units, static_cast<uint32_t>(span), gqa, splits, &ns, &cnt_bytes, &part_bytes);
    L.nsplit = ns;
    L.max_blocks_per_cta = (span + ns - 1) / ns + 1;
    HS_CHECK_CONFIG(L.max_blocks_per_cta <= 8192,
                    "decode_attention: %d blocks per CTA exceeds the index stage; use more splits",
                    L.max_blocks_per_cta);
    if ((st = fill_decode_maps(L, k, v))) return st;
    // The combine mailbox must read as empty (zero) before every launch that uses
    // it; its launches leave it so, but plain split partials must never land on
    // it.  A caller's workspace serves one (k, gqa, splits) geometry:
    // [counters][mailbox sized for the largest row chunk][plain partials].  The
    // per-stream workspaces serve any geometry, so the mailbox gets its own.
    uint8_t* ws;
    const uint32_t gmax = q_rows < 8 ? q_rows : 8;
    if (user_ws != nullptr) {
        int ns_max;
        size_t cnt_max, part_max;
        decode_geometry(L.n_units, static_cast<uint32_t>(span), gmax, splits, &ns_max, &cnt_max, &part_max);
        HS_CHECK_CONFIG(user_ws_bytes >= cnt_max + part_max,
                        "decode_attention: workspace of %llu bytes is smaller than the %llu needed",
                        static_cast<unsigned long long>(user_ws_bytes),
                        static_cast<unsigned long long>(cnt_max + part_max));
        ws = static_cast<uint8_t*>(user_ws);
        L.mailbox = reinterpret_cast<unsigned long long*>(ws + cnt_bytes);
        L.partial = reinterpret_cast<float*>(ws + cnt_bytes + decode_mailbox_bytes(L.n_units, ns, gmax));
    } else {
        ws = static_cast<uint8_t*>(workspace(s, cnt_bytes + decode_plain_bytes(L.n_units, ns, gqa), kWsDecode, &st));
        if (st) return st;
        L.mailbox = nullptr;  // allocated below when the launch combines cooperatively
        L.partial = reinterpret_cast<float*>(ws + cnt_bytes);
    }
    L.counters = reinterpret_cast<int*>(ws);
    L.out = out;
    L.out_mode = out_mode;
    // The parallel combine spins on the unit's arrivals: only when the whole grid
    // fits at once (occupancy of this smem plan); it is then launched cooperatively
    // so residency is guaranteed, not assumed (decode.cu launch_t).
    L.coop_combine = static_cast<int64_t>(ns) * L.n_units <= static_cast<int64_t>(hs::decode_resident_ctas(L, sm_count()));
    if (const char* env = getenv("HS_DECODE_COOP")) L.coop_combine = L.coop_combine && atoi(env) != 0;
    if (L.coop_combine && user_ws == nullptr) {
        L.mailbox = static_cast<unsigned long long*>(
            workspace(s, decode_mailbox_bytes(L.n_units, ns, gqa), kWsMailbox, &st));
        if (st) return st;
    }
    if (const char* env = getenv("HS_DECODE_MAILBOX"))  // tools: A/B of the tagged-mailbox combine
        if (atoi(env) == 0) L.mailbox = nullptr;
    L.blk_ctr = L.counters + 2 * L.n_units;
    // splits == 0 (auto): the unit's CTAs claim blocks dynamically (balanced across
    // SMs, summation order varies run to run).  An explicit split count keeps the
    // static, deterministic partition of attention.hpp:380-381.
    // Only for short per-CTA ranges (configs[1]: 114 blocks): there the load
    // balance decides the step time.  Long ranges (1M tokens: 910 blocks per
    // CTA) stream faster as contiguous static ranges (measured 382 vs 475 us).
    L.dynamic = splits == 0 && L.debug_stream_only == 0 && L.prefetch_distance == 0 && span / ns <= kDynamicMaxBlocks;
    if (const char* env = getenv("HS_DECODE_DYNAMIC")) L.dynamic = L.dynamic && atoi(env) != 0;
    // Units interleaved over the grid (measured: configs[1] 57.3 -> 55.4 us, the
    // per-unit finishing times no longer follow the GPC a unit landed on)
    L.interleave = 1;
    if (const char* env = getenv("HS_DECODE_INTERLEAVE")) L.interleave = atoi(env) != 0;
    L.cta_times = nullptr;
    static long long* times = nullptr;
    const char* tpath = getenv("HS_DECODE_TIMES");  // tools: per-CTA timeline dump
    if (tpath) {
        if (!times) cudaMalloc(&times, 65536 * 16 * sizeof(long long));
        cudaMemsetAsync(times, 0, 65536 * 16 * sizeof(long long), s);
        L.cta_times = times;
    }
    cudaError_t e = hs::launch_decode(L, s);
    count_launch();
    if (e != cudaSuccess) return cuda_fail(e, "decode launch");
    if (tpath) {
        const size_t n = static_cast<size_t>(L.n_units) * ns * 16;
        std::vector<long long> host(n);
        cudaStreamSynchronize(s);
        cudaMemcpy(host.data(), times, n * sizeof(long long), cudaMemcpyDeviceToHost);
        if (FILE* f = fopen(tpath, "wb")) {
            fwrite(host.data(), sizeof(long long), n, f);
            fclose(f);
        }
    }
    return HS_OK;
}

HS_API hs_status hs_decode(const void* q, const hs_device_cache* k, const hs_device_cache* v,
                           const void* k_tail, const void* v_tail, uint32_t tail, uint32_t gqa,
                           float scale, uint32_t splits, float* out, void* stream) {
    HS_CHECK_CONFIG(k != nullptr, "decode_attention: null key cache");
    return decode_common(q, k, v, k_tail, v_tail, tail, gqa, scale, splits, 0, k->logical_blocks, 1, out, 0,
                         nullptr, 0, stream);
}

HS_API hs_status hs_decode_workspace_bytes(const hs_device_cache* k, uint32_t gqa, uint32_t splits,
                                           uint64_t* bytes) {
    HS_CHECK_CONFIG(k != nullptr && bytes != nullptr, "decode_attention: null argument");
    int ns;
    size_t cnt, part;
    decode_geometry(k->n_units, k->logical_blocks, gqa < 8 ? gqa : 8, splits, &ns, &cnt, &part);
    *bytes = cnt + part;
    return HS_OK;
}

HS_API hs_status hs_decode_ws(const void* q, const hs_device_cache* k, const hs_device_cache* v,
                              const void* k_tail, const void* v_tail, uint32_t tail, uint32_t gqa, float scale,
                              uint32_t splits, float* out, void* workspace_ptr, uint64_t workspace_bytes,
                              void* stream) {
    HS_CHECK_CONFIG(k != nullptr, "decode_attention: null key cache");
    HS_CHECK_CONFIG(workspace_ptr != nullptr, "decode_attention: null workspace");
    return decode_common(q, k, v, k_tail, v_tail, tail, gqa, scale, splits, 0, k->logical_blocks, 1, out, 0,
                         workspace_ptr, workspace_bytes, stream);
}

HS_API hs_status hs_decode_partial(const void* q, const hs_device_cache* k, const hs_device_cache* v,
                                   const void* k_tail, const void* v_tail, uint32_t tail, uint32_t gqa,
                                   float scale, uint32_t block_begin, uint32_t block_end, int include_tail,
                                   float* partial, void* stream) {
    return decode_common(q, k, v, k_tail, v_tail, tail, gqa, scale, 0, block_begin, block_end, include_tail,
                         partial, 1, nullptr, 0, stream);
}

HS_API hs_status hs_decode_combine(const float* partials, uint32_t n_parts, uint32_t n_units, uint32_t gqa,
                                   uint32_t d, float* out, void* stream) {
    HS_CHECK_CONFIG(partials && out, "decode_combine: null argument");
    HS_CHECK_CONFIG(n_parts >= 1 && n_units >= 1 && gqa >= 1 && d >= 1, "decode_combine: empty shape");
    cudaError_t e = hs::launch_combine(partials, n_parts, n_units, gqa, d, out, static_cast<cudaStream_t>(stream));
    count_launch();
    if (e != cudaSuccess) return cuda_fail(e, "combine launch");
    return HS_OK;
}

HS_API hs_status hs_prefill(const void* q, uint32_t n_q, uint32_t gqa, const hs_device_cache* k,
                            const hs_device_cache* v, const void* k_tail, const void* v_tail, uint32_t tail,
                            int causal, float scale, float* out, void* stream) {
    hs_status st = check_pair(k, v);
    if (st) return st;
    HS_CHECK_CONFIG(q != nullptr && out != nullptr, "prefill_attention: null argument");
    HS_CHECK_CONFIG(gqa >= 1 && n_q >= 1, "prefill_attention: empty query set");
    const uint64_t n_kv = static_cast<uint64_t>(k->logical_blocks) * k->block_size + tail;
    HS_CHECK_CONFIG(n_kv > 0, "prefill_attention: empty key/value cache");
    HS_CHECK_CONFIG(!causal || n_kv >= n_q, "prefill_attention: causal queries exceed key sequence");
    HS_CHECK_CONFIG(tail == 0 || (k_tail != nullptr && v_tail != nullptr), "prefill_attention: null dense tail");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!specialised(k))
        return generic_attention(q, n_q, gqa, k, v, k_tail, v_tail, tail, causal, scale, 0, k->logical_blocks, 1, out,
                                 0, s);
    HS_CHECK_CONFIG(k->dense_count + k->sparse_count == k->logical_blocks &&
                        v->dense_count + v->sparse_count == v->logical_blocks,
                    "prefill_attention: caches with spare pool slots (per-unit counts) are decode-only");
    HS_CHECK_CONFIG(k->logical_blocks / 2 + 8 <= 4096,
                    "prefill_attention: %u blocks exceed the kernel's key-tile list (max 8184 blocks)",
                    k->logical_blocks);
    HS_CHECK_CONFIG(k->logical_blocks == 0 || k->slot_block != nullptr, "prefill_attention: key cache needs slot_block");
    hs::PrefillLaunch L{};
    L.bf16 = k->dtype == HS_DTYPE_BF16;
    L.n_units = k->n_units;
    L.nb = k->logical_blocks;
    L.gqa = gqa;
    L.n_q = n_q;
    // GQA stacking: hg heads of one KV head per CTA x 128 / hg queries
    // each.  At N = 128 columns per CTA the K/V traffic per column is the same for
    // every hg (a CTA stages the tiles its own 128 columns see), so hg = 1 is the
    // default; measured neutral to -4% at 64K.  Stacking that
    // shares tiles needs N > 128, which TMEM (two S^T buffers + O^T) cannot hold.
    L.hg = 1;
    if (const char* env = getenv("HS_PREFILL_HG")) {  // tests / tools: the stacked layouts
        const int g = atoi(env);
        if ((g == 1 || g == 2 || g == 4) && gqa % g == 0) L.hg = g;
    }
    L.qt = 128 / L.hg;
    L.tail = static_cast<int>(tail);
    L.n_tail_blocks = static_cast<int>((tail + hs::kBlock - 1) / hs::kBlock);
    L.k_tail = k_tail;
    L.v_tail = v_tail;
    L.causal = causal;
    L.k_dense_count = k->dense_count;
    L.k_sparse_count = k->sparse_count;
    L.v_dense_count = v->dense_count;
    L.v_sparse_count = v->sparse_count;
    L.scale_log2 = scale * 1.4426950408889634f;
    L.q = q;
    L.k_index = k->index_map;
    L.v_index = v->index_map;
    L.k_slot_block = k->slot_block;
    L.k_meta = k->meta_pool;
    L.v_meta = v->meta_pool;
    {
        const size_t kb = static_cast<size_t>(k->n_units) * k->sparse_count * 1024;
        const size_t vb = static_cast<size_t>(v->n_units) * v->sparse_count * 2048;
        const size_t tb = static_cast<size_t>(k->n_units) * L.n_tail_blocks * hs::kBlock * hs::kHeadDim * 2;
        // bf16 caches: fp16 copy of the V pools for the ping-pong kernel (PrefillLaunch::v16)
        L.v16 = L.bf16 && getenv("HS_PREFILL_BF16_HILO") == nullptr;
        const size_t vd16 = L.v16 ? static_cast<size_t>(v->n_units) * v->dense_count * hs::kBlock * hs::kHeadDim * 2 : 0;
        const size_t vn16 = L.v16 ? static_cast<size_t>(v->n_units) * v->sparse_count * hs::kBlock * hs::kHeadDim : 0;
        const size_t a256 = 256;
        const size_t nredo = static_cast<size_t>((n_q + L.qt - 1) / L.qt) * (gqa / L.hg) * k->n_units * sizeof(int);
        uint8_t* ws = static_cast<uint8_t*>(
            workspace(s, kb + vb + 2 * tb + vd16 + vn16 + nredo + 5 * a256, kWsPrefill, &st));
        if (st) return st;
        L.k_meta_hw = reinterpret_cast<uint16_t*>(ws);
        L.v_meta_hw = reinterpret_cast<uint16_t*>(ws + kb);
        L.k_tail_ws = reinterpret_cast<uint16_t*>(ws + kb + vb);
        L.v_tail_ws = reinterpret_cast<uint16_t*>(ws + kb + vb + tb);
        uint8_t* p16 = ws + ((kb + vb + 2 * tb + a256 - 1) / a256) * a256;
        L.v16_dense = reinterpret_cast<uint16_t*>(p16);
        L.v16_nnz = reinterpret_cast<uint16_t*>(p16 + vd16);
        L.v16_scale = reinterpret_cast<int*>(p16 + vd16 + vn16);
        L.redo = reinterpret_cast<int*>(p16 + ((vd16 + vn16 + 2 * sizeof(int) + a256 - 1) / a256) * a256);
        L.v_dense_src = v->dense_pool;
        L.v_nnz_src = v->nnz_pool;
    }
    L.out = out;
    static long long* trace = nullptr;
    if (getenv("HS_PREFILL_TRACE")) {
        if (!trace) cudaMalloc(&trace, 4096 * 16 * sizeof(long long));
        cudaMemsetAsync(trace, 0, 4096 * 16 * sizeof(long long), s);
        L.trace = trace;
    }
    static int* dbg = nullptr;
    if (getenv("HS_DEBUG_WAIT")) {
        if (!dbg) cudaMalloc(&dbg, 64);
        cudaMemsetAsync(dbg, 0, 64, s);
        L.dbg = dbg;
    }
    L.mode = 0;
    if (const char* env = getenv("HS_PREFILL_MODE")) L.mode = atoi(env);
    const uint64_t U = k->n_units;
    bool ok = make_map_q(&L.tm_q, q, n_q, U * gqa, static_cast<uint32_t>(L.qt), static_cast<uint32_t>(L.hg));
    // K tiles are two consecutive pool slots (128 rows) per TMA; a single-block
    // tile's second half is masked in the kernel (and zero-filled past the pool).
    ok &= make_map(&L.tm_knnz, k->nnz_pool, 64, U * k->sparse_count * 64, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    ok &= make_map_halves(&L.tm_kden, k->dense_pool, U * k->dense_count * 64, 128);
    const void* vnnz = L.v16 ? static_cast<const void*>(L.v16_nnz) : v->nnz_pool;
    const void* vden = L.v16 ? static_cast<const void*>(L.v16_dense) : v->dense_pool;
    if (L.v16 && v->sparse_count == 0) vnnz = nullptr;
    if (L.v16 && v->dense_count == 0) vden = nullptr;
    ok &= make_map(&L.tm_vnnz, vnnz, 32, U * v->sparse_count * 128, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B);
    ok &= make_map(&L.tm_vden, vden, 64, U * v->dense_count * 128, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    ok &= make_map(&L.tm_vnnz2, vnnz, 32, U * v->sparse_count * 128, 32, 256, CU_TENSOR_MAP_SWIZZLE_64B);
    ok &= make_map(&L.tm_vden2, vden, 64, U * v->dense_count * 128, 64, 256, CU_TENSOR_MAP_SWIZZLE_128B);
    const uint64_t ntb = static_cast<uint64_t>(L.n_tail_blocks);
    ok &= make_map_halves(&L.tm_ktail, ntb ? L.k_tail_ws : nullptr, U * ntb * 64, 128);
    ok &= make_map(&L.tm_vtail, ntb ? L.v_tail_ws : nullptr, 64, U * ntb * 128, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!ok) return fail(HS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    int n_kernels = 0;
    cudaError_t e = hs::launch_prefill(L, s, &n_kernels);
    count_launch(n_kernels);
    if (e != cudaSuccess) return cuda_fail(e, "prefill launch");
    if (L.trace) {
        static std::vector<long long> host(4096 * 16);
        cudaStreamSynchronize(s);
        cudaMemcpy(host.data(), L.trace, host.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        if (FILE* f = fopen(getenv("HS_PREFILL_TRACE"), "wb")) {
            fwrite(host.data(), sizeof(long long), host.size(), f);
            fclose(f);
        }
    }
    if (L.dbg) {
        int h[16] = {0};
        cudaStreamSynchronize(s);
        cudaMemcpy(h, L.dbg, sizeof h, cudaMemcpyDeviceToHost);
        if (getenv("HS_DEBUG_COUNTS"))
            fprintf(stderr, "prefill counts: slow %d rescale %d grow %d\n", h[8], h[9], h[10]);
        if (h[0]) return fail(HS_ERR_CUDA, "prefill watchdog: barrier tag %d parity %d block %d thread %d", h[0], h[1], h[2], h[3]);
    }
    return HS_OK;
}

}  // extern "C"
