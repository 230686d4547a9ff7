// hierasparse_b200.hpp — C++ host layer of the B200-native HieraSparse hot path.
//
// Keeps the reference's `hierasparse::` API surface for the hot path
// (/root/reference/proj/include/hierasparse: pruner.hpp, compressed_cache.hpp,
// attention.hpp) over device-resident pools, and calls the sm_100a kernels
// through the C ABI in hierasparse_b200.h.  Header-only; link
// libhierasparse_b200.so and the CUDA runtime.
//
//   reference                                   this header (namespace hierasparse::b200)
//   SparsityConfig (masks.hpp:73-99)            SparsityConfig
//   CompressedCache (compressed_cache.hpp:37)   DeviceCompressedCache (RAII, n_units units)
//   prune_cache (pruner.hpp:165-176)            prune_cache            (+ fused compression)
//   fused_magnitude_compress (:262-267)         fused_magnitude_compress
//   decompress (:271-298)                       decompress
//   measure_size (:303-310)                     DeviceCompressedCache::measure_size
//   decode_attention (attention.hpp:360-409)    decode_attention
//   attend_range -> SplitPartial (:249-304)     decode_partial / decode_combine
//   prefill_attention (:323-354)                prefill_attention
//   ConfigError / DataError / IoError           same names (errors.hpp:10-25), plus CudaError
//
// Host-data overloads (`*_host`) take any Tensor2D-like type (members rows,
// cols, data: the reference's Tensor2D, tensor.hpp:16-31), round it once to the
// 16-bit storage type, run the device path and copy results back, so the
// reference's own test shapes run against the GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hierasparse_b200.h"

namespace hierasparse::b200 {

// ----------------------------------------------------------------- errors ---
struct ConfigError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(hs_status s) {
    switch (s) {
        case HS_OK: return;
        case HS_ERR_CONFIG: throw ConfigError(hs_last_error());
        case HS_ERR_DATA: throw DataError(hs_last_error());
        case HS_ERR_IO: throw IoError(hs_last_error());
        default: throw CudaError(hs_last_error());
    }
}
inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

enum class DType { kBF16 = HS_DTYPE_BF16, kF16 = HS_DTYPE_F16 };
enum class GroupAxis { kChannel = HS_AXIS_CHANNEL, kSequence = HS_AXIS_SEQUENCE };  // masks.hpp:19-22

// masks.hpp:73-99 with the fixed 2:4 pattern.
struct SparsityConfig {
    double s_key = 0.0;
    double s_value = 0.0;
    std::size_t block_size = 64;
    std::size_t sink_tokens = 0;
    std::size_t local_window = 0;

    hs_sparsity_config c() const {
        return hs_sparsity_config{s_key, s_value, static_cast<uint32_t>(block_size), 0u, sink_tokens, local_window};
    }
};

// measure_size (compressed_cache.hpp:303-310), bytes per unit at 2 B/element.
struct SizeBreakdown {
    std::size_t size_idx = 0, size_den = 0, size_nnz = 0, size_e = 0;
    std::size_t total() const { return size_idx + size_den + size_nnz + size_e; }
};

// ------------------------------------------------------- device storage ---
template <class T>
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t n) : n_(n) {
        if (n) check_cuda(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
    }
    ~DeviceBuffer() {
        if (p_) cudaFree(p_);
    }
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            if (p_) cudaFree(p_);
            p_ = std::exchange(o.p_, nullptr);
            n_ = std::exchange(o.n_, 0);
        }
        return *this;
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    T* get() const { return p_; }
    std::size_t size() const { return n_; }
    std::vector<T> to_host() const {
        std::vector<T> h(n_);
        if (n_) check_cuda(cudaMemcpy(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
        return h;
    }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

// CompressedCache (compressed_cache.hpp:37-110) for n_units (request, KV head)
// units in the canonical layout of hierarchical storage (see hierasparse_b200.h).
class DeviceCompressedCache {
public:
    DeviceCompressedCache(DType dtype, GroupAxis axis, uint32_t n_units, uint32_t logical_blocks,
                          uint32_t dense_count, uint32_t sparse_count, uint32_t head_dim = 128,
                          uint32_t block_size = 64)
        : d_{static_cast<hs_dtype>(dtype), static_cast<hs_axis>(axis), head_dim, block_size, n_units,
             logical_blocks, dense_count, sparse_count, nullptr, nullptr, nullptr, nullptr, nullptr} {
        uint64_t idx, den, nnz, meta, sb;
        check(hs_cache_bytes(&d_, &idx, &den, &nnz, &meta, &sb));
        index_ = DeviceBuffer<uint8_t>(idx);
        dense_ = DeviceBuffer<uint8_t>(den);
        nnz_ = DeviceBuffer<uint8_t>(nnz);
        meta_ = DeviceBuffer<uint8_t>(meta);
        slot_ = DeviceBuffer<uint8_t>(sb);
        flags_ = DeviceBuffer<uint8_t>(static_cast<std::size_t>(n_units) * logical_blocks);
        losses_ = DeviceBuffer<double>(static_cast<std::size_t>(n_units) * logical_blocks);
        d_.index_map = reinterpret_cast<int16_t*>(index_.get());
        d_.dense_pool = dense_.get();
        d_.nnz_pool = nnz_.get();
        d_.meta_pool = reinterpret_cast<uint16_t*>(meta_.get());
        d_.slot_block = reinterpret_cast<int32_t*>(slot_.get());
    }
    const hs_device_cache& desc() const { return d_; }
    hs_device_cache& desc() { return d_; }
    uint32_t n_units() const { return d_.n_units; }
    uint32_t logical_blocks() const { return d_.logical_blocks; }
    uint32_t dense_count() const { return d_.dense_count; }
    uint32_t sparse_count() const { return d_.sparse_count; }
    std::size_t sequence_length() const { return static_cast<std::size_t>(d_.logical_blocks) * d_.block_size; }
    GroupAxis axis() const { return static_cast<GroupAxis>(d_.axis); }
    DType dtype() const { return static_cast<DType>(d_.dtype); }
    uint8_t* flags() const { return flags_.get(); }
    double* losses() const { return losses_.get(); }

    SizeBreakdown measure_size() const {  // per unit
        const std::size_t be = static_cast<std::size_t>(d_.block_size) * d_.head_dim;
        return SizeBreakdown{static_cast<std::size_t>(d_.logical_blocks) * 2, d_.dense_count * be * 2,
                             d_.sparse_count * (be / 2) * 2, d_.sparse_count * (be / 16) * 2};
    }

    // Unit u's arrays copied to the host (index map, 16-bit pools, metadata).
    struct HostUnit {
        std::vector<int16_t> index_map;
        std::vector<uint16_t> dense_pool, nnz_pool, meta_pool;  // raw 16-bit storage
    };
    HostUnit unit_to_host(uint32_t u) const {
        HostUnit h;
        const std::size_t be = static_cast<std::size_t>(d_.block_size) * d_.head_dim;
        auto copy = [](auto& dst, const void* base, std::size_t offset_elems, std::size_t n) {
            dst.resize(n);
            const auto* src = static_cast<const uint8_t*>(base) + offset_elems * sizeof(dst[0]);
            if (n) check_cuda(cudaMemcpy(dst.data(), src, n * sizeof(dst[0]), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
        };
        copy(h.index_map, d_.index_map, static_cast<std::size_t>(u) * d_.logical_blocks, d_.logical_blocks);
        copy(h.dense_pool, d_.dense_pool, u * d_.dense_count * be, d_.dense_count * be);
        copy(h.nnz_pool, d_.nnz_pool, u * d_.sparse_count * (be / 2), d_.sparse_count * (be / 2));
        copy(h.meta_pool, d_.meta_pool, u * d_.sparse_count * (be / 16), d_.sparse_count * (be / 16));
        return h;
    }

private:
    hs_device_cache d_;
    DeviceBuffer<uint8_t> index_, dense_, nnz_, meta_, slot_, flags_;
    DeviceBuffer<double> losses_;
};

// ------------------------------------------------------------ compression ---
// Pool geometry before any data is seen (pruner.hpp:106-108, masks.hpp:93-98).
struct PoolCounts {
    uint32_t logical_blocks, dense_count, sparse_count, prefix_blocks, suffix_blocks;
};
inline PoolCounts pool_counts(std::size_t rows, const SparsityConfig& cfg, double sparsity) {
    PoolCounts p{};
    const hs_sparsity_config c = cfg.c();
    check(hs_pool_counts(rows, &c, sparsity, &p.logical_blocks, &p.dense_count, &p.sparse_count, &p.prefix_blocks,
                         &p.suffix_blocks));
    return p;
}

// hierarchical_mask_for + fused_magnitude_compress for one cache kind of every
// unit: src = device [n_units][rows][head_dim] 16-bit, token-major.  The block
// losses land in out.losses() when the selection ranks them or with_losses;
// a static selection (quota 0 or every prunable block) otherwise skips them
// (the reference's HierarchicalMask carries none) and leaves NaN.
inline DeviceCompressedCache compress_one(const void* src, DType dtype, uint32_t n_units, std::size_t rows,
                                          const SparsityConfig& cfg, double sparsity, GroupAxis axis,
                                          cudaStream_t stream = nullptr, uint32_t head_dim = 128,
                                          bool with_losses = false) {
    const PoolCounts p = pool_counts(rows, cfg, sparsity);
    DeviceCompressedCache out(dtype, axis, n_units, p.logical_blocks, p.dense_count, p.sparse_count, head_dim,
                              static_cast<uint32_t>(cfg.block_size));
    const hs_sparsity_config c = cfg.c();
    const bool static_sel =
        p.sparse_count == 0 || p.sparse_count == p.logical_blocks - p.prefix_blocks - p.suffix_blocks;
    double* losses = out.losses();
    if (static_sel && !with_losses) {
        check_cuda(cudaMemsetAsync(losses, 0xFF, sizeof(double) * n_units * p.logical_blocks, stream),
                   "cudaMemsetAsync");  // all-ones doubles: NaN, "not computed"
        losses = nullptr;
    }
    check(hs_prune_compress(src, rows * head_dim, rows, &c, sparsity, &out.desc(), losses, out.flags(), stream));
    return out;
}

// prune_cache (pruner.hpp:165-176) followed by compression of both caches:
// key along channels at S_K, value along the sequence at S_V.
inline std::pair<DeviceCompressedCache, DeviceCompressedCache> prune_cache(const void* key, const void* value,
                                                                           DType dtype, uint32_t n_units,
                                                                           std::size_t rows,
                                                                           const SparsityConfig& cfg,
                                                                           cudaStream_t stream = nullptr) {
    return {compress_one(key, dtype, n_units, rows, cfg, cfg.s_key, GroupAxis::kChannel, stream),
            compress_one(value, dtype, n_units, rows, cfg, cfg.s_value, GroupAxis::kSequence, stream)};
}

// Device status word (hierasparse_b200.h "status words"): the data-validating
// entry points record the reference's DataErrors here asynchronously.
class StatusWord {
public:
    explicit StatusWord(cudaStream_t stream = nullptr) : w_(1) {
        check_cuda(cudaMemsetAsync(w_.get(), 0, sizeof(uint64_t), stream), "cudaMemsetAsync");
    }
    uint64_t* get() const { return w_.get(); }
    // Synchronises on `stream` and throws what the reference would have thrown.
    void check(cudaStream_t stream = nullptr) const {
        uint64_t h = 0;
        check_cuda(cudaMemcpyAsync(&h, w_.get(), sizeof h, cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync");
        check_cuda(cudaStreamSynchronize(stream), "status word");
        hierasparse::b200::check(hs_status_word_decode(h));
    }

private:
    DeviceBuffer<uint64_t> w_;
};

// fused_magnitude_compress (compressed_cache.hpp:262-267) under an explicit
// BlockMask: flags device u8 [n_units][nb], 1 = dense; dense_count per unit.
// status == nullptr: checked (synchronising) like the reference; otherwise the
// ConfigError of a mismatched dense count is left in *status (asynchronous).
inline DeviceCompressedCache fused_magnitude_compress(const void* src, const uint8_t* flags_dev,
                                                      uint32_t dense_count, DType dtype, uint32_t n_units,
                                                      std::size_t rows, GroupAxis axis, std::size_t block_size = 64,
                                                      cudaStream_t stream = nullptr, uint32_t head_dim = 128,
                                                      StatusWord* status = nullptr) {
    if (block_size == 0 || rows % block_size) throw ConfigError("compress: sequence length not divisible by block_size");
    const uint32_t nb = static_cast<uint32_t>(rows / block_size);
    DeviceCompressedCache out(dtype, axis, n_units, nb, dense_count, nb - dense_count, head_dim,
                              static_cast<uint32_t>(block_size));
    StatusWord own(stream);
    StatusWord* st = status ? status : &own;
    check(hs_compress_with_flags(src, rows * head_dim, rows, flags_dev, &out.desc(), st->get(), stream));
    if (!status) own.check(stream);
    return out;
}

// compress (compressed_cache.hpp:196-225) under an explicit HierarchicalMask:
// element mask device u8 [n_units][rows][head_dim] + BlockMask flags.  Groups of
// sparse blocks keeping != 2 elements throw DataError (or land in *status).
inline DeviceCompressedCache compress(const void* src, const uint8_t* element_mask_dev, const uint8_t* flags_dev,
                                      uint32_t dense_count, DType dtype, uint32_t n_units, std::size_t rows,
                                      GroupAxis axis, std::size_t block_size = 64, cudaStream_t stream = nullptr,
                                      uint32_t head_dim = 128, StatusWord* status = nullptr) {
    if (block_size == 0 || rows % block_size) throw ConfigError("compress: sequence length not divisible by block_size");
    const uint32_t nb = static_cast<uint32_t>(rows / block_size);
    DeviceCompressedCache out(dtype, axis, n_units, nb, dense_count, nb - dense_count, head_dim,
                              static_cast<uint32_t>(block_size));
    StatusWord own(stream);
    StatusWord* st = status ? status : &own;
    check(hs_compress_with_mask(src, rows * head_dim, rows, element_mask_dev, rows * head_dim, flags_dev,
                                &out.desc(), st->get(), stream));
    if (!status) own.check(stream);
    return out;
}

// decompress (compressed_cache.hpp:271-298) into dst [n_units][rows][d].
inline void decompress(const DeviceCompressedCache& c, void* dst, cudaStream_t stream = nullptr,
                       StatusWord* status = nullptr) {
    StatusWord own(stream);
    StatusWord* st = status ? status : &own;
    check(hs_decompress(&c.desc(), dst, st->get(), stream));
    if (!status) own.check(stream);
}

// Decode-phase re-prune (pipeline.hpp:227-240: decompress -> prune_cache at the
// decode sparsity -> compress) in one pass over c's pools.  A corrupt input
// throws decompress's DataError (status == nullptr) or is left in *status.
inline DeviceCompressedCache recompress(const DeviceCompressedCache& c, const SparsityConfig& cfg, double sparsity,
                                        cudaStream_t stream = nullptr, StatusWord* status = nullptr) {
    const hs_device_cache& in = c.desc();
    const PoolCounts p = pool_counts(static_cast<std::size_t>(in.logical_blocks) * in.block_size, cfg, sparsity);
    DeviceCompressedCache out(static_cast<DType>(in.dtype), static_cast<GroupAxis>(in.axis), in.n_units,
                              p.logical_blocks, p.dense_count, p.sparse_count, in.head_dim,
                              static_cast<uint32_t>(cfg.block_size));
    const hs_sparsity_config cc = cfg.c();
    StatusWord own(stream);
    StatusWord* st = status ? status : &own;
    check(hs_recompress(&in, &cc, sparsity, &out.desc(), out.losses(), out.flags(), st->get(), stream));
    if (!status) own.check(stream);
    return out;
}

// Dense-tail growth: the cache re-pruned over its blocks followed by tail_rows
// (whole blocks) of tail tokens tail [n_units][tail_rows][d] (device, unit
// stride tail_unit_stride elements; 0 = tail_rows * d) in one pass.
inline DeviceCompressedCache absorb_tail(const DeviceCompressedCache& c, const void* tail, std::size_t tail_rows,
                                         const SparsityConfig& cfg, double sparsity, cudaStream_t stream = nullptr,
                                         std::size_t tail_unit_stride = 0, StatusWord* status = nullptr) {
    const hs_device_cache& in = c.desc();
    const std::size_t rows = static_cast<std::size_t>(in.logical_blocks) * in.block_size + tail_rows;
    const PoolCounts p = pool_counts(rows, cfg, sparsity);
    DeviceCompressedCache out(static_cast<DType>(in.dtype), static_cast<GroupAxis>(in.axis), in.n_units,
                              p.logical_blocks, p.dense_count, p.sparse_count, in.head_dim,
                              static_cast<uint32_t>(cfg.block_size));
    const hs_sparsity_config cc = cfg.c();
    StatusWord own(stream);
    StatusWord* st = status ? status : &own;
    check(hs_absorb_tail(&in, tail, tail_unit_stride ? tail_unit_stride : tail_rows * in.head_dim, tail_rows, &cc,
                         sparsity, &out.desc(), out.losses(), out.flags(), st->get(), stream));
    if (!status) own.check(stream);
    return out;
}

// -------------------------------------------------------------- attention ---
// decode_attention (attention.hpp:360-409): q [n_units][gqa][d] -> out fp32.
inline void decode_attention(const void* q, const DeviceCompressedCache& k, const DeviceCompressedCache& v,
                             uint32_t gqa, float scale, float* out, cudaStream_t stream = nullptr,
                             uint32_t splits = 0, const void* k_tail = nullptr, const void* v_tail = nullptr,
                             uint32_t tail = 0) {
    check(hs_decode(q, &k.desc(), &v.desc(), k_tail, v_tail, tail, gqa, scale, splits, out, stream));
}

// attend_range over blocks [begin, end) (+ tail) -> packed SplitPartial
// [n_units][gqa][d+2] = (O, m, l) (attention.hpp:249-304, :65-69).
inline void decode_partial(const void* q, const DeviceCompressedCache& k, const DeviceCompressedCache& v,
                           uint32_t gqa, float scale, uint32_t block_begin, uint32_t block_end, bool include_tail,
                           float* partial, cudaStream_t stream = nullptr, const void* k_tail = nullptr,
                           const void* v_tail = nullptr, uint32_t tail = 0) {
    check(hs_decode_partial(q, &k.desc(), &v.desc(), k_tail, v_tail, tail, gqa, scale, block_begin, block_end,
                            include_tail ? 1 : 0, partial, stream));
}

// LSE combine (attention.hpp:387-407): partials [n_parts][n_units][gqa][d+2].
inline void decode_combine(const float* partials, uint32_t n_parts, uint32_t n_units, uint32_t gqa, float* out,
                           cudaStream_t stream = nullptr, uint32_t d = 128) {
    check(hs_decode_combine(partials, n_parts, n_units, gqa, d, out, stream));
}

// prefill_attention (attention.hpp:323-354): q [n_units][gqa][n_q][d] -> out fp32,
// over the compressed caches followed by an optional dense tail
// k_tail / v_tail [n_units][tail][d] (CacheView::dense_tail, attention.hpp:19-31).
inline void prefill_attention(const void* q, uint32_t n_q, uint32_t gqa, const DeviceCompressedCache& k,
                              const DeviceCompressedCache& v, bool causal, float scale, float* out,
                              cudaStream_t stream = nullptr, const void* k_tail = nullptr,
                              const void* v_tail = nullptr, uint32_t tail = 0) {
    check(hs_prefill(q, n_q, gqa, &k.desc(), &v.desc(), k_tail, v_tail, tail, causal ? 1 : 0, scale, out, stream));
}

// flop_and_byte_count byte side (attention.hpp:415-467) for one unit.
inline std::size_t decode_bytes_moved(const DeviceCompressedCache& k, const DeviceCompressedCache& v,
                                      std::size_t tail = 0) {
    constexpr std::size_t kHeader = 38;  // container.hpp:42
    return 2 * kHeader + k.measure_size().total() + v.measure_size().total() + 2 * tail * 128 * 2;
}

// ------------------------------------------------- host-data convenience ---
// RNE float -> 16-bit storage bits (bf16 / IEEE binary16), the single rounding
// of the synthetic inputs both the kernels and the fp32 oracle see.
inline uint16_t to_bits(float x, DType t) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if (t == DType::kBF16) {
        if ((u & 0x7FFFFFFFu) > 0x7F800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
        u += 0x7FFFu + ((u >> 16) & 1u);
        return static_cast<uint16_t>(u >> 16);
    }
    const uint32_t sign = (u >> 16) & 0x8000u;
    u &= 0x7FFFFFFFu;
    if (u >= 0x7F800000u) return static_cast<uint16_t>(sign | (u > 0x7F800000u ? 0x7E00u : 0x7C00u));
    if (u >= 0x477FF000u) return static_cast<uint16_t>(sign | 0x7C00u);  // rounds to infinity
    uint32_t r, rem, half;
    if (u < 0x38800000u) {  // half subnormal: units of 2^-24
        const uint32_t e = u >> 23;
        if (e < 102) return static_cast<uint16_t>(sign);
        const uint32_t m = (u & 0x7FFFFFu) | 0x800000u, shift = 126 - e;
        r = m >> shift;
        rem = m & ((1u << shift) - 1u);
        half = 1u << (shift - 1);
    } else {
        r = (u - 0x38000000u) >> 13;
        rem = u & 0x1FFFu;
        half = 0x1000u;
    }
    if (rem > half || (rem == half && (r & 1u))) ++r;
    return static_cast<uint16_t>(sign | r);
}
inline float from_bits(uint16_t b, DType t) {
    if (t == DType::kBF16) {
        const uint32_t u = static_cast<uint32_t>(b) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    }
    const uint32_t sign = (b & 0x8000u) << 16, e = (b >> 10) & 0x1Fu, m = b & 0x3FFu;
    uint32_t u;
    if (e == 0) {
        if (m == 0) {
            u = sign;
        } else {
            int ee = -1;
            uint32_t mm = m;
            do {
                ++ee;
                mm <<= 1;
            } while (!(mm & 0x400u));
            u = sign | ((112 - ee) << 23) | ((mm & 0x3FFu) << 13);
        }
    } else if (e == 31) {
        u = sign | 0x7F800000u | (m << 13);
    } else {
        u = sign | ((e + 112) << 23) | (m << 13);
    }
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// Upload a list of Tensor2D-like matrices (rows x head_dim each) as one device
// [n_units][rows][head_dim] 16-bit array.
template <class Tensor>
DeviceBuffer<uint16_t> upload_units(const std::vector<const Tensor*>& units, DType t) {
    if (units.empty()) throw ConfigError("upload: no units");
    const std::size_t per = units[0]->rows * units[0]->cols;
    std::vector<uint16_t> h(per * units.size());
    for (std::size_t u = 0; u < units.size(); ++u) {
        if (units[u]->rows * units[u]->cols != per) throw ConfigError("upload: unit shapes differ");
        for (std::size_t i = 0; i < per; ++i) h[u * per + i] = to_bits(units[u]->data[i], t);
    }
    DeviceBuffer<uint16_t> d(h.size());
    check_cuda(cudaMemcpy(d.get(), h.data(), h.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    return d;
}

// Host-side views: a list of per-unit Tensor2D-like matrices (the reference's
// Tensor2D per (request, KV head) unit; every unit of a call has the same shape).
template <class Tensor>
using UnitList = std::vector<const Tensor*>;

namespace detail {
template <class Tensor>
std::vector<Tensor> download_units(const DeviceBuffer<float>& out, std::size_t n_units, std::size_t rows,
                                   std::size_t cols) {
    const auto h = out.to_host();
    std::vector<Tensor> res;
    res.reserve(n_units);
    for (std::size_t u = 0; u < n_units; ++u) {
        Tensor o(rows, cols);
        std::copy(h.begin() + u * rows * cols, h.begin() + (u + 1) * rows * cols, o.data.begin());
        res.push_back(std::move(o));
    }
    return res;
}
template <class Tensor>
DeviceBuffer<uint16_t> upload_tails(const UnitList<Tensor>& tails, DType t, std::size_t n_units,
                                    uint32_t* tail_rows) {
    *tail_rows = 0;
    if (tails.empty()) return DeviceBuffer<uint16_t>();
    if (tails.size() != n_units) throw ConfigError("attention: one dense tail per unit");
    *tail_rows = static_cast<uint32_t>(tails[0]->rows);
    if (*tail_rows == 0) return DeviceBuffer<uint16_t>();
    return upload_units<Tensor>(tails, t);
}
}  // namespace detail

// decode_attention over every unit with host tensors: queries[u] (gqa x d), the
// device caches of all units and optional dense tails (tail x d per unit) ->
// one output Tensor2D (gqa x d) per unit.
template <class Tensor>
std::vector<Tensor> decode_attention_host(const UnitList<Tensor>& queries, const DeviceCompressedCache& k,
                                          const DeviceCompressedCache& v, float scale, uint32_t splits = 0,
                                          const UnitList<Tensor>& k_tails = {},
                                          const UnitList<Tensor>& v_tails = {}) {
    if (queries.size() != k.n_units()) throw ConfigError("decode_attention: one query matrix per unit");
    const DType t = k.dtype();
    const std::size_t gqa = queries[0]->rows, d = queries[0]->cols;
    auto qd = upload_units<Tensor>(queries, t);
    uint32_t tail = 0, tail_v = 0;
    auto kt = detail::upload_tails<Tensor>(k_tails, t, k.n_units(), &tail);
    auto vt = detail::upload_tails<Tensor>(v_tails, t, k.n_units(), &tail_v);
    if (tail != tail_v) throw ConfigError("attention: key/value token counts differ");
    DeviceBuffer<float> out(queries.size() * gqa * d);
    decode_attention(qd.get(), k, v, static_cast<uint32_t>(gqa), scale, out.get(), nullptr, splits, kt.get(),
                     vt.get(), tail);
    check_cuda(cudaDeviceSynchronize(), "decode_attention");
    return detail::download_units<Tensor>(out, queries.size(), gqa, d);
}

// One unit (the reference's decode_attention signature shape).
template <class Tensor>
Tensor decode_attention_host(const Tensor& queries, const DeviceCompressedCache& k, const DeviceCompressedCache& v,
                             float scale, uint32_t splits = 0) {
    if (k.n_units() != 1) throw ConfigError("decode_attention_host: one unit per call");
    return std::move(decode_attention_host<Tensor>(UnitList<Tensor>{&queries}, k, v, scale, splits)[0]);
}

// prefill_attention over every unit and query head with host tensors:
// queries[u * gqa + g] (n_q x d), optional dense tails per unit -> one output
// Tensor2D (n_q x d) per (unit, query head), in the same order.
template <class Tensor>
std::vector<Tensor> prefill_attention_host(const UnitList<Tensor>& queries, uint32_t gqa,
                                           const DeviceCompressedCache& k, const DeviceCompressedCache& v,
                                           bool causal, float scale, const UnitList<Tensor>& k_tails = {},
                                           const UnitList<Tensor>& v_tails = {}) {
    if (gqa == 0 || queries.size() != static_cast<std::size_t>(k.n_units()) * gqa)
        throw ConfigError("prefill_attention: n_units x gqa query matrices expected");
    const DType t = k.dtype();
    const std::size_t n_q = queries[0]->rows, d = queries[0]->cols;
    auto qd = upload_units<Tensor>(queries, t);
    uint32_t tail = 0, tail_v = 0;
    auto kt = detail::upload_tails<Tensor>(k_tails, t, k.n_units(), &tail);
    auto vt = detail::upload_tails<Tensor>(v_tails, t, k.n_units(), &tail_v);
    if (tail != tail_v) throw ConfigError("attention: key/value token counts differ");
    DeviceBuffer<float> out(queries.size() * n_q * d);
    prefill_attention(qd.get(), static_cast<uint32_t>(n_q), gqa, k, v, causal, scale, out.get(), nullptr, kt.get(),
                      vt.get(), tail);
    check_cuda(cudaDeviceSynchronize(), "prefill_attention");
    return detail::download_units<Tensor>(out, queries.size(), n_q, d);
}

template <class Tensor>
Tensor prefill_attention_host(const Tensor& queries, const DeviceCompressedCache& k, const DeviceCompressedCache& v,
                              bool causal, float scale) {
    if (k.n_units() != 1) throw ConfigError("prefill_attention_host: one unit per call");
    return std::move(prefill_attention_host<Tensor>(UnitList<Tensor>{&queries}, 1, k, v, causal, scale)[0]);
}

}  // namespace hierasparse::b200
