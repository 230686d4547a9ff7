// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference
// headers (arxiv 2604.16864, /root/reference/proj/include/hierasparse).  Built by
// oracle/Makefile into oracle/_ref/libhs_ref.so; no reference source is copied
// into this repository.  Exports the ref_* half of oracle/hs_oracle.h.
//
// Each entry converts plain arrays to the reference's own types
// (Tensor2D tensor.hpp:16-31, CompressedCache compressed_cache.hpp:37-110,
// CacheView / AttentionWorkload attention.hpp:22-41), calls the reference
// function named in the comment, and copies the result back out.
#include <cstring>
#include <exception>
#include <string>

#include "hierasparse/hierasparse.hpp"
#include "hs_oracle.h"

using namespace hierasparse;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const DataError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

Tensor2D to_tensor(const float* p, std::size_t rows, std::size_t cols) {
    Tensor2D t(rows, cols);
    if (rows != 0 && cols != 0) std::memcpy(t.data.data(), p, rows * cols * sizeof(float));
    return t;
}

SparsityConfig to_cfg(const hso_config* c) {
    SparsityConfig s;
    s.s_key = c->s_key;
    s.s_value = c->s_value;
    s.block_size = c->block_size;
    s.sink_tokens = c->sink_tokens;
    s.local_window = c->local_window;
    return s;
}

CompressedCache to_cache(const hso_cache* c) {
    CompressedCache cc;
    cc.cfg.block_size = c->block_size;
    cc.axis = c->axis == 0 ? GroupAxis::kChannel : GroupAxis::kSequence;
    cc.head_dim = c->head_dim;
    cc.logical_blocks = c->logical_blocks;
    cc.index_map.assign(c->index_map, c->index_map + c->logical_blocks);
    cc.dense_count = c->dense_count;
    cc.sparse_count = c->sparse_count;
    cc.dense_pool.assign(c->dense_pool, c->dense_pool + c->dense_count * cc.dense_block_elems());
    cc.nnz_pool.assign(c->nnz_pool, c->nnz_pool + c->sparse_count * cc.nnz_block_elems());
    cc.meta_pool.assign(c->meta_pool, c->meta_pool + c->sparse_count * cc.meta_words_per_block());
    return cc;
}

void from_cache(const CompressedCache& cc, hso_cache* c) {
    c->axis = cc.axis == GroupAxis::kChannel ? 0 : 1;
    c->head_dim = cc.head_dim;
    c->block_size = cc.cfg.block_size;
    c->logical_blocks = cc.logical_blocks;
    c->dense_count = cc.dense_count;
    c->sparse_count = cc.sparse_count;
    std::memcpy(c->index_map, cc.index_map.data(), cc.index_map.size() * sizeof(int16_t));
    std::memcpy(c->dense_pool, cc.dense_pool.data(), cc.dense_pool.size() * sizeof(float));
    std::memcpy(c->nnz_pool, cc.nnz_pool.data(), cc.nnz_pool.size() * sizeof(float));
    std::memcpy(c->meta_pool, cc.meta_pool.data(), cc.meta_pool.size() * sizeof(uint16_t));
}

// CacheView over an optional compressed prefix plus the dense tail.
struct Views {
    CompressedCache kc, vc;
    bool has_k = false, has_v = false;
    CacheView k, v;
    Views(const hso_cache* kp, const hso_cache* vp, const float* kt, const float* vt,
          std::size_t tail, std::size_t d) {
        if (kp) { kc = to_cache(kp); has_k = true; }
        if (vp) { vc = to_cache(vp); has_v = true; }
        k.compressed = has_k ? &kc : nullptr;
        v.compressed = has_v ? &vc : nullptr;
        k.dense_tail = tail ? to_tensor(kt, tail, d) : Tensor2D(0, d);
        v.dense_tail = tail ? to_tensor(vt, tail, d) : Tensor2D(0, d);
    }
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_derive_seed(uint64_t base, uint64_t stream) { return derive_seed(base, stream); }

uint64_t ref_head_seed(uint64_t base, size_t head, size_t role) {
    return detail::head_seed(base, head, role);
}

void ref_random_gaussian(size_t rows, size_t cols, uint64_t seed, float scale, float* out) {
    const Tensor2D t = random_gaussian(rows, cols, seed, scale);
    std::memcpy(out, t.data.data(), rows * cols * sizeof(float));
}

// detail::hierarchical_mask_for (pruner.hpp:121-158) then compress
// (compressed_cache.hpp:196) or fused_magnitude_compress (:262).
int ref_prune_compress(const float* x, size_t rows, size_t cols, const hso_config* cfg, int axis,
                       double sparsity, int fused, hso_cache* out, uint8_t* flags,
                       double* losses, uint8_t* element_mask) {
    return guarded([&] {
        const Tensor2D t = to_tensor(x, rows, cols);
        const SparsityConfig sc = to_cfg(cfg);
        sc.validate();
        detail::check_config(cols % sc.pattern.m_group == 0,
                             "prune_cache: head dimension not divisible by m_group");
        const GroupAxis ax = axis == 0 ? GroupAxis::kChannel : GroupAxis::kSequence;
        const HierarchicalMask hm = detail::hierarchical_mask_for(t, ax, sparsity, sc);
        std::memcpy(flags, hm.block.flags.data(), hm.block.flags.size());
        std::memcpy(losses, hm.block.losses.data(), hm.block.losses.size() * sizeof(double));
        if (element_mask) std::memcpy(element_mask, hm.element.bits.data(), hm.element.bits.size());
        const CompressedCache cc = fused ? fused_magnitude_compress(t, hm.block, sc, ax)
                                         : compress(t, hm, sc, ax);
        from_cache(cc, out);
    });
}

int ref_compress_with_flags(const float* x, size_t rows, size_t cols, const hso_config* cfg,
                            int axis, const uint8_t* flags, hso_cache* out) {
    return guarded([&] {
        const Tensor2D t = to_tensor(x, rows, cols);
        BlockMask bm;
        const std::size_t nb = cfg->block_size ? rows / cfg->block_size : 0;
        bm.flags.assign(flags, flags + nb);
        bm.losses.assign(nb, 0.0);
        const CompressedCache cc = fused_magnitude_compress(
            t, bm, to_cfg(cfg), axis == 0 ? GroupAxis::kChannel : GroupAxis::kSequence);
        from_cache(cc, out);
    });
}

// compress (compressed_cache.hpp:196-225) under an explicit HierarchicalMask.
int ref_compress_with_mask(const float* x, size_t rows, size_t cols, const hso_config* cfg, int axis,
                           const uint8_t* element_mask, const uint8_t* flags, hso_cache* out) {
    return guarded([&] {
        const Tensor2D t = to_tensor(x, rows, cols);
        HierarchicalMask hm;
        const std::size_t nb = cfg->block_size ? rows / cfg->block_size : 0;
        hm.block.flags.assign(flags, flags + nb);
        hm.block.losses.assign(nb, 0.0);
        hm.element = ElementMask(rows, cols, 0);
        for (std::size_t r = 0; r < rows; ++r)
            for (std::size_t c = 0; c < cols; ++c) hm.element.set(r, c, element_mask[r * cols + c] != 0);
        const CompressedCache cc = compress(t, hm, to_cfg(cfg), axis == 0 ? GroupAxis::kChannel : GroupAxis::kSequence);
        from_cache(cc, out);
    });
}

int ref_decompress(const hso_cache* c, float* out) {
    return guarded([&] {
        const Tensor2D t = decompress(to_cache(c));
        std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
    });
}

// attend_range (attention.hpp:249-304).
int ref_attend_rows(const float* q, size_t rows, size_t d, const hso_cache* k, const hso_cache* v,
                    const float* k_tail, const float* v_tail, size_t tail, size_t block_begin,
                    size_t block_end, int include_tail, float scale, const int64_t* qpos,
                    float* out_t, float* m_s, float* l_s) {
    return guarded([&] {
        Views views(k, v, k_tail, v_tail, tail, d);
        std::vector<std::ptrdiff_t> qp;
        if (qpos) qp.assign(qpos, qpos + rows);
        const SplitPartial p = attend_range(to_tensor(q, rows, d), views.k, views.v, block_begin,
                                            block_end, include_tail != 0, scale, qp);
        std::memcpy(out_t, p.output_t.data.data(), p.output_t.data.size() * sizeof(float));
        std::memcpy(m_s, p.m_s.data(), rows * sizeof(float));
        std::memcpy(l_s, p.l_s.data(), rows * sizeof(float));
    });
}

// decode_attention (attention.hpp:360-409).
int ref_decode(const float* q, size_t n_q, size_t d, const hso_cache* k, const hso_cache* v,
               const float* k_tail, const float* v_tail, size_t tail, float scale, size_t splits,
               size_t gqa_group, float* out) {
    return guarded([&] {
        Views views(k, v, k_tail, v_tail, tail, d);
        AttentionWorkload w;
        w.queries = to_tensor(q, n_q, d);
        w.key_cache = views.k;
        w.value_cache = views.v;
        w.causal = false;
        w.scale = scale;
        w.gqa_group = gqa_group;
        w.phase = Phase::kDecode;
        const Tensor2D o = decode_attention(w, splits);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    });
}

// prefill_attention (attention.hpp:323-354).
int ref_prefill(const float* q, size_t n_q, size_t d, const hso_cache* k, const hso_cache* v,
                const float* k_tail, const float* v_tail, size_t tail, int causal, float scale,
                size_t b_r, float* out) {
    return guarded([&] {
        Views views(k, v, k_tail, v_tail, tail, d);
        AttentionWorkload w;
        w.queries = to_tensor(q, n_q, d);
        w.key_cache = views.k;
        w.value_cache = views.v;
        w.causal = causal != 0;
        w.scale = scale;
        w.phase = Phase::kPrefill;
        const std::size_t bc = k ? k->block_size : 64;
        const Tensor2D o = prefill_attention(w, TileConfig{b_r, bc});
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    });
}

// dense_attention_oracle (attention.hpp:84-115).
int ref_dense_attention(const float* q, size_t n_q, const float* k, const float* v, size_t n_kv,
                        size_t d, int causal, float scale, float* out) {
    return guarded([&] {
        const Tensor2D o = dense_attention_oracle(to_tensor(q, n_q, d), to_tensor(k, n_kv, d),
                                                  to_tensor(v, n_kv, d), causal != 0, scale);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    });
}

// flop_and_byte_count (attention.hpp:426-467).
int ref_flop_and_byte_count(size_t n_q, size_t d, const hso_cache* k, const hso_cache* v,
                            size_t tail, int causal, uint64_t* flops, uint64_t* bytes) {
    return guarded([&] {
        std::vector<float> zeros(tail * d, 0.0f);
        Views views(k, v, zeros.data(), zeros.data(), tail, d);
        AttentionWorkload w;
        w.queries = Tensor2D(n_q, d);
        w.key_cache = views.k;
        w.value_cache = views.v;
        w.causal = causal != 0;
        const OpCounts c = flop_and_byte_count(w);
        *flops = c.flops;
        *bytes = c.bytes_moved;
    });
}

// serialize (container.hpp:119-148): bytes of one cache; *len = size (call with
// out = NULL to size the buffer).
int ref_serialize(const hso_cache* c, uint8_t* out, size_t cap, size_t* len) {
    return guarded([&] {
        const std::vector<std::uint8_t> b = serialize(to_cache(c));
        *len = b.size();
        if (out != nullptr && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    });
}

// parse (container.hpp:150-250): 0 when the bytes are a valid container, the
// reference's error code otherwise (DataError -> 4); decoded geometry out.
int ref_parse(const uint8_t* bytes, size_t len, size_t* logical_blocks, size_t* dense_count,
              size_t* sparse_count) {
    return guarded([&] {
        const std::vector<std::uint8_t> b(bytes, bytes + len);
        const CompressedCache c = parse(b);
        *logical_blocks = c.logical_blocks;
        *dense_count = c.dense_count;
        *sparse_count = c.sparse_count;
    });
}

}  // extern "C"
