// TEST INFRASTRUCTURE ONLY — C++ parity test of the host layer
// (include/hierasparse_b200.hpp) against the UNMODIFIED reference headers
// (/root/reference/proj/include, compiled in at build time by tests/cpp/Makefile),
// written the way the reference's own tests are (proj/tests/acceptance.cpp
// prints [PASS]/[FAIL] per criterion).  Same seeded inputs (random_gaussian,
// head_seed roles of pipeline.hpp:168-169, :249), rounded once to bf16/fp16:
//   1. compression: index map, pools and metadata bit-identical to
//      prune_cache + fused_magnitude_compress (pruner.hpp:165, compressed_cache.hpp:262)
//   2. decode_attention within max-abs 2e-2 / mean-rel 1e-3 (attention.hpp:360)
//   3. prefill_attention (causal) within the same bar (attention.hpp:323)
//   4. errors map to the reference taxonomy (errors.hpp:10-25)
//   5. the fused decode-phase recompress equals decompress -> prune_cache -> compress
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "hierasparse/hierasparse.hpp"
#include "hierasparse_b200.hpp"

namespace ref = hierasparse;
namespace gpu = hierasparse::b200;

static int g_fail = 0;
static void report(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++g_fail;
}

static ref::Tensor2D rounded(ref::Tensor2D t, gpu::DType d) {
    for (float& v : t.data) v = gpu::from_bits(gpu::to_bits(v, d), d);
    return t;
}

static std::uint64_t head_seed(std::uint64_t seed, std::size_t head, std::size_t role) {
    return ref::derive_seed(ref::derive_seed(seed, head), role);  // pipeline.hpp:131-133
}

static void err_stats(const ref::Tensor2D& got, const ref::Tensor2D& want, double& mx, double& mr) {
    double se = 0, sr = 0;
    mx = 0;
    for (std::size_t i = 0; i < want.data.size(); ++i) {
        const double e = std::fabs(static_cast<double>(got.data[i]) - want.data[i]);
        mx = std::max(mx, e);
        se += e;
        sr += std::fabs(static_cast<double>(want.data[i]));
    }
    mr = se / std::max(sr, 1e-30);
}

static bool pools_equal(const ref::CompressedCache& r, const gpu::DeviceCompressedCache& g, gpu::DType d) {
    const auto h = g.unit_to_host(0);
    if (r.index_map != h.index_map) return false;
    if (r.dense_pool.size() != h.dense_pool.size() || r.nnz_pool.size() != h.nnz_pool.size()) return false;
    for (std::size_t i = 0; i < r.dense_pool.size(); ++i)
        if (gpu::to_bits(r.dense_pool[i], d) != h.dense_pool[i]) return false;
    for (std::size_t i = 0; i < r.nnz_pool.size(); ++i)
        if (gpu::to_bits(r.nnz_pool[i], d) != h.nnz_pool[i]) return false;
    return r.meta_pool == h.meta_pool;
}

int main() {
    const std::size_t d = 128;
    const float scale = 1.0f / std::sqrt(static_cast<float>(d));
    struct Case {
        std::size_t L;
        double s;
        std::size_t sink, window;
        gpu::DType dt;
    };
    const Case cases[] = {{4096, 1.0, 0, 0, gpu::DType::kBF16},
                          {2048, 0.5, 64, 256, gpu::DType::kF16},
                          {1024, 0.0, 0, 0, gpu::DType::kBF16},
                          {1024, 0.75, 0, 0, gpu::DType::kF16}};
    for (const Case& c : cases) {
        const std::string tag = "L=" + std::to_string(c.L) + " S=" + std::to_string(c.s).substr(0, 4) +
                                (c.dt == gpu::DType::kBF16 ? " bf16" : " f16");
        const ref::Tensor2D key = rounded(ref::random_gaussian(c.L, d, head_seed(1, 0, 0)), c.dt);
        const ref::Tensor2D val = rounded(ref::random_gaussian(c.L, d, head_seed(1, 0, 1)), c.dt);
        ref::SparsityConfig rcfg;
        rcfg.s_key = rcfg.s_value = c.s;
        rcfg.sink_tokens = c.sink;
        rcfg.local_window = c.window;
        // reference: prune_cache -> fused_magnitude_compress
        const auto masks = ref::prune_cache(key, val, rcfg);
        const ref::CompressedCache rk = ref::fused_magnitude_compress(key, masks.first.block, rcfg,
                                                                      ref::GroupAxis::kChannel);
        const ref::CompressedCache rv = ref::fused_magnitude_compress(val, masks.second.block, rcfg,
                                                                      ref::GroupAxis::kSequence);
        // B200 host layer
        gpu::SparsityConfig gcfg{c.s, c.s, 64, c.sink, c.window};
        auto kd = gpu::upload_units<ref::Tensor2D>({&key}, c.dt);
        auto vd = gpu::upload_units<ref::Tensor2D>({&val}, c.dt);
        auto [gk, gv] = gpu::prune_cache(kd.get(), vd.get(), c.dt, 1, c.L, gcfg);
        gpu::check_cuda(cudaDeviceSynchronize(), "prune_cache");
        report(pools_equal(rk, gk, c.dt) && pools_equal(rv, gv, c.dt), "compression bit-exact " + tag);
        const auto ms = ref::measure_size(rk);
        const auto gs = gk.measure_size();
        report(ms.size_idx == gs.size_idx && ms.size_den == gs.size_den && ms.size_nnz == gs.size_nnz &&
                   ms.size_e == gs.size_e,
               "measure_size " + tag);

        // decode-phase re-prune (pipeline.hpp:227-240): decompress -> prune_cache at
        // S_dec -> compress, against the fused one-pass recompress
        {
            ref::SparsityConfig dcfg = rcfg;
            dcfg.s_key = dcfg.s_value = c.s < 1.0 ? 1.0 : 0.5;
            const ref::Tensor2D dk = ref::decompress(rk), dv = ref::decompress(rv);
            const auto dm = ref::prune_cache(dk, dv, dcfg);
            const ref::CompressedCache rk2 = ref::fused_magnitude_compress(dk, dm.first.block, dcfg,
                                                                           ref::GroupAxis::kChannel);
            const ref::CompressedCache rv2 = ref::fused_magnitude_compress(dv, dm.second.block, dcfg,
                                                                           ref::GroupAxis::kSequence);
            gpu::SparsityConfig gdec{dcfg.s_key, dcfg.s_value, 64, c.sink, c.window};
            const auto gk2 = gpu::recompress(gk, gdec, dcfg.s_key);
            const auto gv2 = gpu::recompress(gv, gdec, dcfg.s_value);
            gpu::check_cuda(cudaDeviceSynchronize(), "recompress");
            report(pools_equal(rk2, gk2, c.dt) && pools_equal(rv2, gv2, c.dt),
                   "decode-phase recompress bit-exact " + tag);
        }

        // decode: 4 GQA rows (pipeline.hpp:247-251)
        ref::Tensor2D q(4, d);
        for (std::size_t g = 0; g < 4; ++g) {
            const ref::Tensor2D qg = ref::random_gaussian(1, d, head_seed(1, 0, 32 + g));
            std::copy(qg.data.begin(), qg.data.end(), q.data.begin() + g * d);
        }
        q = rounded(q, c.dt);
        ref::AttentionWorkload w;
        w.queries = q;
        w.key_cache.compressed = &rk;
        w.value_cache.compressed = &rv;
        w.scale = scale;
        w.gqa_group = 4;
        w.phase = ref::Phase::kDecode;
        const ref::Tensor2D want = ref::decode_attention(w, 1);
        const ref::Tensor2D got = gpu::decode_attention_host(q, gk, gv, scale);
        double mx, mr;
        err_stats(got, want, mx, mr);
        report(mx < 2e-2 && mr < 1e-3, "decode_attention " + tag + " (max-abs " + std::to_string(mx) +
                                           ", mean-rel " + std::to_string(mr) + ")");

        // prefill: the last 256 query rows, causal (attention.hpp:342-346)
        if (c.dt == gpu::DType::kF16) {
            const ref::Tensor2D qp = rounded(ref::random_gaussian(256, d, head_seed(1, 0, 2)), c.dt);
            ref::AttentionWorkload wp;
            wp.queries = qp;
            wp.key_cache.compressed = &rk;
            wp.value_cache.compressed = &rv;
            wp.scale = scale;
            wp.causal = true;
            const ref::Tensor2D pw = ref::prefill_attention(wp, ref::TileConfig{});
            const ref::Tensor2D pg = gpu::prefill_attention_host(qp, gk, gv, true, scale);
            err_stats(pg, pw, mx, mr);
            report(mx < 2e-2 && mr < 1e-3, "prefill_attention causal " + tag + " (max-abs " + std::to_string(mx) +
                                               ", mean-rel " + std::to_string(mr) + ")");
        }
        if (&c == &cases[0]) {
            bool threw = false;
            try {
                gpu::decode_attention_host(q, gv, gk, scale);  // swapped caches
            } catch (const gpu::ConfigError&) {
                threw = true;
            }
            report(threw, "swapped caches raise ConfigError");
            threw = false;
            try {
                gpu::pool_counts(100, gcfg, 1.0);  // 100 rows: not a multiple of B
            } catch (const gpu::ConfigError&) {
                threw = true;
            }
            report(threw, "ragged sequence raises ConfigError");
        }
    }
    // Multi-unit prefill with dense tails and GQA 2 through the host overloads,
    // against the reference's prefill_attention per (unit, query head) with
    // CacheView::dense_tail (attention.hpp:19-31, :289-297).
    {
        const std::size_t U = 2, G = 2, L = 512, T = 37, NQ = 200;
        const gpu::DType dt = gpu::DType::kF16;
        ref::SparsityConfig rcfg;
        rcfg.s_key = rcfg.s_value = 0.5;
        gpu::SparsityConfig gcfg{0.5, 0.5, 64, 0, 0};
        std::vector<ref::Tensor2D> keys, vals, ktails, vtails, qs;
        for (std::size_t u = 0; u < U; ++u) {
            const ref::Tensor2D kf = rounded(ref::random_gaussian(L + T, d, head_seed(7, u, 0)), dt);
            const ref::Tensor2D vf = rounded(ref::random_gaussian(L + T, d, head_seed(7, u, 1)), dt);
            keys.push_back(ref::slice_rows(kf, 0, L));
            vals.push_back(ref::slice_rows(vf, 0, L));
            ktails.push_back(ref::slice_rows(kf, L, L + T));
            vtails.push_back(ref::slice_rows(vf, L, L + T));
            for (std::size_t g = 0; g < G; ++g)
                qs.push_back(rounded(ref::random_gaussian(NQ, d, head_seed(7, u, 2 + g)), dt));
        }
        std::vector<const ref::Tensor2D*> kp, vp, ktp, vtp, qp;
        for (std::size_t u = 0; u < U; ++u) {
            kp.push_back(&keys[u]);
            vp.push_back(&vals[u]);
            ktp.push_back(&ktails[u]);
            vtp.push_back(&vtails[u]);
        }
        for (auto& q : qs) qp.push_back(&q);
        auto kd = gpu::upload_units<ref::Tensor2D>(kp, dt);
        auto vd = gpu::upload_units<ref::Tensor2D>(vp, dt);
        auto [gk, gv] = gpu::prune_cache(kd.get(), vd.get(), dt, U, L, gcfg);
        const auto got = gpu::prefill_attention_host<ref::Tensor2D>(qp, G, gk, gv, true, scale, ktp, vtp);
        bool ok = got.size() == U * G;
        double worst_mx = 0, worst_mr = 0;
        for (std::size_t u = 0; u < U && ok; ++u) {
            const auto masks = ref::prune_cache(keys[u], vals[u], rcfg);
            const ref::CompressedCache rk = ref::fused_magnitude_compress(keys[u], masks.first.block, rcfg,
                                                                          ref::GroupAxis::kChannel);
            const ref::CompressedCache rv = ref::fused_magnitude_compress(vals[u], masks.second.block, rcfg,
                                                                          ref::GroupAxis::kSequence);
            for (std::size_t g = 0; g < G; ++g) {
                ref::AttentionWorkload w;
                w.queries = qs[u * G + g];
                w.key_cache.compressed = &rk;
                w.key_cache.dense_tail = ktails[u];
                w.value_cache.compressed = &rv;
                w.value_cache.dense_tail = vtails[u];
                w.scale = scale;
                w.causal = true;
                const ref::Tensor2D want = ref::prefill_attention(w, ref::TileConfig{});
                double mx, mr;
                err_stats(got[u * G + g], want, mx, mr);
                worst_mx = std::max(worst_mx, mx);
                worst_mr = std::max(worst_mr, mr);
            }
        }
        report(ok && worst_mx < 2e-2 && worst_mr < 1e-3,
               "prefill_attention multi-unit, GQA 2, dense tails (max-abs " + std::to_string(worst_mx) +
                   ", mean-rel " + std::to_string(worst_mr) + ")");

        // decode over the same units with tails: the multi-unit host overload
        std::vector<ref::Tensor2D> dq;
        std::vector<const ref::Tensor2D*> dqp;
        for (std::size_t u = 0; u < U; ++u) dq.push_back(rounded(ref::random_gaussian(4, d, head_seed(7, u, 32)), dt));
        for (auto& q : dq) dqp.push_back(&q);
        const auto dgot = gpu::decode_attention_host<ref::Tensor2D>(dqp, gk, gv, scale, 0, ktp, vtp);
        worst_mx = worst_mr = 0;
        for (std::size_t u = 0; u < U; ++u) {
            const auto masks = ref::prune_cache(keys[u], vals[u], rcfg);
            const ref::CompressedCache rk = ref::fused_magnitude_compress(keys[u], masks.first.block, rcfg,
                                                                          ref::GroupAxis::kChannel);
            const ref::CompressedCache rv = ref::fused_magnitude_compress(vals[u], masks.second.block, rcfg,
                                                                          ref::GroupAxis::kSequence);
            ref::AttentionWorkload w;
            w.queries = dq[u];
            w.key_cache.compressed = &rk;
            w.key_cache.dense_tail = ktails[u];
            w.value_cache.compressed = &rv;
            w.value_cache.dense_tail = vtails[u];
            w.scale = scale;
            w.gqa_group = 4;
            w.phase = ref::Phase::kDecode;
            double mx, mr;
            err_stats(dgot[u], ref::decode_attention(w, 3), mx, mr);
            worst_mx = std::max(worst_mx, mx);
            worst_mr = std::max(worst_mr, mr);
        }
        report(worst_mx < 2e-2 && worst_mr < 1e-3,
               "decode_attention multi-unit with dense tails (max-abs " + std::to_string(worst_mx) + ")");
    }

    // compress under an explicit HierarchicalMask (compressed_cache.hpp:196-225):
    // the pruner's own masks -> bit-identical pools; a 3-kept group -> DataError.
    {
        const std::size_t L = 1024;
        const gpu::DType dt = gpu::DType::kBF16;
        const ref::Tensor2D key = rounded(ref::random_gaussian(L, d, head_seed(9, 0, 0)), dt);
        const ref::Tensor2D val = rounded(ref::random_gaussian(L, d, head_seed(9, 0, 1)), dt);
        ref::SparsityConfig rcfg;
        rcfg.s_key = rcfg.s_value = 0.5;
        const auto masks = ref::prune_cache(key, val, rcfg);
        bool ok = true;
        for (int which = 0; which < 2; ++which) {
            const ref::Tensor2D& x = which == 0 ? key : val;
            const auto& hm = which == 0 ? masks.first : masks.second;
            const ref::GroupAxis ax = which == 0 ? ref::GroupAxis::kChannel : ref::GroupAxis::kSequence;
            const ref::CompressedCache rc = ref::compress(x, hm, rcfg, ax);
            auto xd = gpu::upload_units<ref::Tensor2D>({&x}, dt);
            gpu::DeviceBuffer<uint8_t> em(L * d), fl(L / 64);
            gpu::check_cuda(cudaMemcpy(em.get(), hm.element.bits.data(), L * d, cudaMemcpyHostToDevice), "H2D");
            gpu::check_cuda(cudaMemcpy(fl.get(), hm.block.flags.data(), L / 64, cudaMemcpyHostToDevice), "H2D");
            uint32_t dense = 0;
            for (auto f : hm.block.flags) dense += f != 0;
            const auto gc = gpu::compress(xd.get(), em.get(), fl.get(), dense, dt, 1, L,
                                          which == 0 ? gpu::GroupAxis::kChannel : gpu::GroupAxis::kSequence);
            ok = ok && pools_equal(rc, gc, dt);
            if (which == 0) {
                std::vector<uint8_t> bad = hm.element.bits;
                std::size_t b = 0;
                while (hm.block.flags[b]) ++b;  // first sparse block
                bad[(b * 64 + 5) * d + 8 + 3] = 1;  // stored row 5, group 2: three or more kept
                bad[(b * 64 + 5) * d + 8 + 0] = 1;
                bad[(b * 64 + 5) * d + 8 + 1] = 1;
                gpu::check_cuda(cudaMemcpy(em.get(), bad.data(), L * d, cudaMemcpyHostToDevice), "H2D");
                bool threw = false;
                try {
                    gpu::compress(xd.get(), em.get(), fl.get(), dense, dt, 1, L, gpu::GroupAxis::kChannel);
                } catch (const gpu::DataError& e) {
                    threw = std::string(e.what()).find("more than n_keep") != std::string::npos;
                }
                report(threw, "compress: a group keeping 3 elements raises DataError");
            }
        }
        report(ok, "compress under the pruner's HierarchicalMask bit-exact");
    }

    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
    return g_fail ? 1 : 0;
}
