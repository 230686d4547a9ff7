// Attention over pooled HieraSparse caches for shapes outside the tcgen05 /
// mma.sp kernels' specialisation (block_size != 64 or head_dim != 128).
//
// Reference semantics: attend_range (attention.hpp:249-304) with the online
// softmax of :171-239 and finalize_rows (:309-317): a query row at absolute
// position qpos sees keys <= qpos when causal (attention.hpp:183-185,
// :342-346), blocks past qpos are skipped (:275), the dense tail follows the
// blocks (:289-297).  One warp per query row on CUDA cores: the row's scores
// are warp dot products, every lane owns d/32 output channels, and 2:4 blocks
// are expanded from their canonical codes (nm_metadata.hpp:42-46) on the fly
// (expand_sparse, nm_metadata.hpp:119-143).  fp32 throughout.  This is the
// generality path (the reference's own test shapes); the specialised kernels
// carry the benchmarked configurations.
#include "common.cuh"
#include "kernels.h"

namespace hs {
namespace {

constexpr int kWarps = 4;
constexpr int kMaxJ = kGenericMaxHeadDim / 32;

template <typename T>
__device__ __forceinline__ float ld16(const void* p, uint64_t i) {
    return F16Traits<T>::to_float(static_cast<const uint16_t*>(p)[i]);
}

// Element (stored row sr, stored column sc) of pool slot `e` (index-map entry)
// of a cache whose stored blocks are srows x scols.
template <typename T>
__device__ __forceinline__ float pool_elem(int e, int u, int dc, int sc_count, const void* dense, const void* nnz,
                                           const uint16_t* meta, int BE, int scols, int sr, int sc) {
    const int slot = (e > 0 ? e : -e) - 1;
    if (e > 0) return ld16<T>(dense, (static_cast<uint64_t>(u) * dc + slot) * BE + sr * scols + sc);
    const uint64_t sb = static_cast<uint64_t>(u) * sc_count + slot;
    const int gi = sr * (scols / 4) + (sc >> 2), pos = sc & 3;
    const uint32_t code = (meta[sb * (BE / 16) + (gi >> 2)] >> (4 * (gi & 3))) & 0xFu;
    const int p0 = code & 3, p1 = code >> 2;
    if (pos == p0) return ld16<T>(nnz, sb * (BE / 2) + 2 * gi);
    if (pos == p1) return ld16<T>(nnz, sb * (BE / 2) + 2 * gi + 1);
    return 0.f;
}

template <typename T>
__global__ void __launch_bounds__(32 * kWarps) generic_attn_kernel(const GenericAttnLaunch L) {
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int g = blockIdx.y, u = blockIdx.z;
    if (row >= L.n_q) return;
    const int d = L.d, B = L.B, BE = B * d, J = (d + 31) / 32;
    const int64_t n_kv = static_cast<int64_t>(L.nb) * B + L.tail;
    const int64_t qpos = n_kv - L.n_q + row;  // attention.hpp:342-346
    const uint64_t qoff = ((static_cast<uint64_t>(u) * L.gqa + g) * L.n_q + row) * d;
    float q[kMaxJ], acc[kMaxJ];
#pragma unroll
    for (int j = 0; j < kMaxJ; ++j) {
        const int c = lane + 32 * j;
        q[j] = (j < J && c < d) ? ld16<T>(L.q, qoff + c) : 0.f;
        acc[j] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    auto visit = [&](float s, auto vload) {
        s *= L.scale;
        const float mn = fmaxf(m, s);
        const float alpha = expf(m - mn);  // m = -inf: 0
        const float p = expf(s - mn);
        l = l * alpha + p;
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
            const int c = lane + 32 * j;
            if (j < J && c < d) acc[j] = acc[j] * alpha + p * vload(c);
        }
        m = mn;
    };
    auto dot = [&](auto kload) {
        float part = 0.f;
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
            const int c = lane + 32 * j;
            if (j < J && c < d) part += q[j] * kload(c);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        return part;
    };
    const int16_t* kidx = L.k_index + static_cast<int64_t>(u) * L.nb;
    const int16_t* vidx = L.v_index + static_cast<int64_t>(u) * L.nb;
    for (int b = L.block_begin; b < L.block_end; ++b) {
        if (L.causal && static_cast<int64_t>(b) * B > qpos) break;  // block-causal skip (attention.hpp:275)
        const int ke = kidx[b], ve = vidx[b];
        for (int kk = 0; kk < B; ++kk) {
            if (L.causal && static_cast<int64_t>(b) * B + kk > qpos) break;
            // K stored [B][d] (token-major), V stored transposed [d][B] (compressed_cache.hpp:160-166)
            const float s = dot([&](int c) {
                return pool_elem<T>(ke, u, L.k_dense_count, L.k_sparse_count, L.k_dense, L.k_nnz, L.k_meta, BE, d, kk, c);
            });
            visit(s, [&](int c) {
                return pool_elem<T>(ve, u, L.v_dense_count, L.v_sparse_count, L.v_dense, L.v_nnz, L.v_meta, BE, B, c, kk);
            });
        }
    }
    if (L.include_tail) {
        const uint64_t toff = static_cast<uint64_t>(u) * L.tail * d;
        for (int tt = 0; tt < L.tail; ++tt) {
            if (L.causal && static_cast<int64_t>(L.nb) * B + tt > qpos) break;
            const float s = dot([&](int c) { return ld16<T>(L.k_tail, toff + static_cast<uint64_t>(tt) * d + c); });
            visit(s, [&](int c) { return ld16<T>(L.v_tail, toff + static_cast<uint64_t>(tt) * d + c); });
        }
    }
    const uint64_t ooff = (static_cast<uint64_t>(u) * L.gqa + g) * L.n_q + row;
    if (L.out_mode == 0) {
        const float inv = l > 0.f ? 1.f / l : 0.f;  // finalize_rows (attention.hpp:309-317)
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
            const int c = lane + 32 * j;
            if (j < J && c < d) L.out[ooff * d + c] = acc[j] * inv;
        }
    } else {
        float* po = L.out + ooff * (d + 2);
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
            const int c = lane + 32 * j;
            if (j < J && c < d) po[c] = acc[j];
        }
        if (lane == 0) {
            po[d] = m;
            po[d + 1] = l;
        }
    }
}

}  // namespace

cudaError_t launch_generic_attention(const GenericAttnLaunch& L, cudaStream_t s) {
    if (L.n_q <= 0 || L.gqa <= 0 || L.n_units <= 0) return cudaSuccess;
    const dim3 grid((L.n_q + kWarps - 1) / kWarps, L.gqa, L.n_units);
    if (L.bf16) generic_attn_kernel<__nv_bfloat16><<<grid, 32 * kWarps, 0, s>>>(L);
    else generic_attn_kernel<__half><<<grid, 32 * kWarps, 0, s>>>(L);
    return cudaGetLastError();
}

}  // namespace hs
