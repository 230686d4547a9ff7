// Hierarchical pruning + pooled 2:4 compression on B200 (HBM-bound integer /
// byte work, no tensor cores).
//
// Reference contract (bit-exact): pruner.hpp:40-176 (element_mask, block_loss,
// select_blocks, hierarchical_mask_for) and compressed_cache.hpp:133-267
// (assemble_cache, fused_magnitude_compress).  Pipeline per cache kind:
//
//   static selection (quota 0 or all prunable, known on the host):
//     pack<with losses>, each CTA deriving its own slot     (source read once)
//   loss-driven selection (0 < quota < prunable):
//     classify (losses) -> radix select + slot assignment (a CTA per unit) -> pack
//   explicit BlockMask / ElementMask: assign_slots -> pack
//
// Layout: source [unit][rows][d] token-major 16-bit.  One CTA per 64x128 block
// (16 KB): one bulk copy into shared memory, coalesced stores of the stored
// layouts.
#include "common.cuh"
#include "kernels.h"

namespace hs {
namespace {

constexpr int kThreads = 256;
#ifndef HS_COMPRESS_MINB
#define HS_COMPRESS_MINB 8  // 32 registers: 8 CTAs per SM (+4% at S = 1 against 6)
#endif

// Top-2-of-4 by magnitude with the stable-sort tie rule (pruner.hpp:53-74):
// element i is kept iff #{j: |x_j|>|x_i|} + #{j<i: |x_j|==|x_i|} < 2.
// Returns the 4-bit keep mask.
__device__ __forceinline__ uint32_t keep_mask4(uint32_t m0, uint32_t m1, uint32_t m2,
                                               uint32_t m3) {
    const uint32_t r0 = (m1 > m0) + (m2 > m0) + (m3 > m0);
    const uint32_t r1 = (m0 >= m1) + (m2 > m1) + (m3 > m1);
    const uint32_t r2 = (m0 >= m2) + (m1 >= m2) + (m3 > m2);
    const uint32_t r3 = (m0 >= m3) + (m1 >= m3) + (m2 >= m3);
    return (r0 < 2) | ((r1 < 2) << 1) | ((r2 < 2) << 2) | ((r3 < 2) << 3);
}

// Canonical 4-bit group code (nm_metadata.hpp:42-46, :81-83): first kept
// position in the low 2 bits.  Also returns the two kept positions.
__device__ __forceinline__ uint32_t group_code(uint32_t keep, uint32_t& p0, uint32_t& p1) {
    p0 = __ffs(keep) - 1;
    p1 = __ffs(keep & (keep - 1)) - 1;
    return p0 | (p1 << 2);
}

// Top-2-of-4 of one group given as two packed words (lo = g0 | g1 << 16,
// hi = g2 | g3 << 16), branch-free.  Keys (|g_i| << 2) | (3 - i) are distinct
// and order exactly like the reference's stable descending sort (larger
// magnitude first, ties to the lower index, pruner.hpp:63-66), so a 4-element
// min/max network yields the two kept positions (canonical code, first kept
// index in the low 2 bits, nm_metadata.hpp:42-46), the kept pair packed by one
// byte permute, and the two pruned magnitudes straight from the low keys.
struct Sel2of4 {
    uint32_t code;   // p0 | p1 << 2, p0 < p1
    uint32_t kept;   // g[p0] | g[p1] << 16
    uint32_t pr_lo;  // magnitude bits of the smaller pruned element
    uint32_t pr_hi;  // magnitude bits of the larger pruned element
};
__device__ __forceinline__ Sel2of4 select2of4(uint32_t lo, uint32_t hi) {
    const uint32_t k0 = ((lo & 0x7FFFu) << 2) | 3u, k1 = ((lo >> 14) & 0x1FFFCu) | 2u;
    const uint32_t k2 = ((hi & 0x7FFFu) << 2) | 1u, k3 = (hi >> 14) & 0x1FFFCu;
    const uint32_t a = max(k0, k1), b = min(k0, k1), c = max(k2, k3), d = min(k2, k3);
    const uint32_t t1 = max(a, c), t2 = max(min(a, c), max(b, d));
    const uint32_t b1 = min(b, d), b2 = min(max(b, d), min(a, c));
    const uint32_t pa = 3u - (t1 & 3u), pb = 3u - (t2 & 3u);
    const uint32_t p0 = min(pa, pb), p1 = max(pa, pb);
    Sel2of4 r;
    r.code = p0 | (p1 << 2);
    r.kept = __byte_perm(lo, hi, 0x1010u + p0 * 0x22u + p1 * 0x2200u);
    r.pr_lo = b1 >> 2;
    r.pr_hi = b2 >> 2;
    return r;
}

// Exact-loss bookkeeping.  Every 16-bit float is M * 2^e with integer M below
// 2^(mant+1); a double sum of such terms is exact in any order while the total
// stays below 2^(53 + e_min), and then equals the reference's sequential double
// sum bit for bit (pruner.hpp:85-87).  We track e_min/e_max of the nonzero
// pruned terms and fall back to a sequential sum when the bound can fail.
template <typename T>
__device__ __forceinline__ int unit_exp(uint32_t mag) {
    constexpr int mant = F16Traits<T>::kMantBits;
    const int E = static_cast<int>(mag >> mant);
    return (E ? E : 1) - F16Traits<T>::kExpBias - mant;
}

struct LossAcc {
    double sum = 0.0;
    uint32_t min_mag = 0xFFFFu;  // smallest nonzero pruned magnitude (16-bit pattern)
};

template <typename T>
__device__ __forceinline__ void loss_add(LossAcc& a, uint16_t bits) {
    const uint32_t mag = mag16(bits);
    if (mag == 0) return;
    a.min_mag = min(a.min_mag, mag);
    a.sum += fabs(static_cast<double>(F16Traits<T>::to_float(bits)));
}

// Both pruned elements of a group (magnitude bits, lo <= hi).
template <typename T>
__device__ __forceinline__ void loss_add_pair(LossAcc& a, uint32_t lo, uint32_t hi) {
#ifdef HS_XP_NO_LOSS
    if (lo != 0x12345u) return;  // timing experiment only
#endif
    a.min_mag = min(a.min_mag, lo ? lo : (hi ? hi : 0xFFFFu));
    a.sum += static_cast<double>(F16Traits<T>::to_float(static_cast<uint16_t>(lo))) +
             static_cast<double>(F16Traits<T>::to_float(static_cast<uint16_t>(hi)));
}

// Classify pass (losses only): the pruned pairs of two 2:4 groups at once in
// 16-bit SIMD lanes (lane k = group k).  Each group is (glo.lo, glo.hi, ghi.lo,
// ghi.hi); its pruned values are its two smallest magnitudes.  Positions do not
// matter for the loss -- tied magnitudes are the same value -- so the keys carry
// no index bits and one min/max network serves both groups (16 ALU ops for two
// groups instead of ~50 for select2of4 twice).
template <typename T>
__device__ __forceinline__ void loss_add_groups2(LossAcc& a, uint32_t& mm, uint32_t g0lo, uint32_t g0hi,
                                                 uint32_t g1lo, uint32_t g1hi) {
    constexpr uint32_t kMag = 0x7FFF7FFFu;
    const uint32_t P = __byte_perm(g0lo, g1lo, 0x5410u) & kMag, Q = __byte_perm(g0lo, g1lo, 0x7632u) & kMag;
    const uint32_t R = __byte_perm(g0hi, g1hi, 0x5410u) & kMag, S = __byte_perm(g0hi, g1hi, 0x7632u) & kMag;
    const uint32_t x = __vmaxu2(P, Q), y = __vminu2(P, Q), z = __vmaxu2(R, S), w = __vminu2(R, S);
    const uint32_t s1 = __vminu2(y, w);                            // smallest (per lane)
    const uint32_t s2 = __vminu2(__vmaxu2(y, w), __vminu2(x, z));  // second smallest
    // smallest nonzero pruned magnitude, kept as (m - 1) per lane (0 wraps to 0xFFFF)
    mm = __vminu2(mm, __vminu2(__vsub2(s1, 0x00010001u), __vsub2(s2, 0x00010001u)));
#ifdef HS_XP_NO_LOSS
    if (s1 != 0x12345u) return;  // timing experiment only
#endif
    a.sum += (static_cast<double>(F16Traits<T>::to_float(static_cast<uint16_t>(s1))) +
              static_cast<double>(F16Traits<T>::to_float(static_cast<uint16_t>(s2)))) +
             (static_cast<double>(F16Traits<T>::to_float(static_cast<uint16_t>(s1 >> 16))) +
              static_cast<double>(F16Traits<T>::to_float(static_cast<uint16_t>(s2 >> 16))));
}
// Fold the packed (m - 1) minimum into LossAcc::min_mag (0xFFFF = none).
__device__ __forceinline__ void loss_fold_min(LossAcc& a, uint32_t mm) {
    const uint32_t m = min(mm & 0xFFFFu, mm >> 16) + 1u;  // 0x10000: no nonzero term
    a.min_mag = min(a.min_mag, m);
}

// Reduce LossAcc across the CTA; thread 0 gets the total.  Returns true on
// thread 0 when the parallel sum is provably the reference's sequential one:
// every term is an integer multiple of u = 2^unit_exp(min nonzero magnitude),
// so every partial sum in any order is K * u with K <= total / u; below 2^53
// units all of them are exact doubles, the reference's included.
template <typename T>
__device__ bool loss_reduce(LossAcc& a, double* s_sum, int* s_min, int*) {
    for (int o = 16; o > 0; o >>= 1) {
        a.sum += __shfl_xor_sync(0xffffffffu, a.sum, o);
        a.min_mag = min(a.min_mag, static_cast<uint32_t>(__shfl_xor_sync(0xffffffffu, a.min_mag, o)));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_sum[w] = a.sum;
        s_min[w] = static_cast<int>(a.min_mag);
    }
    __syncthreads();
    bool exact = false;
    if (threadIdx.x == 0) {
        double s = 0.0;
        uint32_t mn = 0xFFFFu;
        for (int i = 0; i < kThreads / 32; ++i) {
            s += s_sum[i];
            mn = min(mn, static_cast<uint32_t>(s_min[i]));
        }
        a.sum = s;
        exact = mn == 0xFFFFu || s < ldexp(1.0, 53 + unit_exp<T>(mn));
    }
    return exact;
}

// g[p] for p in [0, 4) without local-memory indexing.
__device__ __forceinline__ uint32_t pick4(uint16_t g0, uint16_t g1, uint16_t g2, uint16_t g3, uint32_t p) {
    return p == 0 ? g0 : (p == 1 ? g1 : (p == 2 ? g2 : g3));
}

__device__ __forceinline__ const uint16_t* unit_src(const uint16_t* src, uint64_t stride, int u) {
    return src + static_cast<uint64_t>(u) * stride;
}

// Sequential reference-order loss (pruner.hpp:85-87) for the rare blocks whose
// exponent spread defeats the exact-sum bound.  Logical row-major order;
// at(r, c) returns the logical element.
template <typename T, int AXIS, typename At>
__device__ double sequential_loss_at(At at) {
    double loss = 0.0;
    for (int r = 0; r < kBlock; ++r) {
        for (int c = 0; c < kHeadDim; ++c) {
            uint32_t m[4];
            int pos;
            if (AXIS == 0) {
                const int g0 = c & ~3;
                for (int i = 0; i < 4; ++i) m[i] = mag16(at(r, g0 + i));
                pos = c & 3;
            } else {
                const int r0 = r & ~3;
                for (int i = 0; i < 4; ++i) m[i] = mag16(at(r0 + i, c));
                pos = r & 3;
            }
            const uint32_t keep = keep_mask4(m[0], m[1], m[2], m[3]);
            if (!((keep >> pos) & 1u))
                loss += fabs(static_cast<double>(F16Traits<T>::to_float(at(r, c))));
        }
    }
    return loss;
}
template <typename T, int AXIS>
__device__ double sequential_loss(const uint16_t* blk /*[64][128] logical*/) {
    return sequential_loss_at<T, AXIS>([&](int r, int c) { return blk[r * kHeadDim + c]; });
}

// ---------------------------------------------------------------------------
// Per-block work.  MODE: 0 = losses only (classify), 1 = pack, 2 = pack + losses.
// ---------------------------------------------------------------------------
struct PackArgs {
    const uint16_t* src;
    uint64_t src_stride;      // elements per unit
    int nb;
    int dense_count;
    int sparse_count;
    const int16_t* index_map; // [u][nb] (modes 1, 2)
    uint16_t* dense_pool;
    uint16_t* nnz_pool;
    uint16_t* meta_pool;
    double* losses;           // [u][nb] (modes 0, 2)
    // SRC 1: the source is itself a compressed cache of the same geometry
    // (decode-phase re-prune, pipeline.hpp:227-240): blocks are expanded on the
    // fly (decompress semantics, compressed_cache.hpp:271-298), never
    // materialised dense in HBM.
    const int16_t* in_index;
    int in_nb;                // blocks of the input cache; blocks >= in_nb read src
    int in_dense_count, in_sparse_count;
    const uint16_t* in_dense;
    const uint16_t* in_nnz;
    const uint16_t* in_meta;
    unsigned long long* status; // SRC 1: decompress's DataErrors (status word, kernels.h reasons)
    const uint8_t* element_mask;  // mask_pack_kernel: explicit ElementMask u8 [u][rows][d]
    uint64_t mask_unit_stride;
    int B, d;                     // block size and head dim (generic-shape kernels)
    // Static selection resolved in the pack kernel (no assign_slots launch): block b
    // is dense iff protected (b < prefix or b >= nb - suffix) or !all_sparse; the
    // CTA derives its slot and writes its own index-map entry, slot_block entry
    // and flag (the same values assign_slots_kernel writes).
    int static_sel, prefix, suffix, all_sparse;
    int reverse;                  // block order last-to-first (L2 reuse after a classify pass)
    int16_t* index_out;
    int32_t* slot_block_out;
    uint8_t* flags_out;
};

// One stored 2:4 group (kept pair word, 4-bit code) back to its four logical
// values as two packed words (expand_sparse, nm_metadata.hpp:119-143).
__device__ __forceinline__ void expand_group(uint32_t kept, uint32_t code, uint32_t& lo, uint32_t& hi,
                                             bool& bad) {
    const uint32_t p0 = code & 3u, p1 = code >> 2, klo = kept & 0xFFFFu, khi = kept >> 16;
    bad |= p1 <= p0;
    auto at = [&](uint32_t i) { return i == p0 ? klo : (i == p1 ? khi : 0u); };
    lo = at(0) | (at(1) << 16);
    hi = at(2) | (at(3) << 16);
}

// Logical element (r, c) of input block b of unit u (decompress semantics,
// compressed_cache.hpp:271-298; invalid entries read as zero).
template <int AXIS>
__device__ uint16_t logical_in(const PackArgs& a, int u, int b, int r, int c) {
    const int e = a.in_index[static_cast<int64_t>(u) * a.in_nb + b];
    const int slot = (e > 0 ? e : -e) - 1;
    if (e == 0 || (e > 0 && slot >= a.in_dense_count) || (e < 0 && slot >= a.in_sparse_count)) return 0;
    const int sr = AXIS == 0 ? r : c, sc = AXIS == 0 ? c : r;
    const int scols = AXIS == 0 ? kHeadDim : kBlock;
    if (e > 0) return a.in_dense[(static_cast<uint64_t>(u) * a.in_dense_count + slot) * (kBlock * kHeadDim) + sr * scols + sc];
    const uint64_t sb = static_cast<uint64_t>(u) * a.in_sparse_count + slot;
    const uint16_t* nnz = a.in_nnz + sb * (kBlock * kHeadDim / 2) + sr * (scols / 2);
    const uint16_t* meta = a.in_meta + sb * (kBlock * kHeadDim / 16) + sr * (scols / 16);
    const int g = sc >> 2, pos = sc & 3;
    const uint32_t code = (meta[g >> 2] >> (4 * (g & 3))) & 0xF;
    const int p0 = code & 3, p1 = code >> 2;
    return pos == p0 ? nnz[2 * g] : (pos == p1 ? nnz[2 * g + 1] : static_cast<uint16_t>(0));
}
template <typename T, int AXIS>
__device__ double sequential_loss_in(const PackArgs& a, int u, int b) {
    return sequential_loss_at<T, AXIS>([&](int r, int c) { return logical_in<AXIS>(a, u, b, r, c); });
}

template <typename T, int AXIS, int MODE, int SRC>
__global__ void __launch_bounds__(kThreads, HS_COMPRESS_MINB) block_kernel(PackArgs a) {
    // reverse: walk the blocks last-to-first (the pack pass after a classify pass
    // that read the source first-to-last: its last ~100 MB are still in L2)
    const int b = a.reverse ? static_cast<int>(gridDim.x - 1 - blockIdx.x) : static_cast<int>(blockIdx.x);
    const int u = a.reverse ? static_cast<int>(gridDim.y - 1 - blockIdx.y) : static_cast<int>(blockIdx.y);
    const int t = threadIdx.x;
    // SRC 1: blocks past the input cache come from the dense source (a tail's
    // full blocks absorbed into the cache)
    const bool from_src = SRC == 0 || b >= a.in_nb;
    const uint16_t* blk = from_src ? unit_src(a.src, a.src_stride, u) +
                                         static_cast<uint64_t>(b - (SRC == 0 ? 0 : a.in_nb)) * kBlock * kHeadDim
                                   : nullptr;
    __shared__ double s_sum[kThreads / 32];
    __shared__ int s_min[kThreads / 32];
    // SRC 0: the 16 KB source block lands in shared memory by one bulk copy issued
    // first thing (no registers hold in-flight data, so the 32-register budget
    // keeps 8 CTAs per SM while every CTA's block is in flight at once)
    __shared__ __align__(128) uint16_t tile[kBlock * kHeadDim];
    __shared__ __align__(8) uint64_t s_bar;
    if (SRC == 0) {
        if (t == 0) {
            mbar_init(&s_bar, 1);
            fence_barrier_init();
            mbar_arrive_expect_tx(&s_bar, kBlock * kHeadDim * 2);
            tma_bulk_g2s(tile, blk, kBlock * kHeadDim * 2, &s_bar);
        }
        __syncthreads();  // barrier initialised before anyone waits on it
    }
    // SRC 1: the input block (dense slot or nnz + metadata of a sparse slot)
    int in_e = 0;
    const uint16_t *in_den = nullptr, *in_nnz = nullptr, *in_meta = nullptr;
    bool in_bad = false;
    if (SRC == 1 && !from_src) {
        in_e = a.in_index[static_cast<int64_t>(u) * a.in_nb + b];
        const int slot = (in_e > 0 ? in_e : -in_e) - 1;
        if (in_e == 0 || (in_e > 0 && slot >= a.in_dense_count) || (in_e < 0 && slot >= a.in_sparse_count)) {
            if (t == 0)
                record_status(a.status, static_cast<uint64_t>(u) * a.nb + b,
                              in_e == 0 ? kReasonZeroEntry : in_e > 0 ? kReasonDanglingDense : kReasonDanglingSparse);
            in_e = 0;  // read as zeros
        } else if (in_e > 0) {
            in_den = a.in_dense + (static_cast<uint64_t>(u) * a.in_dense_count + slot) * (kBlock * kHeadDim);
        } else {
            const uint64_t sb = static_cast<uint64_t>(u) * a.in_sparse_count + slot;
            in_nnz = a.in_nnz + sb * (kBlock * kHeadDim / 2);
            in_meta = a.in_meta + sb * (kBlock * kHeadDim / 16);
        }
    }

    bool dense = false;
    int slot = 0;
    if (MODE != 0 && a.static_sel) {
        const bool prot = b < a.prefix || b >= a.nb - a.suffix;
        dense = prot || !a.all_sparse;
        slot = !a.all_sparse ? b : !prot ? b - a.prefix : b < a.prefix ? b : a.prefix + (b - (a.nb - a.suffix));
        if (t == 0) {
            const int64_t ub = static_cast<int64_t>(u) * a.nb;
            a.index_out[ub + b] = static_cast<int16_t>(dense ? slot + 1 : -(slot + 1));
            if (a.slot_block_out) a.slot_block_out[ub + (dense ? slot : a.dense_count + slot)] = b;
            if (a.flags_out) a.flags_out[ub + b] = static_cast<uint8_t>(dense);
        }
    } else if (MODE != 0) {
        const int e = a.index_map[static_cast<int64_t>(u) * a.nb + b];
        dense = e > 0;
        slot = (e > 0 ? e : -e) - 1;
        // a block mask whose dense count differs from the pool capacity was
        // reported by assign_slots_kernel; never write past a pool
        if (e == 0 || slot >= (dense ? a.dense_count : a.sparse_count)) {
            if (SRC == 0) mbar_wait(&s_bar, 0);  // no bulk copy may outlive the CTA
            return;
        }
    }
    if (SRC == 0) mbar_wait(&s_bar, 0);
    constexpr bool kLoss = MODE != 1;
    LossAcc acc;
    uint32_t mm = 0xFFFFFFFFu;  // MODE 0: packed (min nonzero pruned magnitude - 1)

    if (SRC == 1 && in_e < 0 && (MODE == 0 || !dense)) {
        // A stored 2:4 block re-pruned (decode-phase re-prune): expanded, every
        // group holds its two kept values and two zeros, so its pruned terms are
        // zeros (loss exactly 0.0, pruner.hpp:85-87) and top-2-of-4 keeps the
        // same positions unless a kept value is itself zero (then the tie rule may
        // move a code).  Such blocks are copied stored-to-stored (nnz + metadata,
        // 9 KB) instead of expanded and re-selected; the metadata is still
        // validated like unpack_metadata (nm_metadata.hpp:107).
        constexpr int kNnzVec = kBlock * kHeadDim / 2 / 8, kMetaVec = kBlock * kHeadDim / 16 / 8;  // uint4 counts
        const uint4* sn = reinterpret_cast<const uint4*>(in_nnz);
        const uint4* sm = reinterpret_cast<const uint4*>(in_meta);
        bool bad_codes = false, zero_kept = false;
        uint4 nv[kNnzVec / kThreads], mv = make_uint4(0u, 0u, 0u, 0u);
        auto has_zero = [](uint32_t w) { return (w & 0x7FFFu) == 0u || (w & 0x7FFF0000u) == 0u; };
        auto codes_bad = [](uint32_t w) {
            bool bad = false;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t nib = (w >> (4 * i)) & 0xFu;
                bad |= (nib >> 2) <= (nib & 3u);
            }
            return bad;
        };
        if (t < kMetaVec) {
            mv = sm[t];
            bad_codes = codes_bad(mv.x) || codes_bad(mv.y) || codes_bad(mv.z) || codes_bad(mv.w);
        }
        if (MODE != 0) {
#pragma unroll
            for (int i = 0; i < kNnzVec / kThreads; ++i) {
                nv[i] = sn[t + i * kThreads];
                zero_kept |= has_zero(nv[i].x) || has_zero(nv[i].y) || has_zero(nv[i].z) || has_zero(nv[i].w);
            }
        }
        if (!__syncthreads_or(zero_kept)) {
            if (MODE != 0) {
                const uint64_t sb = static_cast<uint64_t>(u) * a.sparse_count + slot;
                uint4* dn = reinterpret_cast<uint4*>(a.nnz_pool + sb * (kBlock * kHeadDim / 2));
                uint4* dm = reinterpret_cast<uint4*>(a.meta_pool + sb * (kBlock * kHeadDim / 16));
#pragma unroll
                for (int i = 0; i < kNnzVec / kThreads; ++i) dn[t + i * kThreads] = nv[i];
                if (t < kMetaVec) dm[t] = mv;
            }
            if (bad_codes) record_status(a.status, static_cast<uint64_t>(u) * a.nb + b, kReasonCodesOrder);
            if (kLoss && t == 0) a.losses[static_cast<int64_t>(u) * a.nb + b] = 0.0;
            return;
        }
    }

    if (AXIS == 0) {
        // Key cache: groups of 4 channels along a token row, stored layout = logical.
        const int c = t & 15;  // 16-byte chunk: channels 8c..8c+7 (groups 2c, 2c+1)
        // all four rows' loads first (memory-level parallelism), then the selection
        uint4 vr[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int r = p * 16 + (t >> 4);
            uint4& v = vr[p];
            if (SRC == 0) {
                v = *reinterpret_cast<const uint4*>(tile + r * kHeadDim + c * 8);
            } else if (from_src) {
                v = *reinterpret_cast<const uint4*>(blk + r * kHeadDim + c * 8);
            } else if (in_e > 0) {
                v = *reinterpret_cast<const uint4*>(in_den + r * kHeadDim + c * 8);
            } else if (in_e < 0) {
                // stored K row r: groups 2c, 2c+1 at nnz[4c..4c+3], codes in metadata byte c
                const uint2 kp = *reinterpret_cast<const uint2*>(in_nnz + r * (kHeadDim / 2) + c * 4);
                const uint32_t mb = reinterpret_cast<const uint8_t*>(in_meta + r * (kHeadDim / 16))[c];
                expand_group(kp.x, mb & 0xFu, v.x, v.y, in_bad);
                expand_group(kp.y, mb >> 4, v.z, v.w, in_bad);
            } else {
                v = make_uint4(0u, 0u, 0u, 0u);
            }
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int r = p * 16 + (t >> 4);
            const uint4 v = vr[p];
            if (MODE != 0 && dense) {
                uint16_t* dst = a.dense_pool + (static_cast<uint64_t>(u) * a.dense_count + slot) * (kBlock * kHeadDim);
                *reinterpret_cast<uint4*>(dst + r * kHeadDim + c * 8) = v;
            }
            if (MODE == 1 && dense) continue;
            if (MODE == 0) {
                loss_add_groups2<T>(acc, mm, v.x, v.y, v.z, v.w);
                continue;
            }
            const Sel2of4 s0 = select2of4(v.x, v.y), s1 = select2of4(v.z, v.w);
            const uint32_t meta_byte = s0.code | (s1.code << 4);
            if (kLoss) {
                loss_add_pair<T>(acc, s0.pr_lo, s0.pr_hi);
                loss_add_pair<T>(acc, s1.pr_lo, s1.pr_hi);
            }
            if (MODE != 0 && !dense) {
                const uint64_t sb = static_cast<uint64_t>(u) * a.sparse_count + slot;
                uint16_t* nnz = a.nnz_pool + sb * (kBlock * kHeadDim / 2);
                *reinterpret_cast<uint2*>(nnz + r * (kHeadDim / 2) + c * 4) = make_uint2(s0.kept, s1.kept);
                uint8_t* meta = reinterpret_cast<uint8_t*>(a.meta_pool + sb * (kBlock * kHeadDim / 16));
                meta[r * (kHeadDim / 8) + c] = static_cast<uint8_t>(meta_byte);
            }
        }
    } else {
        // Value cache: groups of 4 tokens down a channel; stored transposed [d][B].
        const int c = t & 127;  // channel
        const int h = t >> 7;   // token half: groups 8h..8h+7
        if (SRC == 0) {
            // staged by the bulk copy
        } else if (from_src) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int chunk = t + i * kThreads;  // 1024 chunks of 8 elements
                reinterpret_cast<uint4*>(tile)[chunk] = reinterpret_cast<const uint4*>(blk)[chunk];
            }
        } else if (in_e > 0) {
            // stored V^T [d][B]: channel c, tokens 32h..32h+31
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 w = *reinterpret_cast<const uint4*>(in_den + c * kBlock + 32 * h + 8 * q);
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    tile[(32 * h + 8 * q + 2 * j) * kHeadDim + c] = static_cast<uint16_t>(ws[j] & 0xFFFFu);
                    tile[(32 * h + 8 * q + 2 * j + 1) * kHeadDim + c] = static_cast<uint16_t>(ws[j] >> 16);
                }
            }
        } else {
            // stored channel c: token groups 8h..8h+7 at nnz[16h..16h+15], codes in 2 words
            uint32_t kv[8];
            const uint4 k0 = *reinterpret_cast<const uint4*>(in_nnz + c * (kBlock / 2) + 16 * h);
            const uint4 k1 = *reinterpret_cast<const uint4*>(in_nnz + c * (kBlock / 2) + 16 * h + 8);
            kv[0] = k0.x; kv[1] = k0.y; kv[2] = k0.z; kv[3] = k0.w;
            kv[4] = k1.x; kv[5] = k1.y; kv[6] = k1.z; kv[7] = k1.w;
            const uint32_t codes = in_e < 0 ? *reinterpret_cast<const uint32_t*>(in_meta + c * (kBlock / 16) + 2 * h) : 0u;
#pragma unroll
            for (int gi = 0; gi < 8; ++gi) {
                uint32_t lo = 0u, hi = 0u;
                if (in_e < 0) expand_group(kv[gi], (codes >> (4 * gi)) & 0xFu, lo, hi, in_bad);
                const int r0 = 32 * h + 4 * gi;
                tile[r0 * kHeadDim + c] = static_cast<uint16_t>(lo & 0xFFFFu);
                tile[(r0 + 1) * kHeadDim + c] = static_cast<uint16_t>(lo >> 16);
                tile[(r0 + 2) * kHeadDim + c] = static_cast<uint16_t>(hi & 0xFFFFu);
                tile[(r0 + 3) * kHeadDim + c] = static_cast<uint16_t>(hi >> 16);
            }
        }
        __syncthreads();
        if (MODE != 0 && dense) {
            uint16_t* dst = a.dense_pool + (static_cast<uint64_t>(u) * a.dense_count + slot) * (kBlock * kHeadDim) +
                            c * kBlock + 32 * h;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = 32 * h + 8 * q + 2 * j;
                    w[j] = tile[r * kHeadDim + c] | (static_cast<uint32_t>(tile[(r + 1) * kHeadDim + c]) << 16);
                }
                reinterpret_cast<uint4*>(dst)[q] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        if (MODE == 0) {
#pragma unroll
            for (int gi = 0; gi < 8; gi += 2) {
                const int r0 = 32 * h + 4 * gi;
                auto word = [&](int r) {
                    return tile[r * kHeadDim + c] | (static_cast<uint32_t>(tile[(r + 1) * kHeadDim + c]) << 16);
                };
                loss_add_groups2<T>(acc, mm, word(r0), word(r0 + 2), word(r0 + 4), word(r0 + 6));
            }
        } else if (!(MODE == 1 && dense)) {
            uint32_t vals[8];
            uint32_t meta = 0;
#pragma unroll
            for (int gi = 0; gi < 8; ++gi) {
                const int r0 = 32 * h + 4 * gi;
                const uint32_t lo = tile[r0 * kHeadDim + c] | (static_cast<uint32_t>(tile[(r0 + 1) * kHeadDim + c]) << 16);
                const uint32_t hi = tile[(r0 + 2) * kHeadDim + c] | (static_cast<uint32_t>(tile[(r0 + 3) * kHeadDim + c]) << 16);
                const Sel2of4 sg = select2of4(lo, hi);
                meta |= sg.code << (4 * gi);
                vals[gi] = sg.kept;
                if (kLoss) loss_add_pair<T>(acc, sg.pr_lo, sg.pr_hi);
            }
            if (MODE != 0 && !dense) {
                const uint64_t sb = static_cast<uint64_t>(u) * a.sparse_count + slot;
                uint16_t* nnz = a.nnz_pool + sb * (kBlock * kHeadDim / 2) + c * (kBlock / 2) + 16 * h;
                reinterpret_cast<uint4*>(nnz)[0] = make_uint4(vals[0], vals[1], vals[2], vals[3]);
                reinterpret_cast<uint4*>(nnz)[1] = make_uint4(vals[4], vals[5], vals[6], vals[7]);
                uint16_t* mp = a.meta_pool + sb * (kBlock * kHeadDim / 16) + c * (kBlock / 16) + 2 * h;
                *reinterpret_cast<uint32_t*>(mp) = meta;
            }
        }
    }

    if (SRC == 1 && in_bad) record_status(a.status, static_cast<uint64_t>(u) * a.nb + b, kReasonCodesOrder);
    if (kLoss) {
        if (MODE == 0) loss_fold_min(acc, mm);
        const bool exact = loss_reduce<T>(acc, s_sum, s_min, nullptr);
        if (t == 0) {
            double loss = acc.sum;
            // (SRC 1: every stored 2:4 group keeps its two largest magnitudes and
            // zeros elsewhere, so the pruned terms of the re-prune are those of a
            // decompressed block; the rare inexact case re-expands it)
            if (!exact) loss = from_src ? sequential_loss<T, AXIS>(blk) : sequential_loss_in<T, AXIS>(a, u, b);
            a.losses[static_cast<int64_t>(u) * a.nb + b] = loss;
        }
    }
}

// compress (compressed_cache.hpp:196-225): pack under an explicit ElementMask
// (u8 [u][rows][d] logical, nonzero = kept).  Dense-flagged blocks are copied
// verbatim (the mask is not consulted); every group of a sparse block must keep
// exactly n_keep = 2 elements, else the first offending group in the
// reference's order (block, stored row, group) is recorded as "keeps more" /
// "keeps fewer" (:216-223).  Same thread layout as block_kernel.
template <int AXIS>
__global__ void __launch_bounds__(kThreads) mask_pack_kernel(PackArgs a) {
    const int b = blockIdx.x, u = blockIdx.y, t = threadIdx.x;
    const int e = a.index_map[static_cast<int64_t>(u) * a.nb + b];
    const bool dense = e > 0;
    const int slot = (e > 0 ? e : -e) - 1;
    if (e == 0 || slot >= (dense ? a.dense_count : a.sparse_count)) return;
    const uint16_t* blk = unit_src(a.src, a.src_stride, u) + static_cast<uint64_t>(b) * kBlock * kHeadDim;
    const uint8_t* mblk = a.element_mask + static_cast<uint64_t>(u) * a.mask_unit_stride +
                          static_cast<uint64_t>(b) * kBlock * kHeadDim;
    constexpr int kGroupsPerBlock = kBlock * kHeadDim / 4;
    const uint64_t key0 = (static_cast<uint64_t>(u) * a.nb + b) * kGroupsPerBlock;
    // one 2:4 group from its four 16-bit values (lo = g0 | g1 << 16, hi = g2 | g3 << 16)
    // and mask nibble: kept pair (ascending positions), code, validity
    auto pack = [&](uint32_t lo, uint32_t hi, uint32_t m, uint64_t gkey, uint32_t& kept) -> uint32_t {
        const int n = __popc(m);
        if (n != 2) {
            record_status(a.status, key0 + gkey, n > 2 ? kReasonKeepsMore : kReasonKeepsFewer);
            kept = 0u;
            return 0u;
        }
        const uint32_t p0 = __ffs(m) - 1, p1 = __ffs(m & (m - 1)) - 1;
        kept = __byte_perm(lo, hi, 0x1010u + p0 * 0x22u + p1 * 0x2200u);
        return p0 | (p1 << 2);
    };
    auto nib = [](uint32_t w) {  // 4 mask bytes -> nibble of their nonzero flags
        uint32_t r = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) r |= static_cast<uint32_t>(((w >> (8 * k)) & 0xFFu) != 0u) << k;
        return r;
    };
    if (AXIS == 0) {
        const int c = t & 15;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int r = p * 16 + (t >> 4);
            const uint4 v = *reinterpret_cast<const uint4*>(blk + r * kHeadDim + c * 8);
            if (dense) {
                uint16_t* dst = a.dense_pool + (static_cast<uint64_t>(u) * a.dense_count + slot) * (kBlock * kHeadDim);
                *reinterpret_cast<uint4*>(dst + r * kHeadDim + c * 8) = v;
                continue;
            }
            const uint2 mw = *reinterpret_cast<const uint2*>(mblk + r * kHeadDim + c * 8);
            uint32_t k0, k1;
            const uint32_t c0 = pack(v.x, v.y, nib(mw.x), r * (kHeadDim / 4) + 2 * c, k0);
            const uint32_t c1 = pack(v.z, v.w, nib(mw.y), r * (kHeadDim / 4) + 2 * c + 1, k1);
            const uint64_t sb = static_cast<uint64_t>(u) * a.sparse_count + slot;
            uint16_t* nnz = a.nnz_pool + sb * (kBlock * kHeadDim / 2);
            *reinterpret_cast<uint2*>(nnz + r * (kHeadDim / 2) + c * 4) = make_uint2(k0, k1);
            uint8_t* meta = reinterpret_cast<uint8_t*>(a.meta_pool + sb * (kBlock * kHeadDim / 16));
            meta[r * (kHeadDim / 8) + c] = static_cast<uint8_t>(c0 | (c1 << 4));
        }
    } else {
        // stored transposed [d][B]: channel c, token groups 8h..8h+7
        const int c = t & 127, h = t >> 7;
        if (dense) {
            uint16_t* dst = a.dense_pool + (static_cast<uint64_t>(u) * a.dense_count + slot) * (kBlock * kHeadDim) +
                            c * kBlock + 32 * h;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = 32 * h + 8 * q + 2 * j;
                    w[j] = blk[r * kHeadDim + c] | (static_cast<uint32_t>(blk[(r + 1) * kHeadDim + c]) << 16);
                }
                reinterpret_cast<uint4*>(dst)[q] = make_uint4(w[0], w[1], w[2], w[3]);
            }
            return;
        }
        uint32_t vals[8], meta = 0;
#pragma unroll
        for (int gi = 0; gi < 8; ++gi) {
            const int r0 = 32 * h + 4 * gi;
            const uint32_t lo = blk[r0 * kHeadDim + c] | (static_cast<uint32_t>(blk[(r0 + 1) * kHeadDim + c]) << 16);
            const uint32_t hi = blk[(r0 + 2) * kHeadDim + c] | (static_cast<uint32_t>(blk[(r0 + 3) * kHeadDim + c]) << 16);
            uint32_t m = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) m |= static_cast<uint32_t>(mblk[(r0 + k) * kHeadDim + c] != 0) << k;
            meta |= pack(lo, hi, m, c * (kBlock / 4) + 8 * h + gi, vals[gi]) << (4 * gi);
        }
        const uint64_t sb = static_cast<uint64_t>(u) * a.sparse_count + slot;
        uint16_t* nnz = a.nnz_pool + sb * (kBlock * kHeadDim / 2) + c * (kBlock / 2) + 16 * h;
        reinterpret_cast<uint4*>(nnz)[0] = make_uint4(vals[0], vals[1], vals[2], vals[3]);
        reinterpret_cast<uint4*>(nnz)[1] = make_uint4(vals[4], vals[5], vals[6], vals[7]);
        uint16_t* mp = a.meta_pool + sb * (kBlock * kHeadDim / 16) + c * (kBlock / 16) + 2 * h;
        *reinterpret_cast<uint32_t*>(mp) = meta;
    }
}

// select_blocks (pruner.hpp:94-117) as a rank: block i (prunable) is sparse iff
// #{j prunable: L_j < L_i or (L_j == L_i and j < i)} < quota.  The order is a
// strict total order with NaN above +inf (ties to the lower index), so exactly
// quota blocks are flagged whatever the losses hold (a NaN loss comes from 3+
// NaNs in one 2:4 group); the reference's std::stable_sort with `<` has no
// defined order for NaN (pruner.hpp:111-113) but also flags exactly quota.
__device__ __forceinline__ bool loss_before(double lj, int j, double li, int i) {
    const bool nj = isnan(lj), ni = isnan(li);
    if (nj || ni) return (!nj && ni) || (nj && ni && j < i);
    return lj < li || (lj == li && j < i);
}
__global__ void __launch_bounds__(256) rank_kernel(const double* losses, int nb, int prefix,
                                                   int suffix, int quota, uint8_t* flags) {
    const int u = blockIdx.y;
    const int i = blockIdx.x * 256 + threadIdx.x;
    const double* L = losses + static_cast<int64_t>(u) * nb;
    __shared__ double tile[1024];
    const int lo = prefix, hi = nb - suffix;
    const double li = (i < nb) ? L[i] : 0.0;
    int rank = 0;
    for (int j0 = lo; j0 < hi; j0 += 1024) {
        __syncthreads();
        for (int j = threadIdx.x; j < 1024 && j0 + j < hi; j += 256) tile[j] = L[j0 + j];
        __syncthreads();
        const int n = min(1024, hi - j0);
        for (int j = 0; j < n; ++j) rank += loss_before(tile[j], j0 + j, li, i);
    }
    if (i < nb) {
        const bool prunable = i >= lo && i < hi;
        flags[static_cast<int64_t>(u) * nb + i] = (prunable && rank < quota) ? 0 : 1;
    }
}

// Slot assignment in block order (assemble_cache, compressed_cache.hpp:156-185):
// index_map = +(dense rank + 1) or -(sparse rank + 1); slot_block inverts it.
// flags_in == nullptr selects the static pattern (protected dense, prunable
// sparse iff all_sparse).
// A BlockMask whose dense count differs from the pool capacity (explicit masks
// only) is a ConfigError recorded in the status word; slots past a pool are
// then never written (block kernels skip them, slot_block stays in range).
__device__ __forceinline__ void assign_slots_cta(int u, const uint8_t* flags_in, int nb, int prefix, int suffix, int all_sparse,
                                                 int dense_count, int16_t* index_map, int32_t* slot_block,
                                                 uint8_t* flags_out, unsigned long long* status, int sparse_capacity) {
    const int t = threadIdx.x;
    const int per = (nb + 1023) / 1024;
    const int b0 = min(nb, t * per), b1 = min(nb, b0 + per);
    auto flag_of = [&](int b) -> int {
        if (flags_in) return flags_in[static_cast<int64_t>(u) * nb + b] != 0;
        const bool prot = b < prefix || b >= nb - suffix;
        return prot || !all_sparse;
    };
    int nd = 0;
    for (int b = b0; b < b1; ++b) nd += flag_of(b);
    // block exclusive scan of nd
    __shared__ int warp_sums[32];
    int x = nd;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if ((t & 31) >= o) x += y;
    }
    if ((t & 31) == 31) warp_sums[t >> 5] = x;
    __syncthreads();
    if (t < 32) {
        int w = warp_sums[t];
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (t >= o) w += y;
        }
        warp_sums[t] = w;
    }
    __syncthreads();
    int dense_before = x - nd + ((t >> 5) ? warp_sums[(t >> 5) - 1] : 0);
    int sparse_before = b0 - dense_before;
    // pools hold dense_count dense and nb_capacity - dense_count sparse slots per unit
    if (t == 0 && (warp_sums[31] > dense_count || nb - warp_sums[31] > sparse_capacity))
        record_status(status, 0, kReasonMaskCount);
    int16_t* im = index_map + static_cast<int64_t>(u) * nb;
    int32_t* sb = slot_block ? slot_block + static_cast<int64_t>(u) * nb : nullptr;
    for (int b = b0; b < b1; ++b) {
        const int f = flag_of(b);
        if (f) {
            im[b] = static_cast<int16_t>(dense_before + 1);
            if (sb && dense_before < dense_count) sb[dense_before] = b;
            ++dense_before;
        } else {
            im[b] = static_cast<int16_t>(-(sparse_before + 1));
            if (sb && dense_count + sparse_before < nb && sparse_before < sparse_capacity)
                sb[dense_count + sparse_before] = b;
            ++sparse_before;
        }
        if (flags_out) flags_out[static_cast<int64_t>(u) * nb + b] = static_cast<uint8_t>(f);
    }
}
__global__ void __launch_bounds__(1024) assign_slots_kernel(const uint8_t* flags_in, int nb, int prefix, int suffix, int all_sparse,
                                                 int dense_count, int16_t* index_map, int32_t* slot_block,
                                                 uint8_t* flags_out, unsigned long long* status, int sparse_capacity) {
    assign_slots_cta(blockIdx.x, flags_in, nb, prefix, suffix, all_sparse, dense_count, index_map, slot_block,
                     flags_out, status, sparse_capacity);
}

// The same selection by radix select (one 1024-thread CTA per unit): the
// quota-th smallest orderable key T is found digit by digit (8 passes of an 8-bit
// shared-memory histogram over the keys still matching the prefix), then a block
// is sparse iff its key is below T, or equals T and it is among the first
// `remaining` such blocks in index order (block-wide scans).  The key maps the
// strict total order above onto unsigned integers: -0.0 -> +0.0 (the reference's
// `<` treats them as equal), NaN above +inf.  Thread t keeps the keys of
// prunable blocks t, t + 1024, ... in registers.  (A bitonic sort of the same pairs in one CTA
// was issue-bound: 33 us per cache of 2048 blocks; radix select ~4 us.)
constexpr int kSelectThreads = 1024, kSelectKpt = 16;
constexpr int kSortMaxBlocks = kSelectThreads * kSelectKpt;  // 16384 blocks (1M tokens)
__device__ __forceinline__ unsigned long long loss_key(double l) {
    if (isnan(l)) return ~0ull;
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(l == 0.0 ? 0.0 : l));
    return (b >> 63) ? ~b : (b | (1ull << 63));
}
// Block-wide exclusive scan of v over 1024 threads; total in *total.
__device__ __forceinline__ int block_exclusive_scan(int v, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int t = s_warp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        s_warp[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    *total = s_warp[31];
    const int r = x - v + (w ? s_warp[w - 1] : 0);
    __syncthreads();  // s_warp is reused by the next scan
    return r;
}
// Slots (assign_slots_cta) are assigned in the same CTA when index_map != nullptr.
struct SlotOut {
    int dense_count, sparse_capacity;
    int16_t* index_map;
    int32_t* slot_block;
    uint8_t* flags_out;
};
__global__ void __launch_bounds__(kSelectThreads) radix_select_kernel(const double* losses, int nb, int prefix,
                                                                      int suffix, int quota, uint8_t* flags,
                                                                      SlotOut so) {
    __shared__ int s_hist[256];
    __shared__ int s_warp[32];
    __shared__ int s_digit, s_remaining;
    const int u = blockIdx.x, tid = threadIdx.x;
    const double* L = losses + static_cast<int64_t>(u) * nb;
    uint8_t* F = flags + static_cast<int64_t>(u) * nb;
    const int lo = prefix, hi = nb - suffix, np = max(0, hi - lo);
    for (int b = tid; b < nb; b += kSelectThreads)
        if (b < lo || b >= hi) F[b] = 1;  // protected blocks stay dense
    auto assign = [&]() {
        if (so.index_map == nullptr) return;
        __syncthreads();  // every flag of this unit written (CTA-scope ordering of the global stores)
        assign_slots_cta(u, flags, nb, 0, 0, 0, so.dense_count, so.index_map, so.slot_block, so.flags_out, nullptr,
                         so.sparse_capacity);
    };
    if (quota <= 0 || quota >= np) {  // nothing to rank: all prunable dense / all sparse
        for (int i = tid; i < np; i += kSelectThreads) F[lo + i] = quota <= 0 ? 1 : 0;
        assign();
        return;
    }
    // key k of this thread is prunable block i = tid + k * 1024 (every warp holds keys)
    const int nk = (np + kSelectThreads - 1) / kSelectThreads;
    unsigned long long key[kSelectKpt];
#pragma unroll
    for (int k = 0; k < kSelectKpt; ++k) {
        const int i = tid + k * kSelectThreads;
        key[k] = k < nk && i < np ? loss_key(L[lo + i]) : 0ull;
    }
    unsigned long long pval = 0, pmask = 0;
    int remaining = quota;  // selections still to make among keys matching the prefix
    for (int shift = 56; shift >= 0; shift -= 8) {
        if (tid < 256) s_hist[tid] = 0;
        __syncthreads();
        // warp-aggregated increments: the leading digits of similar losses coincide,
        // so per-key atomics on one bin would serialise
#pragma unroll
        for (int k = 0; k < kSelectKpt; ++k) {
            if (k >= nk) break;
            const int i = tid + k * kSelectThreads;
            const bool in = i < np && (key[k] & pmask) == pval;
            const int dg = in ? static_cast<int>((key[k] >> shift) & 0xFF) : 256;
            const unsigned grp = __match_any_sync(0xffffffffu, dg);
            if (in && (tid & 31) == __ffs(grp) - 1) atomicAdd(&s_hist[dg], __popc(grp));
        }
        __syncthreads();
        if (tid < 32) {  // warp 0: the digit where the running count reaches `remaining`
            int c[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) sum += (c[j] = s_hist[8 * tid + j]);
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += y;
            }
            int before = incl - sum;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (before < remaining && remaining <= before + c[j]) {
                    s_digit = 8 * tid + j;
                    s_remaining = remaining - before;
                }
                before += c[j];
            }
        }
        __syncthreads();
        pval |= static_cast<unsigned long long>(s_digit) << shift;
        pmask |= 0xFFull << shift;
        remaining = s_remaining;
        __syncthreads();  // s_digit / s_remaining read before the next pass writes them
    }
    // T = pval: every key below T is selected, and the first `remaining` keys equal
    // to T in index order (ties to the lower block index): index order is (k, tid).
    int base = 0;
#pragma unroll
    for (int k = 0; k < kSelectKpt; ++k) {
        if (k >= nk) break;
        const int i = tid + k * kSelectThreads;
        const bool valid = i < np;
        const bool eq = valid && key[k] == pval;
        int total;
        const int rank = base + block_exclusive_scan(eq ? 1 : 0, s_warp, &total);
        base += total;
        if (valid) F[lo + i] = (key[k] < pval || (eq && rank < remaining)) ? 0 : 1;
    }
    assign();
}
// so.index_map != nullptr: the slots are assigned too (*assigned = true) when the
// radix-select kernel runs; the quadratic fallback leaves them to assign_slots_kernel.
static cudaError_t launch_rank(const double* losses, int n_units, int nb, int prefix, int suffix, int quota,
                               uint8_t* flags, cudaStream_t s, SlotOut so = SlotOut{}, bool* assigned = nullptr) {
    if (assigned) *assigned = false;
    const int np = nb - prefix - suffix;
    if (np <= kSortMaxBlocks && getenv("HS_RANK_QUADRATIC") == nullptr) {
        radix_select_kernel<<<n_units, kSelectThreads, 0, s>>>(losses, nb, prefix, suffix, quota, flags, so);
        if (assigned) *assigned = so.index_map != nullptr;
    } else {
        rank_kernel<<<dim3((nb + 255) / 256, n_units), 256, 0, s>>>(losses, nb, prefix, suffix, quota, flags);
    }
    return cudaGetLastError();
}

// decompress (compressed_cache.hpp:271-298): pools -> logical [rows][d].
template <int AXIS>
__global__ void __launch_bounds__(kThreads) decompress_kernel(const int16_t* index_map, int nb,
                                                              int dense_count, int sparse_count,
                                                              const uint16_t* dense_pool,
                                                              const uint16_t* nnz_pool,
                                                              const uint16_t* meta_pool,
                                                              uint16_t* dst, unsigned long long* status) {
    const int b = blockIdx.x, u = blockIdx.y, t = threadIdx.x;
    const int e = index_map[static_cast<int64_t>(u) * nb + b];
    const int slot = (e > 0 ? e : -e) - 1;
    uint16_t* out = dst + (static_cast<uint64_t>(u) * nb + b) * kBlock * kHeadDim;
    const uint64_t key = static_cast<uint64_t>(u) * nb + b;
    if (e == 0 || (e > 0 && slot >= dense_count) || (e < 0 && slot >= sparse_count)) {
        if (t == 0)
            record_status(status, key, e == 0 ? kReasonZeroEntry : e > 0 ? kReasonDanglingDense : kReasonDanglingSparse);
        return;
    }
    bool bad = false;
    for (int i = t; i < kBlock * kHeadDim; i += kThreads) {
        // stored coordinates (sr, sc) of logical element i = (lr, lc)
        const int lr = i / kHeadDim, lc = i % kHeadDim;
        const int sr = AXIS == 0 ? lr : lc, sc = AXIS == 0 ? lc : lr;
        const int scols = AXIS == 0 ? kHeadDim : kBlock;
        uint16_t v;
        if (e > 0) {
            v = dense_pool[(static_cast<uint64_t>(u) * dense_count + slot) * kBlock * kHeadDim + sr * scols + sc];
        } else {
            const uint64_t sb = static_cast<uint64_t>(u) * sparse_count + slot;
            const uint16_t* nnz = nnz_pool + sb * (kBlock * kHeadDim / 2) + sr * (scols / 2);
            const uint16_t* meta = meta_pool + sb * (kBlock * kHeadDim / 16) + sr * (scols / 16);
            const int g = sc >> 2, pos = sc & 3;
            const uint32_t code = (meta[g >> 2] >> (4 * (g & 3))) & 0xF;
            const int p0 = code & 3, p1 = code >> 2;
            bad |= p1 <= p0;  // unpack_metadata: codes not increasing
            v = pos == p0 ? nnz[2 * g] : (pos == p1 ? nnz[2 * g + 1] : static_cast<uint16_t>(0));
        }
        out[i] = v;
    }
    if (bad) record_status(status, key, kReasonCodesOrder);
}

// ---------------------------------------------------------------------------
// Generic shapes (any block_size B and head_dim d that are multiples of 4, the
// reference's own constraints: masks.hpp:87, pruner.hpp:172-173,
// compressed_cache.hpp:118-126).  Same contracts as block_kernel /
// mask_pack_kernel / decompress_kernel (bit-exact pools, losses and errors),
// written over the canonical storage order instead of the B = 64 / d = 128
// register tiling: one CTA per (block, unit); a thread owns whole metadata
// words (4 consecutive groups in stored order), so every word is written once.
// ---------------------------------------------------------------------------
template <int AXIS>
__device__ __forceinline__ void stored_to_logical(int sr, int sc, int& r, int& c) {
    r = AXIS == 0 ? sr : sc;
    c = AXIS == 0 ? sc : sr;
}

// Logical element (r, c) of input block b (decompress semantics) for any shape;
// validity of the entry is checked by the caller.
template <int AXIS>
__device__ uint16_t gen_logical_in(const PackArgs& a, int u, int e, int r, int c, bool& bad) {
    const int B = a.B, d = a.d, BE = B * d;
    const int slot = (e > 0 ? e : -e) - 1;
    const int scols = AXIS == 0 ? d : B;
    const int sr = AXIS == 0 ? r : c, sc = AXIS == 0 ? c : r;
    if (e > 0) return a.in_dense[(static_cast<uint64_t>(u) * a.in_dense_count + slot) * BE + sr * scols + sc];
    const uint64_t sb = static_cast<uint64_t>(u) * a.in_sparse_count + slot;
    const int gi = sr * (scols / 4) + (sc >> 2), pos = sc & 3;
    const uint32_t code = (a.in_meta[sb * (BE / 16) + (gi >> 2)] >> (4 * (gi & 3))) & 0xFu;
    const int p0 = code & 3, p1 = code >> 2;
    bad |= p1 <= p0;
    const uint16_t* nnz = a.in_nnz + sb * (BE / 2);
    return pos == p0 ? nnz[2 * gi] : (pos == p1 ? nnz[2 * gi + 1] : static_cast<uint16_t>(0));
}

template <typename T, int AXIS, int MODE, int SRC, bool MASK>
__global__ void __launch_bounds__(kThreads) gen_block_kernel(PackArgs a) {
    const int b = blockIdx.x, u = blockIdx.y, t = threadIdx.x;
    const int B = a.B, d = a.d, BE = B * d;
    const int scols = AXIS == 0 ? d : B, gpr = scols / 4, G = BE / 4;
    const bool from_src = SRC == 0 || b >= a.in_nb;
    const uint16_t* blk = from_src ? unit_src(a.src, a.src_stride, u) +
                                         static_cast<uint64_t>(b - (SRC == 0 ? 0 : a.in_nb)) * BE
                                   : nullptr;
    __shared__ double s_sum[kThreads / 32];
    __shared__ int s_min[kThreads / 32];
    const uint64_t bkey = static_cast<uint64_t>(u) * a.nb + b;
    int in_e = 0;
    bool in_bad = false;
    if (SRC == 1 && !from_src) {
        in_e = a.in_index[static_cast<int64_t>(u) * a.in_nb + b];
        const int slot = (in_e > 0 ? in_e : -in_e) - 1;
        if (in_e == 0 || (in_e > 0 && slot >= a.in_dense_count) || (in_e < 0 && slot >= a.in_sparse_count)) {
            if (t == 0)
                record_status(a.status, bkey,
                              in_e == 0 ? kReasonZeroEntry : in_e > 0 ? kReasonDanglingDense : kReasonDanglingSparse);
            in_e = 0;
        }
    }
    auto logical = [&](int r, int c) -> uint16_t {
        if (from_src) return blk[r * d + c];
        if (in_e == 0) return 0;
        return gen_logical_in<AXIS>(a, u, in_e, r, c, in_bad);
    };
    bool dense = false;
    int slot = 0;
    if (MODE != 0 && a.static_sel) {
        const bool prot = b < a.prefix || b >= a.nb - a.suffix;
        dense = prot || !a.all_sparse;
        slot = !a.all_sparse ? b : !prot ? b - a.prefix : b < a.prefix ? b : a.prefix + (b - (a.nb - a.suffix));
        if (t == 0) {
            const int64_t ub = static_cast<int64_t>(u) * a.nb;
            a.index_out[ub + b] = static_cast<int16_t>(dense ? slot + 1 : -(slot + 1));
            if (a.slot_block_out) a.slot_block_out[ub + (dense ? slot : a.dense_count + slot)] = b;
            if (a.flags_out) a.flags_out[ub + b] = static_cast<uint8_t>(dense);
        }
    } else if (MODE != 0) {
        const int e = a.index_map[static_cast<int64_t>(u) * a.nb + b];
        dense = e > 0;
        slot = (e > 0 ? e : -e) - 1;
        if (e == 0 || slot >= (dense ? a.dense_count : a.sparse_count)) return;
    }
    constexpr bool kLoss = MODE != 1 && !MASK;
    LossAcc acc;
    if (MODE != 0 && dense) {
        uint16_t* dst = a.dense_pool + (static_cast<uint64_t>(u) * a.dense_count + slot) * BE;
        for (int i = t; i < BE; i += kThreads) {
            int r, c;
            stored_to_logical<AXIS>(i / scols, i % scols, r, c);
            dst[i] = logical(r, c);
        }
    }
    if (kLoss || (MODE != 0 && !dense)) {
        const uint64_t sbk = static_cast<uint64_t>(u) * a.sparse_count + slot;
        const uint8_t* mblk = MASK ? a.element_mask + static_cast<uint64_t>(u) * a.mask_unit_stride +
                                         static_cast<uint64_t>(b) * BE
                                   : nullptr;
        for (int w = t; w < G / 4; w += kThreads) {
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int gi = 4 * w + q, sr = gi / gpr, g = gi % gpr;
                uint32_t v[4], m = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    int r, c;
                    stored_to_logical<AXIS>(sr, 4 * g + i, r, c);
                    v[i] = logical(r, c);
                    if (MASK) m |= static_cast<uint32_t>(mblk[r * d + c] != 0) << i;
                }
                const uint32_t lo = v[0] | (v[1] << 16), hi = v[2] | (v[3] << 16);
                uint32_t code, kept;
                if (MASK) {
                    const int n = __popc(m);
                    if (n != 2) {
                        record_status(a.status, bkey * G + gi, n > 2 ? kReasonKeepsMore : kReasonKeepsFewer);
                        code = kept = 0u;
                    } else {
                        const uint32_t p0 = __ffs(m) - 1, p1 = __ffs(m & (m - 1)) - 1;
                        kept = __byte_perm(lo, hi, 0x1010u + p0 * 0x22u + p1 * 0x2200u);
                        code = p0 | (p1 << 2);
                    }
                } else {
                    const Sel2of4 sel = select2of4(lo, hi);
                    code = sel.code;
                    kept = sel.kept;
                    if (kLoss) loss_add_pair<T>(acc, sel.pr_lo, sel.pr_hi);
                }
                word |= code << (4 * q);
                if (MODE != 0 && !dense)
                    *reinterpret_cast<uint32_t*>(a.nnz_pool + sbk * (BE / 2) + 2 * gi) = kept;
            }
            if (MODE != 0 && !dense) a.meta_pool[sbk * (BE / 16) + w] = static_cast<uint16_t>(word);
        }
    }
    if (SRC == 1 && in_bad) record_status(a.status, bkey, kReasonCodesOrder);
    if (kLoss) {
        const bool exact = loss_reduce<T>(acc, s_sum, s_min, nullptr);
        if (t == 0) {
            double loss = acc.sum;
            if (!exact) {
                // block_loss (pruner.hpp:81-89) in logical row-major order
                loss = 0.0;
                bool dummy = false;
                for (int r = 0; r < B; ++r)
                    for (int c = 0; c < d; ++c) {
                        uint32_t m[4];
                        const int r0 = AXIS == 0 ? r : (r & ~3), c0 = AXIS == 0 ? (c & ~3) : c;
                        for (int i = 0; i < 4; ++i)
                            m[i] = mag16(AXIS == 0 ? logical(r0, c0 + i) : logical(r0 + i, c0));
                        const int pos = AXIS == 0 ? (c & 3) : (r & 3);
                        if (!((keep_mask4(m[0], m[1], m[2], m[3]) >> pos) & 1u))
                            loss += fabs(static_cast<double>(F16Traits<T>::to_float(logical(r, c))));
                    }
                (void)dummy;
            }
            a.losses[static_cast<int64_t>(u) * a.nb + b] = loss;
        }
    }
}

template <int AXIS>
__global__ void __launch_bounds__(kThreads) gen_decompress_kernel(DecompressLaunch L, int B, int d) {
    const int b = blockIdx.x, u = blockIdx.y, t = threadIdx.x;
    const int BE = B * d, scols = AXIS == 0 ? d : B;
    const int e = L.index_map[static_cast<int64_t>(u) * L.nb + b];
    const int slot = (e > 0 ? e : -e) - 1;
    const uint64_t key = static_cast<uint64_t>(u) * L.nb + b;
    if (e == 0 || (e > 0 && slot >= L.dense_count) || (e < 0 && slot >= L.sparse_count)) {
        if (t == 0)
            record_status(L.status, key, e == 0 ? kReasonZeroEntry : e > 0 ? kReasonDanglingDense : kReasonDanglingSparse);
        return;
    }
    const uint16_t* dense = static_cast<const uint16_t*>(L.dense_pool);
    const uint16_t* nnzp = static_cast<const uint16_t*>(L.nnz_pool);
    uint16_t* out = static_cast<uint16_t*>(L.dst) + (static_cast<uint64_t>(u) * L.nb + b) * BE;
    bool bad = false;
    for (int i = t; i < BE; i += kThreads) {
        const int lr = i / d, lc = i % d;
        const int sr = AXIS == 0 ? lr : lc, sc = AXIS == 0 ? lc : lr;
        uint16_t v;
        if (e > 0) {
            v = dense[(static_cast<uint64_t>(u) * L.dense_count + slot) * BE + sr * scols + sc];
        } else {
            const uint64_t sb = static_cast<uint64_t>(u) * L.sparse_count + slot;
            const int gi = sr * (scols / 4) + (sc >> 2), pos = sc & 3;
            const uint32_t code = (L.meta_pool[sb * (BE / 16) + (gi >> 2)] >> (4 * (gi & 3))) & 0xFu;
            const int p0 = code & 3, p1 = code >> 2;
            bad |= p1 <= p0;
            const uint16_t* nnz = nnzp + sb * (BE / 2);
            v = pos == p0 ? nnz[2 * gi] : (pos == p1 ? nnz[2 * gi + 1] : static_cast<uint16_t>(0));
        }
        out[i] = v;
    }
    if (bad) record_status(L.status, key, kReasonCodesOrder);
}

}  // namespace

// ----------------------------------------------------------------- launchers
template <typename T, int SRC>
static void launch_block_kernel_src(int axis, int mode, const PackArgs& a, int n_units, cudaStream_t s) {
    const dim3 grid(a.nb, n_units);
#define HS_LAUNCH(AX, MD) block_kernel<T, AX, MD, SRC><<<grid, kThreads, 0, s>>>(a)
    if (axis == 0) {
        if (mode == 0) HS_LAUNCH(0, 0); else if (mode == 1) HS_LAUNCH(0, 1); else HS_LAUNCH(0, 2);
    } else {
        if (mode == 0) HS_LAUNCH(1, 0); else if (mode == 1) HS_LAUNCH(1, 1); else HS_LAUNCH(1, 2);
    }
#undef HS_LAUNCH
}
template <typename T, int SRC, bool MASK>
static void launch_gen_src(int axis, int mode, const PackArgs& a, int n_units, cudaStream_t s) {
    const dim3 grid(a.nb, n_units);
#define HS_LAUNCH(AX, MD) gen_block_kernel<T, AX, MD, SRC, MASK><<<grid, kThreads, 0, s>>>(a)
    if (axis == 0) {
        if (mode == 0) HS_LAUNCH(0, 0); else if (mode == 1) HS_LAUNCH(0, 1); else HS_LAUNCH(0, 2);
    } else {
        if (mode == 0) HS_LAUNCH(1, 0); else if (mode == 1) HS_LAUNCH(1, 1); else HS_LAUNCH(1, 2);
    }
#undef HS_LAUNCH
}
template <typename T>
static cudaError_t launch_block_kernel(int axis, int mode, const PackArgs& a, int n_units,
                                       cudaStream_t s) {
    if (a.B != kBlock || a.d != kHeadDim) {  // generic shapes
        if (a.element_mask) launch_gen_src<T, 0, true>(axis, 1, a, n_units, s);
        else if (a.in_index) launch_gen_src<T, 1, false>(axis, mode, a, n_units, s);
        else launch_gen_src<T, 0, false>(axis, mode, a, n_units, s);
        return cudaGetLastError();
    }
    if (a.in_index) launch_block_kernel_src<T, 1>(axis, mode, a, n_units, s);
    else launch_block_kernel_src<T, 0>(axis, mode, a, n_units, s);
    return cudaGetLastError();
}

cudaError_t launch_prune_compress(const CompressLaunch& L, cudaStream_t s) {
    PackArgs a{};
    a.src = static_cast<const uint16_t*>(L.src);
    a.src_stride = L.src_unit_stride;
    a.nb = L.nb;
    a.dense_count = L.dense_count;
    a.sparse_count = L.sparse_count;
    a.index_map = L.index_map;
    a.dense_pool = static_cast<uint16_t*>(L.dense_pool);
    a.nnz_pool = static_cast<uint16_t*>(L.nnz_pool);
    a.meta_pool = L.meta_pool;
    a.losses = L.losses;
    a.in_index = L.in_index;
    a.in_nb = L.in_nb;
    a.in_dense_count = L.in_dense_count;
    a.in_sparse_count = L.in_sparse_count;
    a.in_dense = static_cast<const uint16_t*>(L.in_dense);
    a.in_nnz = static_cast<const uint16_t*>(L.in_nnz);
    a.in_meta = L.in_meta;
    a.status = L.status;
    a.element_mask = nullptr;
    a.mask_unit_stride = 0;
    a.B = L.block_size;
    a.d = L.head_dim;
    auto blocks = [&](int mode) {
        return L.bf16 ? launch_block_kernel<__nv_bfloat16>(L.axis, mode, a, L.n_units, s)
                      : launch_block_kernel<__half>(L.axis, mode, a, L.n_units, s);
    };
    cudaError_t err;
    if (L.flags_in) {
        // fused_magnitude_compress under an explicit BlockMask, or compress under
        // an explicit ElementMask + BlockMask (compressed_cache.hpp:196-225).
        assign_slots_kernel<<<L.n_units, 1024, 0, s>>>(L.flags_in, L.nb, 0, 0, 0, L.dense_count,
                                                       L.index_map, L.slot_block, L.flags_out, L.status,
                                                       L.sparse_count);
        if ((err = cudaGetLastError())) return err;
        if (L.element_mask) {
            a.element_mask = L.element_mask;
            a.mask_unit_stride = L.mask_unit_stride;
            if (a.B != kBlock || a.d != kHeadDim) return blocks(1);
            if (L.axis == 0) mask_pack_kernel<0><<<dim3(L.nb, L.n_units), kThreads, 0, s>>>(a);
            else mask_pack_kernel<1><<<dim3(L.nb, L.n_units), kThreads, 0, s>>>(a);
            return cudaGetLastError();
        }
        return blocks(1);
    }
    a.static_sel = 0;
    if (L.static_selection && a.B == kBlock && a.d == kHeadDim) {
        a.static_sel = 1;
        a.prefix = L.prefix;
        a.suffix = L.suffix;
        a.all_sparse = L.all_sparse;
        a.index_out = L.index_map;
        a.slot_block_out = L.slot_block;
        a.flags_out = L.flags_out;
        return blocks(L.losses ? 2 : 1);
    }
    if (L.static_selection) {
        assign_slots_kernel<<<L.n_units, 1024, 0, s>>>(nullptr, L.nb, L.prefix, L.suffix,
                                                       L.all_sparse, L.dense_count, L.index_map,
                                                       L.slot_block, L.flags_out, nullptr, L.sparse_count);
        if ((err = cudaGetLastError())) return err;
        return blocks(L.losses ? 2 : 1);
    }
    // Loss-driven selection: classify -> rank -> assign -> pack.
    if ((err = blocks(0))) return err;
    bool assigned = false;
    const SlotOut so{L.dense_count, L.sparse_count, L.index_map, L.slot_block, L.flags_out};
    if ((err = launch_rank(L.losses, L.n_units, L.nb, L.prefix, L.suffix, L.quota, L.flags_tmp, s, so, &assigned)))
        return err;
    if (!assigned) {
        assign_slots_kernel<<<L.n_units, 1024, 0, s>>>(L.flags_tmp, L.nb, 0, 0, 0, L.dense_count,
                                                       L.index_map, L.slot_block, L.flags_out, nullptr,
                                                       L.sparse_count);
        if ((err = cudaGetLastError())) return err;
    }
    a.reverse = getenv("HS_COMPRESS_FORWARD") == nullptr;  // (tools: A/B of the pack order)
    return blocks(1);
}

cudaError_t launch_select_blocks(const double* losses, int n_units, int nb, int prefix, int suffix, int quota,
                                 uint8_t* flags, cudaStream_t s) {
    return launch_rank(losses, n_units, nb, prefix, suffix, quota, flags, s);
}

cudaError_t launch_block_losses(const CompressLaunch& L, cudaStream_t s) {
    CompressLaunch M = L;
    M.flags_in = nullptr;
    M.static_selection = false;
    PackArgs a{};
    a.src = static_cast<const uint16_t*>(L.src);
    a.src_stride = L.src_unit_stride;
    a.nb = L.nb;
    a.losses = L.losses;
    a.B = L.block_size;
    a.d = L.head_dim;
    return L.bf16 ? launch_block_kernel<__nv_bfloat16>(L.axis, 0, a, L.n_units, s)
                  : launch_block_kernel<__half>(L.axis, 0, a, L.n_units, s);
}

cudaError_t launch_decompress(const DecompressLaunch& L, cudaStream_t s) {
    const dim3 grid(L.nb, L.n_units);
    if (L.block_size != kBlock || L.head_dim != kHeadDim) {
        if (L.axis == 0) gen_decompress_kernel<0><<<grid, kThreads, 0, s>>>(L, L.block_size, L.head_dim);
        else gen_decompress_kernel<1><<<grid, kThreads, 0, s>>>(L, L.block_size, L.head_dim);
        return cudaGetLastError();
    }
    if (L.axis == 0)
        decompress_kernel<0><<<grid, kThreads, 0, s>>>(L.index_map, L.nb, L.dense_count, L.sparse_count,
                                                       static_cast<const uint16_t*>(L.dense_pool),
                                                       static_cast<const uint16_t*>(L.nnz_pool),
                                                       L.meta_pool, static_cast<uint16_t*>(L.dst), L.status);
    else
        decompress_kernel<1><<<grid, kThreads, 0, s>>>(L.index_map, L.nb, L.dense_count, L.sparse_count,
                                                       static_cast<const uint16_t*>(L.dense_pool),
                                                       static_cast<const uint16_t*>(L.nnz_pool),
                                                       L.meta_pool, static_cast<uint16_t*>(L.dst), L.status);
    return cudaGetLastError();
}

}  // namespace hs
