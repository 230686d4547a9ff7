// Split-KV sparse decode attention over pooled HieraSparse caches (sm_100a).
//
// Reference semantics: attend_range (attention.hpp:249-304) over contiguous
// block ranges, online softmax (attention.hpp:171-239), LSE combine
// (attention.hpp:387-407).  Trans-Both orientation: S^T = K_b * Q^T and
// O^T += V_b^T * P^T, so the pruned K and V^T blocks are the 2:4 *A* operand of
// the sparse tensor-core MMA and the canonical metadata words feed the MMA
// metadata register unchanged.
//
// Data path (HBM-bound): every consumer warp streams its own blocks' surviving
// values (TMA 2-D tiles, hardware swizzle) and metadata (1-D bulk copies) through
// a private mbarrier-tracked stage and owns one block at a time.  In auto-split
// mode with short ranges, lane 0 claims the unit's next block with an atomic
// (dynamic balance); otherwise a CTA streams its contiguous static range:
//   GEMM1  mma.sp m16n8k32  K nnz [64 keys x 64] x Q^T (GQA rows stacked on N)
//   softmax in registers (fp32), warp shuffles over the key lanes
//   P^T    movmatrix relayout of the accumulator fragment (the paper's
//          "RelayoutFragment"); bf16 P as a hi+lo pair
//   GEMM2  mma.sp m16n8k32  V^T nnz [128 ch x 32] x P^T
// Dense blocks take the dense m16n8k16 path.  Warps, then CTAs of a unit,
// merge (m, l, O) with the reference combine: cooperatively when the grid is
// resident (every CTA publishes its partial through a tagged mailbox -- slots
// that carry their own validity -- and merges a 32-column slice once the
// unit's partials are in), otherwise in the unit's last CTA.  The 1-D grid
// interleaves units so each unit's splits span every GPC.
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace hs {
namespace {

constexpr int kMaxGqa = 8;

struct StageLayout {
    uint32_t k_bytes, v_bytes, stage_bytes;
};

template <typename T>
__device__ __forceinline__ uint32_t ld_pair(const T* p) {
    return *reinterpret_cast<const uint32_t*>(p);
}

__device__ __forceinline__ uint32_t meta_sel(uint32_t lo_row, uint32_t hi_row, uint32_t half) {
    return __byte_perm(lo_row, hi_row, half ? 0x7632 : 0x5410);
}

template <typename T, int NW, bool HILO>
__global__ void __launch_bounds__(32 * NW) decode_kernel(const __grid_constant__ DecodeLaunch L,
                                                         int spw, StageLayout lay) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[16];
    __shared__ int s_ticket;
    __shared__ uint32_t s_q[kMaxGqa * kHeadDim / 2];  // the unit's query rows (16-bit pairs)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // interleave: a 1-D grid whose consecutive CTAs belong to different units, so
    // every unit's splits spread over all GPCs instead of filling one or two
    const int split = L.interleave ? static_cast<int>(blockIdx.x) / L.n_units : static_cast<int>(blockIdx.x);
    const int u = L.interleave ? static_cast<int>(blockIdx.x) % L.n_units : static_cast<int>(blockIdx.y);
    long long* const ct = L.cta_times ? L.cta_times + 16 * (static_cast<int64_t>(u) * L.nsplit + split) : nullptr;
    if (ct && threadIdx.x == 0) {
        ct[0] = globaltimer();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        ct[15] = smid;
    }
    const int gqa = L.gqa;
    // Block range of this CTA (attention.hpp:380-381 partition of [begin, end)).
    const int span = L.block_end - L.block_begin;
    const int b0 = L.block_begin + static_cast<int>(static_cast<int64_t>(span) * split / L.nsplit);
    const int b1 = L.block_begin + static_cast<int>(static_cast<int64_t>(span) * (split + 1) / L.nsplit);
    const int nblk = b1 - b0;
    const bool with_tail = L.include_tail && split == L.nsplit - 1 && L.tail > 0;

    // Dynamic smem: [index entries of this range (int16 k, v)] [1 KB pad] [ring]
    const uint32_t raw = smem_u32(smem_raw);
    int16_t* s_kidx = reinterpret_cast<int16_t*>(smem_raw);
    int16_t* s_vidx = s_kidx + L.max_blocks_per_cta;
    const uint32_t idx_bytes = static_cast<uint32_t>(L.max_blocks_per_cta) * 4u;
    const uint32_t base = (raw + idx_bytes + 1023u) & ~1023u;
    uint8_t* const base_ptr = smem_raw + (base - raw);

    // The unit's queries: loaded first (they may live in pinned host memory --
    // zero-copy host I/O, DecodePlan(host_io) -- so their latency overlaps the
    // set-up and the first TMA issue), staged in shared memory below.
    const uint32_t* qg = reinterpret_cast<const uint32_t*>(static_cast<const T*>(L.q) +
                                                           static_cast<int64_t>(u) * L.q_rows * kHeadDim);
    const int nqw = gqa * (kHeadDim / 2);
    constexpr int kQW = kMaxGqa * (kHeadDim / 2) / (32 * NW);  // words per thread at most
    uint32_t qw[kQW];
#pragma unroll
    for (int i = 0; i < kQW; ++i) qw[i] = threadIdx.x + i * 32 * NW < nqw ? qg[threadIdx.x + i * 32 * NW] : 0u;
    const int16_t* kidx = L.k_index + static_cast<int64_t>(u) * L.nb;
    const int16_t* vidx = L.v_index + static_cast<int64_t>(u) * L.nb;
    // dynamic block claiming needs the one-slot ring and the fused combine (which
    // re-arms the counters)
    const bool dyn = L.dynamic != 0 && spw == 1 && L.out != nullptr;
    for (int i = threadIdx.x; i < (dyn ? 0 : nblk); i += 32 * NW) {
        s_kidx[i] = kidx[b0 + i];
        s_vidx[i] = vidx[b0 + i];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NW * spw; ++s) mbar_init(&full_bar[s], 1);
        fence_barrier_init();
    }
    __syncthreads();

    // Each consumer warp streams its own blocks (i = warp + NW*k) into its own
    // `spw` ring slots: it issues block k+spw right after finishing block k, so
    // no empty barriers are needed and a waiter is never a phase ahead.
    auto issue_e = [&](int k, int ke, int ve) {
        const int s = warp * spw + k % spw;
        uint8_t* kreg = base_ptr + s * lay.stage_bytes;
        uint8_t* vreg = kreg + lay.k_bytes;
        const uint32_t bytes = (ke > 0 ? 16384u : 9216u) + (ve > 0 ? 16384u : 9216u);
        mbar_arrive_expect_tx(&full_bar[s], bytes);
        if (ke > 0) {
            const int row = (u * L.k_dense_count + ke - 1) * kBlock;
            tma_tile_g2s(kreg, &L.tm_kden, 0, row, &full_bar[s]);
            tma_tile_g2s(kreg + 8192, &L.tm_kden, 64, row, &full_bar[s]);
        } else {
            const int sb = u * L.k_sparse_count + (-ke - 1);
            if (L.debug_stream_only == 2)
                tma_bulk_g2s(kreg, static_cast<const uint16_t*>(L.k_nnz) + static_cast<int64_t>(sb) * 4096, 8192, &full_bar[s]);
            else
                tma_tile_g2s(kreg, &L.tm_knnz, 0, sb * kBlock, &full_bar[s]);
            tma_bulk_g2s(kreg + 8192, L.k_meta + static_cast<int64_t>(sb) * 512, 1024, &full_bar[s]);
        }
        if (ve > 0) {
            const int row = (u * L.v_dense_count + ve - 1) * kHeadDim;
            tma_tile_g2s(vreg, &L.tm_vden, 0, row, &full_bar[s]);
        } else {
            const int sb = u * L.v_sparse_count + (-ve - 1);
            if (L.debug_stream_only == 2)
                tma_bulk_g2s(vreg, static_cast<const uint16_t*>(L.v_nnz) + static_cast<int64_t>(sb) * 4096, 8192, &full_bar[s]);
            else
                tma_tile_g2s(vreg, &L.tm_vnnz, 0, sb * kHeadDim, &full_bar[s]);
            tma_bulk_g2s(vreg + 8192, L.v_meta + static_cast<int64_t>(sb) * 512, 1024, &full_bar[s]);
        }
    };
    auto issue = [&](int k) {
        const int i = warp + NW * k;
        issue_e(k, s_kidx[i], s_vidx[i]);
    };
    // Dynamic mode: the warps of a unit's CTAs claim the unit's blocks one at a
    // time from a per-unit counter, so CTAs on SMs that stream faster take more
    // blocks (static ranges leave the whole unit waiting for its slowest SM).
    // Lane 0 keeps a two-deep lookahead: the claim for block k+2 and the index
    // entries for block k+1 are in flight while block k computes.
    int* const ctr = L.blk_ctr + u;
    const int16_t* const kidx_g = L.k_index + static_cast<int64_t>(u) * L.nb + L.block_begin;
    const int16_t* const vidx_g = L.v_index + static_cast<int64_t>(u) * L.nb + L.block_begin;
    const int span_dyn = dyn ? span : 0;
    int d_cur = -1, d_cur_ke = 0, d_cur_ve = 0;  // block being computed (lane 0)
    int d_nxt = -1, d_nxt_ke = 0, d_nxt_ve = 0;  // next block: entries in flight
    int d_claim = -1;                            // block after next: claim in flight
    // The first block of every warp is static (warp w of split s: block s*NW + w),
    // so the first TMA needs no atomic round trip; later claims start past them.
    const int first_static = L.nsplit * NW;
    auto claim = [&]() {
        const int b = first_static + atomicAdd(ctr, 1);
        return b < span_dyn ? b : -1;
    };
    // L2 prefetch of a future block of this warp (pools are contiguous per slot).
    auto prefetch = [&](int k) {
        const int i = warp + NW * k;
        const int ke = s_kidx[i], ve = s_vidx[i];
        const uint16_t* kd = static_cast<const uint16_t*>(L.k_dense);
        const uint16_t* vd = static_cast<const uint16_t*>(L.v_dense);
        if (ke > 0) {
            prefetch_l2(kd + (static_cast<int64_t>(u) * L.k_dense_count + ke - 1) * (kBlock * kHeadDim), 16384);
        } else {
            const int64_t sb = static_cast<int64_t>(u) * L.k_sparse_count + (-ke - 1);
            prefetch_l2(static_cast<const uint16_t*>(L.k_nnz) + sb * (kBlock * kHeadDim / 2), 8192);
            prefetch_l2(L.k_meta + sb * 512, 1024);
        }
        if (ve > 0) {
            prefetch_l2(vd + (static_cast<int64_t>(u) * L.v_dense_count + ve - 1) * (kBlock * kHeadDim), 16384);
        } else {
            const int64_t sb = static_cast<int64_t>(u) * L.v_sparse_count + (-ve - 1);
            prefetch_l2(static_cast<const uint16_t*>(L.v_nnz) + sb * (kBlock * kHeadDim / 2), 8192);
            prefetch_l2(L.v_meta + sb * 512, 1024);
        }
    };
    int nk = nblk > warp ? (nblk - warp + NW - 1) / NW : 0;  // blocks of this warp (static mode)
    const int pf = L.prefetch_distance;
    if (lane == 0) {
        if (warp == 0) {
            prefetch_tmap(&L.tm_knnz);
            prefetch_tmap(&L.tm_vnnz);
        }
        if (dyn) {
            d_cur = split * NW + warp < span_dyn ? split * NW + warp : -1;
            if (d_cur >= 0) {
                d_cur_ke = kidx_g[d_cur];
                d_cur_ve = vidx_g[d_cur];
                issue_e(0, d_cur_ke, d_cur_ve);
                d_nxt = claim();
                if (d_nxt >= 0) {
                    d_nxt_ke = kidx_g[d_nxt];
                    d_nxt_ve = vidx_g[d_nxt];
                    d_claim = claim();
                }
            }
        } else {
            for (int k = 0; k < spw && k < nk; ++k) issue(k);
            for (int k = spw; k < spw + pf && k < nk; ++k) prefetch(k);
        }
    }
    if (dyn) nk = 1 << 30;  // until the unit's counter runs out
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kQW; ++i)
        if (threadIdx.x + i * 32 * NW < nqw) s_q[threadIdx.x + i * 32 * NW] = qw[i];
    __syncthreads();

    // ------------------------------------------------------- consumers ----
    const int g = lane >> 2, t = lane & 3, half = t & 1;
    float m_run[2] = {-INFINITY, -INFINITY};
    float l_run[2] = {0.f, 0.f};
    float o[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) o[i][k] = 0.f;

    {
        // Q^T fragments for GEMM1 (B operand, k = channel, n = query row g).
        const uint16_t* q = reinterpret_cast<const uint16_t*>(s_q);
        uint32_t qb[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int x = 0; x < 4; ++x)
                qb[j][x] = g < gqa ? s_q[(g * kHeadDim + 32 * j + 8 * x + 2 * t) / 2] : 0u;

        for (int k = 0; k < nk; ++k) {
            const int s = warp * spw + k % spw;
            bool kd, vd;
            if (dyn) {
                if (__shfl_sync(0xffffffffu, d_cur, 0) < 0) break;
                kd = __shfl_sync(0xffffffffu, d_cur_ke, 0) > 0;
                vd = __shfl_sync(0xffffffffu, d_cur_ve, 0) > 0;
            } else {
                const int i = warp + NW * k;
                kd = s_kidx[i] > 0;
                vd = s_vidx[i] > 0;
            }
            mbar_wait(&full_bar[s], (k / spw) & 1);
            if (ct && k == 0 && threadIdx.x == 0) ct[1] = globaltimer();
            if (L.debug_stream_only) {  // pipeline-only measurement mode (tools/)
                __syncwarp();
                if (lane == 0 && k + spw < nk) issue(k + spw);
                __syncwarp();
                continue;
            }
            const uint32_t kreg = base + s * lay.stage_bytes;
            const uint32_t vreg = kreg + lay.k_bytes;

            // ---------------- GEMM1: S^T[64 keys][8 q] ----------------
            float sc[4][4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int k = 0; k < 4; ++k) sc[mi][k] = 0.f;
            const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8;
            const int lch = lane >> 4;
            if (!kd) {
                const uint8_t* kmeta = base_ptr + (kreg - base) + 8192;
                uint32_t e[4][4];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) {
                    const uint4 mlo = *reinterpret_cast<const uint4*>(kmeta + (16 * mi + g) * 16);
                    const uint4 mhi = *reinterpret_cast<const uint4*>(kmeta + (16 * mi + g + 8) * 16);
                    e[mi][0] = meta_sel(mlo.x, mhi.x, half);
                    e[mi][1] = meta_sel(mlo.y, mhi.y, half);
                    e[mi][2] = meta_sel(mlo.z, mhi.z, half);
                    e[mi][3] = meta_sel(mlo.w, mhi.w, half);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t a[4][4];
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) ldmatrix_x4(kreg + sw128(16 * mi + lrow, 2 * j + lch), a[mi]);
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) mma_sp_16832<T>(sc[mi], a[mi], qb[j], e[mi][j]);
                }
            } else {
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        uint32_t a[4];
                        const uint32_t tile = kreg + (kk >> 2) * 8192;
                        ldmatrix_x4(tile + sw128(16 * mi + lrow, 2 * (kk & 3) + lch), a);
                        mma_16816<T>(sc[mi], a, qb[kk >> 1][(kk & 1) * 2], qb[kk >> 1][(kk & 1) * 2 + 1]);
                    }
            }

            // ---------------- online softmax (log2 domain) ----------------
            float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    sc[mi][k] *= L.scale_log2;
                    mx[k & 1] = fmaxf(mx[k & 1], sc[mi][k]);
                }
            float alpha[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 4));
                mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 8));
                mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 16));
                const float mnew = fmaxf(m_run[e], mx[e]);
                alpha[e] = fast_exp2(m_run[e] - mnew);
                m_run[e] = mnew;
            }
            float psum[2] = {0.f, 0.f};
            uint32_t bt_hi[4][2], bt_lo[4][2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                float p[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    p[k] = fast_exp2(sc[mi][k] - m_run[k & 1]);
                    psum[k & 1] += p[k];
                }
                const uint32_t top = F16Traits<T>::pack(p[0], p[1]);
                const uint32_t bot = F16Traits<T>::pack(p[2], p[3]);
                bt_hi[mi][0] = movmatrix_trans(top);
                bt_hi[mi][1] = movmatrix_trans(bot);
                if (HILO) {
                    const float2 th = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&top));
                    const float2 bh = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bot));
                    bt_lo[mi][0] = movmatrix_trans(F16Traits<T>::pack(p[0] - th.x, p[1] - th.y));
                    bt_lo[mi][1] = movmatrix_trans(F16Traits<T>::pack(p[2] - bh.x, p[3] - bh.y));
                }
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) l_run[e] = l_run[e] * alpha[e] + psum[e];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) {
                o[mi][0] *= alpha[0];
                o[mi][2] *= alpha[0];
                o[mi][1] *= alpha[1];
                o[mi][3] *= alpha[1];
            }

            // ---------------- GEMM2: O^T[128 ch][8 q] += V^T P^T ----------------
            if (!vd) {
                const uint8_t* vmeta = base_ptr + (vreg - base) + 8192;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint32_t bh[4] = {bt_hi[2 * j][0], bt_hi[2 * j][1], bt_hi[2 * j + 1][0], bt_hi[2 * j + 1][1]};
                    const uint32_t bl[4] = {bt_lo[2 * j][0], bt_lo[2 * j][1], bt_lo[2 * j + 1][0], bt_lo[2 * j + 1][1]};
#pragma unroll
                    for (int mh = 0; mh < 2; ++mh) {
                        uint32_t a[4][4], e[4];
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const int mi = 4 * mh + x;
                            const uint32_t mlo = *reinterpret_cast<const uint32_t*>(vmeta + (16 * mi + g) * 8 + 4 * j);
                            const uint32_t mhi = *reinterpret_cast<const uint32_t*>(vmeta + (16 * mi + g + 8) * 8 + 4 * j);
                            e[x] = meta_sel(mlo, mhi, half);
                            ldmatrix_x4(vreg + sw64(16 * mi + lrow, 2 * j + lch), a[x]);
                        }
#pragma unroll
                        for (int x = 0; x < 4; ++x) mma_sp_16832<T>(o[4 * mh + x], a[x], bh, e[x]);
                        if (HILO) {
#pragma unroll
                            for (int x = 0; x < 4; ++x) mma_sp_16832<T>(o[4 * mh + x], a[x], bl, e[x]);
                        }
                    }
                }
            } else {
#pragma unroll
                for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        uint32_t a[4];
                        ldmatrix_x4(vreg + sw128(16 * mi + lrow, 2 * kk + lch), a);
                        mma_16816<T>(o[mi], a, bt_hi[kk][0], bt_hi[kk][1]);
                        if (HILO) mma_16816<T>(o[mi], a, bt_lo[kk][0], bt_lo[kk][1]);
                    }
            }
            __syncwarp();  // every lane is done with slot s
            if (dyn) {
                if (lane == 0) {
                    // next block -> TMA; block after next -> entries; new claim
                    if (d_nxt >= 0) issue_e(k + 1, d_nxt_ke, d_nxt_ve);
                    d_cur = d_nxt;
                    d_cur_ke = d_nxt_ke;
                    d_cur_ve = d_nxt_ve;
                    d_nxt = d_claim;
                    if (d_nxt >= 0) {
                        d_nxt_ke = kidx_g[d_nxt];
                        d_nxt_ve = vidx_g[d_nxt];
                        d_claim = claim();
                    }
                }
            } else {
                if (lane == 0 && k + spw < nk) issue(k + spw);
                if (lane == 0 && k + spw + pf < nk) prefetch(k + spw + pf);
            }
            __syncwarp();
        }

        // ---------------- dense tail (attention.hpp:289-297) ----------------
        if (with_tail && warp == 0) {
            const T* kt = static_cast<const T*>(L.k_tail) + static_cast<int64_t>(u) * L.tail * kHeadDim;
            const T* vt = static_cast<const T*>(L.v_tail) + static_cast<int64_t>(u) * L.tail * kHeadDim;
            for (int tok = 0; tok < L.tail; ++tok) {
                float kv[4];
                for (int x = 0; x < 4; ++x)
                    kv[x] = F16Traits<T>::to_float(reinterpret_cast<const uint16_t*>(kt)[tok * kHeadDim + 4 * lane + x]);
                float sv2[2] = {0.f, 0.f};
#pragma unroll
                for (int qq = 0; qq < kMaxGqa; ++qq) {
                    float part = 0.f;
                    if (qq < gqa)
                        for (int x = 0; x < 4; ++x)
                            part += F16Traits<T>::to_float(reinterpret_cast<const uint16_t*>(q)[qq * kHeadDim + 4 * lane + x]) * kv[x];
                    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
                    if (qq == 2 * t) sv2[0] = part * L.scale_log2;
                    if (qq == 2 * t + 1) sv2[1] = part * L.scale_log2;
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float sv = sv2[e];
                    const float mnew = fmaxf(m_run[e], sv);
                    const float al = fast_exp2(m_run[e] - mnew);
                    const float p = fast_exp2(sv - mnew);
                    l_run[e] = l_run[e] * al + (g == 0 ? p : 0.f);
                    m_run[e] = mnew;
#pragma unroll
                    for (int mi = 0; mi < 8; ++mi) {
                        const float v0 = F16Traits<T>::to_float(reinterpret_cast<const uint16_t*>(vt)[tok * kHeadDim + 16 * mi + g]);
                        const float v1 = F16Traits<T>::to_float(reinterpret_cast<const uint16_t*>(vt)[tok * kHeadDim + 16 * mi + g + 8]);
                        o[mi][e] = o[mi][e] * al + p * v0;
                        o[mi][2 + e] = o[mi][2 + e] * al + p * v1;
                    }
                }
            }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            l_run[e] += __shfl_xor_sync(0xffffffffu, l_run[e], 4);
            l_run[e] += __shfl_xor_sync(0xffffffffu, l_run[e], 8);
            l_run[e] += __shfl_xor_sync(0xffffffffu, l_run[e], 16);
        }
    }

    // ---------------- merge warps (attention.hpp:387-407 formula) ----------------
    __syncthreads();  // all stages consumed; reuse the ring as scratch
    if (ct && threadIdx.x == 0) ct[2] = globaltimer();
    float* s_o = reinterpret_cast<float*>(base_ptr);            // [NW][gqa][128]
    float* s_m = s_o + NW * kMaxGqa * kHeadDim;                 // [NW][gqa]
    float* s_l = s_m + NW * kMaxGqa;
    {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int qq = 2 * t + e;
            if (qq < gqa) {
                if (g == 0) {
                    s_m[warp * kMaxGqa + qq] = m_run[e];
                    s_l[warp * kMaxGqa + qq] = l_run[e];
                }
#pragma unroll
                for (int mi = 0; mi < 8; ++mi) {
                    s_o[(warp * kMaxGqa + qq) * kHeadDim + 16 * mi + g] = o[mi][e];
                    s_o[(warp * kMaxGqa + qq) * kHeadDim + 16 * mi + g + 8] = o[mi][2 + e];
                }
            }
        }
    }
    __syncthreads();
    const int nthr = 32 * NW;
    const int stride_p = gqa * (kHeadDim + 2);
    float* part = L.partial + (static_cast<int64_t>(u) * L.nsplit + split) * stride_p;
    constexpr float kLn2 = 0.6931471805599453f;
    // Tagged mailbox (coop combine): every (split, row, column) slot carries its
    // own O, m and l in two single-copy-atomic 64-bit words whose non-zero tags
    // mark them valid, so readers wait on the data itself -- no CTA barrier,
    // release atomic and acquire poll between the stores and the combine's loads
    // (each a device-scope round trip at the end of the step).
    unsigned long long* const mbox = L.coop_combine && L.out != nullptr && L.debug_tail == 0 ? L.mailbox : nullptr;
    if (mbox) {
        unsigned long long* mb = mbox + (static_cast<int64_t>(u) * L.nsplit + split) * gqa * kHeadDim * 2;
        for (int idx = threadIdx.x; idx < gqa * kHeadDim; idx += nthr) {
            const int qq = idx / kHeadDim, c = idx % kHeadDim;
            float M = -INFINITY;
            for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w * kMaxGqa + qq]);
            float acc = 0.f, accl = 0.f;
            for (int w = 0; w < NW; ++w) {
                const float mw = s_m[w * kMaxGqa + qq];
                const float wt = (mw == -INFINITY) ? 0.f : fast_exp2(mw - M);
                acc += wt * s_o[(w * kMaxGqa + qq) * kHeadDim + c];
                accl += wt * s_l[w * kMaxGqa + qq];
            }
            // ~bits(O) is never 0 (0xFFFFFFFF is no arithmetic result), l's tag is 1
            st_relaxed_gpu_v2(mb + 2 * idx,
                              static_cast<unsigned long long>(~__float_as_uint(acc)) |
                                  (static_cast<unsigned long long>(__float_as_uint(M * kLn2)) << 32),
                              static_cast<unsigned long long>(__float_as_uint(accl)) | (1ull << 32));
        }
    }
    for (int idx = threadIdx.x; idx < (mbox ? 0 : gqa * (kHeadDim + 1)); idx += nthr) {
        const int qq = idx / (kHeadDim + 1), c = idx % (kHeadDim + 1);
        float M = -INFINITY;
        for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w * kMaxGqa + qq]);
        float acc = 0.f;
        for (int w = 0; w < NW; ++w) {
            const float mw = s_m[w * kMaxGqa + qq];
            const float wt = (mw == -INFINITY) ? 0.f : fast_exp2(mw - M);
            acc += wt * (c < kHeadDim ? s_o[(w * kMaxGqa + qq) * kHeadDim + c] : s_l[w * kMaxGqa + qq]);
        }
        if (c < kHeadDim) {
            part[qq * (kHeadDim + 2) + c] = acc;
        } else {
            part[qq * (kHeadDim + 2) + kHeadDim] = M * kLn2;   // m in natural-log units
            part[qq * (kHeadDim + 2) + kHeadDim + 1] = acc;    // l
        }
    }
    if (ct && threadIdx.x == 0) ct[3] = globaltimer();
    if (L.out == nullptr) return;

    // ---------------- combine the unit's splits (attention.hpp:387-407) ----------------
    // Latency-bound (it runs once, after the stream): G lanes per output column
    // each fold a strided subset of the splits (their (m, l, O) loads issued
    // together, online LSE over groups of 4), then the G partial (M, acc, l) merge
    // by a butterfly of shuffles -- a handful of dependent steps instead of one
    // thread walking every split (measured ~2 us of the configs[1] step).
    const float* P = L.partial + static_cast<int64_t>(u) * L.nsplit * stride_p;
    // output staging past the merge scratch (free after the loop; up to gqa x d floats)
    float* const s_stage = s_l + NW * kMaxGqa;
    auto combine_slice = [&](int lo, int hi) {
        constexpr float kLog2e = 1.4426950408889634f;
        const int ncols = hi - lo;
        int G = 8;  // lanes per column (a power of two within a warp)
        while (G > 1 && ncols * G > nthr) G >>= 1;
        const int j = threadIdx.x / G, r = threadIdx.x % G, per_round = nthr / G;
        const int rounds = (ncols + per_round - 1) / per_round;
        for (int it = 0; it < rounds; ++it) {
            const int idx = lo + it * per_round + j;
            const bool valid = idx < hi;
            const int qq = valid ? idx / kHeadDim : 0, c = valid ? idx % kHeadDim : 0;
            const float* pq = P + qq * (kHeadDim + 2);
            float M = -INFINITY, acc = 0.f, lsum = 0.f;
            for (int sp0 = r; valid && sp0 < L.nsplit; sp0 += 4 * G) {
                float mv[4], lv[4], ov[4];
                if (mbox) {
                    // all slots' loads in flight together; re-poll only the late ones
                    unsigned long long* pb[4];
                    unsigned long long a[4], b[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const int sp = sp0 + x * G;
                        pb[x] = mbox + ((static_cast<int64_t>(u) * L.nsplit + sp) * gqa * kHeadDim + idx) * 2;
                        a[x] = sp < L.nsplit ? ld_relaxed_gpu_b64(pb[x]) : 0ull;
                        b[x] = sp < L.nsplit ? ld_relaxed_gpu_b64(pb[x] + 1) : 0ull;
                    }
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const bool live = sp0 + x * G < L.nsplit;
                        while (live && (static_cast<uint32_t>(a[x]) == 0u || (b[x] >> 32) == 0u)) {
                            a[x] = ld_relaxed_gpu_b64(pb[x]);
                            b[x] = ld_relaxed_gpu_b64(pb[x] + 1);
                        }
                        mv[x] = live ? __uint_as_float(static_cast<uint32_t>(a[x] >> 32)) : -INFINITY;
                        ov[x] = live ? __uint_as_float(~static_cast<uint32_t>(a[x])) : 0.f;
                        lv[x] = live ? __uint_as_float(static_cast<uint32_t>(b[x])) : 0.f;
                        // this lane is the slot's only reader: leave it empty for the next launch
                        if (live) *reinterpret_cast<ulonglong2*>(pb[x]) = make_ulonglong2(0ull, 0ull);
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const int sp = sp0 + x * G;
                        const float* ps = pq + static_cast<int64_t>(sp) * stride_p;
                        // weak loads: ordered after the producers' release by the acquire
                        // (and its L1 invalidation) plus the CTA barrier
                        mv[x] = sp < L.nsplit ? ps[kHeadDim] : -INFINITY;
                        lv[x] = sp < L.nsplit ? ps[kHeadDim + 1] : 0.f;
                        ov[x] = sp < L.nsplit ? ps[c] : 0.f;
                    }
                }
                const float Mc = fmaxf(fmaxf(M, fmaxf(mv[0], mv[1])), fmaxf(mv[2], mv[3]));
                if (Mc == -INFINITY) continue;  // every split so far empty
                if (M != Mc) {
                    const float sc = M == -INFINITY ? 0.f : fast_exp2((M - Mc) * kLog2e);
                    acc *= sc;
                    lsum *= sc;
                    M = Mc;
                }
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const float wt = mv[x] == -INFINITY ? 0.f : fast_exp2((mv[x] - M) * kLog2e);
                    acc = fmaf(ov[x], wt, acc);
                    lsum = fmaf(lv[x], wt, lsum);
                }
            }
            for (int o = 1; o < G; o <<= 1) {  // merge the G lanes' partial sums
                const float Mo = __shfl_xor_sync(0xffffffffu, M, o);
                const float ao = __shfl_xor_sync(0xffffffffu, acc, o);
                const float lo2 = __shfl_xor_sync(0xffffffffu, lsum, o);
                const float Mn = fmaxf(M, Mo);
                const float w1 = M == -INFINITY ? 0.f : fast_exp2((M - Mn) * kLog2e);
                const float w2 = Mo == -INFINITY ? 0.f : fast_exp2((Mo - Mn) * kLog2e);
                acc = acc * w1 + ao * w2;
                lsum = lsum * w1 + lo2 * w2;
                M = Mn;
            }
            if (!valid || r != 0) continue;
            if (L.out_mode == 0) {
                // staged, then written by consecutive lanes: full 128-byte lines
                // instead of a 16-byte piece per warp (out may be pinned host
                // memory: one PCIe write per line, DecodePlan(host_io))
                s_stage[idx - lo] = acc / lsum;
            } else {
                float* po = L.out + (static_cast<int64_t>(u) * L.q_rows + qq) * (kHeadDim + 2);
                po[c] = acc;
                if (c == 0) {
                    po[kHeadDim] = M;
                    po[kHeadDim + 1] = lsum;
                }
            }
        }
        if (L.out_mode == 0) {
            __syncthreads();
            for (int idx = lo + static_cast<int>(threadIdx.x); idx < hi; idx += nthr)
                L.out[(static_cast<int64_t>(u) * L.q_rows + idx / kHeadDim) * kHeadDim + idx % kHeadDim] =
                    s_stage[idx - lo];
        }
    };
    if (mbox) {
        // Every warp of the CTA finished claiming before the merge barrier; the
        // unit's last CTA past this point re-arms the claim counter.
        int* done = &L.counters[L.n_units + u];
        if (threadIdx.x == nthr - 1 && atomicAdd(done, 1) == L.nsplit - 1) {
            *done = 0;
            if (dyn) *ctr = 0;
        }
        if (ct && threadIdx.x == 0) ct[5] = globaltimer();
        const int n = gqa * kHeadDim;
        // slices on 32-column (128-byte) boundaries: whole output lines per CTA
        auto cut = [&](int sp) { return static_cast<int>(static_cast<int64_t>(n / 32) * sp / L.nsplit) * 32; };
        combine_slice(cut(split), split == L.nsplit - 1 ? n : cut(split + 1));
        if (ct && threadIdx.x == 0) ct[10] = ct[4] = globaltimer();
        return;
    }
    // Publication: the CTA barrier orders every thread's partial stores before
    // thread 0's release atomic on the unit's counter (no device-wide SC fence
    // in all 256 threads, ~0.5 us here); readers acquire the counter.
    __syncthreads();
    if (ct && threadIdx.x == 0) ct[7] = globaltimer();
    if (L.coop_combine) {
        // Whole grid resident (host-checked): every CTA of the unit waits for the
        // unit's last partial, then merges its own slice of the gqa x d outputs, so
        // the combine is one parallel round instead of one CTA's serial pass.
        int* arrive = &L.counters[u];
        int* done = &L.counters[L.n_units + u];
        if (threadIdx.x == 0) {
            atom_add_release_gpu(arrive, 1);
            while (L.debug_tail < 2 && ld_acquire(arrive) < L.nsplit) __nanosleep(64);
        }
        __syncthreads();
        if (ct && threadIdx.x == 0) ct[5] = globaltimer();
        const int n = gqa * kHeadDim;
        const int lo = static_cast<int>(static_cast<int64_t>(n) * split / L.nsplit);
        const int hi = static_cast<int>(static_cast<int64_t>(n) * (split + 1) / L.nsplit);
        if (L.debug_tail == 0) combine_slice(lo, hi);
        if (ct && threadIdx.x == 0) ct[10] = globaltimer();
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(done, 1) == L.nsplit - 1) {
            *arrive = 0;  // every CTA of the unit is past its spin: safe to re-arm
            *done = 0;
            if (dyn) *ctr = 0;  // every warp of the unit has finished claiming
        }
        if (ct && threadIdx.x == 0) ct[4] = globaltimer();
        return;
    }
    // Otherwise the last CTA of the unit to arrive merges everything.
    if (threadIdx.x == 0) s_ticket = atom_add_acq_rel_gpu(&L.counters[u], 1);
    __syncthreads();
    if (s_ticket != L.nsplit - 1) return;
    if (ct && threadIdx.x == 0) ct[5] = globaltimer();
    __threadfence();
    if (ct && threadIdx.x == 0) ct[6] = globaltimer();
    combine_slice(0, gqa * kHeadDim);
    if (threadIdx.x == 0) {
        L.counters[u] = 0;
        if (dyn) *ctr = 0;  // last CTA of the unit: every warp has finished claiming
    }
    if (ct && threadIdx.x == 0) ct[4] = globaltimer();
}

// Standalone LSE combine of n_parts partials (cross-GPU sequence split).
__global__ void combine_kernel(const float* partials, int n_parts, int n_units, int gqa, int d,
                               float* out) {
    const int u = blockIdx.x;
    const int stride_u = gqa * (d + 2);
    constexpr float kLog2e = 1.4426950408889634f;
    for (int idx = threadIdx.x; idx < gqa * d; idx += blockDim.x) {
        const int qq = idx / d, c = idx % d;
        float M = -INFINITY;
        for (int p = 0; p < n_parts; ++p)
            M = fmaxf(M, partials[(static_cast<int64_t>(p) * n_units + u) * stride_u + qq * (d + 2) + d]);
        float acc = 0.f, lsum = 0.f;
        for (int p = 0; p < n_parts; ++p) {
            const float* ps = partials + (static_cast<int64_t>(p) * n_units + u) * stride_u + qq * (d + 2);
            const float wt = ps[d] == -INFINITY ? 0.f : exp2f((ps[d] - M) * kLog2e);
            lsum += ps[d + 1] * wt;
            acc += ps[c] * wt;
        }
        out[(static_cast<int64_t>(u) * gqa + qq) * d + c] = acc / lsum;
    }
}

template <typename T, int NW, bool HILO>
cudaError_t configure_t(size_t smem) {
    auto k = decode_kernel<T, NW, HILO>;
    static int configured_smem = 0;  // per instantiation; raise the opt-in once
    if (static_cast<int>(smem) > configured_smem) {
        cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err) return err;
        configured_smem = static_cast<int>(smem);
    }
    return cudaSuccess;
}

// Resident CTAs of this instantiation at `smem` bytes over the whole device.
template <typename T, int NW, bool HILO>
int resident_t(size_t smem, int sms) {
    static std::mutex mu;
    static std::map<std::pair<size_t, int>, int> cache;  // (smem, device) -> CTAs per SM
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({smem, dev});
    if (it != cache.end()) return it->second * sms;
    if (configure_t<T, NW, HILO>(smem) != cudaSuccess) return 0;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<T, NW, HILO>, 32 * NW, smem) !=
        cudaSuccess)
        return 0;
    cache[{smem, dev}] = per_sm;
    return per_sm * sms;
}

// The cooperative combine spins on the other CTAs of its unit, so it is only
// launched with cudaLaunchAttributeCooperative: the driver then guarantees the
// whole grid is co-resident or refuses the launch (MPS / green-context SM
// limits, concurrent kernels holding SMs), and the caller falls back to the
// last-CTA ticket combine.
template <typename T, int NW, bool HILO>
cudaError_t launch_t(const DecodeLaunch& L, int spw, StageLayout lay, size_t smem,
                     cudaStream_t s) {
    cudaError_t err = configure_t<T, NW, HILO>(smem);
    if (err) return err;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = L.interleave ? dim3(L.nsplit * L.n_units) : dim3(L.nsplit, L.n_units);
    cfg.blockDim = dim3(32 * NW);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = L.coop_combine ? 1 : 0;
    err = cudaLaunchKernelEx(&cfg, decode_kernel<T, NW, HILO>, L, spw, lay);
    if (err != cudaSuccess && L.coop_combine) {
        (void)cudaGetLastError();  // cooperative launch refused: ticket combine instead
        DecodeLaunch L2 = L;
        L2.coop_combine = 0;
        cfg.numAttrs = 0;
        err = cudaLaunchKernelEx(&cfg, decode_kernel<T, NW, HILO>, L2, spw, lay);
    }
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

}  // namespace

int decode_warps() {
    const char* env = getenv("HS_DECODE_WARPS");
    const int w = env ? atoi(env) : 8;
    return w == 4 ? 4 : 8;
}

int decode_ctas_per_sm() {
    const char* env = getenv("HS_DECODE_CTAS_PER_SM");
    return env && atoi(env) == 2 ? 2 : 1;
}

size_t decode_smem_bytes(const DecodeLaunch& L, int* nw_out, int* spw_out, StageLayout* lay_out) {
    StageLayout lay;
    lay.k_bytes = L.k_dense_count > 0 ? 16384u : 9216u;
    lay.v_bytes = L.v_dense_count > 0 ? 16384u : 9216u;
    lay.stage_bytes = lay.k_bytes + lay.v_bytes;
    const uint32_t idx_bytes = static_cast<uint32_t>(L.max_blocks_per_cta) * 4u;
    const uint32_t budget = (decode_ctas_per_sm() == 1 ? 225u : 112u) * 1024u - idx_bytes - 2048u;
    int NW = decode_warps();
    while (NW > 4 && static_cast<uint32_t>(NW) * lay.stage_bytes > budget) NW = 4;  // dense stages are 32 KB
    int spw = static_cast<int>(budget / (NW * lay.stage_bytes));
    if (const char* env = getenv("HS_DECODE_SPW")) spw = atoi(env);
    if (spw * NW > 16) spw = 16 / NW;
    if (spw < 1) spw = 1;
    size_t smem = static_cast<size_t>(NW * spw) * lay.stage_bytes;
    const size_t scratch = (NW * kMaxGqa * kHeadDim + 2 * NW * kMaxGqa) * sizeof(float);
    const size_t combine = 0;  // the split combine works in registers
    if (smem < scratch) smem = scratch;
    if (smem < combine) smem = combine;
    smem += idx_bytes + 1024;
    *nw_out = NW;
    *spw_out = spw;
    *lay_out = lay;
    return smem;
}

int decode_resident_ctas(const DecodeLaunch& L, int sms) {
    int nw, spw;
    StageLayout lay;
    const size_t smem = decode_smem_bytes(L, &nw, &spw, &lay);
    if (nw == 4) return L.bf16 ? resident_t<__nv_bfloat16, 4, true>(smem, sms) : resident_t<__half, 4, false>(smem, sms);
    return L.bf16 ? resident_t<__nv_bfloat16, 8, true>(smem, sms) : resident_t<__half, 8, false>(smem, sms);
}

cudaError_t launch_decode(const DecodeLaunch& L, cudaStream_t s) {
    int nw, spw;
    StageLayout lay;
    const size_t smem = decode_smem_bytes(L, &nw, &spw, &lay);
    if (nw == 4) {
        if (L.bf16) return launch_t<__nv_bfloat16, 4, true>(L, spw, lay, smem, s);
        return launch_t<__half, 4, false>(L, spw, lay, smem, s);
    }
    if (L.bf16) return launch_t<__nv_bfloat16, 8, true>(L, spw, lay, smem, s);
    return launch_t<__half, 8, false>(L, spw, lay, smem, s);
}

cudaError_t launch_combine(const float* partials, int n_parts, int n_units, int gqa, int d,
                           float* out, cudaStream_t s) {
    combine_kernel<<<n_units, 256, 0, s>>>(partials, n_parts, n_units, gqa, d, out);
    return cudaGetLastError();
}

}  // namespace hs
