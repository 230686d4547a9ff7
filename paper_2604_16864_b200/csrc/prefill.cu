// Trans-Both sparse prefill attention on tcgen05 (sm_100a).
//
// Reference semantics: prefill_attention (attention.hpp:323-354) = attend_range
// (:249-304) over every block + finalize_rows (:309-317), online softmax
// (:171-239), causal alignment qpos = n_kv - n_q + i (:342-346).
//
// Orientation: S^T = K_tile * Q^T and O^T += V^T_tile * P^T,
// so the pruned K (2:4 along d) and V^T (2:4 along the sequence) are the sparse
// A operands of tcgen05.mma.sp; accumulators live in TMEM:
//   S^T[128 keys x 128 queries]  (double buffered)   O^T[128 d x 128 queries]
// One CTA = (unit, query head, 128-query tile).  Key tiles are pairs of 64-token
// blocks of the same K kind so GEMM1 runs at M = 128: fully visible
// sparse pairs, then dense pairs, then single/mixed and diagonal blocks (order
// only changes float rounding; attention is order invariant over visible keys).
//
// Warp roles (352 threads):
//   0-7  softmax, two warpgroups: WG g owns query columns 64g..64g+63; warp w
//        reads TMEM lanes 32(w%4).. (key row r of the tile = d row of O^T).
//        Exact per-tile column max (redux.f32 + smem), running max updated only
//        when it grows by > 2^8 (FA4-style lazy rescale), P^T written to smem
//        (MN-major SW128, N-atom g) for GEMM2, O^T / l rescaled only on the rare
//        max update; epilogue normalises O.
//   8    TMA producer: Q once; per key tile K/V pools + canonical metadata.
//   9    MMA issuer: tcgen05.cp metadata -> TMEM, GEMM1 (t), GEMM2 (t-1).
//   10   metadata: permutes canonical 2-bit codes (nm_metadata.hpp:42-46) into
//        the tcgen05 TMEM metadata atom (pinned by tools/probes/umma_probe.cu).
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace hs {
namespace {

constexpr int kThreads = 352;  // 2 softmax warpgroups + TMA + MMA + metadata warps
constexpr int kMaxTiles = 1280;   // key tiles per query tile (<= 32767 blocks / 2 + a few)
constexpr float kTau = 8.0f;      // lazy-rescale threshold (log2 units): P <= 2^8

struct TileInfo {
    int16_t b0, b1;   // logical blocks (b1 = -1: single block, rows 64..127 invalid)
    uint8_t kd;       // K kind of the tile: 1 dense, 0 sparse
    uint8_t vd0, vd1; // V kinds of b0 / b1
    uint8_t diag;     // needs element-level causal masking
};

struct PrefillLayout {
    uint32_t k_bytes, vblk_bytes, stage_bytes, stages;
    uint32_t off_q, off_p, off_stage;
};

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ float redux_max(float v) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}

// P^T element offset (MN-major SW128): N-atom h = q/64 at h*16 KB; key row r at
// (r/8)*1024 + (r%8)*128; 16-byte chunk (q%64)/8 swizzled by r%8.
__device__ __forceinline__ uint32_t pt_chunk_off(int r, int q8 /*query/8 in 0..15*/) {
    const int h = q8 >> 3, c = q8 & 7;
    return h * 16384 + (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
}

// Per-tile event timestamps of CTA (0,0,0) for pipeline analysis (tools only).
__device__ __forceinline__ void trace(const PrefillLaunch& L, int t, int ev) {
    if (L.trace != nullptr && t < 4096 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        L.trace[t * 8 + ev] = clock64();
}

template <typename T, bool HILO>
__global__ void __launch_bounds__(kThreads, 1) prefill_kernel(const __grid_constant__ PrefillLaunch L,
                                                               PrefillLayout lay) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar_q, bar_full[4], bar_meta[4], bar_empty[4];
    __shared__ __align__(8) uint64_t bar_sfull[2], bar_sempty[2], bar_pfull, bar_pempty;
    __shared__ uint32_t s_tmem;
    __shared__ int s_ntiles, s_rescale[2][2];
    __shared__ float s_red[4][128];
    __shared__ float s_mnew[128], s_alpha[128];
    __shared__ TileInfo s_tiles[kMaxTiles];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int n_tiles_q = (L.n_q + 127) / 128;
    const int qt = n_tiles_q - 1 - static_cast<int>(blockIdx.x);  // heaviest causal tiles first
    const int h = blockIdx.y, u = blockIdx.z;
    const int q0 = qt * 128;
    const int n_kv = L.nb * kBlock;  // tail == 0 on this path
    const int off = n_kv - L.n_q;
    const int rows_q = min(128, L.n_q - q0);

    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* const base_ptr = smem_raw + (base - raw);
    const uint32_t sQ = base + lay.off_q, sP = base + lay.off_p, sStage = base + lay.off_stage;

    // ------------------------------------------------------------ setup ----
    if (warp == 9) tmem_alloc(&s_tmem, 512);
    if (tid == 0) {
        mbar_init(&bar_q, 1);
        for (uint32_t s = 0; s < lay.stages; ++s) {
            mbar_init(&bar_full[s], 1);
            mbar_init(&bar_meta[s], 1);
            mbar_init(&bar_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar_sfull[i], 1);
            mbar_init(&bar_sempty[i], 8);
        }
        mbar_init(&bar_pfull, 8);
        mbar_init(&bar_pempty, 1);
        fence_barrier_init();
    }
    if (warp == 8 && lane == 0) {
        // Key-tile list (see header).  Block b is fully visible iff its last key
        // <= the tile's first query position; visible iff its first key <= the last.
        const int16_t* kidx = L.k_index + static_cast<int64_t>(u) * L.nb;
        const int16_t* vidx = L.v_index + static_cast<int64_t>(u) * L.nb;
        const int32_t* sb = L.k_slot_block + static_cast<int64_t>(u) * L.nb;
        int fv_end = L.nb, vis_end = L.nb;
        if (L.causal) {
            fv_end = max(0, min(L.nb, (off + q0 + 1) / kBlock));
            vis_end = min(L.nb, (off + q0 + rows_q - 1) / kBlock + 1);
        }
        // sparse K slots hold blocks in increasing order: count those < fv_end
        int lo = 0, hi = L.k_sparse_count;
        const int32_t* sparse_blocks = sb + L.k_dense_count;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sparse_blocks[mid] < fv_end) lo = mid + 1; else hi = mid;
        }
        const int ns = lo, nd = fv_end - ns;
        int n = 0;
        auto push = [&](int b0, int b1, int kd, int diag) {
            TileInfo ti;
            ti.b0 = static_cast<int16_t>(b0);
            ti.b1 = static_cast<int16_t>(b1);
            ti.kd = static_cast<uint8_t>(kd);
            ti.vd0 = vidx[b0] > 0;
            ti.vd1 = b1 >= 0 ? (vidx[b1] > 0) : 0;
            ti.diag = static_cast<uint8_t>(diag);
            if (n < kMaxTiles) s_tiles[n] = ti;
            ++n;
        };
        for (int i = 0; i + 1 < ns; i += 2) push(sparse_blocks[i], sparse_blocks[i + 1], 0, 0);
        for (int i = 0; i + 1 < nd; i += 2) push(sb[i], sb[i + 1], 1, 0);
        if (ns & 1) push(sparse_blocks[ns - 1], -1, 0, 0);
        if (nd & 1) push(sb[nd - 1], -1, 1, 0);
        for (int b = fv_end; b < vis_end; ++b) {
            const int kd = kidx[b] > 0;
            if (b + 1 < vis_end && (kidx[b + 1] > 0) == kd) {
                push(b, b + 1, kd, 1);
                ++b;
            } else {
                push(b, -1, kd, 1);
            }
        }
        s_ntiles = n;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const int ntiles = min(s_ntiles, kMaxTiles);
    // TMEM columns: S[0] 0..127, S[1] 128..255, O 256..383, E_K[2] 384.., E_V[2] 392..
    const uint32_t tS0 = tmem, tO = tmem + 256, tEK = tmem + 384, tEV = tmem + 392;

    const uint8_t* stage_ptr0 = base_ptr + lay.off_stage;
    auto stage_base = [&](int s) { return sStage + s * lay.stage_bytes; };
    // stage sub-layout
    const uint32_t oK = 0, oV = lay.k_bytes, oKm = lay.k_bytes + 2 * lay.vblk_bytes, oVm = oKm + 2048,
                   oEK = oVm + 2048, oEV = oEK + 2048;

    if (warp == 8) {
        // ------------------------------------------------------- TMA producer
        if (lane == 0) {
            prefetch_tmap(&L.tm_q);
            prefetch_tmap(&L.tm_knnz);
            prefetch_tmap(&L.tm_vnnz);
            const int qrow = (u * L.gqa + h) * L.n_q + q0;
            mbar_arrive_expect_tx(&bar_q, 32768);
            tma_tile_g2s(base_ptr + lay.off_q, &L.tm_q, 0, qrow, &bar_q);
            tma_tile_g2s(base_ptr + lay.off_q + 16384, &L.tm_q, 64, qrow, &bar_q);
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % lay.stages;
                mbar_wait_dbg(&bar_empty[s], ((t / lay.stages) & 1) ^ 1, L.dbg, 4);
                const TileInfo ti = s_tiles[t];
                uint8_t* st = const_cast<uint8_t*>(stage_ptr0) + s * lay.stage_bytes;
                uint32_t bytes = 0;
                const int nb_t = ti.b1 >= 0 ? 2 : 1;
                for (int i = 0; i < nb_t; ++i) bytes += ti.kd ? 16384u : 9216u;
                for (int i = 0; i < nb_t; ++i) bytes += (i == 0 ? ti.vd0 : ti.vd1) ? 16384u : 9216u;
                mbar_arrive_expect_tx(&bar_full[s], bytes);
                for (int i = 0; i < nb_t; ++i) {
                    const int b = i == 0 ? ti.b0 : ti.b1;
                    const int ke = L.k_index[static_cast<int64_t>(u) * L.nb + b];
                    if (ti.kd) {
                        const int row = (u * L.k_dense_count + ke - 1) * kBlock;
                        tma_tile_g2s(st + oK + 8192 * i, &L.tm_kden, 0, row, &bar_full[s]);
                        tma_tile_g2s(st + oK + 16384 + 8192 * i, &L.tm_kden, 64, row, &bar_full[s]);
                    } else {
                        const int sbk = u * L.k_sparse_count + (-ke - 1);
                        tma_tile_g2s(st + oK + 8192 * i, &L.tm_knnz, 0, sbk * kBlock, &bar_full[s]);
                        tma_bulk_g2s(st + oKm + 1024 * i, L.k_meta + static_cast<int64_t>(sbk) * 512, 1024,
                                     &bar_full[s]);
                    }
                    const int ve = L.v_index[static_cast<int64_t>(u) * L.nb + b];
                    if (ve > 0) {
                        const int row = (u * L.v_dense_count + ve - 1) * kHeadDim;
                        tma_tile_g2s(st + oV + lay.vblk_bytes * i, &L.tm_vden, 0, row, &bar_full[s]);
                    } else {
                        const int sbv = u * L.v_sparse_count + (-ve - 1);
                        tma_tile_g2s(st + oV + lay.vblk_bytes * i, &L.tm_vnnz, 0, sbv * kHeadDim, &bar_full[s]);
                        tma_bulk_g2s(st + oVm + 1024 * i, L.v_meta + static_cast<int64_t>(sbv) * 512, 1024,
                                     &bar_full[s]);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 10) {
        // ------------------------------------------------ metadata permuter
        // E atom u16 index for (row m, word w): 8(m&7) + ((m>>3)&1) + 128(m>>4)
        // + 64(w&1) + 2(w>>1) (+4 for the second V block); rows m and m+8 are
        // adjacent u16s, so each store writes a (row m, row m+8) pair.
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % lay.stages;
            mbar_wait_dbg(&bar_full[s], (t / lay.stages) & 1, L.dbg, 2);
            const TileInfo ti = s_tiles[t];
            uint8_t* st = const_cast<uint8_t*>(stage_ptr0) + s * lay.stage_bytes;
            if (!ti.kd) {
                const bool single = ti.b1 < 0;
                for (int pidx = lane; pidx < 64; pidx += 32) {  // row pairs (m, m+8)
                    const int m = (pidx & 7) + 16 * (pidx >> 3);
                    uint4 lo4 = make_uint4(0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
                    uint4 hi4 = lo4;
                    if (!(single && m >= 64)) {
                        lo4 = *reinterpret_cast<const uint4*>(st + oKm + (m >> 6) * 1024 + (m & 63) * 16);
                        hi4 = *reinterpret_cast<const uint4*>(st + oKm + ((m + 8) >> 6) * 1024 + ((m + 8) & 63) * 16);
                    }
                    const uint32_t lw[4] = {lo4.x, lo4.y, lo4.z, lo4.w}, hw[4] = {hi4.x, hi4.y, hi4.z, hi4.w};
                    uint16_t* e = reinterpret_cast<uint16_t*>(st + oEK);
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        const uint32_t a = (lw[w >> 1] >> (16 * (w & 1))) & 0xFFFF;
                        const uint32_t b = (hw[w >> 1] >> (16 * (w & 1))) & 0xFFFF;
                        const int idx = 8 * (m & 7) + 128 * (m >> 4) + 64 * (w & 1) + 2 * (w >> 1);
                        *reinterpret_cast<uint32_t*>(e + idx) = a | (b << 16);
                    }
                }
            }
            const int nb_t = ti.b1 >= 0 ? 2 : 1;
            for (int i = 0; i < nb_t; ++i) {
                if (i == 0 ? ti.vd0 : ti.vd1) continue;
                for (int pidx = lane; pidx < 64; pidx += 32) {
                    const int m = (pidx & 7) + 16 * (pidx >> 3);
                    const uint2 lo2 = *reinterpret_cast<const uint2*>(st + oVm + 1024 * i + m * 8);
                    const uint2 hi2 = *reinterpret_cast<const uint2*>(st + oVm + 1024 * i + (m + 8) * 8);
                    const uint32_t lw[2] = {lo2.x, lo2.y}, hw[2] = {hi2.x, hi2.y};
                    uint16_t* e = reinterpret_cast<uint16_t*>(st + oEV);
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const uint32_t a = (lw[w >> 1] >> (16 * (w & 1))) & 0xFFFF;
                        const uint32_t b = (hw[w >> 1] >> (16 * (w & 1))) & 0xFFFF;
                        const int idx = 8 * (m & 7) + 128 * (m >> 4) + 64 * (w & 1) + 2 * (w >> 1) + 4 * i;
                        *reinterpret_cast<uint32_t*>(e + idx) = a | (b << 16);
                    }
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_meta[s]);
        }
    } else if (warp == 9) {
        // ------------------------------------------------------- MMA issuer
        if (lane == 0) {
            const bool bf = std::is_same<T, __nv_bfloat16>::value;
            const uint32_t id_g1_sp = umma_idesc_f16(bf, 128, 128, false, false, true);
            const uint32_t id_g1_de = umma_idesc_f16(bf, 128, 128, false, false, false);
            const uint32_t id_g2_sp = umma_idesc_f16(bf, 128, 128, false, true, true);
            const uint32_t id_g2_de = umma_idesc_f16(bf, 128, 128, false, true, false);
            mbar_wait_dbg(&bar_q, 0, L.dbg, 1);
            tc_fence_after();
            bool o_started = false;
            auto gemm2 = [&](int tp) {
                // O^T += V^T (tile tp) * P^T ; P^T in smem (hi, then lo for bf16)
                const int s = tp % lay.stages;
                const uint32_t st = stage_base(s);
                const TileInfo ti = s_tiles[tp];
                mbar_wait_dbg(&bar_pfull, tp & 1, L.dbg, 7);
                tc_fence_after();
                trace(L, tp, 5);
                const int nb_t = ti.b1 >= 0 ? 2 : 1;
                for (int pass = 0; pass < (HILO ? 2 : 1); ++pass) {
                    const uint32_t pbase = sP + pass * 32768;
                    for (int i = 0; i < nb_t; ++i) {
                        const bool vdense = i == 0 ? ti.vd0 : ti.vd1;
                        const uint32_t va = st + oV + lay.vblk_bytes * i;
                        if (vdense) {
                            for (int kk = 0; kk < 4; ++kk) {
                                umma_f16(tO, umma_desc(va + 32 * kk, 16, 1024, kLayoutSW128),
                                         umma_desc(pbase + 8192 * i + 2048 * kk, 16384, 1024, kLayoutSW128),
                                         id_g2_de, o_started);
                                o_started = true;
                            }
                        } else {
                            for (int j = 0; j < 2; ++j) {
                                umma_sp_f16(tO, umma_desc(va + 32 * j, 16, 512, kLayoutSW64),
                                            umma_desc(pbase + 8192 * i + 4096 * j, 16384, 1024, kLayoutSW128),
                                            tEV + 4 * (tp & 1) + 2 * i + j, id_g2_sp, o_started);
                                o_started = true;
                            }
                        }
                    }
                }
                trace(L, tp, 6);
                umma_commit(&bar_pempty);   // P^T buffer and O^T (for the softmax rescale)
                umma_commit(&bar_empty[s]); // K/V stage can be refilled
            };
            for (int t = 0; t < ntiles; ++t) {
                // One stage (bf16 + dense K/V) cannot hold tile t while GEMM2(t-1)
                // still reads tile t-1: drain GEMM2(t-1) first in that case.
                if (lay.stages == 1 && t >= 1) gemm2(t - 1);
                const int s = t % lay.stages, sb = t & 1;
                const uint32_t st = stage_base(s);
                const TileInfo ti = s_tiles[t];
                mbar_wait_dbg(&bar_full[s], (t / lay.stages) & 1, L.dbg, 2);
                mbar_wait_dbg(&bar_meta[s], (t / lay.stages) & 1, L.dbg, 3);
                if (t >= 2) mbar_wait_dbg(&bar_sempty[sb], ((t >> 1) - 1) & 1, L.dbg, 6);
                tc_fence_after();
                trace(L, t, 4);
                // metadata -> TMEM (ordered before the MMAs that read it)
                if (!ti.kd) tmem_cp_128x128b(tEK + 4 * sb, umma_desc(st + oEK, 16, 128, kLayoutNone));
                if (!ti.vd0 || (ti.b1 >= 0 && !ti.vd1))
                    tmem_cp_128x128b(tEV + 4 * sb, umma_desc(st + oEV, 16, 128, kLayoutNone));
                // GEMM1: S^T[sb] = K_tile * Q^T
                const uint32_t tS = tS0 + 128 * sb;
                if (ti.kd) {
                    for (int j = 0; j < 8; ++j)
                        umma_f16(tS, umma_desc(st + oK + (j >> 2) * 16384 + 32 * (j & 3), 16, 1024, kLayoutSW128),
                                 umma_desc(sQ + (j >> 2) * 16384 + 32 * (j & 3), 16, 1024, kLayoutSW128), id_g1_de,
                                 j > 0);
                } else {
                    for (int j = 0; j < 4; ++j)
                        umma_sp_f16(tS, umma_desc(st + oK + 32 * j, 16, 1024, kLayoutSW128),
                                    umma_desc(sQ + (j >> 1) * 16384 + 64 * (j & 1), 16, 1024, kLayoutSW128),
                                    tEK + 4 * sb + j, id_g1_sp, j > 0);
                }
                umma_commit(&bar_sfull[sb]);
                if (lay.stages > 1 && t >= 1) gemm2(t - 1);
            }
            if (ntiles > 0) gemm2(ntiles - 1);
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------- softmax WGs
        const int wg = warp >> 2, wq = warp & 3;
        const int r = 32 * wq + lane;  // TMEM lane = key row of the tile = d row of O^T
        const int cbase = 64 * wg;     // this warpgroup's query columns
        const int bar_id = 1 + wg;
        const uint32_t lane_off = static_cast<uint32_t>(32 * wq) << 16;
        float l_part[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) l_part[c] = 0.f;
        float m_col = -INFINITY;  // running max of column cbase + r (threads r < 64)
        uint8_t* pbuf = base_ptr + lay.off_p;
        for (int t = 0; t < ntiles; ++t) {
            const int sb = t & 1;
            const TileInfo ti = s_tiles[t];
            mbar_wait_dbg(&bar_sfull[sb], (t >> 1) & 1, L.dbg, 5);
            tc_fence_after();
            if (tid == 0) trace(L, t, 0);
            // masks: invalid rows of single-block tiles; causal (attention.hpp:181-190)
            const bool row_valid = r < 64 || ti.b1 >= 0;
            const int key_pos = (r < 64 ? ti.b0 : ti.b1) * kBlock + (r & 63);
            // column c (query q0 + c at position off + q0 + c) sees this key iff c >= c_first
            const int c_first = row_valid ? (ti.diag ? key_pos - off - q0 : 0) : 1 << 30;
            // warp-uniform fast path: every (row, column) of this warp visible
            const bool fast = __all_sync(0xffffffffu, c_first <= cbase);
            const uint32_t tS = tS0 + 128 * sb + lane_off + cbase;
            // pass 1: exact column max of the raw scores (scale > 0 commutes with max);
            // the redux result is warp-uniform, so every lane stores it (no select)
#pragma unroll
            for (int ch = 0; ch < 2; ++ch) {
                uint32_t v[32];
                tmem_ld32(tS + 32 * ch, v);
                tmem_ld_wait();
                float* dst = &s_red[wq][cbase + 32 * ch];
                if (fast) {
#pragma unroll
                    for (int k = 0; k < 32; ++k) dst[k] = redux_max(__uint_as_float(v[k]));
                } else {
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        dst[k] = redux_max(cbase + 32 * ch + k >= c_first ? __uint_as_float(v[k]) : -INFINITY);
                }
            }
            if (r == 0) s_rescale[wg][t & 1] = 0;
            named_bar(bar_id, 128);
            if (r < 64) {
                const int c = cbase + r;
                float tm = fmaxf(fmaxf(s_red[0][c], s_red[1][c]), fmaxf(s_red[2][c], s_red[3][c]));
                tm = tm * L.scale_log2;
                float mnew = m_col, alpha = 1.f;
                if (tm > -INFINITY && (m_col == -INFINITY || tm > m_col + kTau)) {
                    mnew = tm;
                    alpha = m_col == -INFINITY ? 1.f : fast_exp2(m_col - mnew);
                    if (m_col != -INFINITY) s_rescale[wg][t & 1] = 1;
                }
                m_col = mnew;
                s_mnew[c] = mnew;
                s_alpha[c] = alpha;
            }
            named_bar(bar_id, 128);
            if (tid == 0) trace(L, t, 1);
            // P^T buffer free + O^T stable (GEMM2(t-1) complete)
            if (t >= 1) mbar_wait_dbg(&bar_pempty, (t - 1) & 1, L.dbg, 8);
            tc_fence_after();
            if (tid == 0) trace(L, t, 2);
            if (s_rescale[wg][t & 1]) {
#pragma unroll
                for (int cc = 0; cc < 64; ++cc) l_part[cc] *= s_alpha[cbase + cc];
                if (t >= 1) {
#pragma unroll
                    for (int ch = 0; ch < 2; ++ch) {
                        uint32_t v[32];
                        tmem_ld32(tO + lane_off + cbase + 32 * ch, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int k = 0; k < 32; k += 4) {
                            const float4 a4 = *reinterpret_cast<const float4*>(&s_alpha[cbase + 32 * ch + k]);
                            v[k] = __float_as_uint(__uint_as_float(v[k]) * a4.x);
                            v[k + 1] = __float_as_uint(__uint_as_float(v[k + 1]) * a4.y);
                            v[k + 2] = __float_as_uint(__uint_as_float(v[k + 2]) * a4.z);
                            v[k + 3] = __float_as_uint(__uint_as_float(v[k + 3]) * a4.w);
                        }
#pragma unroll
                        for (int k = 0; k < 32; k += 4)
                            tmem_st4(tO + lane_off + cbase + 32 * ch + k, v[k], v[k + 1], v[k + 2], v[k + 3]);
                    }
                    tmem_st_wait();
                }
            }
            // pass 2: probabilities, row sums, P^T (+ residual for bf16)
#pragma unroll
            for (int ch = 0; ch < 2; ++ch) {
                uint32_t v[32];
                tmem_ld32(tS + 32 * ch, v);
                tmem_ld_wait();
#pragma unroll
                for (int g8 = 0; g8 < 4; ++g8) {
                    const int q8 = (cbase >> 3) + 4 * ch + g8;  // 8-query chunk index in 0..15
                    const float4 ma = *reinterpret_cast<const float4*>(&s_mnew[8 * q8]);
                    const float4 mb = *reinterpret_cast<const float4*>(&s_mnew[8 * q8 + 4]);
                    const float mm[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
                    float p[8];
                    if (fast) {
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            p[k] = fast_exp2(fmaf(__uint_as_float(v[8 * g8 + k]), L.scale_log2, -mm[k]));
                    } else {
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const float x = fmaf(__uint_as_float(v[8 * g8 + k]), L.scale_log2, -mm[k]);
                            const int cc = 8 * q8 + k;
                            p[k] = (cc >= c_first && mm[k] != -INFINITY) ? fast_exp2(x) : 0.f;
                        }
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) l_part[32 * ch + 8 * g8 + k] += p[k];
                    const uint4 hi = make_uint4(F16Traits<T>::pack(p[0], p[1]), F16Traits<T>::pack(p[2], p[3]),
                                                F16Traits<T>::pack(p[4], p[5]), F16Traits<T>::pack(p[6], p[7]));
                    *reinterpret_cast<uint4*>(pbuf + pt_chunk_off(r, q8)) = hi;
                    if (HILO) {
                        float rr[8];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t w = (&hi.x)[k];
                            rr[2 * k] = p[2 * k] - F16Traits<T>::to_float(static_cast<uint16_t>(w & 0xFFFF));
                            rr[2 * k + 1] = p[2 * k + 1] - F16Traits<T>::to_float(static_cast<uint16_t>(w >> 16));
                        }
                        const uint4 lo = make_uint4(F16Traits<T>::pack(rr[0], rr[1]), F16Traits<T>::pack(rr[2], rr[3]),
                                                    F16Traits<T>::pack(rr[4], rr[5]), F16Traits<T>::pack(rr[6], rr[7]));
                        *reinterpret_cast<uint4*>(pbuf + 32768 + pt_chunk_off(r, q8)) = lo;
                    }
                }
            }
            if (tid == 0) trace(L, t, 3);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_sempty[sb]);  // this warp is done with S^T[sb]
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_pfull);
        }
        // ---------------------------------------------------- epilogue ----
        if (ntiles > 0) mbar_wait_dbg(&bar_pempty, (ntiles - 1) & 1, L.dbg, 8);
        tc_fence_after();
        // l[c] = sum over the 128 key lanes of l_part[c]: transpose through smem
        float* s_l = reinterpret_cast<float*>(base_ptr + lay.off_stage) + wg * (128 * 65);
        named_bar(bar_id, 128);
#pragma unroll
        for (int c = 0; c < 64; ++c) s_l[r * 65 + c] = l_part[c];
        named_bar(bar_id, 128);
        if (r < 64) {
            float lsum = 0.f;
            for (int k = 0; k < 128; ++k) lsum += s_l[k * 65 + r];
            s_alpha[cbase + r] = lsum > 0.f ? 1.f / lsum : 0.f;
        }
        named_bar(bar_id, 128);
        float* out = L.out + (static_cast<int64_t>(u * L.gqa + h) * L.n_q + q0) * kHeadDim;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
            uint32_t v[32];
            tmem_ld32(tO + lane_off + cbase + 32 * ch, v);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int c = cbase + 32 * ch + k;
                if (c < rows_q) out[c * kHeadDim + r] = __uint_as_float(v[k]) * s_alpha[c];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) tmem_dealloc(tmem, 512);
}

}  // namespace

cudaError_t launch_prefill(const PrefillLaunch& L, cudaStream_t s) {
    PrefillLayout lay;
    const bool hilo = L.bf16;
    lay.k_bytes = L.k_dense_count > 0 ? 32768u : 16384u;
    lay.vblk_bytes = L.v_dense_count > 0 ? 16384u : 9216u;
    lay.vblk_bytes = (lay.vblk_bytes + 1023u) & ~1023u;
    lay.stage_bytes = lay.k_bytes + 2 * lay.vblk_bytes + 8192u;
    lay.off_q = 0;
    lay.off_p = 32768;
    lay.off_stage = 32768 + (hilo ? 65536u : 32768u);
    const uint32_t budget = 227u * 1024u - 16384u /*static smem*/ - 1024u - lay.off_stage;
    uint32_t stages = budget / lay.stage_bytes;
    if (stages > 4) stages = 4;
    if (stages < 1) return cudaErrorInvalidConfiguration;
    lay.stages = stages;
    size_t smem = lay.off_stage + static_cast<size_t>(stages) * lay.stage_bytes + 1024;
    const size_t epi = lay.off_stage + 2 * 128 * 65 * 4 + 1024;
    if (smem < epi) smem = epi;
    const dim3 grid((L.n_q + 127) / 128, L.gqa, L.n_units);
    if (L.bf16) {
        auto k = prefill_kernel<__nv_bfloat16, true>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
        k<<<grid, kThreads, smem, s>>>(L, lay);
    } else {
        auto k = prefill_kernel<__half, false>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
        k<<<grid, kThreads, smem, s>>>(L, lay);
    }
    return cudaGetLastError();
}

}  // namespace hs
