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
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace hs {
namespace {

constexpr int kThreads = 352;  // 2 softmax warpgroups + TMA + MMA + metadata warps

constexpr float kTau = 8.0f;      // lazy-rescale threshold (log2 units): P <= 2^8

// One key tile = one or two 64-token blocks of the same K kind.  8 bytes:
//   ke0   K index-map entry of the first block (sign = kind, |ke0|-1 = pool slot);
//         the second block of a pair is always the next slot of the same pool
//   ve0/1 V index-map entries of the two blocks (ve1 == 0: single-block tile,
//         TMEM rows 64..127 invalid)
//   dblk  first block of a diagonal tile (pair = dblk, dblk+1) needing element
//         causal masks, -1 otherwise
struct TileInfo {
    int16_t ke0, ve0, ve1, dblk;
};

// Shared-memory plan (bytes from the 1024-aligned base):
//   Q [128 q][128 d] (SW128, two 64-column atoms)            off_q
//   P^T buffers (n_pbuf x p_bytes; bf16 adds a residual half)  off_p
//   K ring (nk x k_stage): nnz or dense 128-key tile; sparse stages carry the
//          canonical metadata (+k_meta) and its TMEM-atom permutation (+k_e)
//   V ring (nv x v_stage): two 64-key V^T blocks of vblk bytes; metadata + E
//   tile list (TileInfo x tile_cap)
// K and V are separate rings: a K stage is recycled as soon as GEMM1 of its
// tile completes, a V stage after GEMM2, so neither waits for the other.
struct PrefillLayout {
    uint32_t off_q, off_p, p_bytes, n_pbuf;
    uint32_t off_k, k_stage, nk, k_meta, k_e;
    uint32_t off_v, v_stage, nv, vblk, v_meta, v_e;
    uint32_t off_tiles, tile_cap;
};

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Barrier over `n` threads of named barrier `id` that also ORs a predicate.
__device__ __forceinline__ bool bar_red_or(int id, bool v) {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
        "barrier.cta.red.or.pred p, %2, 128, q;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "r"(static_cast<uint32_t>(v)), "r"(id)
        : "memory");
    return r != 0;
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
        L.trace[t * 16 + ev] = clock64();
}

template <typename T, bool HILO>
__global__ void __launch_bounds__(kThreads, 1) prefill_kernel(const __grid_constant__ PrefillLaunch L,
                                                               PrefillLayout lay) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar_q, bar_kfull[4], bar_kmeta[4], bar_kempty[4];
    __shared__ __align__(8) uint64_t bar_vfull[4], bar_vmeta[4], bar_vempty[4];
    __shared__ __align__(8) uint64_t bar_sfull[2], bar_sempty[2], bar_pfull[2], bar_pempty[2];
    __shared__ uint32_t s_tmem;
    __shared__ int s_ntiles;
    __shared__ float s_red[4][128];
    __shared__ float s_mnew[128], s_alpha[128], s_mrun[128];

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
    const uint32_t sQ = base + lay.off_q, sP = base + lay.off_p;
    const uint32_t sK = base + lay.off_k, sV = base + lay.off_v;
    TileInfo* const s_tiles = reinterpret_cast<TileInfo*>(base_ptr + lay.off_tiles);
    const int nk = static_cast<int>(lay.nk), nv = static_cast<int>(lay.nv);

    // ------------------------------------------------------------ setup ----
    if (warp == 9) tmem_alloc(&s_tmem, 512);
    if (tid == 0) {
        mbar_init(&bar_q, 1);
        for (int s = 0; s < nk; ++s) {
            mbar_init(&bar_kfull[s], 1);
            mbar_init(&bar_kmeta[s], 1);
            mbar_init(&bar_kempty[s], 1);
        }
        for (int s = 0; s < nv; ++s) {
            mbar_init(&bar_vfull[s], 1);
            mbar_init(&bar_vmeta[s], 1);
            mbar_init(&bar_vempty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar_sfull[i], 1);
            mbar_init(&bar_sempty[i], 8);
            mbar_init(&bar_pfull[i], 8);
            mbar_init(&bar_pempty[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 8) {
        // Key-tile list (see header).  Block b is fully visible iff its last key
        // <= the tile's first query position; visible iff its first key <= the last.
        // The kind-grouped pairs are index arithmetic over the slot lists, so the
        // 32 lanes fill them in parallel; lane 0 appends the few odd/diagonal tiles.
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
        const int cap = static_cast<int>(lay.tile_cap);
        auto make = [&](int b0, int b1, int diag) {
            TileInfo ti;
            ti.ke0 = kidx[b0];
            ti.ve0 = vidx[b0];
            ti.ve1 = b1 >= 0 ? vidx[b1] : int16_t(0);
            ti.dblk = static_cast<int16_t>(diag ? b0 : -1);
            return ti;
        };
        const int nsp = ns >> 1, ndp = nd >> 1;
        for (int i = lane; i < nsp + ndp && i < cap; i += 32) {
            s_tiles[i] = i < nsp ? make(sparse_blocks[2 * i], sparse_blocks[2 * i + 1], 0)
                                 : make(sb[2 * (i - nsp)], sb[2 * (i - nsp) + 1], 0);
        }
        if (lane == 0) {
            int n = nsp + ndp;
            auto push = [&](int b0, int b1, int diag) {
                if (n < cap) s_tiles[n] = make(b0, b1, diag);
                ++n;
            };
            if (ns & 1) push(sparse_blocks[ns - 1], -1, 0);
            if (nd & 1) push(sb[nd - 1], -1, 0);
            for (int b = fv_end; b < vis_end; ++b) {
                const int kd = kidx[b] > 0;
                if (b + 1 < vis_end && (kidx[b + 1] > 0) == kd) {
                    push(b, b + 1, 1);
                    ++b;
                } else {
                    push(b, -1, 1);
                }
            }
            s_ntiles = min(n, cap);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    // P^T buffers: tile t uses buffer t % npb; its barrier phase is (t / npb) & 1.
    const int npb = static_cast<int>(lay.n_pbuf);
    auto pbuf_of = [npb](int t) { return npb == 2 ? (t & 1) : 0; };
    auto pphase = [npb](int t) { return static_cast<uint32_t>((npb == 2 ? (t >> 1) : t) & 1); };
    const int ntiles = s_ntiles;
    // TMEM columns: S[0] 0..127, S[1] 128..255, O 256..383, E_K[2] 384.., E_V[2] 392..
    const uint32_t tS0 = tmem, tO = tmem + 256, tEK = tmem + 384, tEV = tmem + 392;

    const int warp_u = warp_id_uniform();
    // Values read from smem are per-thread registers to the compiler; broadcasting
    // them from lane 0 makes them provably warp-uniform, so the descriptor / TMA
    // arithmetic below stays in uniform registers and the single-thread
    // tcgen05 / TMA instructions issue without R2UR waterfall loops.
    auto uni = [](int v) { return __shfl_sync(0xffffffffu, v, 0); };
    // Canonical 2-bit metadata rows -> tcgen05 TMEM metadata atom.  E atom u16
    // index for (row m, word w): 8(m&7) + ((m>>3)&1) + 128(m>>4) + 64(w&1) +
    // 2(w>>1) (+4 for the second V block); rows m and m+8 are adjacent u16s, so
    // each store writes a (row m, row m+8) pair.
    auto permute_k_meta = [&](const uint8_t* meta, uint8_t* e, bool single) {
        for (int pidx = lane; pidx < 64; pidx += 32) {  // row pairs (m, m+8)
            const int m = (pidx & 7) + 16 * (pidx >> 3);
            uint4 lo4 = make_uint4(0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
            uint4 hi4 = lo4;
            if (!(single && m >= 64)) {
                lo4 = *reinterpret_cast<const uint4*>(meta + m * 16);
                hi4 = *reinterpret_cast<const uint4*>(meta + (m + 8) * 16);
            }
            const uint32_t lw[4] = {lo4.x, lo4.y, lo4.z, lo4.w}, hw[4] = {hi4.x, hi4.y, hi4.z, hi4.w};
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const uint32_t a = (lw[w >> 1] >> (16 * (w & 1))) & 0xFFFF;
                const uint32_t b = (hw[w >> 1] >> (16 * (w & 1))) & 0xFFFF;
                const int idx = 8 * (m & 7) + 128 * (m >> 4) + 64 * (w & 1) + 2 * (w >> 1);
                *reinterpret_cast<uint32_t*>(reinterpret_cast<uint16_t*>(e) + idx) = a | (b << 16);
            }
        }
    };
    auto permute_v_meta = [&](const uint8_t* meta, uint8_t* e, int i) {
        for (int pidx = lane; pidx < 64; pidx += 32) {
            const int m = (pidx & 7) + 16 * (pidx >> 3);
            const uint2 lo2 = *reinterpret_cast<const uint2*>(meta + 1024 * i + m * 8);
            const uint2 hi2 = *reinterpret_cast<const uint2*>(meta + 1024 * i + (m + 8) * 8);
            const uint32_t lw[2] = {lo2.x, lo2.y}, hw[2] = {hi2.x, hi2.y};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const uint32_t a = (lw[w >> 1] >> (16 * (w & 1))) & 0xFFFF;
                const uint32_t b = (hw[w >> 1] >> (16 * (w & 1))) & 0xFFFF;
                const int idx = 8 * (m & 7) + 128 * (m >> 4) + 64 * (w & 1) + 2 * (w >> 1) + 4 * i;
                *reinterpret_cast<uint32_t*>(reinterpret_cast<uint16_t*>(e) + idx) = a | (b << 16);
            }
        }
    };
    if (warp_u == 8) {
        // ------------------------------------------- K producer + K metadata
        // Issue K(t), then permute the metadata of K(t-1) (one tile behind, so the
        // TMA of the next tile is in flight while this warp waits for a landing;
        // with a single stage K(t+1) needs K(t) consumed, so no lag).
        const int lag = nk >= 2 ? 1 : 0;
        if (elect_one()) {
            prefetch_tmap(&L.tm_q);
            prefetch_tmap(&L.tm_knnz);
            prefetch_tmap(&L.tm_kden);
            const int qrow = (u * L.gqa + h) * L.n_q + q0;
            mbar_arrive_expect_tx(&bar_q, 32768);
            tma_tile_g2s(base_ptr + lay.off_q, &L.tm_q, 0, qrow, &bar_q);
            tma_tile_g2s(base_ptr + lay.off_q + 16384, &L.tm_q, 64, qrow, &bar_q);
        }
        __syncwarp();
        auto meta_of = [&](int t) {
            const int s = t % nk;
            mbar_wait_dbg(&bar_kfull[s], (t / nk) & 1, L.dbg, 2);
            const TileInfo ti = s_tiles[t];
            if (ti.ke0 < 0) {
                uint8_t* st = base_ptr + lay.off_k + s * lay.k_stage;
                permute_k_meta(st + lay.k_meta, st + lay.k_e, ti.ve1 == 0);
                fence_async_smem();
            }
            __syncwarp();
            if (lane == 0) {
                trace(L, t, 8);
                mbar_arrive(&bar_kmeta[s]);
            }
        };
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % nk;
            const TileInfo ti = s_tiles[t];
            const int ke0 = uni(ti.ke0), two = uni(ti.ve1 != 0);
            mbar_wait_dbg(&bar_kempty[s], ((t / nk) & 1) ^ 1, L.dbg, 4);
            if (lane == 0) trace(L, t, 7);
            if (elect_one()) {
                uint8_t* st = base_ptr + lay.off_k + s * lay.k_stage;
                // both blocks (consecutive slots) in one 128-row box per column half
                if (ke0 > 0) {
                    mbar_arrive_expect_tx(&bar_kfull[s], 32768u);
                    const int row = (u * L.k_dense_count + ke0 - 1) * kBlock;
                    tma_tile_g2s(st, &L.tm_kden, 0, row, &bar_kfull[s]);
                    tma_tile_g2s(st + 16384, &L.tm_kden, 64, row, &bar_kfull[s]);
                } else {
                    mbar_arrive_expect_tx(&bar_kfull[s], 16384u + 1024u * (1 + two));
                    const int sbk = u * L.k_sparse_count + (-ke0 - 1);
                    tma_tile_g2s(st, &L.tm_knnz, 0, sbk * kBlock, &bar_kfull[s]);
                    tma_bulk_g2s(st + lay.k_meta, L.k_meta + static_cast<int64_t>(sbk) * 512, 1024 * (1 + two),
                                 &bar_kfull[s]);
                }
            }
            __syncwarp();
            if (t >= lag) meta_of(t - lag);
        }
        for (int t = max(0, ntiles - lag); t < ntiles; ++t) meta_of(t);
    } else if (warp_u == 10) {
        // ------------------------------------------- V producer + V metadata
        const int lag = nv >= 2 ? 1 : 0;
        if (elect_one()) {
            prefetch_tmap(&L.tm_vnnz);
            prefetch_tmap(&L.tm_vden);
        }
        __syncwarp();
        auto meta_of = [&](int t) {
            const int s = t % nv;
            mbar_wait_dbg(&bar_vfull[s], (t / nv) & 1, L.dbg, 2);
            const TileInfo ti = s_tiles[t];
            uint8_t* st = base_ptr + lay.off_v + s * lay.v_stage;
            bool any = false;
            if (ti.ve0 < 0) { permute_v_meta(st + lay.v_meta, st + lay.v_e, 0); any = true; }
            if (ti.ve1 < 0) { permute_v_meta(st + lay.v_meta, st + lay.v_e, 1); any = true; }
            if (any) fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_vmeta[s]);
        };
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % nv;
            const TileInfo ti = s_tiles[t];
            const int ve0 = uni(ti.ve0), ve1 = uni(ti.ve1);
            mbar_wait_dbg(&bar_vempty[s], ((t / nv) & 1) ^ 1, L.dbg, 4);
            if (elect_one()) {
                uint8_t* st = base_ptr + lay.off_v + s * lay.v_stage;
                const int nb_t = ve1 != 0 ? 2 : 1;
                uint32_t bytes = ve0 > 0 ? 16384u : 9216u;
                if (nb_t == 2) bytes += ve1 > 0 ? 16384u : 9216u;
                mbar_arrive_expect_tx(&bar_vfull[s], bytes);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int ve = i == 0 ? ve0 : ve1;
                    if (i == 1 && nb_t == 1) break;
                    if (ve > 0) {
                        const int row = (u * L.v_dense_count + ve - 1) * kHeadDim;
                        tma_tile_g2s(st + lay.vblk * i, &L.tm_vden, 0, row, &bar_vfull[s]);
                    } else {
                        const int sbv = u * L.v_sparse_count + (-ve - 1);
                        tma_tile_g2s(st + lay.vblk * i, &L.tm_vnnz, 0, sbv * kHeadDim, &bar_vfull[s]);
                        tma_bulk_g2s(st + lay.v_meta + 1024 * i, L.v_meta + static_cast<int64_t>(sbv) * 512, 1024,
                                     &bar_vfull[s]);
                    }
                }
            }
            __syncwarp();
            if (t >= lag) meta_of(t - lag);
        }
        for (int t = max(0, ntiles - lag); t < ntiles; ++t) meta_of(t);
    } else if (warp_u == 9) {
        // ------------------------------------------------------- MMA issuer
        const bool bf = std::is_same<T, __nv_bfloat16>::value;
        const uint32_t id_g1_sp = umma_idesc_f16(bf, 128, 128, false, false, true);
        const uint32_t id_g1_de = umma_idesc_f16(bf, 128, 128, false, false, false);
        const uint32_t id_g2_sp = umma_idesc_f16(bf, 128, 128, false, true, true);
        const uint32_t id_g2_de = umma_idesc_f16(bf, 128, 128, false, true, false);
        mbar_wait_dbg(&bar_q, 0, L.dbg, 1);
        tc_fence_after();
        // Descriptor bases (start address in 16-byte units in the low 14 bits:
        // adding (bytes >> 4) advances the start address).
        const uint64_t dQ = umma_desc(sQ, 16, 1024, kLayoutSW128);
        const uint64_t dK = umma_desc(sK, 16, 1024, kLayoutSW128);
        const uint64_t dVden = umma_desc(sV, 16, 1024, kLayoutSW128);
        const uint64_t dVsp = umma_desc(sV, 16, 512, kLayoutSW64);
        const uint64_t dP = umma_desc(sP, 16384, 1024, kLayoutSW128);
        const uint64_t dEK = umma_desc(sK + lay.k_e, 16, 128, kLayoutNone);
        const uint64_t dEV = umma_desc(sV + lay.v_e, 16, 128, kLayoutNone);
        const uint32_t kst16 = lay.k_stage >> 4, vst16 = lay.v_stage >> 4, vblk16 = lay.vblk >> 4;
        bool o_started = false;
        auto gemm2 = [&](int tp) {
            // O^T += V^T (tile tp) * P^T ; P^T in smem (hi, then lo for bf16)
            const int s = tp % nv;
            const TileInfo ti = s_tiles[tp];
            const int ve0 = uni(ti.ve0), ve1 = uni(ti.ve1);
            mbar_wait_dbg(&bar_vmeta[s], (tp / nv) & 1, L.dbg, 3);
            mbar_wait_dbg(&bar_pfull[pbuf_of(tp)], pphase(tp), L.dbg, 7);
            tc_fence_after();
            if (lane == 0) trace(L, tp, 5);
            if (elect_one()) {
                const int nb_t = (L.mode & 2) ? 0 : ve1 != 0 ? 2 : 1;
                const uint64_t so = static_cast<uint64_t>(s) * vst16;
                if (ve0 < 0 || ve1 < 0) tmem_cp_128x128b(tEV + 4 * (tp & 1), dEV + so);
#pragma unroll
                for (int pass = 0; pass < (HILO ? 2 : 1); ++pass) {
                    for (int i = 0; i < nb_t; ++i) {
                        const bool vdense = (i == 0 ? ve0 : ve1) > 0;
                        const uint64_t pb = dP + (pbuf_of(tp) * lay.p_bytes + pass * 32768 + 8192 * i) / 16;
                        if (vdense) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                umma_f16(tO, dVden + so + i * vblk16 + 2 * kk, pb + 128 * kk, id_g2_de, o_started);
                                o_started = true;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                umma_sp_f16(tO, dVsp + so + i * vblk16 + 2 * j, pb + 256 * j,
                                            tEV + 4 * (tp & 1) + 2 * i + j, id_g2_sp, o_started);
                                o_started = true;
                            }
                        }
                    }
                }
                umma_commit(&bar_pempty[pbuf_of(tp)]);  // P^T buffer free; O^T through tile tp final
                umma_commit(&bar_vempty[s]);            // V stage can be refilled
            }
            __syncwarp();
            o_started = true;
            if (lane == 0) trace(L, tp, 6);
        };
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % nk, sb = t & 1;
            const TileInfo ti = s_tiles[t];
            const int ke0 = uni(ti.ke0);
            if (lane == 0) trace(L, t, 11);
            mbar_wait_dbg(&bar_kmeta[s], (t / nk) & 1, L.dbg, 3);  // K landed (+ metadata permuted)
            if (lane == 0) trace(L, t, 10);
            if (t >= 2) mbar_wait_dbg(&bar_sempty[sb], ((t >> 1) - 1) & 1, L.dbg, 6);
            tc_fence_after();
            if (lane == 0) trace(L, t, 4);
            if (elect_one()) {
                const uint64_t so = static_cast<uint64_t>(s) * kst16;
                // metadata -> TMEM (ordered before the MMAs that read it)
                if (ke0 < 0) tmem_cp_128x128b(tEK + 4 * sb, dEK + so);
                // GEMM1: S^T[sb] = K_tile * Q^T
                const uint32_t tS = tS0 + 128 * sb;
                if (L.mode & 2) {
                } else if (ke0 > 0) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        umma_f16(tS, dK + so + (j >> 2) * 1024 + 2 * (j & 3), dQ + (j >> 2) * 1024 + 2 * (j & 3),
                                 id_g1_de, j > 0);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        umma_sp_f16(tS, dK + so + 2 * j, dQ + (j >> 1) * 1024 + 4 * (j & 1), tEK + 4 * sb + j,
                                    id_g1_sp, j > 0);
                }
                umma_commit(&bar_sfull[sb]);
                umma_commit(&bar_kempty[s]);  // K stage can be refilled once GEMM1(t) read it
            }
            __syncwarp();
            if (t >= 1) gemm2(t - 1);
        }
        if (ntiles > 0) gemm2(ntiles - 1);
    } else {
        // ------------------------------------------------------- softmax WGs
        // S^T is read from TMEM once per tile and released at once (GEMM1(t+2) may
        // reuse the buffer).  The running column max m lives in smem; in steady
        // state a tile needs no cross-lane reduction at all: every thread checks
        // x = s*scale*log2e - m <= tau for its own values, and one bar.red.or per
        // warpgroup confirms it (P <= 2^tau fits fp16).  Only when some column grows
        // past m + tau (first visible tile, rare later) the slow path computes the
        // exact column max (redux.f32 + smem), updates m and rescales O^T and l.
        const int wg = warp >> 2, wq = warp & 3;
        const int r = 32 * wq + lane;  // TMEM lane = key row of the tile = d row of O^T
        const int cbase = 64 * wg;     // this warpgroup's query columns
        const int bar_id = 1 + wg;
        const uint32_t lane_off = static_cast<uint32_t>(32 * wq) << 16;
        float l_part[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) l_part[c] = 0.f;
        if (r < 64) s_mrun[cbase + r] = -INFINITY;
        named_bar(bar_id, 128);
        uint8_t* const pbuf0 = base_ptr + lay.off_p;
        const float sl2 = L.scale_log2;
        for (int t = 0; t < ntiles; ++t) {
            const int sb = t & 1;
            const TileInfo ti = s_tiles[t];
            mbar_wait_dbg(&bar_sfull[sb], (t >> 1) & 1, L.dbg, 5);
            tc_fence_after();
            if (tid == 0) trace(L, t, 0);
            if (L.mode & 1) {  // tools: pipeline without the softmax
                if (t >= npb) mbar_wait_dbg(&bar_pempty[pbuf_of(t)], pphase(t - npb), L.dbg, 8);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&bar_sempty[sb]);
                    mbar_arrive(&bar_pfull[pbuf_of(t)]);
                }
                continue;
            }
            // masks: invalid rows of single-block tiles; causal (attention.hpp:181-190)
            const bool row_valid = r < 64 || ti.ve1 != 0;
            const int key_pos = ti.dblk * kBlock + r;  // diagonal pairs are consecutive blocks
            // column c (query q0 + c at position off + q0 + c) sees this key iff c >= c_first
            const int c_first = row_valid ? (ti.dblk >= 0 ? key_pos - off - q0 : 0) : 1 << 30;
            // The warpgroup's 64 columns are processed as two 32-column halves
            // (32 score registers live at a time next to the 64 partial sums).
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int c0 = cbase + 32 * hf;  // first column of this half
                const uint32_t tS = tS0 + 128 * sb + lane_off + c0;
                // warp-uniform fast path: every (row, column) of this warp visible
                const bool fast = __all_sync(0xffffffffu, c_first <= c0);
                float x[32];
                auto load_s = [&]() {
                    uint32_t v[32];
                    tmem_ld32(tS, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 32; ++k) x[k] = __uint_as_float(v[k]);
                };
                load_s();
                // x <- s*scale*log2e - m (masked: -inf); does any value exceed m + tau?
#pragma unroll
                for (int k = 0; k < 32; k += 4) {
                    const float4 m4 = *reinterpret_cast<const float4*>(&s_mrun[c0 + k]);
                    x[k] = fmaf(x[k], sl2, -m4.x);
                    x[k + 1] = fmaf(x[k + 1], sl2, -m4.y);
                    x[k + 2] = fmaf(x[k + 2], sl2, -m4.z);
                    x[k + 3] = fmaf(x[k + 3], sl2, -m4.w);
                }
                if (!fast) {
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        if (c0 + k < c_first) x[k] = -INFINITY;
                }
                float xmax = -INFINITY;
#pragma unroll
                for (int k = 0; k < 32; k += 4)
                    xmax = fmaxf(fmaxf(xmax, fmaxf(x[k], x[k + 1])), fmaxf(x[k + 2], x[k + 3]));
                if (bar_red_or(bar_id, !(xmax <= kTau))) {
                    // ---- slow path: exact column max of this half-tile, update m (lazy
                    // rule).  (!(xmax <= tau) also catches a NaN from m = -inf.)
                    load_s();
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const bool vis = fast || c0 + k >= c_first;
                        x[k] = vis ? x[k] * sl2 : -INFINITY;  // s*scale*log2e (scale > 0 commutes with max)
                        s_red[wq][c0 + k] = redux_max(x[k]);
                    }
                    named_bar(bar_id, 128);
                    bool resc = false;
                    if (r < 32) {
                        const int c = c0 + r;
                        const float tm = fmaxf(fmaxf(s_red[0][c], s_red[1][c]), fmaxf(s_red[2][c], s_red[3][c]));
                        const float mo = s_mrun[c];
                        float mnew = mo, alpha = 1.f;
                        if (tm > -INFINITY && (mo == -INFINITY || tm > mo + kTau)) {
                            mnew = tm;
                            if (mo != -INFINITY) {
                                alpha = fast_exp2(mo - mnew);
                                resc = true;
                            }
                        }
                        s_mnew[c] = mnew;
                        s_alpha[c] = alpha;
                    }
                    resc = bar_red_or(bar_id, resc);
                    if (r < 32) s_mrun[c0 + r] = s_mnew[c0 + r];
                    // x <- x - m_new (masked stay -inf; columns with no visible key yet stay -inf)
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const float mn = s_mnew[c0 + k];
                        x[k] = mn == -INFINITY ? -INFINITY : x[k] - mn;
                    }
                    if (resc) {
                        // O^T (GEMM2(t-1) complete) and l rescale for the grown columns
                        if (t >= 1) mbar_wait_dbg(&bar_pempty[pbuf_of(t - 1)], pphase(t - 1), L.dbg, 8);
                        tc_fence_after();
#pragma unroll
                        for (int k = 0; k < 32; ++k) l_part[32 * hf + k] *= s_alpha[c0 + k];
                        if (t >= 1) {
                            uint32_t v[32];
                            tmem_ld32(tO + lane_off + c0, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                v[k] = __float_as_uint(__uint_as_float(v[k]) * s_alpha[c0 + k]);
#pragma unroll
                            for (int k = 0; k < 32; k += 4)
                                tmem_st4(tO + lane_off + c0 + k, v[k], v[k + 1], v[k + 2], v[k + 3]);
                            tmem_st_wait();
                        }
                    }
                    named_bar(bar_id, 128);  // s_mnew / s_alpha reads done before the next slow path
                }
                if (hf == 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bar_sempty[sb]);  // this warp is done with S^T[sb]
                }
                if (tid == 0) trace(L, t, 1);
                // P^T buffer free + O^T stable (GEMM2(t-1) complete)
                if (hf == 0 && t >= npb) mbar_wait_dbg(&bar_pempty[pbuf_of(t)], pphase(t - npb), L.dbg, 8);
                if (tid == 0) trace(L, t, 2);
                // probabilities, partial column sums, P^T (+ residual for bf16)
#pragma unroll
                for (int g8 = 0; g8 < 4; ++g8) {
                    const int q8 = (c0 >> 3) + g8;  // 8-query chunk index in 0..15
                    float p[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        p[k] = fast_exp2(x[8 * g8 + k]);  // exp2(-inf) = 0
                        l_part[32 * hf + 8 * g8 + k] += p[k];
                    }
                    const uint4 hi = make_uint4(F16Traits<T>::pack(p[0], p[1]), F16Traits<T>::pack(p[2], p[3]),
                                                F16Traits<T>::pack(p[4], p[5]), F16Traits<T>::pack(p[6], p[7]));
                    uint8_t* const pbuf = pbuf0 + pbuf_of(t) * lay.p_bytes;
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
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_pfull[pbuf_of(t)]);
        }
        // ---------------------------------------------------- epilogue ----
        if (ntiles > 0) mbar_wait_dbg(&bar_pempty[pbuf_of(ntiles - 1)], pphase(ntiles - 1), L.dbg, 8);
        tc_fence_after();
        // l[c] = sum over the 128 key lanes of l_part[c]: transpose through smem
        float* s_l = reinterpret_cast<float*>(base_ptr + lay.off_k) + wg * (128 * 65);
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

int prefill_tile_cap(int nb) { return nb / 2 + 8; }

cudaError_t launch_prefill(const PrefillLaunch& L, cudaStream_t s) {
    PrefillLayout lay;
    const bool hilo = L.bf16;
    // K stage: dense 128x128 tile, or 128x64 nnz + 2 KB metadata + 2 KB E atom.
    const bool kden = L.k_dense_count > 0, vden = L.v_dense_count > 0;
    lay.k_meta = 16384u;
    lay.k_e = 18432u;
    lay.k_stage = kden ? 32768u : 20480u;
    // V stage: two V^T blocks (dense 128x64 or nnz 128x32) + 2 KB metadata + 2 KB E.
    lay.vblk = vden ? 16384u : 9216u;
    lay.v_meta = 2 * lay.vblk;
    lay.v_e = lay.v_meta + 2048u;
    lay.v_stage = lay.v_e + 2048u;
    lay.tile_cap = static_cast<uint32_t>(prefill_tile_cap(L.nb));
    const uint32_t tiles_bytes = (lay.tile_cap * sizeof(TileInfo) + 1023u) & ~1023u;
    lay.off_q = 0;
    lay.off_p = 32768;
    lay.p_bytes = hilo ? 65536u : 32768u;  // P^T (hi [+ lo]) per buffer
    const uint32_t budget = 227u * 1024u - 8192u /*static smem*/ - 1024u /*align*/ - tiles_bytes;
    // Preference order: 2 K + 2 V stages with two P^T buffers, then fewer P^T
    // buffers, then shallower rings.
    const uint32_t plans[][3] = {{2, 3, 3}, {2, 2, 3}, {2, 3, 2}, {2, 2, 2}, {1, 2, 2}, {2, 2, 1}, {2, 1, 2},
                                 {1, 2, 1}, {1, 1, 2}, {1, 1, 1}};
    bool ok = false;
    for (const auto& pl : plans) {
        const uint32_t need = 32768u + pl[0] * lay.p_bytes + pl[1] * lay.k_stage + pl[2] * lay.v_stage;
        if (need <= budget) {
            lay.n_pbuf = pl[0];
            lay.nk = pl[1];
            lay.nv = pl[2];
            ok = true;
            break;
        }
    }
    if (!ok) return cudaErrorInvalidConfiguration;
    if (const char* env = getenv("HS_PREFILL_PLAN")) {  // tools: "pbuf,nk,nv"
        unsigned a, b, c;
        if (sscanf(env, "%u,%u,%u", &a, &b, &c) == 3) {
            lay.n_pbuf = a;
            lay.nk = b;
            lay.nv = c;
        }
    }
    lay.off_k = lay.off_p + lay.n_pbuf * lay.p_bytes;
    lay.off_v = lay.off_k + lay.nk * lay.k_stage;
    lay.off_tiles = lay.off_v + lay.nv * lay.v_stage;
    size_t smem = lay.off_tiles + tiles_bytes + 1024;
    const size_t epi = lay.off_k + 2 * 128 * 65 * 4 + 1024;
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
