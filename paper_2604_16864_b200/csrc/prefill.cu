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
// Warp roles (608 threads, 19 warps, 96 registers):
//   0-15 softmax.  fp16 (ping-pong): two 8-warp groups take alternate tiles
//        (group g: S^T buffer g, P^T buffer g, GEMM1 bias operand g); warp
//        (g, wq, ch) covers key lanes 32 wq.. and query columns 64 ch..; row sums
//        l come from the tensor core.  bf16 (lockstep): 4 warpgroups of 32 query
//        columns work on every tile, l in registers.  Both: the running max is
//        folded into GEMM1 as a rank-1 bias MMA (x = S^T * scale log2e), a tile
//        needs no cross-lane reduction unless a column grows past m + tau
//        (FA4-style lazy rescale), P^T is written to smem (MN-major SW128) for
//        GEMM2, a quarter of the exponentials can run on the FMA pipe.
//   16   TMA producer: tile list, Q once, K tiles (3-D box for dense) and V
//        tiles (256-row box for consecutive slots) with prepared metadata atoms.
//   17   GEMM1 issuer: tcgen05.cp metadata -> TMEM, bias MMA + K Q^T (mma.sp for
//        2:4 tiles); TMEM owner.
//   18   GEMM2 issuer: O^T += V^T P^T (+ the l MMA P^T x ones in ping-pong mode).
// See DESIGN.md section 3.3 for the measured bounds and the rejected variants.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace hs {
namespace {

#ifndef HS_PREFILL_WG
#define HS_PREFILL_WG 4
#endif
constexpr int kSoftWG = HS_PREFILL_WG;     // lockstep softmax warpgroups (each owns kCols query columns)
constexpr int kCols = 128 / kSoftWG;       // query columns per softmax thread
constexpr int kSoftWarps = 4 * kSoftWG;
constexpr int kWarpK = kSoftWarps;         // TMA producer: tile list, Q and K tiles
constexpr int kWarpMma = kSoftWarps + 1;   // tcgen05 issuer of GEMM1 (S^T = K Q^T), TMEM owner
constexpr int kWarpMma2 = kSoftWarps + 2;  // tcgen05 issuer of GEMM2 (O^T += V^T P^T)
constexpr int kWarpV = kSoftWarps + 3;     // TMA producer: V tiles
// One warp issues a TMA operation every ~180 cycles at best (the mbarrier /
// address chain, tools/probes/tma_ops.cu), so each tile's loads are as few
// operations as the slot layout allows.  HS_PREFILL_SPLIT_PRODUCER moves the V
// loads to a 20th warp (measured 3% slower: the softmax, not the producer,
// bounds the full kernel, and the extra warp shares its SM sub-partition).
#ifndef HS_PREFILL_SPLIT_PRODUCER
constexpr int kThreads = 32 * (kSoftWarps + 3);
#else
constexpr int kThreads = 32 * (kSoftWarps + 4);
#endif

// Ping-pong softmax state (static shared memory of the PP instantiation).
struct __align__(16) PPShared {
    unsigned long long s_mcur[128];  // shared running max: orderable(m) << 32 | bias bits
    float s_red2[2][4][128];         // slow-path column maxima [group][lane quarter][column]
    float s_dl[2][128];              // slow path: m_t - m_used [group][column]
    float s_mt[2][2][128];           // m of a published tile [group][slot][column]
    float s_al[2][128];              // rescale factors exp2(m_{t-1} - m_t) [group][column]
    int s_ver[2];                    // m version per column half (bumped on growth)
    int s_vsnap[2][2];               // [group][half] version snapshot broadcast
    int s_tdone[2][2][2];            // last tile published per [group][slot][half]
};
struct PPNone {
    int unused;
};
#ifndef HS_PREFILL_G2FIRST
#define HS_PREFILL_G2FIRST 0  // measured: +1.5% at S=1, -2% at S=0 (64K); off
#endif
constexpr bool kG2First = HS_PREFILL_G2FIRST != 0;  // issue GEMM2(t-2) before GEMM1(t)
constexpr uint32_t kBiasBytes = 4 * 2048;  // ones + bias[2] GEMM1 operands + fp16 ones for the l MMA (16-byte rows)
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
    uint32_t off_bias;  // ones [128 x 16] + two bias operands [128 x 16] (16-byte rows, K halves aliased)
};

// Monotone float <-> uint32 map (for atomicMax on possibly negative floats).
__device__ __forceinline__ uint32_t ord_f32(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
    return __uint_as_float((o >> 31) ? (o & 0x7FFFFFFFu) : ~o);
}

// CTA-scope release / acquire on a shared-memory word (cross-warp ordering flags).
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// TMEM -> fp32 registers, 16 columns starting at taddr (the softmax's S^T halves).
__device__ __forceinline__ void tmem_ld16_f(uint32_t taddr, float* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]),
          "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11]), "=f"(r[12]), "=f"(r[13]), "=f"(r[14]), "=f"(r[15])
        : "r"(taddr));
}

// TMEM -> registers: this warp's 32 lanes x N consecutive 32-bit columns.
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]) {
    if constexpr (N == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    } else if constexpr (N == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else {
#pragma unroll
        for (int c = 0; c < N; c += 32) tmem_ld32(taddr + c, *reinterpret_cast<uint32_t(*)[32]>(&r[c]));
    }
}

// Blackwell packed fp32: (x0, x1) <- (x0, x1) * b + (c0, c1) in one FFMA2.
__device__ __forceinline__ void ffma2(float& x0, float& x1, float b, float c0, float c1) {
    asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %2};\n\t"
        "mov.b64 rc, {%3, %4};\n\tfma.rn.f32x2 ra, ra, rb, rc;\n\tmov.b64 {%0, %1}, ra;\n\t}"
        : "+f"(x0), "+f"(x1)
        : "f"(b), "f"(c0), "f"(c1));
}
// (a0, a1) += (b0, b1) in one FADD2.
__device__ __forceinline__ void fadd2(float& a0, float& a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
        "add.rn.f32x2 ra, ra, rb;\n\tmov.b64 {%0, %1}, ra;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "f"(b0), "f"(b1));
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// 2^x on the FMA pipe for x <= tau (+inf excluded, -inf -> 0): round-to-nearest
// split x = j + f (magic-number add), degree-5 minimax-style polynomial for 2^f on
// [-1/2, 1/2] (relative error ~2e-7, below fp16/bf16 P rounding), 2^j by an
// integer add into the exponent field.  Offloads the MUFU / MIO queue, which the
// exponentials otherwise saturate (ncu: MUFU.EX2 stalls on mio).
__device__ __forceinline__ float exp2_fma(float x) {
    x = fmaxf(x, -127.f);
    const float y = x + 12582912.f;  // 1.5 * 2^23: j in the low mantissa bits
    const float j = y - 12582912.f;
    const float f = x - j;
    float p = 1.3333558e-3f;
    p = fmaf(p, f, 9.6181291e-3f);
    p = fmaf(p, f, 5.5504109e-2f);
    p = fmaf(p, f, 2.4022651e-1f);
    p = fmaf(p, f, 6.9314718e-1f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(y) << 23));
}
// exp2_fma on a pair with packed f32x2 arithmetic (FADD2 / FFMA2): half the
// instructions of two scalar calls.
__device__ __forceinline__ void exp2_fma2(float& x0, float& x1) {
    x0 = fmaxf(x0, -127.f);
    x1 = fmaxf(x1, -127.f);
    float y0 = x0, y1 = x1;
    fadd2(y0, y1, 12582912.f, 12582912.f);    // 1.5 * 2^23: j in the low mantissa bits
    float j0 = y0, j1 = y1;
    fadd2(j0, j1, -12582912.f, -12582912.f);
    float f0 = x0, f1 = x1;
    fadd2(f0, f1, -j0, -j1);
    float p0 = f0, p1 = f1;
    ffma2(p0, p1, 1.3333558e-3f, 9.6181291e-3f, 9.6181291e-3f);  // (c5 f + c4)
    float q0 = p0, q1 = p1;
    // Horner: p <- p * f + c (f per lane): packed multiply by the pair f
    auto step = [&](float c) {
        asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
            "mov.b64 rc, {%4, %4};\n\tfma.rn.f32x2 ra, ra, rb, rc;\n\tmov.b64 {%0, %1}, ra;\n\t}"
            : "+f"(q0), "+f"(q1)
            : "f"(f0), "f"(f1), "f"(c));
    };
    (void)p0;
    (void)p1;
    step(5.5504109e-2f);
    step(2.4022651e-1f);
    step(6.9314718e-1f);
    step(1.0f);
    x0 = __int_as_float(__float_as_int(q0) + (__float_as_int(y0) << 23));
    x1 = __int_as_float(__float_as_int(q1) + (__float_as_int(y1) << 23));
}

#ifndef HS_PREFILL_POLY
#define HS_PREFILL_POLY 2  // of every 8 exponentials, this many run on the FMA pipe
#endif
constexpr int kPolyPer8 = HS_PREFILL_POLY;  // default for the lockstep softmax
static_assert(kPolyPer8 % 2 == 0, "polynomial exponentials run in packed pairs");

#ifndef HS_PREFILL_EXP_F16X2
#define HS_PREFILL_EXP_F16X2 0  // sm_100a splits f16x2 ex2 into two MUFU ops: no gain
#endif
constexpr bool kExpF16x2 = HS_PREFILL_EXP_F16X2 != 0;
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
    uint32_t r;
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
    return r;
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

// Canonical 2-bit metadata (nm_metadata.hpp:42-46: row m of a stored block has
// 8 (K) or 4 (V) u16 words) -> the tcgen05 TMEM metadata atom, so the prefill
// kernel copies it smem -> TMEM with tcgen05.cp and no per-tile shuffling.
// Atom u16 index of (row m, word w): 8(m&7) + ((m>>3)&1) + 128(m>>4) + 64(w&1)
// + 2(w>>1) (pinned by tools/probes/umma_probe.cu).  K: 1 KB per block (a pair
// of consecutive slots is the 2 KB atom of a 128-row tile).  V: 2 KB per block,
// 16-byte lane rows of which the first 8 bytes are used (one tcgen05.cp per
// block into its own 4-column group).
__global__ void __launch_bounds__(128) meta_atom_kernel(const uint16_t* __restrict__ k_meta, int k_blocks,
                                                        const uint16_t* __restrict__ v_meta, int v_blocks,
                                                        uint16_t* __restrict__ k_hw, uint16_t* __restrict__ v_hw) {
    const int b = blockIdx.x, m = threadIdx.x;  // one CTA per block, one thread per stored row
    auto idx = [](int m, int w) { return 8 * (m & 7) + ((m >> 3) & 1) + 128 * (m >> 4) + 64 * (w & 1) + 2 * (w >> 1); };
    if (b < k_blocks) {
        if (m < 64) {
            const uint4 row = *reinterpret_cast<const uint4*>(k_meta + static_cast<int64_t>(b) * 512 + m * 8);
            const uint32_t wd[4] = {row.x, row.y, row.z, row.w};
            uint16_t* dst = k_hw + static_cast<int64_t>(b) * 512;
#pragma unroll
            for (int w = 0; w < 8; ++w) dst[idx(m, w)] = static_cast<uint16_t>(wd[w >> 1] >> (16 * (w & 1)));
        }
    } else {
        const int vb = b - k_blocks;
        const uint2 row = *reinterpret_cast<const uint2*>(v_meta + static_cast<int64_t>(vb) * 512 + m * 4);
        const uint32_t wd[2] = {row.x, row.y};
        uint16_t* dst = v_hw + static_cast<int64_t>(vb) * 1024;
#pragma unroll
        for (int w = 0; w < 4; ++w) dst[idx(m, w)] = static_cast<uint16_t>(wd[w >> 1] >> (16 * (w & 1)));
        if (m < 64) *reinterpret_cast<uint2*>(dst + 16 * m + 4) = make_uint2(0u, 0u);  // unused halves of
        if (m < 64) *reinterpret_cast<uint2*>(dst + 16 * m + 12) = make_uint2(0u, 0u); // the 16-byte rows
    }
}

// The dense tail (attention.hpp:289-297) as extra dense blocks nb, nb+1, ...:
// K rows copied token-major ([B][d], the dense K block layout), V transposed to
// [d][B] (the dense V^T block layout), both zero padded to whole blocks.  One CTA
// per (tail block, unit); 128 threads = one token row (K) / one channel (V).
// bf16 magnitude bits -> fp16 bits of x * 2^-e (round to nearest even).
__device__ __forceinline__ uint16_t bf16_to_f16_scaled(uint16_t b, int e) {
    const float f = ldexpf(__uint_as_float(static_cast<uint32_t>(b) << 16), -e);
    return __half_as_ushort(__float2half_rn(f));
}

__global__ void __launch_bounds__(128) tail_prep_kernel(const uint16_t* __restrict__ k_tail,
                                                        const uint16_t* __restrict__ v_tail, int tail, int ntb,
                                                        uint16_t* __restrict__ k_ws, uint16_t* __restrict__ v_ws,
                                                        const int* __restrict__ v16_scale) {
    const int tb = blockIdx.x, u = blockIdx.y, c = threadIdx.x;
    const uint16_t* kt = k_tail + static_cast<int64_t>(u) * tail * kHeadDim;
    const uint16_t* vt = v_tail + static_cast<int64_t>(u) * tail * kHeadDim;
    uint16_t* kw = k_ws + (static_cast<int64_t>(u) * ntb + tb) * kBlock * kHeadDim;
    uint16_t* vw = v_ws + (static_cast<int64_t>(u) * ntb + tb) * kBlock * kHeadDim;
    const int e = v16_scale ? v16_scale[1] : 0;
    for (int i = 0; i < kBlock; ++i) {
        const int tok = tb * kBlock + i;
        const bool in = tok < tail;
        kw[i * kHeadDim + c] = in ? kt[static_cast<int64_t>(tok) * kHeadDim + c] : uint16_t(0);
        const uint16_t vb = in ? vt[static_cast<int64_t>(tok) * kHeadDim + c] : uint16_t(0);
        vw[c * kBlock + i] = v16_scale ? bf16_to_f16_scaled(vb, e) : vb;  // V^T of the tail (fp16 on the v16 path)
    }
}

// The v16 path's scale: the largest bf16 magnitude of the V pools and tail
// (integer order of the low 15 bits is magnitude order).
__global__ void __launch_bounds__(256) v16_absmax_kernel(const uint32_t* __restrict__ a, int64_t na,
                                                         const uint32_t* __restrict__ b, int64_t nb,
                                                         const uint16_t* __restrict__ tail, int64_t nt, int* scale) {
    uint32_t m = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < na + nb + nt; i += stride) {
        uint32_t w;
        if (i < na) w = a[i];
        else if (i < na + nb) w = b[i - na];
        else w = tail[i - na - nb];
        m = max(m, max(w & 0x7FFFu, (w >> 16) & 0x7FFFu));
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(reinterpret_cast<unsigned*>(scale), m);
}

// fp16 copy of the bf16 V pools scaled by 2^-e, e chosen so the largest magnitude
// lands in [2^14, 2^15): every value in fp16's normal range after scaling
// converts exactly (bf16 has 8 significant bits, fp16 11); values more than 2^28
// below the largest round at 2^-25 of it.  Inf / NaN: e = 0.
__global__ void __launch_bounds__(256) v16_convert_kernel(const uint32_t* __restrict__ a, uint32_t* __restrict__ a16,
                                                          int64_t na, const uint32_t* __restrict__ b,
                                                          uint32_t* __restrict__ b16, int64_t nb, int* scale) {
    const uint32_t mb = static_cast<uint32_t>(scale[0]);
    const int ex = static_cast<int>(mb >> 7);
    const int e = (mb == 0 || ex >= 0xFF) ? 0 : (ex == 0 ? -126 : ex - 127) - 14;
    if (blockIdx.x == 0 && threadIdx.x == 0) scale[1] = e;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < na + nb; i += stride) {
        const bool first = i < na;
        const uint32_t w = first ? a[i] : b[i - na];
        const uint32_t r = bf16_to_f16_scaled(static_cast<uint16_t>(w & 0xFFFFu), e) |
                           (static_cast<uint32_t>(bf16_to_f16_scaled(static_cast<uint16_t>(w >> 16), e)) << 16);
        if (first) a16[i] = r;
        else b16[i - na] = r;
    }
}

template <typename T, bool HILO, bool DBG, bool PP, int POLY = kPolyPer8, bool SAFE = false>
__global__ void __launch_bounds__(kThreads, 1) prefill_kernel(const __grid_constant__ PrefillLaunch L,
                                                               PrefillLayout lay) {
    // DBG: tools-only instrumentation (per-tile trace, watchdog waits, mode
    // switches); the production instantiation compiles all of it out.
    int* const dbgp = DBG ? L.dbg : nullptr;
    const int mode = DBG ? L.mode : 0;
    // bf16 caches on the ping-pong path: GEMM2 (and the l MMA) in fp16 over the
    // fp16 V^T copy, P^T in fp16 (PrefillLaunch::v16)
    constexpr bool V16 = PP && std::is_same<T, __nv_bfloat16>::value;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar_q, bar_kfull[4], bar_kempty[4];
    __shared__ __align__(8) uint64_t bar_vfull[4], bar_vempty[4];
    __shared__ __align__(8) uint64_t bar_sfull[2], bar_sempty[2], bar_pfull[2], bar_pempty[2];
    __shared__ uint32_t s_tmem;
    __shared__ int s_ntiles;
    // 16-byte aligned: per-column arrays are read as 4-wide vectors (a 4-byte shift of
    // this block once cost ~8% at S = 1 through scalarised shared accesses)
    __shared__ __align__(16) float s_red[4][128];
    __shared__ __align__(16) float s_delta[128];
    __shared__ __align__(16) float s_alpha[128];
    __shared__ __align__(16) float s_mrun[128];
    __shared__ __align__(16) float s_mused[2][128];
    __shared__ uint16_t s_bq[128];
    __shared__ int s_g2_issued;  // GEMM2 tiles issued (kG2First ordering)
    __shared__ typename std::conditional<PP, PPShared, PPNone>::type pps;  // ping-pong softmax state
    __shared__ int s_bad;        // ping-pong: some output row of this CTA came out non-finite

    if constexpr (SAFE) {  // only the CTAs the fast pass flagged
        if (L.redo[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] == 0) return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    // Columns: hg stacked query heads x QT queries (column c = head h0 + c / QT,
    // query q0 + c % QT; QT a power of two, QT * hg = 128)
    const int QT = L.qt, qmask = L.qt - 1, qshift = __ffs(L.qt) - 1;
    const int n_tiles_q = (L.n_q + QT - 1) / QT;
    const int qt = n_tiles_q - 1 - static_cast<int>(blockIdx.x);  // heaviest causal tiles first
    const int h0 = blockIdx.y * L.hg, u = blockIdx.z;
    const int q0 = qt * QT;
    const int n_kv = L.nb * kBlock + L.tail;  // blocked prefix + dense tail
    const int off = n_kv - L.n_q;
    const int rows_q = min(QT, L.n_q - q0);
    // output row of column c (valid iff (c & qmask) < rows_q)
    auto out_row = [&](int c) {
        return L.out + (static_cast<int64_t>(u * L.gqa + h0 + (c >> qshift)) * L.n_q + q0 + (c & qmask)) * kHeadDim;
    };

    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* const base_ptr = smem_raw + (base - raw);
    const uint32_t sQ = base + lay.off_q, sP = base + lay.off_p;
    const uint32_t sK = base + lay.off_k, sV = base + lay.off_v;
    TileInfo* const s_tiles = reinterpret_cast<TileInfo*>(base_ptr + lay.off_tiles);
    const int nk = static_cast<int>(lay.nk), nv = static_cast<int>(lay.nv);

    // ------------------------------------------------------------ setup ----
    if (warp == kWarpMma) tmem_alloc(&s_tmem, 512);
    if (tid == 0) {
        s_g2_issued = 0;
        s_bad = 0;
        mbar_init(&bar_q, 1);
        for (int s = 0; s < nk; ++s) {
            mbar_init(&bar_kfull[s], 1);
            mbar_init(&bar_kempty[s], 1);
        }
        for (int s = 0; s < nv; ++s) {
            mbar_init(&bar_vfull[s], 1);
            mbar_init(&bar_vempty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar_sfull[i], 1);
            mbar_init(&bar_sempty[i], PP ? kSoftWarps / 2 : kSoftWarps);  // PP: one 8-warp group per buffer
            mbar_init(&bar_pfull[i], PP ? kSoftWarps / 2 : kSoftWarps);
            mbar_init(&bar_pempty[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == kWarpK) {
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
            // dense tail blocks nb.. (dense K and V from the tail workspace; always masked)
            const int last_q = off + q0 + rows_q - 1;
            for (int tb = 0; tb < L.n_tail_blocks; tb += 2) {
                if (L.causal && (L.nb + tb) * kBlock > last_q) break;
                const bool pair = tb + 1 < L.n_tail_blocks && (!L.causal || (L.nb + tb + 1) * kBlock <= last_q);
                TileInfo ti;
                ti.ke0 = 1;
                ti.ve0 = 1;
                ti.ve1 = pair ? int16_t(1) : int16_t(0);
                ti.dblk = static_cast<int16_t>(L.nb + tb);
                if (n < cap) s_tiles[n] = ti;
                ++n;
            }
            s_ntiles = min(n, cap);
        }
    }
    if (warp < kSoftWarps) {
        // GEMM1 operands of the stabiliser term (see the softmax header): A = ones,
        // B[sb] row c = 8 copies of -m_c / (16 scale log2e) (m unset: 0).
        uint4* ob = reinterpret_cast<uint4*>(base_ptr + lay.off_bias);
        const uint32_t one = F16Traits<T>::pack(1.f, 1.f);
        const uint32_t one16 = F16Traits<__half>::pack(1.f, 1.f);  // the l MMA's B operand (fp16 P^T)
        for (int i = tid; i < (V16 ? 4 : 3) * 128; i += 32 * kSoftWarps)  // (fp16 ones: V16 only)
            ob[i] = i < 128 ? make_uint4(one, one, one, one)
                            : i >= 384 ? make_uint4(one16, one16, one16, one16) : make_uint4(0u, 0u, 0u, 0u);
        if (tid < 128) {
            s_mused[0][tid] = PP ? -INFINITY : 0.f;
            s_mused[1][tid] = PP ? -INFINITY : 0.f;
        }
        if constexpr (PP) {
            if (tid < 128) {
                pps.s_mcur[tid] = static_cast<unsigned long long>(ord_f32(-INFINITY)) << 32;
                pps.s_mt[0][0][tid] = pps.s_mt[0][1][tid] = pps.s_mt[1][0][tid] = pps.s_mt[1][1][tid] = -INFINITY;
            }
            if (tid < 8) (&pps.s_tdone[0][0][0])[tid] = -1;
            if (tid < 2) pps.s_ver[tid] = 0;
        }
        fence_async_smem();
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
    // TMEM columns: S[0] 0..127, S[1] 128..255, O 256..383, E_K[2] 384..391, E_V[2] 392..407
    const uint32_t tS0 = tmem, tO = tmem + 256, tEK = tmem + 384, tEV = tmem + 392;

    const int warp_u = warp_id_uniform();
    // Values read from smem are per-thread registers to the compiler; broadcasting
    // them from lane 0 makes them provably warp-uniform, so the descriptor / TMA
    // arithmetic below stays in uniform registers and the single-thread
    // tcgen05 / TMA instructions issue without R2UR waterfall loops.
    auto uni = [](int v) { return __shfl_sync(0xffffffffu, v, 0); };
#ifndef HS_PREFILL_SPLIT_PRODUCER
    if (warp_u == kWarpK) {
#else
    if (warp_u == kWarpK || warp_u == kWarpV) {
#endif
        // -------------------------------------------------------- producers
        if (warp_u == kWarpK && elect_one()) {
            prefetch_tmap(&L.tm_q);
            prefetch_tmap(&L.tm_knnz);
            prefetch_tmap(&L.tm_kden);
            mbar_arrive_expect_tx(&bar_q, 32768);  // [half][hg heads x QT queries][64]
            tma_tile4_g2s(base_ptr + lay.off_q, &L.tm_q, 0, q0, u * L.gqa + h0, 0, &bar_q);
        }
#ifndef HS_PREFILL_SPLIT_PRODUCER
        if (elect_one()) {
#else
        if (warp_u == kWarpV && elect_one()) {
#endif
            prefetch_tmap(&L.tm_vnnz);
            prefetch_tmap(&L.tm_vden);
            prefetch_tmap(&L.tm_vnnz2);
            prefetch_tmap(&L.tm_vden2);
        }
        __syncwarp();
        auto issue_k = [&](int t) {
            const int s = t % nk;
            const TileInfo ti = s_tiles[t];
            const int ke0 = uni(ti.ke0), two = uni(ti.ve1 != 0), dblk = uni(ti.dblk);
            mbar_wait_dbg(&bar_kempty[s], ((t / nk) & 1) ^ 1, dbgp, 4);
            if (DBG && lane == 0) trace(L, t, 7);
            if (elect_one()) {
                uint8_t* st = base_ptr + lay.off_k + s * lay.k_stage;
                // both blocks (consecutive slots) in one 128-row box per column half
                // dense: both 64-column halves in one 3-D box ([half][row][64])
                if (dblk >= L.nb) {  // dense tail blocks
                    mbar_arrive_expect_tx(&bar_kfull[s], 32768u);
                    const int row = (u * L.n_tail_blocks + dblk - L.nb) * kBlock;
                    tma_tile3_g2s(st, &L.tm_ktail, 0, row, 0, &bar_kfull[s]);
                } else if (ke0 > 0) {
                    mbar_arrive_expect_tx(&bar_kfull[s], 32768u);
                    const int row = (u * L.k_dense_count + ke0 - 1) * kBlock;
                    tma_tile3_g2s(st, &L.tm_kden, 0, row, 0, &bar_kfull[s]);
                } else {
                    mbar_arrive_expect_tx(&bar_kfull[s], 16384u + 1024u * (1 + two));
                    const int sbk = u * L.k_sparse_count + (-ke0 - 1);
                    tma_tile_g2s(st, &L.tm_knnz, 0, sbk * kBlock, &bar_kfull[s]);
                    tma_bulk_g2s(st + lay.k_e, L.k_meta_hw + static_cast<int64_t>(sbk) * 512, 1024 * (1 + two),
                                 &bar_kfull[s]);
                }
            }
            __syncwarp();
        };
        auto issue_v = [&](int t) {
            const int s = t % nv;
            const TileInfo ti = s_tiles[t];
            const int ve0 = uni(ti.ve0), ve1 = uni(ti.ve1), vdblk = uni(ti.dblk);
            mbar_wait_dbg(&bar_vempty[s], ((t / nv) & 1) ^ 1, dbgp, 4);
            if (elect_one()) {
                uint8_t* st = base_ptr + lay.off_v + s * lay.v_stage;
                const int nb_t = ve1 != 0 ? 2 : 1;
                uint32_t bytes = ve0 > 0 ? 16384u : 8192u + 2048u;
                if (nb_t == 2) bytes += ve1 > 0 ? 16384u : 8192u + 2048u;
                mbar_arrive_expect_tx(&bar_vfull[s], bytes);
                // two consecutive pool slots of one kind: one 256-row box (+ one 4 KB
                // metadata copy); otherwise one operation per block
                // (sparse pairs only when the stage holds nnz blocks back to back)
                if (nb_t == 2 && vdblk < L.nb && ve0 > 0 && ve1 == ve0 + 1) {
                    const int row = (u * L.v_dense_count + ve0 - 1) * kHeadDim;
                    tma_tile_g2s(st, &L.tm_vden2, 0, row, &bar_vfull[s]);
                } else if (nb_t == 2 && vdblk < L.nb && ve0 < 0 && ve1 == ve0 - 1 && lay.vblk == 8192u) {
                    const int sbv = u * L.v_sparse_count + (-ve0 - 1);
                    tma_tile_g2s(st, &L.tm_vnnz2, 0, sbv * kHeadDim, &bar_vfull[s]);
                    tma_bulk_g2s(st + lay.v_e, L.v_meta_hw + static_cast<int64_t>(sbv) * 1024, 4096, &bar_vfull[s]);
                } else
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int ve = i == 0 ? ve0 : ve1;
                    if (i == 1 && nb_t == 1) break;
                    if (vdblk >= L.nb) {  // dense tail block vdblk + i
                        const int row = (u * L.n_tail_blocks + vdblk - L.nb + i) * kHeadDim;
                        tma_tile_g2s(st + lay.vblk * i, &L.tm_vtail, 0, row, &bar_vfull[s]);
                    } else if (ve > 0) {
                        const int row = (u * L.v_dense_count + ve - 1) * kHeadDim;
                        tma_tile_g2s(st + lay.vblk * i, &L.tm_vden, 0, row, &bar_vfull[s]);
                    } else {
                        const int sbv = u * L.v_sparse_count + (-ve - 1);
                        tma_tile_g2s(st + lay.vblk * i, &L.tm_vnnz, 0, sbv * kHeadDim, &bar_vfull[s]);
                        tma_bulk_g2s(st + lay.v_e + 2048 * i, L.v_meta_hw + static_cast<int64_t>(sbv) * 1024, 2048,
                                     &bar_vfull[s]);
                    }
                }
            }
            __syncwarp();
        };
#ifndef HS_PREFILL_SPLIT_PRODUCER
        for (int t = 0; t < ntiles; ++t) {
            issue_k(t);
            if (t >= 1) issue_v(t - 1);
        }
        if (ntiles > 0) issue_v(ntiles - 1);
#else
        if (warp_u == kWarpK) {
            for (int t = 0; t < ntiles; ++t) issue_k(t);
        } else {
            for (int t = 0; t < ntiles; ++t) issue_v(t);
        }
#endif
    } else if (warp_u == kWarpMma || warp_u == kWarpMma2) {
        // ------------------------------------------------------ MMA issuers
        // kWarpMma issues GEMM1 (S^T = K Q^T) per tile, kWarpMma2 GEMM2
        // (O^T += V^T P^T): the two chains wait on different barriers (K / S
        // buffer vs V / P^T), so neither stalls the other's issue.  Each
        // tcgen05.commit tracks the MMAs of its own thread only.
        const bool bf = std::is_same<T, __nv_bfloat16>::value;
        const bool bf2 = bf && !V16;  // GEMM2 / l MMA format (fp16 on the v16 path)
        const uint32_t id_g1_sp = umma_idesc_f16(bf, 128, 128, false, false, true);
        const uint32_t id_g1_de = umma_idesc_f16(bf, 128, 128, false, false, false);
        const uint32_t id_g2_sp = umma_idesc_f16(bf2, 128, 128, false, true, true);
        const uint32_t id_g2_de = umma_idesc_f16(bf2, 128, 128, false, true, false);
        mbar_wait_dbg(&bar_q, 0, dbgp, 1);
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
        // ones / bias operands: K-major, no swizzle, 16-byte rows (SBO 128 B per 8
        // rows); LBO 0 aliases the two 8-element K halves (the rows are constant)
        const uint32_t sBias = base + lay.off_bias;
        const uint64_t dOnes = umma_desc(sBias, 0, 128, kLayoutNone);
        const uint64_t dOnesL = V16 ? umma_desc(sBias + 3 * 2048, 0, 128, kLayoutNone) : dOnes;  // l MMA ones
        const uint64_t dBias = umma_desc(sBias + 2048, 0, 128, kLayoutNone);
        const uint32_t kst16 = lay.k_stage >> 4, vst16 = lay.v_stage >> 4, vblk16 = lay.vblk >> 4;
        bool o_started = false;
        auto gemm2 = [&](int tp) {
            // O^T += V^T (tile tp) * P^T ; P^T in smem (hi, then lo for bf16)
            const int s = tp % nv;
            const TileInfo ti = s_tiles[tp];
            const int ve0 = uni(ti.ve0), ve1 = uni(ti.ve1);
            mbar_wait_dbg(&bar_vfull[s], (tp / nv) & 1, dbgp, 3);
            mbar_wait_dbg(&bar_pfull[pbuf_of(tp)], pphase(tp), dbgp, 7);
            tc_fence_after();
            if (DBG && lane == 0) trace(L, tp, 5);
            if (elect_one()) {
                const int nb_t = (mode & 2) ? 0 : ve1 != 0 ? 2 : 1;
                const uint64_t so = static_cast<uint64_t>(s) * vst16;
                if (ve0 < 0) tmem_cp_128x128b(tEV + 8 * (tp & 1), dEV + so);
                if (ve1 < 0) tmem_cp_128x128b(tEV + 8 * (tp & 1) + 4, dEV + so + 128);
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
                                            tEV + 8 * (tp & 1) + 4 * i + j, id_g2_sp, o_started);
                                o_started = true;
                            }
                        }
                    }
                }
                if constexpr (PP) {
                umma_commit(&bar_vempty[s]);  // V stage free once the O^T MMAs are done
#ifndef HS_PREFILL_XP_NO_LMMA
                {   // row sums l[q] += sum_k P^T[q][k]: P^T as an MN-major A operand, ones as B (N = 16)
                    const uint32_t id_l = umma_idesc_f16(bf2, 128, 16, true, false, false);
                    const uint64_t pa = dP + (pbuf_of(tp) * lay.p_bytes) / 16;
#pragma unroll
                    for (int pass = 0; pass < (HILO ? 2 : 1); ++pass)
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            umma_f16(tmem + 416u, pa + pass * 2048 + 128 * kk, dOnesL, id_l, tp > 0 || pass > 0 || kk > 0);
                }
#endif
                umma_commit(&bar_pempty[pbuf_of(tp)]);  // P^T buffer free; O^T and l through tile tp final
                } else {
                umma_commit(&bar_pempty[pbuf_of(tp)]);  // P^T buffer free; O^T through tile tp final
                umma_commit(&bar_vempty[s]);            // V stage can be refilled
                }
            }
            __syncwarp();
            if (kG2First && lane == 0) st_release(&s_g2_issued, tp + 1);
            o_started = true;
            if (DBG && lane == 0) trace(L, tp, 6);
        };
        if (warp_u == kWarpMma2) {
            for (int tp = 0; tp < ntiles; ++tp) gemm2(tp);
        } else
        for (int t = 0; t < ntiles; ++t) {
            const int s = t % nk, sb = t & 1;
            const TileInfo ti = s_tiles[t];
            const int ke0 = uni(ti.ke0);
            if (DBG && lane == 0) trace(L, t, 11);
            mbar_wait_dbg(&bar_kfull[s], (t / nk) & 1, dbgp, 3);  // K tile + metadata atom landed
            if (DBG && lane == 0) trace(L, t, 10);
            if (t >= 2) mbar_wait_dbg(&bar_sempty[sb], ((t >> 1) - 1) & 1, dbgp, 6);
            if (kG2First && t >= 2) {
                // GEMM2(t-2) enters the tensor pipe ahead of GEMM1(t): the P^T buffer
                // softmax(t) writes is then free in time (GEMM1 still runs a tile ahead)
                while (ld_acquire_cta(&s_g2_issued) < t - 1) __nanosleep(32);
            }
            tc_fence_after();
            if (DBG && lane == 0) trace(L, t, 4);
            if (elect_one()) {
                const uint64_t so = static_cast<uint64_t>(s) * kst16;
                // metadata -> TMEM (ordered before the MMAs that read it)
                if (ke0 < 0) tmem_cp_128x128b(tEK + 4 * sb, dEK + so);
                // GEMM1: S^T[sb] = K_tile * Q^T
                const uint32_t tS = tS0 + 128 * sb;
                // S^T = ones * bias[sb]^T (the -m_c / (scale log2e) stabiliser of every
                // column) + K_tile * Q^T
                if (!(mode & 2)) umma_f16(tS, dOnes, dBias + sb * 128, id_g1_de, 0u);
                if (mode & 2) {
                } else if (ke0 > 0) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        umma_f16(tS, dK + so + (j >> 2) * 1024 + 2 * (j & 3), dQ + (j >> 2) * 1024 + 2 * (j & 3),
                                 id_g1_de, 1u);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        umma_sp_f16(tS, dK + so + 2 * j, dQ + (j >> 1) * 1024 + 4 * (j & 1), tEK + 4 * sb + j,
                                    id_g1_sp, 1u);
                }
                umma_commit(&bar_sfull[sb]);
                umma_commit(&bar_kempty[s]);  // K stage can be refilled once GEMM1(t) read it
            }
            __syncwarp();
        }
    } else if constexpr (PP) {
        // ------------------------------------------- ping-pong softmax ----
        // Two groups of 8 warps take alternate tiles: group g handles t = g (mod 2)
        // with S^T buffer g, P^T buffer g and GEMM1 bias operand g, so one group's
        // exponentials overlap the other's TMEM load and reduction.  Warp (g, wq,
        // ch) covers key lanes 32 wq.. and query columns 64 ch..; its 4 warps (one
        // per lane quarter) form a "quad" with its own named barrier.  The row sums
        // l are accumulated by the tensor core (GEMM2 warp: P^T x ones).
        //
        // Running max: one shared value per column (s_mcur, grown with atomicMax,
        // version-counted per column half).  A quad's fast path needs its bias
        // snapshot to be current (version match) and every value <= tau; otherwise
        // its slow path grows m_cur where needed, re-reads it, corrects x and
        // refreshes its bias.  Every tile publishes the m it used (version +
        // values); before its P^T is released to GEMM2, the next tile's quad
        // compares versions and, when they differ, rescales O^T and l between
        // GEMM2(t-1) and GEMM2(t) by exp2(m_{t-1} - m_t).
        auto& s_mcur = pps.s_mcur;
        auto& s_red2 = pps.s_red2;
        auto& s_dl = pps.s_dl;
        auto& s_mt = pps.s_mt;
        auto& s_al = pps.s_al;
        auto& s_ver = pps.s_ver;
        auto& s_vsnap = pps.s_vsnap;
        auto& s_tdone = pps.s_tdone;
        const int grp = warp >> 3, wq = warp & 3, ch = (warp >> 2) & 1;
        const int r = 32 * wq + lane;
        const int c0 = 64 * ch;
        const int bar_id = 1 + 2 * grp + ch;
        const uint32_t lane_off = static_cast<uint32_t>(32 * wq) << 16;
        const uint32_t tL = tmem + 416u;
        const uint32_t pt_base_h = static_cast<uint32_t>(ch) * 16384u + (r >> 3) * 1024 + (r & 7) * 128;
        const uint32_t r7 = r & 7;
        uint8_t* const pbuf0 = base_ptr + lay.off_p;
        uint4* const bias_rows = reinterpret_cast<uint4*>(base_ptr + lay.off_bias + 2048);
        const float sl2 = L.scale_log2;
        bool pending = true;        // quad-uniform: some column of the quad has no max yet
        int bver = -1;              // version of the m values in this group's bias snapshot
        for (int t = grp; t < ntiles; t += 2) {
            const int sb = grp, slot = (t >> 1) & 1;
            const TileInfo ti = s_tiles[t];
            mbar_wait_dbg(&bar_sfull[sb], (t >> 1) & 1, dbgp, 21);
            tc_fence_after();
            if (DBG && (mode & 1)) {  // tools: the TMA + MMA pipeline without the softmax
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_sempty[sb]);
                if (t >= 2) mbar_wait_dbg(&bar_pempty[sb], ((t >> 1) - 1) & 1, dbgp, 22);
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_pfull[sb]);
                continue;
            }
            const bool tr0 = DBG && lane == 0 && wq == 0 && ch == 0;  // one tracing thread per group
            if (tr0) trace(L, t, 0);
            float x[64];
            tmem_ld16_f(tS0 + 128 * sb + lane_off + c0, x);
            tmem_ld16_f(tS0 + 128 * sb + lane_off + c0 + 16, x + 16);
            tmem_ld16_f(tS0 + 128 * sb + lane_off + c0 + 32, x + 32);
            tmem_ld16_f(tS0 + 128 * sb + lane_off + c0 + 48, x + 48);
            tmem_ld_wait();
            if (tr0) trace(L, t, 1);
            int c_first = 0;
            bool fast = true;
            if (ti.dblk >= 0 || ti.ve1 == 0) {
                const int key_pos = ti.dblk * kBlock + r;
                const bool row_valid = (r < 64 || ti.ve1 != 0) && (ti.dblk < 0 || key_pos < n_kv);
                c_first = row_valid ? ((L.causal && ti.dblk >= 0) ? key_pos - off - q0 : 0) : 1 << 30;
                fast = __all_sync(0xffffffffu, c_first <= (QT > 64 ? (c0 & qmask) : 0));
            }
#pragma unroll
            for (int k = 0; k < 64; k += 2) ffma2(x[k], x[k + 1], sl2, 0.f, 0.f);  // s*scale*log2e - m_used
            if (!fast) {
#pragma unroll
                for (int k = 0; k < 64; ++k)
                    if (((c0 + k) & qmask) < c_first) x[k] = -INFINITY;
            }
            bool slow = pending || *reinterpret_cast<volatile int*>(&s_ver[ch]) != bver;
            if (!slow) {
                float m8[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float m = max3f(x[8 * j], x[8 * j + 1], x[8 * j + 2]);
                    m = max3f(m, x[8 * j + 3], x[8 * j + 4]);
                    m = max3f(m, x[8 * j + 5], x[8 * j + 6]);
                    m8[j] = fmaxf(m, x[8 * j + 7]);
                }
                const float xmax =
                    max3f(max3f(m8[0], m8[1], m8[2]), max3f(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
                slow = !(xmax <= kTau);
            }
            const bool slow_q = bar_red_or(bar_id, slow);
            if (tr0) trace(L, t, 2);
            if (slow_q) {
                if (DBG && dbgp && r == 0) atomicAdd(dbgp + 8, 1);
                // ---- slow path (quad): x is relative to m_used[grp]
#pragma unroll
                for (int k = 0; k < 64; ++k) s_red2[grp][wq][c0 + k] = redux_max(x[k]);
                named_bar(bar_id, 128);
                bool grew = false;
                if (r < 64) {
                    const int c = c0 + r;
                    const float tm = fmaxf(fmaxf(s_red2[grp][0][c], s_red2[grp][1][c]),
                                           fmaxf(s_red2[grp][2][c], s_red2[grp][3][c]));
                    const float mu = s_mused[grp][c];
                    const float tabs = tm + (mu == -INFINITY ? 0.f : mu);  // absolute column max
                    const float mc = unord_f32(static_cast<uint32_t>(
                        *reinterpret_cast<volatile unsigned long long*>(&s_mcur[c]) >> 32));
                    if (tm > -INFINITY && (mc == -INFINITY || tabs > mc + kTau)) {
                        const float b = F16Traits<T>::round(fminf(fmaxf(-tabs / (16.f * sl2), -60000.f), 60000.f));
                        const float mnew = -16.f * b * sl2;
                        const uint32_t bb = F16Traits<T>::pack(b, b) & 0xFFFFu;
                        atomicMax(&s_mcur[c], (static_cast<unsigned long long>(ord_f32(mnew)) << 32) | bb);
                        grew = true;
                    }
                }
                grew = bar_red_or(bar_id, grew);  // every atomicMax of the quad done
                if (DBG && dbgp && grew && r == 0) atomicAdd(dbgp + 10, 1);
                if (r == 0) {
                    if (grew) atomicAdd(&s_ver[ch], 1);
                    s_vsnap[grp][ch] = *reinterpret_cast<volatile int*>(&s_ver[ch]);
                }
                named_bar(bar_id, 128);
                bver = s_vsnap[grp][ch];  // values read below are at least this recent
                bool pend = false;
                if (r < 64) {
                    const int c = c0 + r;
                    const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(&s_mcur[c]);
                    const float mt = unord_f32(static_cast<uint32_t>(cur >> 32));
                    const float mu = s_mused[grp][c];
                    s_dl[grp][c] = mt == -INFINITY ? 0.f : mt - (mu == -INFINITY ? 0.f : mu);
                    s_mused[grp][c] = mt;
                    const uint32_t w = mt == -INFINITY ? 0u : static_cast<uint32_t>(cur & 0xFFFFu) * 0x10001u;
                    bias_rows[sb * 128 + c] = make_uint4(w, w, w, w);  // GEMM1(t+2) reads it after sempty
                    pend = mt == -INFINITY;
                    fence_async_smem();
                }
                pending = bar_red_or(bar_id, pend);  // also publishes s_dl / s_mused / bias rows
#pragma unroll
                for (int k = 0; k < 64; ++k) x[k] -= s_dl[grp][c0 + k];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_sempty[sb]);  // S^T[sb] consumed
            if (t >= 2) mbar_wait_dbg(&bar_pempty[sb], ((t >> 1) - 1) & 1, dbgp, 22);  // P^T[sb] free (GEMM2(t-2) done)
            if (tr0) trace(L, t, 3);
            uint8_t* const pbuf = pbuf0 + sb * lay.p_bytes;
#pragma unroll
            for (int g8 = 0; g8 < 8; ++g8) {
                float p[8];
#pragma unroll
                for (int k = 0; k < 8 - POLY; ++k) p[k] = fast_exp2(x[8 * g8 + k]);
#pragma unroll
                for (int k = 8 - POLY; k < 8; k += 2) {
                    p[k] = x[8 * g8 + k];
                    p[k + 1] = x[8 * g8 + k + 1];
                    exp2_fma2(p[k], p[k + 1]);
                }
                using PT = typename std::conditional<V16, __half, T>::type;  // P^T element type
                const uint4 hi = make_uint4(F16Traits<PT>::pack(p[0], p[1]), F16Traits<PT>::pack(p[2], p[3]),
                                            F16Traits<PT>::pack(p[4], p[5]), F16Traits<PT>::pack(p[6], p[7]));
                const uint32_t pto = pt_base_h + ((static_cast<uint32_t>(g8) ^ r7) << 4);
#ifdef HS_PREFILL_XP_NO_PSTORE
                if (hi.x == 0x7fff7fffu)  // experiment: keep the math, drop the P^T stores
#endif
                *reinterpret_cast<uint4*>(pbuf + pto) = hi;
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
                    *reinterpret_cast<uint4*>(pbuf + 32768 + pto) = lo;
                }
            }
            if (tr0) trace(L, t, 12);
            bool need = false;
            if constexpr (!SAFE) {
            // ---- publish the m this tile used; O^T / l to it when tile t-1 used another
            // (between GEMM2(t-1) and GEMM2(t)).  Per-column compare of exact values:
            // a version match alone does not imply equal values across the groups.
            if (r < 64) s_mt[grp][slot][c0 + r] = s_mused[grp][c0 + r];
            need = false;
            if (t >= 1) {
                const int pg = grp ^ 1, ps = ((t - 1) >> 1) & 1;
                if (lane == 0) {
                    long long spins = 0;
                    while (ld_acquire_cta(&s_tdone[pg][ps][ch]) != t - 1) {
                        __nanosleep(32);
                        if (DBG && dbgp && ++spins > (1ll << 22)) {
                            if (atomicCAS(dbgp, 0, 25) == 0) {
                                dbgp[1] = ld_acquire_cta(&s_tdone[pg][ps][ch]);
                                dbgp[2] = static_cast<int>(blockIdx.x + 1000 * blockIdx.y + 100000 * blockIdx.z);
                                dbgp[3] = static_cast<int>(threadIdx.x) + 10000 * t;
                                __threadfence_system();
                            }
                            asm volatile("trap;");
                        }
                    }
                }
                __syncwarp();
                if (tr0) trace(L, t, 13);
                if (r < 64) need = s_mt[pg][ps][c0 + r] != s_mused[grp][c0 + r];
            }
            need = bar_red_or(bar_id, need);  // also: this quad's s_mt values are all stored
            if (r == 0) st_release(&s_tdone[grp][slot][ch], t);
            } else {
            // ---- SAFE pass: the tile's m is m_t = max(m_used, m_{t-1}) per column, so
            // O^T / l are only ever rescaled by exp2(m_{t-1} - m_t) <= 1 (between
            // GEMM2(t-1) and GEMM2(t)).  When the other group grew a column after this
            // group's snapshot (m_{t-1} > m_used; this group's next tile sees the
            // version bump), the P^T values just stored are lowered to m_t instead.
            if (t >= 1) {
                const int pg = grp ^ 1, ps = ((t - 1) >> 1) & 1;
                if (lane == 0) {
                    while (ld_acquire_cta(&s_tdone[pg][ps][ch]) != t - 1) __nanosleep(32);
                }
                __syncwarp();
                if (r < 64) {
                    const int c = c0 + r;
                    const float mp = s_mt[pg][ps][c], mu = s_mused[grp][c];
                    // mu = -inf: every logit of the column so far is masked (P = 0)
                    const float me = mu == -INFINITY ? mp : fmaxf(mu, mp);
                    const float pscale = (mu != -INFINITY && me > mu) ? fast_exp2(mu - me) : 1.f;
                    const float al = (mp == -INFINITY || me == mp) ? 1.f : fast_exp2(mp - me);
                    s_mt[grp][slot][c] = me;
                    // P^T factor in the slow path's scratch (every read of it is behind
                    // the slow path's last quad barrier)
                    s_red2[grp][0][c] = pscale;
                    s_al[grp][c] = al;
                    need = pscale != 1.f || al != 1.f;
                }
            } else if (r < 64) {
                s_mt[grp][slot][c0 + r] = s_mused[grp][c0 + r];
            }
            need = bar_red_or(bar_id, need);  // also: this quad's s_mt / P^T factors / s_al values are all stored
            if (r == 0) st_release(&s_tdone[grp][slot][ch], t);
            }
            if (need) {
                if (DBG && dbgp && r == 0) atomicAdd(dbgp + 9, 1);
                if constexpr (SAFE) {  // P^T of this tile to m_t (this thread's own chunks; 1 where unchanged)
                    uint8_t* const pbuf = pbuf0 + sb * lay.p_bytes;
                    using PT = typename std::conditional<V16, __half, T>::type;
#pragma unroll 1
                    for (int g8 = 0; g8 < 8; ++g8) {
                        uint4* const pp = reinterpret_cast<uint4*>(pbuf + pt_base_h + ((static_cast<uint32_t>(g8) ^ r7) << 4));
                        uint4 w = *pp;
                        uint32_t* wv = &w.x;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const float a = F16Traits<PT>::to_float(static_cast<uint16_t>(wv[k] & 0xFFFF)) *
                                            s_red2[grp][0][c0 + 8 * g8 + 2 * k];
                            const float b = F16Traits<PT>::to_float(static_cast<uint16_t>(wv[k] >> 16)) *
                                            s_red2[grp][0][c0 + 8 * g8 + 2 * k + 1];
                            wv[k] = F16Traits<PT>::pack(a, b);
                        }
                        *pp = w;
                    }
                }
                const int pg = grp ^ 1, ps = ((t - 1) >> 1) & 1;
                mbar_wait_dbg(&bar_pempty[pg], ((t - 1) >> 1) & 1, dbgp, 23);  // GEMM2(t-1) complete
                tc_fence_after();
                if constexpr (!SAFE) {
                    if (r < 64) {
                        const int c = c0 + r;
                        const float mp = s_mt[pg][ps][c], mt = s_mused[grp][c];
                        s_al[grp][c] = (mp == -INFINITY || mt == -INFINITY) ? 1.f : fast_exp2(mp - mt);
                    }
                    named_bar(bar_id, 128);
                }
                (void)ps;
#pragma unroll 1
                for (int k8 = 0; k8 < 64; k8 += 8) {
                    uint32_t v[8];
                    tmem_ld_cols<8>(tO + lane_off + c0 + k8, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 8; ++k) v[k] = __float_as_uint(__uint_as_float(v[k]) * s_al[grp][c0 + k8 + k]);
                    tmem_st4(tO + lane_off + c0 + k8, v[0], v[1], v[2], v[3]);
                    tmem_st4(tO + lane_off + c0 + k8 + 4, v[4], v[5], v[6], v[7]);
                }
                if ((wq >> 1) == ch) {  // this lane quarter holds l of queries 32 wq + lane
                    uint32_t lv;
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(lv) : "r"(tL + lane_off));
                    tmem_ld_wait();
                    const float ln = __uint_as_float(lv) * s_al[grp][r];
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tL + lane_off),
                                 "r"(__float_as_uint(ln)));
                }
                tmem_st_wait();
                tc_fence_before();
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_pfull[sb]);
            if (tr0) trace(L, t, 14);
        }
        // ---- epilogue: O^T / l after the last GEMM2 (l from the row-sum accumulator),
        // by the group of the last tile: it already waited on that P^T buffer's
        // previous phase, so the parity wait below cannot alias an older phase
        const int egrp = ntiles > 0 ? (ntiles - 1) & 1 : 0;
        if (grp == egrp) {
            if (ntiles > 0) mbar_wait_dbg(&bar_pempty[egrp], ((ntiles - 1) >> 1) & 1, dbgp, 24);
            tc_fence_after();
            if ((wq >> 1) == ch) {
                uint32_t lv = 0;
                if (ntiles > 0) {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(lv) : "r"(tL + lane_off));
                    tmem_ld_wait();
                }
                const float l = __uint_as_float(lv);
                s_alpha[r] = l > 0.f ? 1.f / l : 0.f;
            }
            named_bar(5, 256);  // the epilogue group only (ids 1-4 are the quads' barriers)
            const int v_exp = V16 ? L.v16_scale[1] : 0;  // O^T was accumulated over V * 2^-v_exp
            bool bad = false;  // a non-finite row: flag this CTA for the SAFE pass
#pragma unroll 1
            for (int k16 = 0; k16 < 64; k16 += 16) {
                float v[16];
                tmem_ld16_f(tO + lane_off + c0 + k16, v);
                tmem_ld_wait();
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int c = c0 + k16 + k;
                    const float o = v[k] * s_alpha[c];
                    const bool cv = (c & qmask) < rows_q;
                    bad |= cv && !(fabsf(o) <= 3.4e38f);
                    if (cv) out_row(c)[r] = ntiles > 0 ? (V16 ? ldexpf(o, v_exp) : o) : 0.f;
                }
            }
            if (!SAFE && bad) s_bad = 1;  // published to L.redo after the final barrier
        }
    } else {
        // ------------------------------------------------------- softmax WGs
        // kSoftWG warpgroups; WG g owns query columns [kCols*g, kCols*(g+1)); warp
        // w reads TMEM lanes 32(w%4).. (key row r of the tile = d row of O^T).
        // S^T is read from TMEM once per tile and released at once.  The running
        // column max m lives in smem; in steady state a tile needs no cross-lane
        // reduction: every thread checks x = s*scale*log2e - m <= tau for its own
        // values, one bar.red.or per warpgroup confirms it (P <= 2^tau fits fp16).
        // Only when a column grows past m + tau (first visible tile, rare later)
        // the slow path computes the exact column max (redux.f32 + smem), updates
        // m and rescales O^T and the partial sums.
        const int wg = warp >> 2, wq = warp & 3;
        const int r = 32 * wq + lane;  // TMEM lane = key row of the tile = d row of O^T
        const int c0 = kCols * wg;     // this warpgroup's first query column
        const int bar_id = 1 + wg;
        static_assert(kCols % 32 == 0, "P^T chunk offsets assume c0/8 is a multiple of 4");
        const uint32_t pt_r3 = static_cast<uint32_t>(r & 3) << 4;
        const uint32_t pt_base = pt_chunk_off(r, c0 >> 3) - ((static_cast<uint32_t>((c0 >> 3) & 7) ^ (r & 7)) << 4) +
                                 ((static_cast<uint32_t>((c0 >> 3) & 4) ^ (r & 4)) << 4);
        const uint32_t lane_off = static_cast<uint32_t>(32 * wq) << 16;
        float l_part[kCols];
#pragma unroll
        for (int c = 0; c < kCols; ++c) l_part[c] = 0.f;
        if (r < kCols) {
            s_mrun[c0 + r] = -INFINITY;
            s_bq[c0 + r] = 0;
        }
        named_bar(bar_id, 128);
        uint8_t* const pbuf0 = base_ptr + lay.off_p;
        uint4* const bias_rows = reinterpret_cast<uint4*>(base_ptr + lay.off_bias + 2048);
        const float sl2 = L.scale_log2;
        // Warpgroup-uniform state: `pending` while some column of this warpgroup
        // has no running max yet; bit b of `dirty` while bias[b] (the stabiliser
        // GEMM1 folds into S buffer b) differs from the running max.
        bool pending = true;
        uint32_t dirty = 0;
        for (int t = 0; t < ntiles; ++t) {
            const int sb = t & 1;
            const TileInfo ti = s_tiles[t];
            mbar_wait_dbg(&bar_sfull[sb], (t >> 1) & 1, dbgp, 5);
            tc_fence_after();
            if (DBG && tid == 0) trace(L, t, 0);
            if (DBG && tid == 256) trace(L, t, 15);  // warpgroup 2's view of the same tile
            if (mode & 1) {  // tools: pipeline without the softmax
                if (t >= npb) mbar_wait_dbg(&bar_pempty[pbuf_of(t)], pphase(t - npb), dbgp, 8);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&bar_sempty[sb]);
                    mbar_arrive(&bar_pfull[pbuf_of(t)]);
                }
                continue;
            }
            float x[kCols];
            tmem_ld16_f(tS0 + 128 * sb + lane_off + c0, x);
            tmem_ld16_f(tS0 + 128 * sb + lane_off + c0 + 16, x + 16);
            tmem_ld_wait();
            if (DBG && tid == 0) trace(L, t, 12);
            // masks: invalid rows of single-block tiles; causal (attention.hpp:181-190)
            // (a full off-diagonal pair -- most tiles -- is visible everywhere: no mask work)
            int c_first = 0;
            bool fast = true;
            if (ti.dblk >= 0 || ti.ve1 == 0) {
                const int key_pos = ti.dblk * kBlock + r;  // diagonal / tail pairs are consecutive blocks
                // rows past a single block or past the end of the tail hold no key
                const bool row_valid = (r < 64 || ti.ve1 != 0) && (ti.dblk < 0 || key_pos < n_kv);
                // column c (query q0 + c at position off + q0 + c) sees this key iff c >= c_first
                c_first = row_valid ? ((L.causal && ti.dblk >= 0) ? key_pos - off - q0 : 0) : 1 << 30;
                // warp-uniform fast path: every (row, column) of this warp visible
                fast = __all_sync(0xffffffffu, c_first <= (QT > kCols ? (c0 & qmask) : 0));
            }
            // S^T holds s + bias[sb] = s - m_used/(scale log2e), so x = S^T * scale log2e
            // = s*scale*log2e - m_used: no per-column operand in the steady state
#pragma unroll
            for (int k = 0; k < kCols; k += 2) ffma2(x[k], x[k + 1], sl2, 0.f, 0.f);
            if (!fast) {
#pragma unroll
                for (int k = 0; k < kCols; ++k)
                    if (((c0 + k) & qmask) < c_first) x[k] = -INFINITY;
            }
            bool slow = pending || ((dirty >> sb) & 1u);
            if (!slow) {
                // four independent 3-input max chains (short dependency depth), then merge
                static_assert(kCols == 32, "max tree laid out for 32 columns");
                float m4[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float m = max3f(x[8 * j], x[8 * j + 1], x[8 * j + 2]);
                    m = max3f(m, x[8 * j + 3], x[8 * j + 4]);
                    m = max3f(m, x[8 * j + 5], x[8 * j + 6]);
                    m4[j] = fmaxf(m, x[8 * j + 7]);
                }
                const float xmax = fmaxf(max3f(m4[0], m4[1], m4[2]), m4[3]);
                if (DBG && tid == 0) trace(L, t, 13);
                slow = bar_red_or(bar_id, !(xmax <= kTau));
            }
            if (DBG && tid == 0) trace(L, t, 14);
            if (slow) {
                // ---- slow path: a column grew past m + tau, a column has no max
                // yet, or S[sb] was built with a stale stabiliser.  x is relative
                // to m_used[sb]; the exact column max decides the new m.
#pragma unroll
                for (int k = 0; k < kCols; ++k) s_red[wq][c0 + k] = redux_max(x[k]);
                named_bar(bar_id, 128);
                bool resc = false, changed = false, pend = false;
                if (r < kCols) {
                    const int c = c0 + r;
                    const float tm = fmaxf(fmaxf(s_red[0][c], s_red[1][c]), fmaxf(s_red[2][c], s_red[3][c]));
                    const float mu = s_mused[sb][c], mo = s_mrun[c];
                    const float tabs = tm + mu;  // absolute column max (log2 units)
                    float mnew = mo, alpha = 1.f;
                    if (tm > -INFINITY && (mo == -INFINITY || tabs > mo + kTau)) {
                        // the stabiliser is what the bias operand can hold exactly
                        const float b = F16Traits<T>::round(fminf(fmaxf(-tabs / (16.f * sl2), -60000.f), 60000.f));
                        s_bq[c] = static_cast<uint16_t>(F16Traits<T>::pack(b, b) & 0xFFFFu);
                        mnew = -16.f * b * sl2;
                        if (mo != -INFINITY) {
                            alpha = fast_exp2(mo - mnew);
                            resc = true;
                        }
                        changed = true;
                    }
                    s_delta[c] = mnew == -INFINITY ? 0.f : mnew - mu;
                    s_alpha[c] = alpha;
                    s_mrun[c] = mnew;
                    pend = mnew == -INFINITY;
                }
                changed = bar_red_or(bar_id, changed);
                resc = bar_red_or(bar_id, resc);
                pending = bar_red_or(bar_id, pend);
                if (changed) dirty = 3u;
                // x <- x - (m_new - m_used): relative to the running max
#pragma unroll
                for (int k = 0; k < kCols; ++k) x[k] -= s_delta[c0 + k];
                if (resc) {
                    // O^T (GEMM2(t-1) complete) and l rescale for the grown columns
                    if (t >= 1) mbar_wait_dbg(&bar_pempty[pbuf_of(t - 1)], pphase(t - 1), dbgp, 8);
                    tc_fence_after();
#pragma unroll
                    for (int k = 0; k < kCols; ++k) l_part[k] *= s_alpha[c0 + k];
                    if (t >= 1) {
#pragma unroll 1
                        for (int k8 = 0; k8 < kCols; k8 += 8) {  // 8 columns at a time: low register pressure
                            uint32_t v[8];
                            tmem_ld_cols<8>(tO + lane_off + c0 + k8, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int k = 0; k < 8; ++k)
                                v[k] = __float_as_uint(__uint_as_float(v[k]) * s_alpha[c0 + k8 + k]);
                            tmem_st4(tO + lane_off + c0 + k8, v[0], v[1], v[2], v[3]);
                            tmem_st4(tO + lane_off + c0 + k8 + 4, v[4], v[5], v[6], v[7]);
                        }
                        tmem_st_wait();
                    }
                }
                named_bar(bar_id, 128);  // s_red / s_delta / s_alpha reads done before reuse
            }
            if ((dirty >> sb) & 1u) {
                // GEMM1(t+2) reads bias[sb] once every warp released S[sb]: refresh it
                if (r < kCols) {
                    const int c = c0 + r;
                    const uint32_t w = s_bq[c] * 0x10001u;
                    bias_rows[sb * 128 + c] = make_uint4(w, w, w, w);
                    const float m = s_mrun[c];
                    s_mused[sb][c] = m == -INFINITY ? 0.f : m;  // no max yet: bias 0
                    fence_async_smem();
                }
                dirty &= ~(1u << sb);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_sempty[sb]);  // this warp is done with S^T[sb]
            if (DBG && tid == 0) trace(L, t, 1);
            // P^T buffer free (GEMM2 of its previous tile complete)
            if (t >= npb) mbar_wait_dbg(&bar_pempty[pbuf_of(t)], pphase(t - npb), dbgp, 8);
            if (DBG && tid == 0) trace(L, t, 2);
            // probabilities, partial column sums, P^T (+ residual for bf16)
            uint8_t* const pbuf = pbuf0 + pbuf_of(t) * lay.p_bytes;
#pragma unroll
            for (int g8 = 0; g8 < kCols / 8; ++g8) {
                // pt_chunk_off(r, c0/8 + g8) with c0/8 a multiple of 4: only the low two
                // chunk bits vary with g8, so one XOR + add per chunk
                const uint32_t pto = pt_base + ((static_cast<uint32_t>(g8) << 4) ^ pt_r3);
                if constexpr (!HILO && kExpF16x2) {
                    // fp16 P: two exponentials per MUFU op (ex2.approx.f16x2 on x
                    // rounded to fp16; x <= tau keeps the argument error small where
                    // P is large), the packed result is the stored P^T chunk.
                    uint32_t ph[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        ph[k] = ex2_f16x2(pack_f16x2(x[8 * g8 + 2 * k], x[8 * g8 + 2 * k + 1]));
                        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&ph[k]));
                        l_part[8 * g8 + 2 * k] += f.x;
                        l_part[8 * g8 + 2 * k + 1] += f.y;
                    }
                    *reinterpret_cast<uint4*>(pbuf + pto) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
                    continue;
                }
                float p[8];
#pragma unroll
                for (int k = 0; k < 8 - POLY; ++k) p[k] = fast_exp2(x[8 * g8 + k]);  // exp2(-inf) = 0
#pragma unroll
                for (int k = 8 - POLY; k < 8; k += 2) {
                    p[k] = x[8 * g8 + k];
                    p[k + 1] = x[8 * g8 + k + 1];
                    exp2_fma2(p[k], p[k + 1]);
                }
#pragma unroll
                for (int k = 0; k < 8; k += 2) fadd2(l_part[8 * g8 + k], l_part[8 * g8 + k + 1], p[k], p[k + 1]);
                const uint4 hi = make_uint4(F16Traits<T>::pack(p[0], p[1]), F16Traits<T>::pack(p[2], p[3]),
                                            F16Traits<T>::pack(p[4], p[5]), F16Traits<T>::pack(p[6], p[7]));
                *reinterpret_cast<uint4*>(pbuf + pto) = hi;
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
                    *reinterpret_cast<uint4*>(pbuf + 32768 + pto) = lo;
                }
            }
            if (DBG && tid == 0) trace(L, t, 3);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_pfull[pbuf_of(t)]);
        }
        // ---------------------------------------------------- epilogue ----
        if (ntiles > 0) mbar_wait_dbg(&bar_pempty[pbuf_of(ntiles - 1)], pphase(ntiles - 1), dbgp, 8);
        tc_fence_after();
        // l[c] = sum over the 128 key lanes of l_part[c]: transpose through smem
        // (P^T buffers and the K ring are free: every GEMM has completed)
        float* s_l = reinterpret_cast<float*>(base_ptr + lay.off_p) + wg * (128 * (kCols + 1));
#pragma unroll
        for (int c = 0; c < kCols; ++c) s_l[r * (kCols + 1) + c] = l_part[c];
        named_bar(bar_id, 128);
        if (r < kCols) {
            float lsum = 0.f;
            for (int k = 0; k < 128; ++k) lsum += s_l[k * (kCols + 1) + r];
            s_alpha[c0 + r] = lsum > 0.f ? 1.f / lsum : 0.f;
        }
        named_bar(bar_id, 128);
        {
            uint32_t v[kCols];
            tmem_ld_cols<kCols>(tO + lane_off + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < kCols; ++k) {
                const int c = c0 + k;
                if ((c & qmask) < rows_q) out_row(c)[r] = __uint_as_float(v[k]) * s_alpha[c];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kWarpMma) tmem_dealloc(tmem, 512);
    if (PP && !SAFE && tid == 0 && s_bad) L.redo[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = 1;
}

}  // namespace

int prefill_tile_cap(int nb, int ntb) { return nb / 2 + ntb / 2 + 10; }

cudaError_t launch_prefill(const PrefillLaunch& L, cudaStream_t s, int* n_kernels) {
    PrefillLayout lay;
    *n_kernels = 0;
    const bool hilo = L.bf16 && !L.v16;
    // K stage: dense 128x128 tile, or 128x64 nnz + 2 KB metadata + 2 KB E atom.
    const bool kden = L.k_dense_count > 0 || L.n_tail_blocks > 0, vden = L.v_dense_count > 0 || L.n_tail_blocks > 0;
    lay.k_meta = 0;  // unused: the metadata atoms come prepared (meta_atom_kernel)
    lay.k_e = 16384u;
    lay.k_stage = kden ? 32768u : 18432u;
    // V stage: two V^T blocks (dense 128x64 or nnz 128x32) + 2 KB metadata + 2 KB E.
    lay.vblk = vden ? 16384u : 8192u;
    lay.v_meta = 0;  // unused: the metadata atoms come prepared (meta_atom_kernel)
    lay.v_e = 2 * lay.vblk;
    lay.v_stage = lay.v_e + 4096u;
    lay.tile_cap = static_cast<uint32_t>(prefill_tile_cap(L.nb, L.n_tail_blocks));
    const uint32_t tiles_bytes = (lay.tile_cap * sizeof(TileInfo) + 127u) & ~127u;
    // the fp16 ones operand of the row-sum MMA exists only on the bf16 (v16) path
    const uint32_t bias_bytes = L.v16 ? kBiasBytes : kBiasBytes - 2048u;
    // static shared memory of the two kernel families (queried once): the plans use
    // the real figure, not an estimate -- a few KB decide whether a dense-stage
    // plan keeps two V stages at 128K
    static int static_pp = -1, static_ls = -1;
    if (static_pp < 0) {
        cudaFuncAttributes fa{};
        static_pp = cudaFuncGetAttributes(&fa, prefill_kernel<__half, false, false, true, 2>) == cudaSuccess
                        ? static_cast<int>(fa.sharedSizeBytes) : 12288;
        static_ls = cudaFuncGetAttributes(&fa, prefill_kernel<__half, false, false, false>) == cudaSuccess
                        ? static_cast<int>(fa.sharedSizeBytes) : 8192;
        (void)cudaGetLastError();
    }
    lay.off_q = 0;
    lay.off_p = 32768;
    lay.p_bytes = hilo ? 65536u : 32768u;  // P^T (hi [+ lo]) per buffer
    // Preference order: 2 K + 2 V stages with two P^T buffers, then fewer P^T
    // buffers, then shallower rings.
    // V(t) is consumed a softmax period after K(t), so one V stage is enough to
    // keep two P^T buffers (softmax(t+1) never waits for GEMM2(t)) when dense
    // tiles leave no room for both.
    const uint32_t plans[][3] = {{2, 3, 3}, {2, 2, 3}, {2, 3, 2}, {2, 2, 2}, {2, 3, 1}, {2, 2, 1}, {1, 2, 2},
                                 {2, 1, 2}, {1, 2, 1}, {1, 1, 2}, {1, 1, 1}};
    // The ping-pong softmax moves the bound to the rings: it prefers two V stages
    // over two K stages when dense stages leave room for only three.
    const uint32_t plans_pp[][3] = {{2, 3, 3}, {2, 2, 3}, {2, 3, 2}, {2, 2, 2}, {2, 1, 3}, {2, 1, 2}, {2, 3, 1},
                                    {2, 2, 1}};
    auto choose = [&](uint32_t static_bytes, bool for_pp) {
        const uint32_t budget = 227u * 1024u - static_bytes - 1024u /*align*/ - tiles_bytes - bias_bytes;
        const uint32_t(*list)[3] = for_pp ? plans_pp : plans;
        const int n = for_pp ? static_cast<int>(sizeof(plans_pp) / sizeof(plans_pp[0]))
                             : static_cast<int>(sizeof(plans) / sizeof(plans[0]));
        for (int i = 0; i < n; ++i) {
            const uint32_t* pl = list[i];
            const uint32_t need = 32768u + pl[0] * lay.p_bytes + pl[1] * lay.k_stage + pl[2] * lay.v_stage;
            if (need <= budget) {
                lay.n_pbuf = pl[0];
                lay.nk = pl[1];
                lay.nv = pl[2];
                return true;
            }
        }
        return false;
    };
    // The ping-pong softmax (alternate tiles per 8-warp group, row sums on the
    // tensor core) needs one P^T buffer per group: fp16 P (bf16 P^T is hi + lo,
    // 64 KB a buffer) and a plan with two buffers.  Measured at 64K: +11% on
    // fully 2:4 caches (softmax-bound), +1-2% with dense stages (ring-bound, hence
    // the two-V-stage plan preference above).
    const uint32_t st_pp = static_cast<uint32_t>(static_pp) + 128u, st_ls = static_cast<uint32_t>(static_ls) + 128u;
    bool pp = !hilo && getenv("HS_PREFILL_NO_PP") == nullptr && choose(st_pp, true) && lay.n_pbuf == 2;
    if (getenv("HS_PREFILL_FORCE_PP")) pp = !hilo && choose(st_pp, true) && lay.n_pbuf == 2;  // tools
    if (!pp && !choose(st_ls, false)) return cudaErrorInvalidConfiguration;
    if (const char* env = getenv("HS_PREFILL_PLAN")) {  // tools: "pbuf,nk,nv"
        unsigned a, b, c;
        if (sscanf(env, "%u,%u,%u", &a, &b, &c) == 3) {
            lay.n_pbuf = a;
            lay.nk = b;
            lay.nv = c;
            pp = pp && a == 2;
        }
    }
    if (getenv("HS_PREFILL_VERBOSE"))  // tools
        fprintf(stderr, "prefill plan: pp %d pbuf %u nk %u (stage %u) nv %u (stage %u) hg %d\n", (int)pp, lay.n_pbuf,
                lay.nk, lay.k_stage, lay.nv, lay.v_stage, L.hg);
    lay.off_k = lay.off_p + lay.n_pbuf * lay.p_bytes;
    lay.off_v = lay.off_k + lay.nk * lay.k_stage;
    lay.off_tiles = lay.off_v + lay.nv * lay.v_stage;
    lay.off_bias = lay.off_tiles + tiles_bytes;
    size_t smem = lay.off_bias + bias_bytes + 1024;
    const size_t epi = lay.off_p + kSoftWG * 128 * (kCols + 1) * 4 + 1024;  // lockstep epilogue scratch
    if (!pp && smem < epi) smem = epi;
    {
        const int kb = L.n_units * L.k_sparse_count, vb = L.n_units * L.v_sparse_count;
        if (kb + vb > 0) {
            meta_atom_kernel<<<kb + vb, 128, 0, s>>>(L.k_meta, kb, L.v_meta, vb, L.k_meta_hw, L.v_meta_hw);
            ++*n_kernels;
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
    }
    if (L.v16) {
        if (!pp) return cudaErrorInvalidConfiguration;  // the fp16 V copy serves the ping-pong kernel only
        const int64_t na = static_cast<int64_t>(L.n_units) * L.v_dense_count * kBlock * kHeadDim / 2;
        const int64_t nb = static_cast<int64_t>(L.n_units) * L.v_sparse_count * kBlock * kHeadDim / 4;
        const int64_t nt = static_cast<int64_t>(L.n_units) * L.tail * kHeadDim;
        cudaError_t e = cudaMemsetAsync(L.v16_scale, 0, 2 * sizeof(int), s);
        if (e != cudaSuccess) return e;
        const int grid = 148 * 8;
        v16_absmax_kernel<<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(L.v_dense_src), na,
                                               static_cast<const uint32_t*>(L.v_nnz_src), nb,
                                               static_cast<const uint16_t*>(L.v_tail), nt, L.v16_scale);
        v16_convert_kernel<<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(L.v_dense_src),
                                                reinterpret_cast<uint32_t*>(L.v16_dense), na,
                                                static_cast<const uint32_t*>(L.v_nnz_src),
                                                reinterpret_cast<uint32_t*>(L.v16_nnz), nb, L.v16_scale);
        *n_kernels += 2;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (L.n_tail_blocks > 0) {
        tail_prep_kernel<<<dim3(L.n_tail_blocks, L.n_units), 128, 0, s>>>(
            static_cast<const uint16_t*>(L.k_tail), static_cast<const uint16_t*>(L.v_tail), L.tail, L.n_tail_blocks,
            L.k_tail_ws, L.v_tail_ws, L.v16 ? L.v16_scale : nullptr);
        ++*n_kernels;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (L.hg < 1 || L.hg > 4 || (L.hg & (L.hg - 1)) || L.gqa % L.hg || L.qt * L.hg != 128)
        return cudaErrorInvalidValue;
    const dim3 grid((L.n_q + L.qt - 1) / L.qt, L.gqa / L.hg, L.n_units);
    const bool dbg = L.trace != nullptr || L.dbg != nullptr || L.mode != 0;
    auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
        kern<<<grid, kThreads, smem, s>>>(L, lay);
        ++*n_kernels;
        return cudaSuccess;
    };
    // Ping-pong launches: the fast pass, then the SAFE pass over the CTAs it flagged
    // (every other CTA of the SAFE grid exits at once; a few microseconds).
    auto launch_pp = [&](auto fast, auto safe) -> cudaError_t {
        cudaError_t e = cudaMemsetAsync(L.redo, 0, sizeof(int) * grid.x * grid.y * grid.z, s);
        if (e) return e;
        if ((e = launch(fast)) != cudaSuccess) return e;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (getenv("HS_PREFILL_NO_SAFE")) return cudaSuccess;  // tools: timing of the fast pass alone
        if (getenv("HS_PREFILL_FORCE_SAFE"))  // tests: every CTA recomputed by the SAFE pass
            if ((e = cudaMemsetAsync(L.redo, 1, sizeof(int) * grid.x * grid.y * grid.z, s)) != cudaSuccess) return e;
        return launch(safe);
    };
    cudaError_t e;
    if (L.bf16 && L.v16 && !kden && !vden)
        e = dbg ? launch(prefill_kernel<__nv_bfloat16, false, true, true, 2>)
                : launch_pp(prefill_kernel<__nv_bfloat16, false, false, true, 2>,
                            prefill_kernel<__nv_bfloat16, false, false, true, 2, true>);
    else if (L.bf16 && L.v16)
        e = dbg ? launch(prefill_kernel<__nv_bfloat16, false, true, true, 0>)
                : launch_pp(prefill_kernel<__nv_bfloat16, false, false, true, 0>,
                            prefill_kernel<__nv_bfloat16, false, false, true, 0, true>);
    else if (L.bf16)
        e = dbg ? launch(prefill_kernel<__nv_bfloat16, true, true, false>)
                : launch(prefill_kernel<__nv_bfloat16, true, false, false>);
    else if (pp && !kden && !vden)  // softmax-bound: a quarter of the exponentials on the FMA pipe
        e = dbg ? launch(prefill_kernel<__half, false, true, true, 2>)
                : launch_pp(prefill_kernel<__half, false, false, true, 2>, prefill_kernel<__half, false, false, true, 2, true>);
    else if (pp)  // ring-bound (dense stages): every exponential on the SFU (2.5% faster than a quarter)
        e = dbg ? launch(prefill_kernel<__half, false, true, true, 0>)
                : launch_pp(prefill_kernel<__half, false, false, true, 0>, prefill_kernel<__half, false, false, true, 0, true>);
    else
        e = dbg ? launch(prefill_kernel<__half, false, true, false>) : launch(prefill_kernel<__half, false, false, false>);
    if (e) return e;
    return cudaGetLastError();
}

}  // namespace hs
