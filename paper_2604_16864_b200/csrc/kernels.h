// Internal launch descriptors shared by the C-ABI layer and the kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hs {

constexpr int kBlock = 64;    // B: tokens per block (masks.hpp:76 default)
constexpr int kHeadDim = 128; // d: Llama-3.1-8B head dim

// Status words (hs_status_word in hierasparse_b200.h): ((kStatusKeyMax - key) << 8) | reason,
// key = position of the offending block / group in the reference's iteration order.
constexpr uint64_t kStatusKeyMax = (uint64_t(1) << 48) - 1;
enum StatusReason : uint32_t {
    kReasonZeroEntry = 1,      // decompress: index map holds a zero entry
    kReasonDanglingDense = 2,  // decompress: dangling dense offset
    kReasonDanglingSparse = 3, // decompress: dangling sparse offset
    kReasonCodesOrder = 4,     // unpack_metadata: corrupt metadata, codes not increasing
    kReasonKeepsMore = 5,      // compress: group keeps more than n_keep elements
    kReasonKeepsFewer = 6,     // compress: group keeps fewer than n_keep elements
    kReasonMaskCount = 7,      // compress: block mask dense count differs from the dense pool (ConfigError)
};

struct CompressLaunch {
    bool bf16;
    int axis;
    int block_size = kBlock, head_dim = kHeadDim;  // != (64, 128): generic-shape kernels
    int n_units;
    int nb;
    int dense_count, sparse_count;
    int prefix, suffix, quota;
    bool static_selection;   // quota is 0 or all prunable blocks
    bool all_sparse;         // static: prunable blocks are sparse
    const void* src;
    uint64_t src_unit_stride;
    const uint8_t* flags_in; // explicit BlockMask (hs_compress_with_flags)
    uint8_t* flags_tmp;      // scratch for loss-driven selection
    uint8_t* flags_out;      // optional
    double* losses;          // optional in static mode, required otherwise
    int16_t* index_map;
    int32_t* slot_block;
    void* dense_pool;
    void* nnz_pool;
    uint16_t* meta_pool;
    // compressed source (decode-phase re-prune); in_index == nullptr: dense src
    const int16_t* in_index;
    int in_nb;  // input blocks; blocks >= in_nb come from src (absorbed tail blocks)
    int in_dense_count, in_sparse_count;
    const void* in_dense;
    const void* in_nnz;
    const uint16_t* in_meta;
    unsigned long long* status;  // decompress's DataErrors / BlockMask count (status word), may be null
    const uint8_t* element_mask; // compress under an explicit ElementMask: u8 [u][rows][d] (mask_unit_stride)
    uint64_t mask_unit_stride;
};
cudaError_t launch_prune_compress(const CompressLaunch& L, cudaStream_t s);
// block_loss (pruner.hpp:81-89) of every block (classify pass only) and
// select_blocks (pruner.hpp:94-117) over given losses (sequence-split pruning).
cudaError_t launch_block_losses(const CompressLaunch& L, cudaStream_t s);
cudaError_t launch_select_blocks(const double* losses, int n_units, int nb, int prefix, int suffix, int quota,
                                 uint8_t* flags, cudaStream_t s);

struct DecompressLaunch {
    int axis, n_units, nb, dense_count, sparse_count;
    const int16_t* index_map;
    const void* dense_pool;
    const void* nnz_pool;
    const uint16_t* meta_pool;
    void* dst;
    unsigned long long* status;
    int block_size = kBlock, head_dim = kHeadDim;
};
cudaError_t launch_decompress(const DecompressLaunch& L, cudaStream_t s);

// Split-KV decode over pooled caches (attention.hpp:249-304, :360-409).
struct DecodeLaunch {
    bool bf16;
    int n_units, nb, gqa, tail;
    int q_rows;              // rows per unit of q / out in memory (>= gqa: GQA groups above 8 run in chunks)
    int k_dense_count, k_sparse_count, v_dense_count, v_sparse_count;
    float scale_log2;        // scale * log2(e)
    const void* q;           // [u][q_rows][d], this launch's rows first
    const int16_t* k_index;  // [u][nb]
    const int16_t* v_index;
    const uint16_t* k_meta;  // [u][sparse][512]
    const uint16_t* v_meta;
    const void* k_nnz;       // pools (for L2 prefetch; TMA reads through the maps)
    const void* v_nnz;
    const void* k_dense;
    const void* v_dense;
    int prefetch_distance;   // blocks per warp prefetched into L2 ahead of the ring
    int debug_stream_only;   // tools only: stream the ring without math
    int debug_tail;          // tools only: 1 = skip the split combine, 2 = also skip the arrival spin (timing)
    const void* k_tail;      // [u][tail][d]
    const void* v_tail;
    // split geometry: unit u, split s covers blocks [nb*s/nsplit, nb*(s+1)/nsplit)
    int nsplit;
    int block_begin, block_end;  // restrict to a block range (partial API)
    int max_blocks_per_cta;      // ceil(span / nsplit): sizes the smem index stage
    int include_tail;
    // outputs
    float* partial;          // [u][nsplit][gqa][d+2] (O, m, l)
    float* out;              // fused combine target or nullptr (split partials only)
    int out_mode;            // 0: normalised [u][gqa][d]; 1: merged partial [u][gqa][d+2]
    int* counters;           // [2u] arrival / done counters for the fused combine
    // coop combine mailbox: [u][nsplit][gqa][d] x {~bits(O) | bits(m) << 32, bits(l) | 1 << 32};
    // zero = empty (each reader clears what it read, so launches leave it zeroed)
    unsigned long long* mailbox;
    int coop_combine;        // every CTA resident: all CTAs of a unit merge in parallel
    int dynamic;             // warps claim the unit's blocks from blk_ctr (no static ranges)
    int interleave;          // 1-D grid, CTA i = (unit i % n_units, split i / n_units)
    int* blk_ctr;            // [u] block claim counters (dynamic mode; reset by the combine)
    long long* cta_times;    // tools only: [grid][5] globaltimer at start / first data / loop end / partial written / combine done
    CUtensorMap tm_knnz, tm_kden, tm_vnnz, tm_vden;
};
cudaError_t launch_decode(const DecodeLaunch& L, cudaStream_t s);
int decode_resident_ctas(const DecodeLaunch& L, int sms);  // co-resident CTAs at L's smem plan
int decode_ctas_per_sm();  // CTAs the decode ring is sized for (1 or 2)
cudaError_t launch_combine(const float* partials, int n_parts, int n_units, int gqa, int d,
                           float* out, cudaStream_t s);

// Causal / non-causal prefill (attention.hpp:323-354).
struct PrefillLaunch {
    bool bf16;
    int n_units, nb, gqa, n_q, tail, causal;
    // GQA stacking: one CTA covers hg query heads of a KV head x qt queries each
    // (hg * qt = 128 columns), so every K/V tile is staged once for hg heads.
    int hg, qt;
    int k_dense_count, k_sparse_count, v_dense_count, v_sparse_count;
    float scale_log2;
    const void* q;
    const int16_t* k_index;
    const int16_t* v_index;
    const int32_t* k_slot_block;
    const uint16_t* k_meta;
    const uint16_t* v_meta;
    uint16_t* k_meta_hw;     // workspace: K metadata in the tcgen05 TMEM atom order, 1 KB / block
    uint16_t* v_meta_hw;     // workspace: V metadata atom rows (8 of 16 bytes used), 2 KB / block
    const void* k_tail;      // [u][tail][d] dense tail (CacheView::dense_tail, attention.hpp:19-31)
    const void* v_tail;
    int n_tail_blocks;       // ceil(tail / 64): the tail enters as dense blocks nb, nb+1, ...
    uint16_t* k_tail_ws;     // workspace: [u][n_tail_blocks * 64][d], zero padded
    uint16_t* v_tail_ws;     // workspace: [u][n_tail_blocks][d][64] (transposed, zero padded)
    // bf16 caches on the ping-pong path: GEMM2 runs in fp16 (P^T fp16 keeps 11
    // mantissa bits; kind::f16 needs A and B of one format), over an fp16 copy of
    // the V pools scaled by 2^-v_exp (exact for every value in fp16's normal range
    // after scaling); the epilogue multiplies by 2^v_exp.
    bool v16;
    const void* v_dense_src;  // the bf16 V pools the copy is made from
    const void* v_nnz_src;
    uint16_t* v16_dense;      // workspace: fp16 V pools (same layouts); the V maps point here
    uint16_t* v16_nnz;
    int* v16_scale;           // workspace: [0] = max bf16 magnitude bits, [1] = v_exp
    float* out;
    // workspace, one int per CTA (zeroed by launch_prefill): the ping-pong kernel
    // flags a CTA whose output rows came out non-finite; a second SAFE pass
    // recomputes exactly those CTAs with the race-free running-max exchange
    int* redo;
    int* dbg;                // optional pipeline watchdog record (debug)
    int mode;                // tools only: 1 = softmax skipped, 2 = MMAs skipped, 3 = both
    long long* trace;        // optional per-tile event clocks of CTA (0,0,0) (tools)
    // tm_q is a 4-D view [half][unit*gqa + head][query][64]: one box {64, qt, hg, 2}
    // lands as the stacked 128-column Q tile (rows past n_q zero-filled).
    // tm_kden / tm_ktail are 3-D views ([half][row][64]: one box per 128x128 tile);
    // tm_vnnz2 / tm_vden2 box two consecutive V pool slots (256 rows).
    CUtensorMap tm_q, tm_knnz, tm_kden, tm_vnnz, tm_vden, tm_ktail, tm_vtail, tm_vnnz2, tm_vden2;
};
// *n_kernels: kernels launched (prep passes, the attention kernel, the SAFE pass)
cudaError_t launch_prefill(const PrefillLaunch& L, cudaStream_t s, int* n_kernels);

// Attention for shapes outside the tcgen05 / mma.sp kernels' specialisation
// (block_size != 64 or head_dim != 128): attend_range (attention.hpp:249-304)
// per query row on CUDA cores, one warp per row, expanding 2:4 blocks from their
// canonical metadata on the fly.  Decode, prefill (causal or not) and partials.
struct GenericAttnLaunch {
    bool bf16;
    int n_units, nb, B, d, gqa, n_q, tail, causal;
    float scale;
    const void* q;           // [u][gqa][n_q][d]
    const int16_t* k_index;
    const int16_t* v_index;
    int k_dense_count, k_sparse_count, v_dense_count, v_sparse_count;
    const void* k_dense;
    const void* k_nnz;
    const uint16_t* k_meta;
    const void* v_dense;
    const void* v_nnz;
    const uint16_t* v_meta;
    const void* k_tail;      // [u][tail][d]
    const void* v_tail;
    int block_begin, block_end, include_tail;
    float* out;              // out_mode 0: [u][gqa][n_q][d]; 1: SplitPartial [u][gqa][n_q][d + 2] (O, m, l)
    int out_mode;
};
cudaError_t launch_generic_attention(const GenericAttnLaunch& L, cudaStream_t s);
constexpr int kGenericMaxHeadDim = 512;

}  // namespace hs
