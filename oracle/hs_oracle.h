/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the HieraSparse hot path.
 *
 * Two libraries export this interface with different symbol prefixes:
 *   hso_*  oracle/hs_oracle.c   plain-C restatement of the reference algorithm
 *                               (each function cites the reference file:line).
 *   ref_*  oracle/ref_capi.cpp  thin extern "C" shim over the UNMODIFIED
 *                               reference headers (/root/reference/proj/include),
 *                               compiled by oracle/Makefile into oracle/_ref/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these.  The product path never does.
 *
 * Conventions (mirroring the reference):
 *   - all values are float32 working values (tensor.hpp:13-15);
 *   - return codes: 0 ok, 2 ConfigError, 4 DataError (errors.hpp:10-20,
 *     exit codes of bench_cli.cpp:21-23); the message is in *_last_error();
 *   - a cache is one CompressedCache (compressed_cache.hpp:37-110) in arrays.
 */
#ifndef HS_ORACLE_H
#define HS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One CompressedCache (compressed_cache.hpp:37-54) as plain arrays.  On
 * output from *_prune_compress the caller supplies arrays with capacity for
 * every block (logical_blocks entries of each pool kind). */
typedef struct {
    int axis;                 /* 0 = kChannel (key), 1 = kSequence (value), masks.hpp:19-22 */
    size_t head_dim;          /* d */
    size_t block_size;        /* B */
    size_t logical_blocks;
    size_t dense_count;
    size_t sparse_count;
    int16_t* index_map;       /* [logical_blocks] */
    float* dense_pool;        /* [dense_count][B*d] stored layout */
    float* nnz_pool;          /* [sparse_count][B*d/2] */
    uint16_t* meta_pool;      /* [sparse_count][B*d/16] */
} hso_cache;

/* SparsityConfig (masks.hpp:73-99) with the fixed 2:4 pattern. */
typedef struct {
    double s_key;
    double s_value;
    size_t block_size;
    size_t sink_tokens;
    size_t local_window;
} hso_config;

#define HSO_DECL(prefix)                                                                     \
    const char* prefix##last_error(void);                                                    \
    uint64_t prefix##derive_seed(uint64_t base, uint64_t stream);                            \
    uint64_t prefix##head_seed(uint64_t base, size_t head, size_t role);                     \
    void prefix##random_gaussian(size_t rows, size_t cols, uint64_t seed, float scale,       \
                                 float* out);                                                \
    int prefix##prune_compress(const float* x, size_t rows, size_t cols,                     \
                               const hso_config* cfg, int axis, double sparsity, int fused,  \
                               hso_cache* out, uint8_t* flags, double* losses,               \
                               uint8_t* element_mask);                                       \
    int prefix##compress_with_flags(const float* x, size_t rows, size_t cols,                \
                                    const hso_config* cfg, int axis, const uint8_t* flags,   \
                                    hso_cache* out);                                         \
    int prefix##compress_with_mask(const float* x, size_t rows, size_t cols,                 \
                                   const hso_config* cfg, int axis,                          \
                                   const uint8_t* element_mask, const uint8_t* flags,        \
                                   hso_cache* out);                                          \
    int prefix##decompress(const hso_cache* c, float* out);                                  \
    int prefix##attend_rows(const float* q, size_t rows, size_t d, const hso_cache* k,       \
                            const hso_cache* v, const float* k_tail, const float* v_tail,    \
                            size_t tail, size_t block_begin, size_t block_end,               \
                            int include_tail, float scale, const int64_t* qpos,              \
                            float* out_t, float* m_s, float* l_s);                           \
    int prefix##decode(const float* q, size_t n_q, size_t d, const hso_cache* k,             \
                       const hso_cache* v, const float* k_tail, const float* v_tail,         \
                       size_t tail, float scale, size_t splits, size_t gqa_group,            \
                       float* out);                                                          \
    int prefix##prefill(const float* q, size_t n_q, size_t d, const hso_cache* k,            \
                        const hso_cache* v, const float* k_tail, const float* v_tail,        \
                        size_t tail, int causal, float scale, size_t b_r, float* out);       \
    int prefix##dense_attention(const float* q, size_t n_q, const float* k, const float* v,  \
                                size_t n_kv, size_t d, int causal, float scale, float* out); \
    int prefix##flop_and_byte_count(size_t n_q, size_t d, const hso_cache* k,                \
                                    const hso_cache* v, size_t tail, int causal,             \
                                    uint64_t* flops, uint64_t* bytes);

HSO_DECL(hso_)
HSO_DECL(ref_)

/* Port-only host helpers. */
/* Pool sizing before any data is seen: pruner.hpp:106-108 and :127-131. */
int hso_pool_counts(size_t rows, size_t block_size, double sparsity, size_t sink_tokens,
                    size_t local_window, size_t* prefix, size_t* suffix, size_t* quota);
/* RNE float -> bfloat16 / binary16 -> float round trip on a buffer (inputs are
 * rounded once so GPU and oracle see identical values). */
void hso_round_bf16(float* x, size_t n);
void hso_round_f16(float* x, size_t n);

#ifdef __cplusplus
}
#endif
#endif
