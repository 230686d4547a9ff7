/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the HieraSparse reference
 * (arxiv 2604.16864, /root/reference/proj/include/hierasparse headers) for the
 * hot path: hierarchical pruning, pooled 2:4 compression, Trans-Both
 * attention (prefill + split-KV decode) and the roofline op counts.
 *
 * Every function restates the reference arithmetic in the reference's own
 * operation order (float32 working values, no FMA contraction — build with
 * -ffp-contract=off like the reference's default x86-64 build), so on the same
 * inputs it agrees with the compiled reference (oracle/_ref) bit for bit; the
 * CPU test suite checks exactly that, plus the reference tests' golden vectors.
 *
 * Parity pinned by: tests/test_oracle.py (golden vectors from
 * proj/tests/test_{metadata,pruner,compressor,attention}.cpp and random
 * cross-checks against oracle/_ref built from the reference sources).
 */
#include "hs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define HSO_OK 0
#define HSO_CONFIG 2
#define HSO_DATA 4

static _Thread_local char g_err[512];

const char* hso_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
#define CHECK_CONFIG(ok, msg) do { if (!(ok)) return fail(HSO_CONFIG, msg); } while (0)
#define CHECK_DATA(ok, msg) do { if (!(ok)) return fail(HSO_DATA, msg); } while (0)

/* ------------------------------------------------------------------------ */
/* Deterministic Gaussian source: tensor.hpp:91-137, pipeline.hpp:131-133.    */
/* ------------------------------------------------------------------------ */

/* derive_seed (tensor.hpp:91-96): splitmix64 finaliser over base + golden*(stream+1). */
uint64_t hso_derive_seed(uint64_t base, uint64_t stream) {
    uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* head_seed (pipeline.hpp:131-133): one stream per (head, role). */
uint64_t hso_head_seed(uint64_t base, size_t head, size_t role) {
    return hso_derive_seed(base, (uint64_t)head * 64 + role);
}

/* std::mt19937_64 (the generator GaussianSource wraps, tensor.hpp:125). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) {
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    static const uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & kUpper) | (g->mt[(i + 1) % 312] & kLower);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* GaussianSource::uniform01 (tensor.hpp:119-122): 53-bit draw in [0,1). */
static double uniform01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

/* random_gaussian (tensor.hpp:131-137) with GaussianSource::next (:102-117):
 * Box-Muller, cos sample first, sin sample cached as the spare. */
void hso_random_gaussian(size_t rows, size_t cols, uint64_t seed, float scale, float* out) {
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    int have_spare = 0;
    float spare = 0.0f;
    const size_t n = rows * cols;
    for (size_t i = 0; i < n; ++i) {
        float v;
        if (have_spare) {
            have_spare = 0;
            v = spare;
        } else {
            double u1 = 0.0;
            do {
                u1 = uniform01(g);
            } while (u1 <= 0.0);
            const double u2 = uniform01(g);
            const double r = sqrt(-2.0 * log(u1));
            const double theta = 2.0 * 3.14159265358979323846 * u2;
            spare = (float)(r * sin(theta));
            have_spare = 1;
            v = (float)(r * cos(theta));
        }
        out[i] = v * scale;
    }
    free(g);
}

/* RNE rounding helpers (fp16.hpp:14-64 semantics for binary16; bfloat16 by
 * the same round-to-nearest-even rule on the top 16 bits). */
static float bf16_round(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return f; /* inf / nan passthrough */
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    u &= 0xFFFF0000u;
    memcpy(&f, &u, 4);
    return f;
}

void hso_round_bf16(float* x, size_t n) {
    for (size_t i = 0; i < n; ++i) x[i] = bf16_round(x[i]);
}

static float f16_round(float f) {
    /* Round a float to the nearest binary16 value (RNE), returned as float. */
    if (isnan(f) || isinf(f)) return f;
    const float a = fabsf(f);
    if (a >= 65520.0f) return copysignf(INFINITY, f); /* overflow past max half + half ulp */
    if (a < 0x1.0p-25f) return copysignf(0.0f, f);    /* below half the min subnormal */
    int e;
    frexpf(a, &e);                  /* a = m * 2^e, m in [0.5, 1) */
    int ulp_exp = e - 11;           /* 11 significant bits */
    if (ulp_exp < -24) ulp_exp = -24; /* subnormal spacing 2^-24 */
    const float ulp = ldexpf(1.0f, ulp_exp);
    const float q = a / ulp;        /* exact: power-of-two scaling */
    float r = rintf(q);             /* round half to even (default rounding mode) */
    return copysignf(r * ulp, f);
}

void hso_round_f16(float* x, size_t n) {
    for (size_t i = 0; i < n; ++i) x[i] = f16_round(x[i]);
}

/* ------------------------------------------------------------------------ */
/* Pruner: pruner.hpp:40-176.                                                 */
/* ------------------------------------------------------------------------ */

/* Per-group top-2 of 4 (element_mask, pruner.hpp:53-74 / fused path
 * compressed_cache.hpp:244-258): stable sort by |x| descending, keep the first
 * two, report positions ascending.  Equivalent rank rule: element i is kept
 * iff #{j : |x_j| > |x_i|} + #{j < i : |x_j| == |x_i|} < 2. */
static void top2_of_4(const float g[4], int kept[2]) {
    int n = 0;
    for (int i = 0; i < 4; ++i) {
        const float ai = fabsf(g[i]);
        int rank = 0;
        for (int j = 0; j < 4; ++j) {
            const float aj = fabsf(g[j]);
            if (aj > ai || (j < i && !(aj > ai) && !(ai > aj))) ++rank;
        }
        if (rank < 2 && n < 2) kept[n++] = i;
    }
}

/* Block selection (select_blocks, pruner.hpp:94-117): among non-protected
 * blocks, floor(S * prunable) lowest-loss blocks become sparse; the stable
 * sort's tie rule is "lower block index first". */
static int cmp_loss_idx(const void* a, const void* b, const double* losses) {
    const size_t ia = *(const size_t*)a, ib = *(const size_t*)b;
    if (losses[ia] < losses[ib]) return -1;
    if (losses[ib] < losses[ia]) return 1;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

static _Thread_local const double* g_sort_losses;
static int cmp_qsort(const void* a, const void* b) { return cmp_loss_idx(a, b, g_sort_losses); }

static int select_blocks(const double* losses, size_t total, double target, size_t prefix,
                         size_t suffix, uint8_t* flags) {
    CHECK_CONFIG(target >= 0.0 && target <= 1.0, "select_blocks: sparsity outside [0, 1]");
    CHECK_CONFIG(prefix + suffix <= total, "select_blocks: protected regions exceed block count");
    for (size_t b = 0; b < total; ++b) flags[b] = 1;
    const size_t prunable = total - prefix - suffix;
    const size_t quota = (size_t)floor(target * (double)prunable);
    if (quota == 0) return HSO_OK;
    size_t* cand = (size_t*)malloc(prunable * sizeof(size_t));
    for (size_t i = 0; i < prunable; ++i) cand[i] = prefix + i;
    /* qsort with the index tie-break reproduces std::stable_sort's order; the
     * comparator reads the losses through a thread-local pointer. */
    g_sort_losses = losses;
    qsort(cand, prunable, sizeof(size_t), cmp_qsort);
    for (size_t i = 0; i < quota; ++i) flags[cand[i]] = 0;
    free(cand);
    return HSO_OK;
}

int hso_pool_counts(size_t rows, size_t block_size, double sparsity, size_t sink_tokens,
                    size_t local_window, size_t* prefix, size_t* suffix, size_t* quota) {
    CHECK_CONFIG(block_size > 0 && block_size % 4 == 0,
                 "SparsityConfig: block_size must be a positive multiple of m_group");
    CHECK_CONFIG(sparsity >= 0.0 && sparsity <= 1.0, "SparsityConfig: sparsity outside [0, 1]");
    CHECK_CONFIG(rows % block_size == 0,
                 "prune_cache: sequence length not divisible by block_size");
    const size_t nblocks = rows / block_size;
    /* masks.hpp:93-98 rounding, pruner.hpp:130-131 clamping. */
    size_t p = (sink_tokens + block_size - 1) / block_size;
    size_t s = (local_window + block_size - 1) / block_size;
    if (p > nblocks) p = nblocks;
    if (s > nblocks - p) s = nblocks - p;
    *prefix = p;
    *suffix = s;
    *quota = (size_t)floor(sparsity * (double)(nblocks - p - s));
    return HSO_OK;
}

/* Logical (row, col) of the i-th element of group g in stored row sr of block b
 * (compressed_cache.hpp:203-207 / :247-249). */
static inline void group_elem(int axis, size_t B, size_t b, size_t sr, size_t g, size_t i,
                              size_t* lr, size_t* lc) {
    if (axis == 0) {
        *lr = b * B + sr;
        *lc = g * 4 + i;
    } else {
        *lr = b * B + g * 4 + i;
        *lc = sr;
    }
}

/* assemble_cache (compressed_cache.hpp:133-188) specialised to the fused
 * magnitude path (:232-267): blocks in order, dense blocks copied in stored
 * layout (value cache transposed), sparse blocks keep each group's top-2 and
 * pack 2-bit codes (nm_metadata.hpp:63-88). */
static int assemble(const float* x, size_t rows, size_t cols, size_t B, int axis,
                    const uint8_t* flags, const uint8_t* emask, hso_cache* c) {
    CHECK_CONFIG(B > 0 && B % 4 == 0,
                 "SparsityConfig: block_size must be a positive multiple of m_group");
    CHECK_CONFIG(rows % B == 0, "compress: sequence length not divisible by block_size");
    CHECK_CONFIG(((axis == 0) ? cols : B) % 4 == 0,
                 "compress: grouping axis not divisible by m_group");
    const size_t nblocks = rows / B;
    const size_t srows = axis == 0 ? B : cols;
    const size_t scols = axis == 0 ? cols : B;
    const size_t belems = B * cols;
    const size_t words = (belems / 4 * 2 + 7) / 8;
    c->axis = axis;
    c->head_dim = cols;
    c->block_size = B;
    c->logical_blocks = nblocks;
    c->dense_count = 0;
    c->sparse_count = 0;
    for (size_t b = 0; b < nblocks; ++b) {
        if (flags[b]) {
            CHECK_CONFIG(c->dense_count < 32767, "compress: dense pool exceeds int16 index capacity");
            float* dst = c->dense_pool + c->dense_count * belems;
            for (size_t sr = 0; sr < srows; ++sr)
                for (size_t sc = 0; sc < scols; ++sc) {
                    const size_t lr = axis == 0 ? sr : sc, lc = axis == 0 ? sc : sr;
                    dst[sr * scols + sc] = x[(b * B + lr) * cols + lc];
                }
            ++c->dense_count;
            c->index_map[b] = (int16_t)c->dense_count;
        } else {
            CHECK_CONFIG(c->sparse_count < 32767, "compress: sparse pool exceeds int16 index capacity");
            float* nnz = c->nnz_pool + c->sparse_count * (belems / 2);
            uint16_t* meta = c->meta_pool + c->sparse_count * words;
            memset(meta, 0, words * sizeof(uint16_t));
            size_t code = 0, v = 0;
            for (size_t sr = 0; sr < srows; ++sr) {
                for (size_t g = 0; g < scols / 4; ++g) {
                    float grp[4];
                    for (size_t i = 0; i < 4; ++i) {
                        size_t lr, lc;
                        group_elem(axis, B, b, sr, g, i, &lr, &lc);
                        grp[i] = x[lr * cols + lc];
                    }
                    int kept[2];
                    if (emask) {
                        /* compress (compressed_cache.hpp:208-223): the mask's kept
                         * elements in ascending position; exactly n_keep = 2 */
                        int n = 0;
                        for (size_t i = 0; i < 4; ++i) {
                            size_t lr, lc;
                            group_elem(axis, B, b, sr, g, i, &lr, &lc);
                            if (emask[lr * cols + lc]) {
                                if (n >= 2) return fail(HSO_DATA, "compress: group keeps more than n_keep elements");
                                kept[n++] = (int)i;
                            }
                        }
                        if (n != 2) return fail(HSO_DATA, "compress: group keeps fewer than n_keep elements");
                    } else {
                        top2_of_4(grp, kept);
                    }
                    for (int i = 0; i < 2; ++i) {
                        nnz[v++] = grp[kept[i]];
                        meta[code / 8] |= (uint16_t)(kept[i] << (2 * (code % 8)));
                        ++code;
                    }
                }
            }
            ++c->sparse_count;
            c->index_map[b] = (int16_t)(-(int)c->sparse_count);
        }
    }
    return HSO_OK;
}

/* hierarchical_mask_for (pruner.hpp:121-158) for one cache, followed by
 * compress / fused_magnitude_compress (compressed_cache.hpp:196-267; the two
 * are field-identical, test_compressor.cpp:114-134).  The per-block loss is
 * block_loss (pruner.hpp:81-89): double sum of pruned |x| in the logical
 * row-major order of the block. */
int hso_prune_compress(const float* x, size_t rows, size_t cols, const hso_config* cfg,
                       int axis, double sparsity, int fused, hso_cache* out, uint8_t* flags,
                       double* losses, uint8_t* element_mask) {
    (void)fused;
    const size_t B = cfg->block_size;
    CHECK_CONFIG(cfg->s_key >= 0.0 && cfg->s_key <= 1.0, "SparsityConfig: s_key outside [0, 1]");
    CHECK_CONFIG(cfg->s_value >= 0.0 && cfg->s_value <= 1.0,
                 "SparsityConfig: s_value outside [0, 1]");
    CHECK_CONFIG(B > 0 && B % 4 == 0,
                 "SparsityConfig: block_size must be a positive multiple of m_group");
    CHECK_CONFIG(cols % 4 == 0, "prune_cache: head dimension not divisible by m_group");
    CHECK_CONFIG(rows % B == 0, "prune_cache: sequence length not divisible by block_size");
    size_t prefix, suffix, quota;
    int rc = hso_pool_counts(rows, B, sparsity, cfg->sink_tokens, cfg->local_window, &prefix,
                             &suffix, &quota);
    if (rc) return rc;
    const size_t nblocks = rows / B;
    uint8_t* keep = (uint8_t*)malloc(B * cols);
    for (size_t b = 0; b < nblocks; ++b) {
        /* element_mask over the block (pruner.hpp:40-77). */
        memset(keep, 0, B * cols);
        const size_t lanes = axis == 0 ? B : cols;
        const size_t groups = (axis == 0 ? cols : B) / 4;
        for (size_t lane = 0; lane < lanes; ++lane) {
            for (size_t g = 0; g < groups; ++g) {
                float grp[4];
                for (size_t i = 0; i < 4; ++i) {
                    const size_t off = g * 4 + i;
                    grp[i] = axis == 0 ? x[(b * B + lane) * cols + off]
                                       : x[(b * B + off) * cols + lane];
                }
                int kept[2];
                top2_of_4(grp, kept);
                for (int i = 0; i < 2; ++i) {
                    const size_t off = g * 4 + (size_t)kept[i];
                    if (axis == 0) keep[lane * cols + off] = 1;
                    else keep[off * cols + lane] = 1;
                }
            }
        }
        /* block_loss (pruner.hpp:81-89). */
        double loss = 0.0;
        for (size_t i = 0; i < B * cols; ++i)
            if (!keep[i]) loss += fabs((double)x[b * B * cols + i]);
        losses[b] = loss;
        if (element_mask) memcpy(element_mask + b * B * cols, keep, B * cols);
    }
    free(keep);
    rc = select_blocks(losses, nblocks, sparsity, prefix, suffix, flags);
    if (rc) return rc;
    if (element_mask) {
        /* dense blocks keep every element (pruner.hpp:150-157). */
        for (size_t b = 0; b < nblocks; ++b)
            if (flags[b]) memset(element_mask + b * B * cols, 1, B * cols);
    }
    return assemble(x, rows, cols, B, axis, flags, NULL, out);
}

/* fused_magnitude_compress (compressed_cache.hpp:262-267) under a given
 * block mask. */
int hso_compress_with_flags(const float* x, size_t rows, size_t cols, const hso_config* cfg,
                            int axis, const uint8_t* flags, hso_cache* out) {
    return assemble(x, rows, cols, cfg->block_size, axis, flags, NULL, out);
}

/* compress (compressed_cache.hpp:196-225) under an explicit element mask
 * (u8 [rows][cols], nonzero = kept) and block mask. */
int hso_compress_with_mask(const float* x, size_t rows, size_t cols, const hso_config* cfg,
                           int axis, const uint8_t* element_mask, const uint8_t* flags, hso_cache* out) {
    return assemble(x, rows, cols, cfg->block_size, axis, flags, element_mask, out);
}

/* ------------------------------------------------------------------------ */
/* Storage access: compressed_cache.hpp:62-110, nm_metadata.hpp:92-143.       */
/* ------------------------------------------------------------------------ */

static size_t stored_rows(const hso_cache* c) { return c->axis == 0 ? c->block_size : c->head_dim; }
static size_t stored_cols(const hso_cache* c) { return c->axis == 0 ? c->head_dim : c->block_size; }
static size_t block_elems(const hso_cache* c) { return c->block_size * c->head_dim; }
static size_t meta_words(const hso_cache* c) { return (block_elems(c) / 4 * 2 + 7) / 8; }

/* expand_stored_block (compressed_cache.hpp:106-109): unpack_metadata
 * (nm_metadata.hpp:92-112, rejecting non-increasing codes) and scatter. */
static int expand_block(const hso_cache* c, size_t slot, float* dense) {
    CHECK_DATA(slot < c->sparse_count, "nnz_block: slot past the sparse pool");
    const size_t sr = stored_rows(c), sc = stored_cols(c);
    const float* nnz = c->nnz_pool + slot * (block_elems(c) / 2);
    const uint16_t* meta = c->meta_pool + slot * meta_words(c);
    memset(dense, 0, sr * sc * sizeof(float));
    size_t code = 0;
    for (size_t r = 0; r < sr; ++r) {
        for (size_t g = 0; g < sc / 4; ++g) {
            int prev = -1;
            for (int i = 0; i < 2; ++i, ++code) {
                const int pos = (meta[code / 8] >> (2 * (code % 8))) & 3;
                CHECK_DATA(i == 0 || pos > prev,
                           "unpack_metadata: corrupt metadata, codes not increasing");
                prev = pos;
                dense[r * sc + g * 4 + (size_t)pos] = nnz[r * (sc / 2) + g * 2 + (size_t)i];
            }
        }
    }
    return HSO_OK;
}

/* Stored-layout dense-equivalent of block b (dense_block or expanded). */
static int stored_block(const hso_cache* c, size_t b, int dense, float* out) {
    const int16_t e = c->index_map[b];
    CHECK_DATA(e != 0, "block_slot: index map holds a zero entry");
    const size_t slot = (size_t)((e > 0 ? e : -e) - 1);
    if (dense) {
        CHECK_DATA(slot < c->dense_count, "dense_block: slot past the dense pool");
        memcpy(out, c->dense_pool + slot * block_elems(c), block_elems(c) * sizeof(float));
        return HSO_OK;
    }
    return expand_block(c, slot, out);
}

/* decompress (compressed_cache.hpp:271-298). */
int hso_decompress(const hso_cache* c, float* out) {
    const size_t B = c->block_size, d = c->head_dim;
    float* st = (float*)malloc(B * d * sizeof(float));
    for (size_t b = 0; b < c->logical_blocks; ++b) {
        const int16_t e = c->index_map[b];
        if (e == 0) { free(st); return fail(HSO_DATA, "decompress: index map holds a zero entry"); }
        const size_t slot = (size_t)((e > 0 ? e : -e) - 1);
        if (e > 0 && slot >= c->dense_count) { free(st); return fail(HSO_DATA, "decompress: dangling dense offset"); }
        if (e < 0 && slot >= c->sparse_count) { free(st); return fail(HSO_DATA, "decompress: dangling sparse offset"); }
        int rc = stored_block(c, b, e > 0, st);
        if (rc) { free(st); return rc; }
        const size_t sr = stored_rows(c), sc = stored_cols(c);
        for (size_t r = 0; r < sr; ++r)
            for (size_t cc = 0; cc < sc; ++cc) {
                const size_t lr = c->axis == 0 ? r : cc, lc = c->axis == 0 ? cc : r;
                out[(b * B + lr) * d + lc] = st[r * sc + cc];
            }
    }
    free(st);
    return HSO_OK;
}

/* ------------------------------------------------------------------------ */
/* Attention engine: attention.hpp:84-409.                                    */
/* ------------------------------------------------------------------------ */

static inline float fmaxref(float a, float b) { return (a < b) ? b : a; } /* std::max */

/* matmul (tensor.hpp:35-50): c[i][j] += a[i][k]*b[k][j], k ascending, c from 0. */
static void matmul(const float* a, size_t ar, size_t ac, const float* b, size_t bc, float* c) {
    memset(c, 0, ar * bc * sizeof(float));
    for (size_t i = 0; i < ar; ++i) {
        const float* arow = a + i * ac;
        float* crow = c + i * bc;
        for (size_t k = 0; k < ac; ++k) {
            const float aik = arow[k];
            const float* brow = b + k * bc;
            for (size_t j = 0; j < bc; ++j) crow[j] += aik * brow[j];
        }
    }
}

/* dense_attention_oracle (attention.hpp:84-115). */
int hso_dense_attention(const float* q, size_t n_q, const float* k, const float* v, size_t n_kv,
                        size_t d, int causal, float scale, float* out) {
    CHECK_CONFIG(n_kv > 0, "oracle: empty key sequence");
    CHECK_CONFIG(!causal || n_kv >= n_q, "oracle: causal queries exceed key sequence");
    float* kt = (float*)malloc(d * n_kv * sizeof(float));
    for (size_t i = 0; i < n_kv; ++i)
        for (size_t j = 0; j < d; ++j) kt[j * n_kv + i] = k[i * d + j];
    float* s = (float*)malloc(n_q * n_kv * sizeof(float));
    matmul(q, n_q, d, kt, n_kv, s);
    const size_t offset = n_kv - n_q;
    for (size_t i = 0; i < n_q; ++i)
        for (size_t j = 0; j < n_kv; ++j) {
            if (causal && j > offset + i) s[i * n_kv + j] = -INFINITY;
            else s[i * n_kv + j] *= scale;
        }
    for (size_t i = 0; i < n_q; ++i) {
        float m = -INFINITY;
        for (size_t j = 0; j < n_kv; ++j) m = fmaxref(m, s[i * n_kv + j]);
        float l = 0.0f;
        for (size_t j = 0; j < n_kv; ++j) {
            const float p = expf(s[i * n_kv + j] - m);
            s[i * n_kv + j] = p;
            l += p;
        }
        for (size_t j = 0; j < n_kv; ++j) s[i * n_kv + j] /= l;
    }
    matmul(s, n_q, n_kv, v, d, out);
    free(kt);
    free(s);
    return HSO_OK;
}

/* block_dense with DispatchPolicy::kAuto (attention.hpp:160-167). */
static int block_is_dense(const hso_cache* c, size_t b, int* dense) {
    if (c->sparse_count == 0) { *dense = 1; return HSO_OK; }
    if (c->dense_count == 0) { *dense = 0; return HSO_OK; }
    CHECK_DATA(c->index_map[b] != 0, "attention: index map holds a zero entry");
    *dense = c->index_map[b] > 0;
    return HSO_OK;
}

typedef struct {
    float* running_max; /* [rows] */
    float* running_sum; /* [rows] */
    float* acc_t;       /* [d][rows] */
} softmax_state;

/* online_softmax_update (attention.hpp:171-239).  scores_t is keys x rows;
 * vt is the value operand V^T as a dense d x keys matrix. */
static void softmax_update(softmax_state* st, float* scores_t, size_t kkeys, size_t rows,
                           size_t d, size_t key_start, float scale, const int64_t* qpos,
                           const float* vt, float* alpha, float* contrib) {
    for (size_t kk = 0; kk < kkeys; ++kk)
        for (size_t q = 0; q < rows; ++q) {
            if (qpos && (int64_t)(key_start + kk) > qpos[q]) scores_t[kk * rows + q] = -INFINITY;
            else scores_t[kk * rows + q] *= scale;
        }
    for (size_t q = 0; q < rows; ++q) {
        alpha[q] = 1.0f;
        float block_max = -INFINITY;
        for (size_t kk = 0; kk < kkeys; ++kk) block_max = fmaxref(block_max, scores_t[kk * rows + q]);
        const float m_new = fmaxref(st->running_max[q], block_max);
        if (m_new == -INFINITY) {
            for (size_t kk = 0; kk < kkeys; ++kk) scores_t[kk * rows + q] = 0.0f;
            alpha[q] = 1.0f;
            continue;
        }
        float row_sum = 0.0f;
        for (size_t kk = 0; kk < kkeys; ++kk) {
            const float p = expf(scores_t[kk * rows + q] - m_new);
            scores_t[kk * rows + q] = p;
            row_sum += p;
        }
        alpha[q] = expf(st->running_max[q] - m_new);
        st->running_sum[q] = st->running_sum[q] * alpha[q] + row_sum;
        st->running_max[q] = m_new;
    }
    for (size_t dd = 0; dd < d; ++dd)
        for (size_t q = 0; q < rows; ++q) st->acc_t[dd * rows + q] *= alpha[q];
    matmul(vt, d, kkeys, scores_t, rows, contrib);
    for (size_t i = 0; i < d * rows; ++i) st->acc_t[i] += contrib[i];
}

static int check_view_pair(const hso_cache* k, const hso_cache* v) {
    const size_t kb = k ? k->logical_blocks : 0, vb = v ? v->logical_blocks : 0;
    const size_t kt = k ? k->logical_blocks * k->block_size : 0;
    const size_t vt = v ? v->logical_blocks * v->block_size : 0;
    CHECK_CONFIG(kt == vt, "attention: key/value token counts differ");
    CHECK_CONFIG(kb == vb, "attention: key/value block counts differ");
    if (k) CHECK_CONFIG(k->axis == 0, "attention: key cache must be channel-grouped");
    if (v) CHECK_CONFIG(v->axis == 1, "attention: value cache must be sequence-grouped");
    if (k && v) CHECK_CONFIG(k->block_size == v->block_size, "attention: key/value block sizes differ");
    return HSO_OK;
}

/* attend_range (attention.hpp:249-304): online softmax over blocks
 * [block_begin, block_end) plus the dense tail, with the block-causal skip. */
int hso_attend_rows(const float* q, size_t rows, size_t d, const hso_cache* k,
                    const hso_cache* v, const float* k_tail, const float* v_tail, size_t tail,
                    size_t block_begin, size_t block_end, int include_tail, float scale,
                    const int64_t* qpos, float* out_t, float* m_s, float* l_s) {
    int rc = check_view_pair(k, v);
    if (rc) return rc;
    const size_t nblocks = k ? k->logical_blocks : 0;
    CHECK_CONFIG(block_end <= nblocks && block_begin <= block_end,
                 "attend_range: block range out of bounds");
    const size_t B = k ? k->block_size : 0;
    softmax_state st = {m_s, l_s, out_t};
    for (size_t r = 0; r < rows; ++r) { m_s[r] = -INFINITY; l_s[r] = 0.0f; }
    memset(out_t, 0, d * rows * sizeof(float));
    float* q_t = (float*)malloc(d * rows * sizeof(float));
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < d; ++c) q_t[c * rows + r] = q[r * d + c];
    int64_t qpos_max = -1;
    if (qpos)
        for (size_t r = 0; r < rows; ++r) if (qpos[r] > qpos_max) qpos_max = qpos[r];
    const size_t maxk = (B > tail ? B : tail) + 1;
    float* kblk = (float*)malloc(maxk * d * sizeof(float));
    float* vblk = (float*)malloc(maxk * d * sizeof(float));
    float* scores = (float*)malloc(maxk * rows * sizeof(float));
    float* contrib = (float*)malloc(d * rows * sizeof(float));
    float* alpha = (float*)malloc((rows + 1) * sizeof(float));
    for (size_t b = block_begin; b < block_end && rc == HSO_OK; ++b) {
        const size_t key_start = b * B;
        if (qpos && (int64_t)key_start > qpos_max) continue;
        int kd, vd;
        if ((rc = block_is_dense(k, b, &kd))) break;
        if ((rc = stored_block(k, b, kd, kblk))) break; /* [B][d] */
        matmul(kblk, B, d, q_t, rows, scores);
        if ((rc = block_is_dense(v, b, &vd))) break;
        if ((rc = stored_block(v, b, vd, vblk))) break; /* [d][B] */
        softmax_update(&st, scores, B, rows, d, key_start, scale, qpos, vblk, alpha, contrib);
    }
    if (rc == HSO_OK && include_tail && tail > 0) {
        const size_t key_start = nblocks * B;
        if (!qpos || (int64_t)key_start <= qpos_max) {
            matmul(k_tail, tail, d, q_t, rows, scores);
            for (size_t t = 0; t < tail; ++t)
                for (size_t c = 0; c < d; ++c) vblk[c * tail + t] = v_tail[t * d + c];
            softmax_update(&st, scores, tail, rows, d, key_start, scale, qpos, vblk, alpha, contrib);
        }
    }
    free(q_t); free(kblk); free(vblk); free(scores); free(contrib); free(alpha);
    return rc;
}

/* decode_attention (attention.hpp:360-409): contiguous split ranges, LSE combine. */
int hso_decode(const float* q, size_t n_q, size_t d, const hso_cache* k, const hso_cache* v,
               const float* k_tail, const float* v_tail, size_t tail, float scale,
               size_t splits, size_t gqa_group, float* out) {
    int rc = check_view_pair(k, v);
    if (rc) return rc;
    CHECK_CONFIG(n_q >= 1, "decode_attention: no query rows");
    CHECK_CONFIG(gqa_group == 0 || n_q == gqa_group,
                 "decode_attention: one query row per head in the GQA group");
    const size_t nblocks = k ? k->logical_blocks : 0;
    CHECK_CONFIG(nblocks * (k ? k->block_size : 0) + tail > 0, "decode_attention: empty cache");
    size_t ns = splits < 1 ? 1 : splits;
    const size_t cap = nblocks < 1 ? 1 : nblocks;
    if (ns > cap) ns = cap;
    float* ot = (float*)malloc(ns * d * n_q * sizeof(float));
    float* ms = (float*)malloc(ns * n_q * sizeof(float));
    float* ls = (float*)malloc(ns * n_q * sizeof(float));
    for (size_t s = 0; s < ns && rc == HSO_OK; ++s) {
        const size_t begin = nblocks * s / ns, end = nblocks * (s + 1) / ns;
        rc = hso_attend_rows(q, n_q, d, k, v, k_tail, v_tail, tail, begin, end, s + 1 == ns,
                             scale, NULL, ot + s * d * n_q, ms + s * n_q, ls + s * n_q);
    }
    float* w = (float*)malloc(ns * sizeof(float));
    for (size_t qq = 0; qq < n_q && rc == HSO_OK; ++qq) {
        float m = -INFINITY;
        for (size_t s = 0; s < ns; ++s) m = fmaxref(m, ms[s * n_q + qq]);
        float l = 0.0f;
        for (size_t s = 0; s < ns; ++s) {
            w[s] = expf(ms[s * n_q + qq] - m);
            l += ls[s * n_q + qq] * w[s];
        }
        if (!(l > 0.0f)) { rc = fail(HSO_DATA, "decode_attention: query row attends no keys"); break; }
        for (size_t dd = 0; dd < d; ++dd) {
            float acc = 0.0f;
            for (size_t s = 0; s < ns; ++s) acc += ot[s * d * n_q + dd * n_q + qq] * w[s];
            out[qq * d + dd] = acc / l;
        }
    }
    free(ot); free(ms); free(ls); free(w);
    return rc;
}

/* prefill_attention (attention.hpp:323-354) + finalize_rows (:309-317). */
int hso_prefill(const float* q, size_t n_q, size_t d, const hso_cache* k, const hso_cache* v,
                const float* k_tail, const float* v_tail, size_t tail, int causal, float scale,
                size_t b_r, float* out) {
    int rc = check_view_pair(k, v);
    if (rc) return rc;
    CHECK_CONFIG(b_r > 0, "prefill_attention: b_r must be positive");
    const size_t n_kv = (k ? k->logical_blocks * k->block_size : 0) + tail;
    CHECK_CONFIG(n_kv > 0, "prefill_attention: empty key/value cache");
    CHECK_CONFIG(!causal || n_kv >= n_q, "prefill_attention: causal queries exceed key sequence");
    const size_t nblocks = k ? k->logical_blocks : 0;
    float* ot = (float*)malloc(d * b_r * sizeof(float));
    float* ms = (float*)malloc(b_r * sizeof(float));
    float* ls = (float*)malloc(b_r * sizeof(float));
    int64_t* qpos = (int64_t*)malloc(b_r * sizeof(int64_t));
    for (size_t t0 = 0; t0 < n_q && rc == HSO_OK; t0 += b_r) {
        const size_t t1 = t0 + b_r < n_q ? t0 + b_r : n_q, rows = t1 - t0;
        for (size_t i = 0; i < rows; ++i) qpos[i] = (int64_t)(n_kv - n_q + t0 + i);
        rc = hso_attend_rows(q + t0 * d, rows, d, k, v, k_tail, v_tail, tail, 0, nblocks, 1,
                             scale, causal ? qpos : NULL, ot, ms, ls);
        for (size_t r = 0; r < rows && rc == HSO_OK; ++r) {
            if (!(ls[r] > 0.0f)) { rc = fail(HSO_DATA, "attention: query row attends no visible keys"); break; }
            for (size_t dd = 0; dd < d; ++dd) out[(t0 + r) * d + dd] = ot[dd * rows + r] / ls[r];
        }
    }
    free(ot); free(ms); free(ls); free(qpos);
    return rc;
}

/* flop_and_byte_count (attention.hpp:426-467) with the 38-byte container
 * header (container.hpp:42) and measure_size (compressed_cache.hpp:303-310). */
int hso_flop_and_byte_count(size_t n_q, size_t d, const hso_cache* k, const hso_cache* v,
                            size_t tail, int causal, uint64_t* flops, uint64_t* bytes) {
    const size_t nblocks = k ? k->logical_blocks : 0;
    const size_t B = k ? k->block_size : 0;
    const size_t prefix = nblocks * B;
    const size_t n_kv = prefix + tail;
    uint64_t f = 0;
    for (size_t i = 0; i < n_q; ++i) {
        const size_t visible = causal ? (n_kv - n_q + i + 1) : n_kv;
        for (size_t b = 0; b < nblocks; ++b) {
            const size_t start = b * B;
            if (start >= visible) break;
            const uint64_t width = (B < visible - start) ? B : visible - start;
            int kd, vd;
            int rc = block_is_dense(k, b, &kd);
            if (rc) return rc;
            rc = block_is_dense(v, b, &vd);
            if (rc) return rc;
            f += width * d * (kd ? 2 : 1);
            f += width * d * (vd ? 2 : 1);
        }
        if (visible > prefix) f += 2 * (uint64_t)(visible - prefix) * d * 2;
    }
    uint64_t by = 0;
    const hso_cache* views[2] = {k, v};
    for (int i = 0; i < 2; ++i) {
        const hso_cache* c = views[i];
        if (c) {
            by += 38;
            by += (uint64_t)c->logical_blocks * 2;
            by += (uint64_t)c->dense_count * block_elems(c) * 2;
            by += (uint64_t)c->sparse_count * (block_elems(c) / 2) * 2;
            by += (uint64_t)c->sparse_count * meta_words(c) * 2;
        }
        by += (uint64_t)tail * d * 2;
    }
    *flops = f;
    *bytes = by;
    return HSO_OK;
}
