// Probe: tcgen05 operand/metadata layouts on B200 (sm_100a).
//  T1 dense  M128 N128 K64,  A K-major SW128, B K-major SW128
//  T2 sparse M128 N128 K128, A compressed K-major SW128, metadata via tcgen05.cp (E atom)
//  T3 sparse  same, metadata via tcgen05.st (register layout)
//  T4 dense  M128 N128 K64,  B MN-major SW128 (the P^T operand of GEMM2)
//  T5 sparse M128 N128 K64,  A compressed K-major SW64 (the V^T nnz tile), tcgen05.st metadata
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include "../../paper_2604_16864_b200/csrc/common.cuh"

using namespace hs;

// element offsets in swizzled K-major tiles (16-bit elements)
__device__ __forceinline__ uint32_t off_k128(int r, int k) {  // rows of 128 B
    return r * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2;
}
__device__ __forceinline__ uint32_t off_k64(int r, int k) {   // rows of 64 B
    return r * 64 + (((k >> 3) ^ ((r >> 1) & 3)) << 4) + (k & 7) * 2;
}

struct Args {
    int test;
    const uint16_t* A;     // logical A [128][K] bf16 (dense) or compressed nnz [128][K/2]
    const uint16_t* meta;  // canonical meta [128][K/16] u16
    const uint16_t* B;     // logical B [N=128][K] bf16 (B[n][k])
    int K;                 // logical K
    float* D;              // [128][128]
};

__global__ void __launch_bounds__(128) probe(Args a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    uint8_t* sA = base;            // 32 KB
    uint8_t* sB = base + 32768;    // 32 KB
    uint8_t* sE = base + 65536;    // 2 KB
    const int K = a.K;
    const bool sparse = a.test == 2 || a.test == 3 || a.test == 5 || a.test == 6;
    // ---- fill A
    if (!sparse) {
        for (int i = tid; i < 128 * K; i += 128) {  // K == 64
            const int r = i / K, k = i % K;
            *reinterpret_cast<uint16_t*>(sA + off_k128(r, k)) = a.A[i];
        }
    } else {
        const int kp = K / 2;  // physical columns
        for (int i = tid; i < 128 * kp; i += 128) {
            const int r = i / kp, k = i % kp;
            const uint32_t o = (a.test >= 5) ? off_k64(r, k) : off_k128(r, k);
            *reinterpret_cast<uint16_t*>(sA + o) = a.A[i];
        }
    }
    // ---- fill B
    if (a.test == 4) {  // MN-major: [K rows][N]; N atoms of 64 at LBO = K*128 bytes
        for (int i = tid; i < 128 * K; i += 128) {
            const int n = i / K, k = i % K;
            const uint32_t o = (n / 64) * (K * 128) + k * 128 + ((((n % 64) >> 3) ^ (k & 7)) << 4) + (n & 7) * 2;
            *reinterpret_cast<uint16_t*>(sB + o) = a.B[i];
        }
    } else {  // K-major: [N rows][K] in K-atoms of 64 elements, atom stride 128*128 B
        for (int i = tid; i < 128 * K; i += 128) {
            const int n = i / K, k = i % K;
            const uint32_t o = (k / 64) * 16384 + off_k128(n, k % 64);
            *reinterpret_cast<uint16_t*>(sB + o) = a.B[i];
        }
    }
    // ---- E atom (T2): u16 index 8*(m&7) + ((m>>3)&1) + 128*(m>>4) + 64*(w&1) + 2*(w>>1)
    if (a.test == 2) {
        const int words = K / 16;
        for (int i = tid; i < 128 * words; i += 128) {
            const int m = i / words, w = i % words;
            const int idx = 8 * (m & 7) + ((m >> 3) & 1) + 128 * (m >> 4) + 64 * (w & 1) + 2 * (w >> 1);
            reinterpret_cast<uint16_t*>(sE)[idx] = a.meta[i];
        }
    }
    if (warp == 0) tmem_alloc(&tbase, 256);
    if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tD = tbase, tE = tbase + 128;
    // ---- T3/T5: metadata via tcgen05.st, lane L = m0 + 8*k1 + 16*m2, column j = k-step
    if (a.test == 3 || a.test >= 5) {
        const int L = tid, m0 = L & 7, k1 = (L >> 3) & 1, m2 = L >> 4;
        const int rlo = m0 + 16 * m2, rhi = rlo + 8, words = K / 16;
        uint32_t v[4] = {0, 0, 0, 0};
        for (int j = 0; j < K / 32; ++j) {
            const int w = 2 * j + k1;
            v[j] = a.meta[rlo * words + w] | (static_cast<uint32_t>(a.meta[rhi * words + w]) << 16);
        }
        tmem_st4(tE + ((32 * warp) << 16), v[0], v[1], v[2], v[3]);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        uint32_t idesc = umma_idesc_f16(true, 128, 128, false, a.test == 4, sparse);
        if (a.test == 6) idesc &= ~(7u << 10);  // B format = F16
        if (a.test == 2) tmem_cp_128x128b(tE, umma_desc(smem_u32(sE), 16, 128, kLayoutNone));
        if (!sparse) {
            for (int j = 0; j < K / 16; ++j) {
                const uint64_t ad = umma_desc(smem_u32(sA) + 32 * j, 16, 1024, kLayoutSW128);
                uint64_t bd;
                if (a.test == 4) bd = umma_desc(smem_u32(sB) + 2048 * j, K * 128, 1024, kLayoutSW128);
                else bd = umma_desc(smem_u32(sB) + 32 * j, 16, 1024, kLayoutSW128);
                umma_f16(tD, ad, bd, idesc, j > 0);
            }
        } else {
            for (int j = 0; j < K / 32; ++j) {
                const uint64_t ad = (a.test >= 5) ? umma_desc(smem_u32(sA) + 32 * j, 16, 512, kLayoutSW64)
                                                  : umma_desc(smem_u32(sA) + 32 * j, 16, 1024, kLayoutSW128);
                const uint64_t bd = umma_desc(smem_u32(sB) + (j / 2) * 16384 + (j % 2) * 64, 16, 1024, kLayoutSW128);
                umma_sp_f16(tD, ad, bd, tE + j, idesc, j > 0);
            }
        }
        umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tD + ((32 * warp) << 16) + 32 * c, r);
        tmem_ld_wait();
        for (int x = 0; x < 32; ++x) a.D[(32 * warp + lane) * 128 + 32 * c + x] = __uint_as_float(r[x]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 256);
}

static uint16_t bf(float x) { uint32_t u; memcpy(&u, &x, 4); u += 0x7FFF + ((u >> 16) & 1); return u >> 16; }
static float fb(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }

int main(int argc, char** argv) {
    srand(7);
    const int only = argc > 1 ? atoi(argv[1]) : 0;
    const char* names[] = {"", "T1 dense K-major SW128", "T2 sparse SW128 meta tcgen05.cp", "T3 sparse SW128 meta tcgen05.st",
                           "T4 dense B MN-major SW128", "T5 sparse A SW64 meta tcgen05.st", "T6 mixed A bf16 x B f16"};
    float* dD; uint16_t *dA, *dB, *dM;
    cudaMalloc(&dD, 128 * 128 * 4); cudaMalloc(&dA, 128 * 128 * 2); cudaMalloc(&dB, 128 * 128 * 2); cudaMalloc(&dM, 128 * 16 * 2);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int test = 1; test <= 6; ++test) {
        if (only && test != only) { for (int i = 0; i < 3; ++i) rand(); continue; }
        const bool sparse = test == 2 || test == 3 || test >= 5;
        const int K = (test == 1 || test >= 4) ? 64 : 128;
        std::vector<float> A(128 * K), B(128 * K);
        std::vector<uint16_t> Ab, Bb(128 * K), meta(128 * K / 16, 0);
        for (int i = 0; i < 128 * K; ++i) B[i] = fb(bf((rand() % 2001 - 1000) / 500.0f));
        for (auto& x : B) {}
        for (int i = 0; i < 128 * K; ++i) Bb[i] = bf(B[i]);
        if (test == 6) for (int i = 0; i < 128 * K; ++i) { float x = (rand() % 2001 - 1000) / 512.0f; B[i] = x; __half h = __float2half_rn(x); B[i] = __half2float(h); memcpy(&Bb[i], &h, 2); }
        if (!sparse) {
            for (int i = 0; i < 128 * K; ++i) { A[i] = fb(bf((rand() % 2001 - 1000) / 500.0f)); Ab.push_back(bf(A[i])); }
        } else {
            for (int r = 0; r < 128; ++r)
                for (int g = 0; g < K / 4; ++g) {
                    int p0 = rand() % 3, p1 = p0 + 1 + rand() % (3 - p0);
                    for (int p = 0; p < 4; ++p) A[r * K + 4 * g + p] = 0.f;
                    float v0 = fb(bf((rand() % 2001 - 1000) / 500.0f)), v1 = fb(bf((rand() % 2001 - 1000) / 500.0f));
                    A[r * K + 4 * g + p0] = v0; A[r * K + 4 * g + p1] = v1;
                    Ab.push_back(bf(v0)); Ab.push_back(bf(v1));
                    meta[r * (K / 16) + g / 4] |= (uint16_t)((p0 | (p1 << 2)) << (4 * (g % 4)));
                }
        }
        cudaMemcpy(dA, Ab.data(), Ab.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, Bb.data(), Bb.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dM, meta.data(), meta.size() * 2, cudaMemcpyHostToDevice);
        cudaMemset(dD, 0, 128 * 128 * 4);
        Args a{test, dA, dM, dB, K, dD};
        probe<<<1, 128, 80 * 1024>>>(a);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> D(128 * 128);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double md = 0, mref = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 128; ++n) {
                double s = 0;
                for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
                md = fmax(md, fabs(s - D[m * 128 + n]));
                mref = fmax(mref, fabs(s));
            }
        printf("%-36s err=%s maxdiff=%.3g (max|ref| %.3g) %s\n", names[test], cudaGetErrorString(e), md, mref,
               (e == cudaSuccess && md < 1e-2) ? "MATCH" : "MISMATCH");
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
