// Probe: TMA operation rate per SM — is the per-SM ingest bound by bytes or by
// operations?  W producer warps per CTA, each with its own ring of STAGES
// buffers, issuing BYTES-sized 1-D bulk copies (KIND 0) or 64 x (BYTES/128)
// SW128 2-D tiles (KIND 1) from an L2-resident buffer; one CTA alone and one
// CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ops tma_ops.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2604_16864_b200/csrc/common.cuh"
using namespace hs;

template <int W, int STAGES, int BYTES, int KIND, int VAR>
__global__ void __launch_bounds__(32 * W) ops(const __grid_constant__ CUtensorMap map, const uint8_t* src,
                                              uint32_t nchunks, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
    __shared__ __align__(8) uint64_t full[W][STAGES];
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int w = 0; w < W; ++w)
            for (int s = 0; s < STAGES; ++s) mbar_init(&full[w][s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint8_t* ring = sm + warp * STAGES * BYTES;
    uint32_t c = (blockIdx.x * 7919u + warp * 131u) & (nchunks - 1);
    long long t0 = clock64();
    for (int i = 0; i < iters + STAGES; ++i) {
        if (i >= STAGES) mbar_wait(&full[warp][(i - STAGES) % STAGES], ((i - STAGES) / STAGES) & 1);
        if (VAR == 3) {  // whole warp, lane 0 issues (no elect / syncwarp)
            if (i < iters && (threadIdx.x & 31) == 0) {
                const int s = i % STAGES;
                mbar_arrive_expect_tx(&full[warp][s], BYTES);
                tma_bulk_g2s(ring + s * BYTES, src + static_cast<size_t>(c) * 16384, BYTES, &full[warp][s]);
            }
        } else if (i < iters && elect_one()) {
            const int s = i % STAGES;
            if (VAR == 1) {
                asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                                 smem_u32(&full[warp][s])), "r"(BYTES) : "memory");
            } else if (VAR == 2) {  // expect_tx without arrive, then the arrive after the copy
                asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                                 smem_u32(&full[warp][s])), "r"(BYTES) : "memory");
            } else {
                mbar_arrive_expect_tx(&full[warp][s], BYTES);
            }
            if (KIND == 1) tma_tile_g2s(ring + s * BYTES, &map, 0, c * (BYTES / 128), &full[warp][s]);
            else tma_bulk_g2s(ring + s * BYTES, src + static_cast<size_t>(c) * 16384, BYTES, &full[warp][s]);
            if (VAR == 2)
                asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[warp][s])) : "memory");
        }
        if (VAR != 3) __syncwarp();
        c = (c + 1) & (nchunks - 1);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn enc;

template <int W, int STAGES, int BYTES, int KIND, int VAR = 0>
void run(uint8_t* src, size_t bytes, int sms, long long* d) {
    CUtensorMap map;
    const cuuint64_t rows = bytes / 128;
    cuuint64_t dims[2] = {64, rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(BYTES / 128)}, es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto k = ops<W, STAGES, BYTES, KIND, VAR>;
    const int smem = W * STAGES * BYTES + 1024;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return;
    const uint32_t nchunks = static_cast<uint32_t>(bytes / 16384);
    for (int grid : {1, sms}) {
        const int iters = 2000;
        k<<<grid, 32 * W, smem>>>(map, src, nchunks, iters, d);
        cudaError_t err = cudaDeviceSynchronize();
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double cyc = static_cast<double>(h[grid / 2]) / (static_cast<double>(iters) * W);
        printf("var%d %s %5d B  warps %d stages %2d grid %3d: %6.1f cyc/op per SM  %6.1f B/clk/SM %s\n",
               VAR, KIND ? "tile" : "bulk", BYTES, W, STAGES, grid, cyc, BYTES / cyc, cudaGetErrorString(err));
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = 16u << 20;
    std::vector<uint32_t> host(bytes / 4);
    uint32_t x = 12345;
    for (auto& v : host) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; v = x; }
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemcpy(src, host.data(), bytes, cudaMemcpyHostToDevice);
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    run<1, 8, 2048, 0, 0>(src, bytes, sms, d);
    run<1, 8, 2048, 0, 1>(src, bytes, sms, d);
    run<1, 8, 2048, 0, 2>(src, bytes, sms, d);
    run<1, 8, 2048, 0, 3>(src, bytes, sms, d);
    run<1, 8, 16384, 1, 0>(src, bytes, sms, d);
    run<1, 8, 16384, 1, 1>(src, bytes, sms, d);
    run<1, 8, 16384, 1, 2>(src, bytes, sms, d);
    return 0;
}
