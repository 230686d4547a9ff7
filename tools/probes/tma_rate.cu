// Probe: TMA (2-D tensor tiles and 1-D bulk copies) latency and per-SM ingest
// from an L2-resident, incompressible buffer: a ring of STAGES buffers per CTA,
// one CTA per SM (or one CTA alone).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_2604_16864_b200/csrc/common.cuh"

using namespace hs;

template <int STAGES, int KIND>  // KIND 0: 2-D tile 64x128 bf16 SW128 (16 KB); 1: bulk 16 KB; 2: bulk 2 KB
__global__ void __launch_bounds__(32) ingest(const __grid_constant__ CUtensorMap map, const uint8_t* src,
                                             uint32_t rows_total, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
    __shared__ __align__(8) uint64_t full[STAGES];
    constexpr uint32_t bytes = KIND == 2 ? 2048u : 16384u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncwarp();
    const uint32_t nchunks = rows_total / 128;  // power of two
    uint32_t c = (blockIdx.x * 7919u) & (nchunks - 1);
    long long t0 = clock64();
    for (int i = 0; i < iters + STAGES; ++i) {
        if (i >= STAGES) mbar_wait(&full[(i - STAGES) % STAGES], ((i - STAGES) / STAGES) & 1);
        if (i < iters && elect_one()) {
            const int s = i % STAGES;
            mbar_arrive_expect_tx(&full[s], bytes);
            if (KIND == 0) tma_tile_g2s(sm + s * 16384, &map, 0, c * 128, &full[s]);
            else tma_bulk_g2s(sm + s * 16384, src + static_cast<size_t>(c) * 16384, bytes, &full[s]);
        }
        __syncwarp();
        c = (c + 1) & (nchunks - 1);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int STAGES, int KIND>
void run(const char* name, const CUtensorMap& map, const uint8_t* src, uint32_t rows, int sms, long long* d) {
    auto k = ingest<STAGES, KIND>;
    const int smem = STAGES * 16384 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int grid : {1, sms}) {
        const int iters = 4000;
        k<<<grid, 32, smem>>>(map, src, rows, iters, d);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<grid, 32, smem>>>(map, src, rows, iters, d);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double bytes = KIND == 2 ? 2048.0 : 16384.0;
        const double cyc = static_cast<double>(h[grid / 2]) / iters;
        printf("%-34s stages %d grid %3d: %7.1f cyc/op  %6.1f B/clk/SM  %6.2f TB/s %s\n", name, STAGES, grid, cyc,
               bytes / cyc, bytes * iters * grid / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t rows = 1u << 16;  // 65536 rows x 128 B = 8 MB... use 256 B rows: 16 MB
    const size_t bytes = static_cast<size_t>(rows) * 256;
    std::vector<uint32_t> host(bytes / 4);
    uint32_t x = 12345;
    for (auto& v : host) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; v = x; }
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemcpy(src, host.data(), bytes, cudaMemcpyHostToDevice);
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {128, rows};  // bf16 elements: 128 per 256-byte row
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    run<1, 0>("tile 64x128 SW128 (16 KB)", map, src, rows, sms, d);
    run<2, 0>("tile 64x128 SW128 (16 KB)", map, src, rows, sms, d);
    run<4, 0>("tile 64x128 SW128 (16 KB)", map, src, rows, sms, d);
    run<8, 0>("tile 64x128 SW128 (16 KB)", map, src, rows, sms, d);
    run<1, 1>("bulk 16 KB", map, src, rows, sms, d);
    run<4, 1>("bulk 16 KB", map, src, rows, sms, d);
    run<8, 1>("bulk 16 KB", map, src, rows, sms, d);
    run<1, 2>("bulk 2 KB", map, src, rows, sms, d);
    run<8, 2>("bulk 2 KB", map, src, rows, sms, d);
    return 0;
}
