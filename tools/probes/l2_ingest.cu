// Probe: L2 -> SM ingest rate with 1-D bulk copies (cp.async.bulk, TMA) from
// an L2-resident buffer, one CTA per SM, a ring of `stages` x `chunk` bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_ingest l2_ingest.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2604_16864_b200/csrc/common.cuh"

using namespace hs;

__global__ void __launch_bounds__(64) ingest(const uint8_t* src, size_t span, int chunk, int stages, int iters,
                                            long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[16];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (warp_id_uniform() == 0) {
        const uint32_t mask = static_cast<uint32_t>(span / chunk) - 1;  // power of two
        uint32_t c = (blockIdx.x * 7919u) & mask;
        long long t0 = clock64();
        for (int i = 0; i < iters + stages; ++i) {
            if (i >= stages) {
                const int s = (i - stages) % stages;
                mbar_wait(&full[s], ((i - stages) / stages) & 1);
            }
            if (i < iters && elect_one()) {
                const int s = i % stages;
                mbar_arrive_expect_tx(&full[s], chunk);
                tma_bulk_g2s(sm + s * chunk, src + static_cast<size_t>(c) * chunk, chunk, &full[s]);
            }
            __syncwarp();
            c = (c + 1) & mask;
        }
        long long t1 = clock64();
        if (tid == 0) out[blockIdx.x] = t1 - t0;
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t span = 32u << 20;
    uint8_t* src;
    cudaMalloc(&src, span);
    cudaMemset(src, 1, span);
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct { int chunk, stages; } cfgs[] = {{4096, 4}, {4096, 16}, {16384, 4}, {16384, 12}, {32768, 6}};
    for (auto cf : cfgs) {
        for (int grid : {1, 16, 74, sms}) {
            const int iters = 2000;
            ingest<<<grid, 64, cf.chunk * cf.stages>>>(src, span, cf.chunk, cf.stages, iters, d);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            ingest<<<grid, 64, cf.chunk * cf.stages>>>(src, span, cf.chunk, cf.stages, iters, d);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<long long> h(grid);
            cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            const double bpc = static_cast<double>(cf.chunk) * iters / h[grid / 2];
            const double tbs = static_cast<double>(cf.chunk) * iters * grid / (ms * 1e-3) / 1e12;
            printf("chunk %6d stages %2d grid %3d: %6.1f B/clk/SM  %6.2f TB/s total %s\n", cf.chunk, cf.stages, grid,
                   bpc, tbs, cudaGetErrorString(err));
        }
    }
    return 0;
}
