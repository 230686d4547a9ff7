// Probe: tcgen05.mma / tcgen05.mma.sp issue rate and group latency on B200 for
// the operand shapes the prefill kernel uses.  One CTA per SM, one issuing
// thread, operands resident in smem (contents irrelevant for timing).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_2604_16864_b200/csrc/common.cuh"

using namespace hs;

struct Cfg {
    const char* name;
    int sparse, N, b_mn, a_sw64, group;  // group: MMAs per commit+wait (0: one commit at the end)
};

template <int SPARSE, int N, int BMN, int ASW64, int GROUP>
__global__ void __launch_bounds__(128) rate(int reps, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    for (int i = tid; i < 96 * 1024 / 4; i += 128)
        reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
    if (warp == 0) tmem_alloc(&tbase, 512);
    if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tD = tbase, tE = tbase + 256;
    tmem_st4(tE + ((32 * warp) << 16), 0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
    tmem_st4(tE + 4 + ((32 * warp) << 16), 0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp_id_uniform() == 0) {
        const uint32_t sA = smem_u32(base), sB = smem_u32(base) + 32768;
        constexpr uint32_t idesc = umma_idesc_f16(false, 128, N, false, BMN, SPARSE);
        uint64_t ad[4], bd[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            ad[j] = ASW64 ? umma_desc(sA + 32 * (j & 1), 16, 512, kLayoutSW64) : umma_desc(sA + 32 * j, 16, 1024, kLayoutSW128);
            bd[j] = BMN ? umma_desc(sB + 2048 * j, 16384, 1024, kLayoutSW128) : umma_desc(sB + 32 * j, 16, 1024, kLayoutSW128);
        }
        uint32_t phase = 0;
        long long t0 = clock64();
        for (int i = 0; i < reps; i += 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (elect_one()) {
                    if (SPARSE) umma_sp_f16(tD, ad[j], bd[j], tE + j, idesc, (i + j) > 0);
                    else umma_f16(tD, ad[j], bd[j], idesc, (i + j) > 0);
                }
                __syncwarp();
                if (GROUP && ((i + j) % GROUP) == GROUP - 1) {
                    if (elect_one()) umma_commit(&bar);
                    __syncwarp();
                    mbar_wait(&bar, phase);
                    phase ^= 1;
                }
            }
        }
        if (!GROUP) {
            if (elect_one()) umma_commit(&bar);
            __syncwarp();
            mbar_wait(&bar, 0);
        }
        long long t1 = clock64();
        if (tid == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int SPARSE, int N, int BMN, int ASW64, int GROUP>
void run(const char* name, int sms, long long* d) {
    auto k = rate<SPARSE, N, BMN, ASW64, GROUP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int reps = 4096;
    for (int grid : {1, sms}) {
        k<<<grid, 128, 100 * 1024>>>(reps, d);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<grid, 128, 100 * 1024>>>(reps, d);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double cyc = static_cast<double>(h[grid / 2]) / reps;
        const double flop = 2.0 * 128 * N * (SPARSE ? 32 : 16);  // logical (dense-equivalent) flops
        const double tflops = flop * reps * grid / (ms * 1e-3) / 1e12;
        printf("%-48s grid %3d: %7.1f cyc/MMA  %6.0f logical flop/clk/SM  %7.1f TFLOPS (event) %s\n", name, grid, cyc,
               flop / cyc, tflops, cudaGetErrorString(err));
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    run<0, 128, 0, 0, 0>("dense  M128 N128 K16  A:K-SW128 B:K-SW128", sms, d);
    run<0, 128, 1, 0, 0>("dense  M128 N128 K16  B:MN-SW128", sms, d);
    run<0, 256, 0, 0, 0>("dense  M128 N256 K16", sms, d);
    run<0, 64, 0, 0, 0>("dense  M128 N64  K16", sms, d);
    run<1, 128, 0, 0, 0>("sparse M128 N128 K32  A:K-SW128 B:K-SW128", sms, d);
    run<1, 128, 1, 1, 0>("sparse M128 N128 K32  A:SW64 B:MN-SW128 (GEMM2)", sms, d);
    run<1, 256, 0, 0, 0>("sparse M128 N256 K32", sms, d);
    run<1, 64, 0, 0, 0>("sparse M128 N64  K32", sms, d);
    run<1, 128, 0, 0, 4>("latency: 4 x sparse N128 + commit/wait", sms, d);
    run<0, 128, 0, 0, 8>("latency: 8 x dense N128 + commit/wait", sms, d);
    run<0, 128, 0, 0, 1>("latency: 1 x dense N128 + commit/wait", sms, d);
    return 0;
}
