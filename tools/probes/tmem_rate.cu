// Probe: TMEM -> register read bandwidth (tcgen05.ld.32x32b.xN) with W warps per
// CTA (W/4 per sub-partition), one CTA per SM; and MUFU.EX2 throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_rate tmem_rate.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2604_16864_b200/csrc/common.cuh"

using namespace hs;

template <int W, int N>
__global__ void __launch_bounds__(32 * W) tmem_read(int iters, long long* out, float* sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&tbase, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t lane_off = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    const uint32_t col = (warp >> 2) * N % 512;
    float acc = 0.f;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < N; c += 32) {
            tmem_ld32(tbase + lane_off + ((col + c) & 511), v);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += __uint_as_float(v[k]);
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int W>
__global__ void __launch_bounds__(32 * W) mufu(int iters, long long* out, float* sink) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = -0.001f * (threadIdx.x + k);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fast_exp2(x[k]) - 1.0f;
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    float a = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) a += x[k];
    if (a == 12345.f) sink[0] = a;
}

template <int W, int N>
void run_tmem(int sms, long long* d, float* sink) {
    const int iters = 2000;
    tmem_read<W, N><<<sms, 32 * W>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(sms);
    cudaMemcpy(h.data(), d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    const double bytes = static_cast<double>(W) * 32 * N * 4 * iters;
    printf("tcgen05.ld 32x32b x32, %2d warps, %3d cols/warp/iter: %6.1f B/clk/SM  (%6.1f cyc per warp-load) %s\n", W, N,
           bytes / h[sms / 2], static_cast<double>(h[sms / 2]) / (iters * N / 32), cudaGetErrorString(e));
}

template <int W>
void run_mufu(int sms, long long* d, float* sink) {
    const int iters = 4000;
    mufu<W><<<sms, 32 * W>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(sms);
    cudaMemcpy(h.data(), d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    const double ops = static_cast<double>(W) * 32 * 8 * iters;
    printf("MUFU.EX2 (+FADD) %2d warps: %6.2f ex2/clk/SM %s\n", W, ops / h[sms / 2], cudaGetErrorString(e));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d;
    float* sink;
    cudaMalloc(&d, sms * sizeof(long long));
    cudaMalloc(&sink, 16);
    run_tmem<4, 32>(sms, d, sink);
    run_tmem<8, 32>(sms, d, sink);
    run_tmem<16, 32>(sms, d, sink);
    run_tmem<16, 64>(sms, d, sink);
    run_tmem<32, 32>(sms, d, sink);
    run_mufu<4>(sms, d, sink);
    run_mufu<8>(sms, d, sink);
    run_mufu<16>(sms, d, sink);
    run_mufu<32>(sms, d, sink);
    return 0;
}
