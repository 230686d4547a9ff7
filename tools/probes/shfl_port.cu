// Does SHFL share the shared-memory data port?  One CTA per SM, 16 warps:
//   mode 0: all warps LDS.128        mode 1: all warps SHFL (fp32 xor)
//   mode 2: 8 warps LDS.128 + 8 warps SHFL concurrently
//   mode 3: all warps redux.sync.add.u32    mode 4: 8 warps LDS.128 + 8 warps REDUX
// Prints per-SM throughput (LDS bytes/clk, SHFL warp-instr/clk) from clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/shfl_port tools/probes/shfl_port.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void __launch_bounds__(512) probe(int mode, long long* out, float* sink) {
    __shared__ __align__(16) float4 buf[2048];  // 32 KB
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2048; i += 512) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    const bool lds = mode == 0 || ((mode == 2 || mode == 4) && warp < 8);
    float4 acc = make_float4(0, 0, 0, 0);
    float v[8];
    unsigned u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = lane + i;
        u[i] = lane * 7 + i;
    }
    __syncthreads();
    const long long t0 = clock64();
    if (lds) {
        int idx = threadIdx.x & 2047;
        for (int it = 0; it < kIters; ++it) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float4 x = buf[(idx + j * 256) & 2047];
                acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
            }
            idx += 37;
        }
    } else if (mode == 3 || mode == 4) {
        for (int it = 0; it < kIters; ++it) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                unsigned r;
                asm volatile("redux.sync.add.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(u[j]));
                u[j] += r;
            }
        }
    } else {
        for (int it = 0; it < kIters; ++it) {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], (j & 3) + 1 + (it & 8));
        }
    }
    const long long t1 = clock64();
    float s = acc.x + acc.y + acc.z + acc.w;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i] + u[i];
    if (s == 12345.f) sink[0] = s;
    if (lane == 0) {
        out[(blockIdx.x * 16 + warp) * 2] = t0;
        out[(blockIdx.x * 16 + warp) * 2 + 1] = t1;
    }
}

int main() {
    long long* d;
    float* sink;
    cudaMalloc(&d, 148 * 16 * 2 * sizeof(long long));
    cudaMalloc(&sink, 4);
    long long h[148 * 16 * 2];
    const char* names[] = {"LDS.128 x16 warps", "SHFL x16 warps", "LDS.128 x8 + SHFL x8", "REDUX.add.u32 x16 warps", "LDS.128 x8 + REDUX x8"};
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) probe<<<148, 512>>>(mode, d, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        // CTA 0: each group's span (min start .. max end)
        long long s_l = 1LL << 62, e_l = 0, s_s = 1LL << 62, e_s = 0;
        for (int w = 0; w < 16; ++w) {
            const bool lds = mode == 0 || ((mode == 2 || mode == 4) && w < 8);
            long long a = h[w * 2], b = h[w * 2 + 1];
            if (lds) { s_l = a < s_l ? a : s_l; e_l = b > e_l ? b : e_l; }
            else { s_s = a < s_s ? a : s_s; e_s = b > e_s ? b : e_s; }
        }
        const int nl = mode == 0 ? 16 : (mode == 2 || mode == 4) ? 8 : 0, ns = 16 - nl;
        printf("%-26s", names[mode]);
        if (nl) {
            double clk = double(e_l - s_l);
            printf(" LDS: %.0f clk, %.1f B/clk/SM", clk, nl * 32.0 * 16 * 8 * kIters / clk);
        }
        if (ns) {
            double clk = double(e_s - s_s);
            printf(" %s: %.0f clk, %.3f warp-instr/clk/SM (%.1f B/clk if 128 B each)", mode >= 3 ? "REDUX" : "SHFL",
                   clk, ns * 8.0 * kIters / clk, ns * 8.0 * kIters * 128 / clk);
        }
        printf("\n");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
