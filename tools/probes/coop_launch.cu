// Launch overhead of the cooperative attribute: event-timed graph replays of a
// near-empty 144 x 256 kernel, plain vs cudaLaunchAttributeCooperative, and the
// same with ~100 KB of dynamic shared memory (the decode plan's footprint).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/coop_launch_bin tools/probes/coop_launch.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); fflush(stdout); return -1.f; } } while (0)

__global__ void tiny(int* p) {
    __shared__ int sm[1];  // (the dynamic shared memory only sets the footprint)
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] < 0) p[blockIdx.x] = 1;
}

static float time_graph(bool coop, int smem, int* p) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(144);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 1 : 0;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaLaunchKernelEx(&cfg, tiny, p));
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    CK(cudaLaunchKernelEx(&cfg, tiny, p));
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    float best = 1e9, sum = 0;
    const int n = 200;
    for (int i = 0; i < n; ++i) {
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        sum += ms;
        best = ms < best ? ms : best;
    }
    printf("coop=%d smem=%6d: mean %.2f us, best %.2f us\n", coop, smem, sum / n * 1e3, best * 1e3);
    fflush(stdout);
    return sum / n;
}

int main() {
    int* p;
    cudaMalloc(&p, 4096);
    if (cudaFuncSetAttribute(tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) printf("attr fail\n");
    for (int rep = 0; rep < 2; ++rep)
        for (int smem : {0, 100 * 1024})
            for (bool coop : {false, true}) time_graph(coop, smem, p);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
