// Probe: which metadata-register layout does mma.sp m16n8k32 (bf16) use on sm_100a?
// Builds a random 2:4 A (16x32), B (32x8), runs the sparse MMA under several
// metadata hypotheses and reports which reproduces the dense product.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// A: 16x32 dense (2:4 along k), B: 32x8, meta16[row][half] 16-bit per (row, k-half)
template <int ORDERED>
__global__ void probe(const float* A, const float* B, const uint16_t* meta16, int hyp, float* C) {
    int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    // compressed A values: row r: for k32 groups j=0..7, two kept values
    __shared__ float Ac[16][16];
    if (lane < 16) {
        int r = lane;
        for (int j = 0; j < 8; ++j) {
            int n = 0;
            for (int p = 0; p < 4; ++p) {
                float v = A[r * 32 + 4 * j + p];
                // kept = positions encoded in meta
                int half = j / 4, jj = j % 4;
                int nib = (meta16[r * 2 + half] >> (4 * jj)) & 0xF;
                int i0 = nib & 3, i1 = nib >> 2;
                if (p == i0 || p == i1) Ac[r][2 * j + (n++)] = v;
            }
        }
    }
    __syncwarp();
    uint32_t a[4], b[4];
    a[0] = pack_bf16(Ac[g][2 * t], Ac[g][2 * t + 1]);
    a[1] = pack_bf16(Ac[g + 8][2 * t], Ac[g + 8][2 * t + 1]);
    a[2] = pack_bf16(Ac[g][2 * t + 8], Ac[g][2 * t + 9]);
    a[3] = pack_bf16(Ac[g + 8][2 * t + 8], Ac[g + 8][2 * t + 9]);
    for (int i = 0; i < 4; ++i)
        b[i] = pack_bf16(B[(2 * t + 8 * i) * 8 + g], B[(2 * t + 8 * i + 1) * 8 + g]);
    uint32_t e = 0;
    int tt = t & 1;
    if (hyp == 0) {  // H_A: thread t: row g k-half t low | row g+8 k-half t high
        e = (uint32_t)meta16[g * 2 + tt] | ((uint32_t)meta16[(g + 8) * 2 + tt] << 16);
    } else if (hyp == 1) {  // H_B: t=0 row g full k32, t=1 row g+8 full k32
        int r = tt == 0 ? g : g + 8;
        e = (uint32_t)meta16[r * 2 + 0] | ((uint32_t)meta16[r * 2 + 1] << 16);
    } else if (hyp == 2) {  // H_C: t: row g k-half t low | row g k-half ... (row g both halves, rows g+8 by t=1)
        e = (uint32_t)meta16[g * 2 + tt] | ((uint32_t)meta16[g * 2 + (1 - tt)] << 16);
    }
    float c[4] = {0, 0, 0, 0};
    if (ORDERED) {
        asm volatile(
            "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.f32.bf16.bf16.f32 "
            "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9,%10,%11}, {%0,%1,%2,%3}, %12, 0x0;\n"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]),
              "r"(b[3]), "r"(e));
    } else {
        asm volatile(
            "mma.sp.sync.aligned.m16n8k32.row.col.f32.bf16.bf16.f32 "
            "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9,%10,%11}, {%0,%1,%2,%3}, %12, 0x0;\n"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]),
              "r"(b[3]), "r"(e));
    }
    C[g * 8 + 2 * t] = c[0];
    C[g * 8 + 2 * t + 1] = c[1];
    C[(g + 8) * 8 + 2 * t] = c[2];
    C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

static float bf(float x) {  // round to bf16
    uint32_t u; memcpy(&u, &x, 4); u += 0x7FFF + ((u >> 16) & 1); u &= 0xFFFF0000u; memcpy(&x, &u, 4); return x;
}

int main() {
    srand(1);
    float hA[16 * 32], hB[32 * 8], ref[16 * 8];
    uint16_t hm[16 * 2];
    for (int r = 0; r < 16; ++r) {
        hm[r * 2] = hm[r * 2 + 1] = 0;
        for (int j = 0; j < 8; ++j) {
            int i0 = rand() % 3, i1 = i0 + 1 + rand() % (3 - i0);
            for (int p = 0; p < 4; ++p)
                hA[r * 32 + 4 * j + p] = (p == i0 || p == i1) ? bf((rand() % 200 - 100) / 37.0f) : 0.f;
            hm[r * 2 + j / 4] |= (uint16_t)((i0 | (i1 << 2)) << (4 * (j % 4)));
        }
    }
    for (int i = 0; i < 32 * 8; ++i) hB[i] = bf((rand() % 200 - 100) / 53.0f);
    for (int r = 0; r < 16; ++r)
        for (int n = 0; n < 8; ++n) {
            double s = 0; for (int k = 0; k < 32; ++k) s += (double)hA[r * 32 + k] * hB[k * 8 + n];
            ref[r * 8 + n] = (float)s;
        }
    float *dA, *dB, *dC; uint16_t* dm;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dC, sizeof ref); cudaMalloc(&dm, sizeof hm);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaMemcpy(dm, hm, sizeof hm, cudaMemcpyHostToDevice);
    for (int ord = 0; ord < 2; ++ord)
        for (int hyp = 0; hyp < 3; ++hyp) {
            float hC[16 * 8];
            cudaMemset(dC, 0, sizeof ref);
            if (ord) probe<1><<<1, 32>>>(dA, dB, dm, hyp, dC); else probe<0><<<1, 32>>>(dA, dB, dm, hyp, dC);
            cudaError_t err = cudaDeviceSynchronize();
            cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
            double md = 0; for (int i = 0; i < 128; ++i) md = fmax(md, fabs(hC[i] - ref[i]));
            printf("ordered=%d hyp=%d err=%s maxdiff=%g %s\n", ord, hyp, cudaGetErrorString(err), md,
                   md < 1e-3 ? "MATCH" : "");
        }
    return 0;
}
