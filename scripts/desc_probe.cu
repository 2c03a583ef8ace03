// Probe: can a K-major SW128 UMMA A operand start at an arbitrary 128-byte row of a
// swizzled tile (descriptor base-offset field)?  One CTA fills a 152 x 64 bf16 tile in
// the SW128 layout (as TMA writes it), then for each row shift s runs D = A[s:s+128] B^T
// (M = 128, N = 32, K = 64) with base_offset = 0 or (s & 7) and compares with a CPU
// product.  usage: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17
//   -I paper_2111_01264_b200/csrc scripts/desc_probe.cu -o /tmp/desc_probe && /tmp/desc_probe
#include <cuda_bf16.h>
#include <cstdio>
#include <cmath>
#include <vector>

#include "common.cuh"

using namespace pq;

constexpr int ROWS = 152, K = 64, N = 32;

__global__ void k_probe(const __nv_bfloat16 *A, const __nv_bfloat16 *B, int shift, int boff, float *D) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_s;
    const int tid = threadIdx.x;
    uint8_t *a_s = sm, *b_s = sm + 32 * 1024;
    // A rows 0..151 and B rows 0..31, 16-byte chunks at the SW128 K-major offsets
    for (int q = tid; q < ROWS * 8; q += blockDim.x) {
        const int r = q >> 3, c = q & 7;
        *reinterpret_cast<uint4 *>(a_s + kmaj_off(r, c)) = *reinterpret_cast<const uint4 *>(A + r * K + c * 8);
    }
    for (int q = tid; q < N * 8; q += blockDim.x) {
        const int r = q >> 3, c = q & 7;
        *reinterpret_cast<uint4 *>(b_s + kmaj_off(r, c)) = *reinterpret_cast<const uint4 *>(B + r * K + c * 8);
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if ((tid >> 5) == 0) tmem_alloc<32>(&tmem_s);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_s;
    if (tid == 0) {
        const uint32_t a0 = smem_u32(a_s) + shift * 128, b0 = smem_u32(b_s);
        for (int j = 0; j < 4; ++j) {
            uint64_t ad = desc_sw128(a0 + j * 32, 0) | ((uint64_t)(boff & 7) << 49);
            uint64_t bd = desc_sw128(b0 + j * 32, 0);
            umma_bf16(tmem, ad, bd, idesc_bf16(N, false, false), j > 0);
        }
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    float v[32];
    const int w = tid >> 5, lane = tid & 31;
    tmem_ld32(tmem + ((uint32_t)(w * 32) << 16), v);
    for (int c = 0; c < N; ++c) D[(w * 32 + lane) * N + c] = v[c];
    tc_fence_before();
    __syncthreads();
    if (w == 0) tmem_dealloc<32>(tmem);
}


// MN-major A: smem rows = K (spatial rows, 0..151), 64 M elements (channels) per 128-byte
// row; the M = 128 operand stacks rows [s0, s0+64) and [s1, s1+64) as its two 64-wide M
// atoms (LBO = (s1 - s0) * 128 bytes).  D[m][n] = sum_k A(m, k) B[n][k] with
// A(m, k) = T[s0 + k][m] (m < 64), T[s1 + k][m - 64] (m >= 64), K = 64.
__global__ void k_probe_mn(const __nv_bfloat16 *T, const __nv_bfloat16 *B, int s0, int s1, float *D) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_s;
    const int tid = threadIdx.x;
    uint8_t *a_s = sm, *b_s = sm + 32 * 1024;
    for (int q = tid; q < ROWS * 8; q += blockDim.x) {
        const int r = q >> 3, c = q & 7;
        *reinterpret_cast<uint4 *>(a_s + kmaj_off(r, c)) = *reinterpret_cast<const uint4 *>(T + r * 64 + c * 8);
    }
    for (int q = tid; q < N * 8; q += blockDim.x) {
        const int r = q >> 3, c = q & 7;
        *reinterpret_cast<uint4 *>(b_s + kmaj_off(r, c)) = *reinterpret_cast<const uint4 *>(B + r * K + c * 8);
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if ((tid >> 5) == 0) tmem_alloc<32>(&tmem_s);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_s;
    if (tid == 0) {
        const uint32_t a0 = smem_u32(a_s) + s0 * 128, b0 = smem_u32(b_s);
        for (int j = 0; j < 4; ++j) {  // K steps of 16 rows = 2048 bytes
            uint64_t ad = desc_sw128(a0 + j * 2048, (uint32_t)(s1 - s0) * 128);
            uint64_t bd = desc_sw128(b0 + j * 32, 0);
            umma_bf16(tmem, ad, bd, idesc_bf16(N, true, false), j > 0);
        }
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    float v[32];
    const int w = tid >> 5, lane = tid & 31;
    tmem_ld32(tmem + ((uint32_t)(w * 32) << 16), v);
    for (int c = 0; c < N; ++c) D[(w * 32 + lane) * N + c] = v[c];
    tc_fence_before();
    __syncthreads();
    if (w == 0) tmem_dealloc<32>(tmem);
}

int main() {
    std::vector<__nv_bfloat16> hA(ROWS * K), hB(N * K);
    std::vector<float> fA(ROWS * K), fB(N * K);
    unsigned s = 12345;
    auto rnd = [&] { s = s * 1664525u + 1013904223u; return ((s >> 9) & 0xFFFF) / 65536.0f - 0.5f; };
    for (int i = 0; i < ROWS * K; ++i) { hA[i] = __float2bfloat16(rnd()); fA[i] = __bfloat162float(hA[i]); }
    for (int i = 0; i < N * K; ++i) { hB[i] = __float2bfloat16(rnd()); fB[i] = __bfloat162float(hB[i]); }
    __nv_bfloat16 *dA, *dB;
    float *dD;
    cudaMalloc(&dA, ROWS * K * 2);
    cudaMalloc(&dB, N * K * 2);
    cudaMalloc(&dD, 128 * N * 4);
    cudaMemcpy(dA, hA.data(), ROWS * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
    const int smem = 64 * 1024;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> hD(128 * N);
    const int shifts[] = {0, 1, 2, 7, 8, 21, 22, 23};
    for (int sh : shifts)
        for (int mode = 0; mode < 2; ++mode) {
            const int boff = mode ? (sh & 7) : 0;
            k_probe<<<1, 128, smem>>>(dA, dB, sh, boff, dD);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("shift %d boff %d: CUDA error %s\n", sh, boff, cudaGetErrorString(e)); return 1; }
            cudaMemcpy(hD.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost);
            double err = 0;
            for (int i = 0; i < 128; ++i)
                for (int n = 0; n < N; ++n) {
                    double ref = 0;
                    for (int k = 0; k < K; ++k) ref += (double)fA[(sh + i) * K + k] * fB[n * K + k];
                    err = fmax(err, fabs(ref - hD[i * N + n]));
                }
            printf("shift %2d base_offset %d: max |err| %.3e %s\n", sh, boff, err, err < 1e-3 ? "OK" : "WRONG");
        }
    cudaFuncSetAttribute(k_probe_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int pairs[][2] = {{0, 64}, {0, 1}, {0, 21}, {21, 22}, {1, 22}, {3, 11}};
    for (auto &pr : pairs) {
        const int s0 = pr[0], s1 = pr[1];
        if (s1 + 64 > ROWS) continue;
        k_probe_mn<<<1, 128, smem>>>(dA, dB, s0, s1, dD);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mn %d/%d: CUDA error %s\n", s0, s1, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(hD.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) {
                    const int row = (m < 64 ? s0 : s1) + k, col = m & 63;
                    ref += (double)fA[row * K + col] * fB[n * K + k];
                }
                err = fmax(err, fabs(ref - hD[m * N + n]));
            }
        printf("MN-major rows %2d / %2d (LBO %4d B): max |err| %.3e %s\n", s0, s1, (s1 - s0) * 128, err,
               err < 1e-3 ? "OK" : "WRONG");
    }
    return 0;
}
