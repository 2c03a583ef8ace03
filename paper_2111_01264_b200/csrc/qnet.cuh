// Nature-CNN Q-network layout shared by the kernels and the C ABI.
//
// Logical parameter order = nn.parameter_bytes order (nn.py:214-220): per layer the
// flattened weight then the bias.  Weight flattening (restatement choice, see
// oracle/natcnn.py): conv1 (out, c, kh, kw) over the planar 4x84x84 input;
// conv2/conv3 (out, kh, kw, c) over NHWC activations; fc1 reads conv3's output
// flattened (h, w, c); fc2 (A, 512).
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace pq {

constexpr int FRAME_BYTES = 84 * 84;  // 7056 = 441 x 16 B
constexpr int REC_INTS = 8;  // replay record: f0..f4, action | terminal << 16, f64 reward (lo, hi)

// Record fields 5..7: the action (< 32) with the bootstrap terminal in bit 16, then the
// reward as the two 32-bit halves of its IEEE f64 bits (the reference keeps a Python
// float, replay.py:19-27).
__host__ __device__ inline int rec_action(int32_t f5) { return f5 & 0xFFFF; }
__host__ __device__ inline bool rec_terminal(int32_t f5) { return (f5 >> 16) & 1; }
#ifdef __CUDACC__
__host__ __device__ inline double rec_reward(int32_t lo, int32_t hi) {
#ifdef __CUDA_ARCH__
    return __hiloint2double(hi, lo);
#else
    uint64_t u = ((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo;
    double d;
    __builtin_memcpy(&d, &u, 8);
    return d;
#endif
}
__host__ __device__ inline void rec_pack(int32_t *f5, int action, bool terminal, double reward) {
#ifdef __CUDA_ARCH__
    const long long u = __double_as_longlong(reward);
#else
    long long u;
    __builtin_memcpy(&u, &reward, 8);
#endif
    f5[0] = action | (terminal ? 1 << 16 : 0);
    f5[1] = (int32_t)(uint32_t)(unsigned long long)u;
    f5[2] = (int32_t)(uint32_t)((unsigned long long)u >> 32);
}
#endif

constexpr int64_t P_W1 = 0, P_B1 = 8192, P_W2 = 8224, P_B2 = 40992, P_W3 = 41056, P_B3 = 77920,
                  P_W4 = 77984, P_B4 = 1683616, P_W5 = 1684128;
__host__ __device__ constexpr int64_t p_b5(int A) { return P_W5 + (int64_t)A * 512; }
__host__ __device__ constexpr int64_t n_params(int A) { return p_b5(A) + A; }
// bf16 shadow (GEMM operand) copies of the conv1..fc1 weights
constexpr int64_t S_W1 = 0, S_W2 = 8192, S_W3 = 40960, S_W4 = 77824;
// W1 again with its K index permuted for the space-to-depth conv1 (TMA engine):
// k = (c, kh, kw) -> k' = ((ty, tx), c, dy, dx) with kh = 4 ty + dy, kw = 4 tx + dx
constexpr int64_t S_W1P = 1683456, S_TOTAL = 1683456 + 8192;
__host__ __device__ inline int w1_perm(int k) {
    const int c = k >> 6, kh = (k >> 3) & 7, kw = k & 7;
    return (((kh >> 2) * 2 + (kw >> 2)) * 4 + c) * 16 + (kh & 3) * 4 + (kw & 3);
}
constexpr int MAX_ACTIONS = 32;
constexpr int MAX_SPLITS = 64;
constexpr int P1_MAX_SPLITS = 148;  // part1 rows: the shifted conv1 weight gradient runs one CTA per SM
constexpr int FC1_SPLITS = 7;  // 49 K-chunks of fc1 -> 7 x 7

}  // namespace pq
