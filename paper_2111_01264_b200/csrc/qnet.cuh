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
constexpr int REC_INTS = 8;           // replay record: f0..f4, action, reward bits, terminal

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
