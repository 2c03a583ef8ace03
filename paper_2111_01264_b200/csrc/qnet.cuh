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
constexpr int64_t S_W1 = 0, S_W2 = 8192, S_W3 = 40960, S_W4 = 77824, S_TOTAL = 1683456;
constexpr int MAX_ACTIONS = 32;
constexpr int MAX_SPLITS = 64;
constexpr int FC1_SPLITS = 7;  // 49 K-chunks of fc1 -> 7 x 7

}  // namespace pq
