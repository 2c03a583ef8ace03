// Implicit-GEMM on the 5th-gen tensor cores (tcgen05 / TMEM), sm_100a.
//
//   D[m, n] = sum_k A[m, k] * B[n, k]      (bf16 operands, fp32 accumulate in TMEM)
//
// One CTA = 128 threads computes a 128 x BN tile.  Operand tiles (BK = 64) are
// gathered straight from the producing layout -- im2col of uint8 frames through the
// replay ring's frame table, im2col of NHWC activations, transposed-conv windows,
// plain matrices -- by cp.async (LDGSTS) into shared memory in the UMMA 128B-swizzled
// canonical layout, K-major or MN-major, so no im2col or transpose is materialised in
// HBM.  The mainloop is a STAGES-deep ring: loads for K-chunk i+STAGES-1 are in flight
// while thread 0 issues the 4 x tcgen05.mma (K = 16) of chunk i and commits them to
// the chunk's mbarrier, which releases the slot for reuse.  Ragged edges zero-fill
// through the cp.async src-size operand.  uint8 frame tiles are copied raw and widened
// to bf16 in shared memory by the thread that loaded them (0..255 is exact in bf16).
// The epilogue reads the accumulator with tcgen05.ld (warp w owns TMEM lanes
// 32w..32w+31 = tile rows) and applies a fused operator (bias / 1/255 scale / ReLU /
// ReLU-mask / split-K partial / transposed store).
//
// A loader exposes src(outer, inner, bytes) -> address of 8 consecutive elements of its
// natural row-major view (inner % 8 == 0), bytes = how many of them exist (0 = zero
// chunk).  K-major operands use (outer, inner) = (mn, k); MN-major operands use
// (outer, inner) = (k, mn).
#pragma once

#include "common.cuh"

namespace pq {

typedef __nv_bfloat16 bf16;

// ------------------------------------------------------------------------ cp.async
PQ_DEV void cp_async16(uint32_t dst, const void *src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes)
                 : "memory");
}
PQ_DEV void cp_async4(uint32_t dst, const void *src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes)
                 : "memory");
}
PQ_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
PQ_DEV void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------------------ loaders
// Exact x / d for 0 <= x < 2^24, 1 <= d < 4096 by one 64-bit multiply-high.
struct FastDiv {
    uint64_t m;
    int d;
    FastDiv() = default;
    __host__ __device__ FastDiv(int dd) : m(((1ull << 40) + (uint64_t)dd - 1) / (uint64_t)dd), d(dd) {}
    PQ_DEV int div(int x) const { return (int)(((uint64_t)(uint32_t)x * m) >> 40); }
};

// Per-CTA context handed to the loaders (frame-slot table in shared memory).
struct LoadCtx {
    const int32_t *table;  // [samples][4] frame slots of the CTA's sample window
    int tb;                // first sample of the window
};

// Addresses are separable into a row part (outer index) and a column part (inner
// index): row(outer) and col(inner) are computed once per thread per row / per
// K-chunk, addr() combines them.  K-major operands keep their rows for the whole
// K loop; MN-major operands keep their column.
struct LoadDense {  // bf16 row-major [rows][cols] with row stride ld (elements)
    static constexpr bool U8 = false, TABLE = false;
    PQ_DEV void at_tile(int) {}
    const bf16 *p;
    int rows, cols, ld;
    struct Row {
        const bf16 *p;
        bool ok;
    };
    struct Col {
        int c, bytes;
    };
    PQ_DEV Row row(int r) const { return {p + (size_t)r * ld, r < rows}; }
    PQ_DEV Col col(int c) const {
        int rem = cols - c;
        return {c, rem <= 0 ? 0 : (rem >= 8 ? 16 : rem * 2)};
    }
    PQ_DEV const void *addr(const Row &R, const Col &Cc, int &bytes, const LoadCtx &) const {
        bytes = R.ok ? Cc.bytes : 0;
        return bytes ? (const void *)(R.p + Cc.c) : (const void *)p;
    }
};

// im2col over NHWC bf16 activations: row m = (b, oy, ox), col k = (kh, kw, c)
struct LoadIm2col {
    static constexpr bool U8 = false, TABLE = false;
    PQ_DEV void at_tile(int) {}
    const bf16 *x;
    int n, H, W, C, KS, S, OH, OW;
    FastDiv f_npix, f_ow, f_kc, f_c;
    struct Row {
        int off;
        bool ok;
    };
    struct Col {
        int off;
        bool ok;
    };
    PQ_DEV Row row(int m) const {
        if (m >= n * OH * OW) return {0, false};
        int b = f_npix.div(m), rem = m - b * OH * OW;
        int oy = f_ow.div(rem), ox = rem - oy * OW;
        return {((b * H + oy * S) * W + ox * S) * C, true};
    }
    PQ_DEV Col col(int k) const {
        if (k >= KS * KS * C) return {0, false};
        int kh = f_kc.div(k), r2 = k - kh * KS * C;
        int kw = f_c.div(r2), c = r2 - kw * C;
        return {(kh * W + kw) * C + c, true};
    }
    PQ_DEV const void *addr(const Row &R, const Col &Cc, int &bytes, const LoadCtx &) const {
        bytes = (R.ok && Cc.ok) ? 16 : 0;
        return bytes ? (const void *)(x + R.off + Cc.off) : (const void *)x;
    }
};

// im2col over uint8 frame stacks addressed through a frame table:
// sample b, channel c -> frame slot refs[map(b) * ref_stride + ref_off + c] (-1 = zero
// frame) inside the frame ring; row m = (b, oy, ox) of the 20x20 conv1 output, col k in
// the space-to-depth order k = ((ty, tx), c, dy, dx), kh = 4 ty + dy, kw = 4 tx + dx
// (qnet.cuh w1_perm), the order the TMA engine's space-to-depth conv1 uses, so both
// engines accumulate identically; an 8-element chunk is two 4-byte runs (rows dy, dy+1).
// Values are the raw bytes 0..255 (exact in bf16); the 1/255 scale is in the epilogue.
// The CTA first stages the slots of its sample window in shared memory (fill()); an
// optional device counter slices the map (graph replay of the epoch index table).
struct LoadFrames {
    static constexpr bool U8 = true, TABLE = true;
    static constexpr int HALF2 = 84;  // second 4-byte run of a chunk: the next frame row
    PQ_DEV void at_tile(int) {}
    const uint8_t *ring;
    const int32_t *refs;
    const int64_t *map;
    const int32_t *counter;
    int counter_add;  // the map row is (*counter + counter_add)
    int map_stride;
    int n, ref_stride, ref_off;
    FastDiv f400, f20;
    struct Row {
        int pix, b;
        bool ok;
    };
    struct Col {
        int c, off;
        bool ok;
    };
    PQ_DEV Row row(int m) const {
        if (m >= n * 400) return {0, 0, false};
        int b = f400.div(m), rem = m - b * 400;
        int oy = f20.div(rem), ox = rem - oy * 20;
        return {oy * 336 + ox * 4, b, true};
    }
    PQ_DEV Col col(int k) const {  // k % 8 == 0: tap (ty, tx), frame c, rows dy, dy + 1
        const int tap = k >> 6, dy = (k >> 2) & 3;
        return {(k >> 4) & 3, (4 * (tap >> 1) + dy) * 84 + 4 * (tap & 1), k < 256};
    }
    PQ_DEV const void *addr(const Row &R, const Col &Cc, int &bytes, const LoadCtx &cx) const {
        bytes = 0;
        if (!R.ok || !Cc.ok) return ring;
        int slot = cx.table[(R.b - cx.tb) * 4 + Cc.c];
        if (slot < 0) return ring;
        bytes = 8;
        return ring + (size_t)slot * 7056 + R.pix + Cc.off;
    }
    // stage frame slots of samples [b_lo, b_hi] (all threads of the CTA)
    PQ_DEV void fill(int b_lo, int b_hi, int32_t *table) const {
        const int64_t base = (map && counter) ? (int64_t)(*counter + counter_add) * map_stride : 0;
        for (int e = threadIdx.x; e < (b_hi - b_lo + 1) * 4; e += blockDim.x) {
            int b = b_lo + (e >> 2), c = e & 3;
            int32_t v = -1;
            if (b < n) {
                int64_t rec = map ? map[base + b] : (int64_t)b;
                v = refs[rec * ref_stride + ref_off + c];
            }
            table[e] = v;
        }
    }
};

// transposed-conv window (data gradient, stride 1): row m = input pixel (b, iy, ix) of an
// H x W layer input, col t = (kh, kw, o); reads dY[b, iy-kh, ix-kw, o] when in range.
struct LoadTConv {
    static constexpr bool U8 = false, TABLE = false;
    PQ_DEV void at_tile(int) {}
    const bf16 *dy;
    int n, H, W, OH, OW, O, KS;
    FastDiv f_npix, f_w, f_ko, f_o;
    struct Row {
        int b, iy, ix;
        bool ok;
    };
    struct Col {
        int kh, kw, o;
        bool ok;
    };
    PQ_DEV Row row(int m) const {
        if (m >= n * H * W) return {0, 0, 0, false};
        int b = f_npix.div(m), rem = m - b * H * W;
        int iy = f_w.div(rem);
        return {b, iy, rem - iy * W, true};
    }
    PQ_DEV Col col(int t) const {
        if (t >= KS * KS * O) return {0, 0, 0, false};
        int kh = f_ko.div(t), r2 = t - kh * KS * O;
        int kw = f_o.div(r2);
        return {kh, kw, r2 - kw * O, true};
    }
    PQ_DEV const void *addr(const Row &R, const Col &Cc, int &bytes, const LoadCtx &) const {
        int oy = R.iy - Cc.kh, ox = R.ix - Cc.kw;
        bytes = (R.ok && Cc.ok && oy >= 0 && ox >= 0 && oy < OH && ox < OW) ? 16 : 0;
        return bytes ? (const void *)(dy + ((size_t)(R.b * OH + oy) * OW + ox) * O + Cc.o)
                     : (const void *)dy;
    }
};

// conv weight W[o][kh][kw][c] viewed as [t = (kh, kw, o)][c] (rows t, contiguous c)
struct LoadWeightT {
    static constexpr bool U8 = false, TABLE = false;
    PQ_DEV void at_tile(int) {}
    const bf16 *w;
    int O, KS, C;
    FastDiv f_ko, f_o;
    struct Row {
        int off;
        bool ok;
    };
    struct Col {
        int c;
        bool ok;
    };
    PQ_DEV Row row(int t) const {
        if (t >= KS * KS * O) return {0, false};
        int kh = f_ko.div(t), r2 = t - kh * KS * O;
        int kw = f_o.div(r2), o = r2 - kw * O;
        return {o * (KS * KS * C) + (kh * KS + kw) * C, true};
    }
    PQ_DEV Col col(int c) const { return {c, c < C}; }
    PQ_DEV const void *addr(const Row &R, const Col &Cc, int &bytes, const LoadCtx &) const {
        bytes = (R.ok && Cc.ok) ? 16 : 0;
        return bytes ? (const void *)(w + R.off + Cc.c) : (const void *)w;
    }
};

// Stride-2 transposed conv split into the 4 parity classes (py, px) of the input pixel:
// a class sees only taps kh = py + 2i, kw = px + 2j (i, j in {0,1}), so the contraction
// is 4 taps x O instead of 16 taps x O.  Grid rows are class-major, tpc tiles per class:
// row m -> class = m / (tpc*128), local row = (b, iy', ix') with iy = 2 iy' + py.
struct LoadTConvP {
    static constexpr bool U8 = false, TABLE = false;
    PQ_DEV void at_tile(int) {}
    const bf16 *dy;
    int n, H2, W2, OH, OW, O, tpc;  // H2 = H / 2
    FastDiv f_per, f_npix, f_w2, f_o;
    struct Row {
        int b, iy2, ix2;
        bool ok;
    };
    struct Col {
        int ty, tx, o;
        bool ok;
    };
    PQ_DEV Row row(int m) const {
        int cls = f_per.div(m), loc = m - cls * tpc * 128;
        if (loc >= n * H2 * W2) return {0, 0, 0, false};
        int b = f_npix.div(loc), rem = loc - b * H2 * W2;
        int iy2 = f_w2.div(rem);
        return {b, iy2, rem - iy2 * W2, true};
    }
    PQ_DEV Col col(int t) const {
        if (t >= 4 * O) return {0, 0, 0, false};
        int tap = f_o.div(t);
        return {tap >> 1, tap & 1, t - tap * O, true};
    }
    PQ_DEV const void *addr(const Row &R, const Col &Cc, int &bytes, const LoadCtx &) const {
        int oy = R.iy2 - Cc.ty, ox = R.ix2 - Cc.tx;
        bytes = (R.ok && Cc.ok && oy >= 0 && ox >= 0 && oy < OH && ox < OW) ? 16 : 0;
        return bytes ? (const void *)(dy + ((size_t)(R.b * OH + oy) * OW + ox) * O + Cc.o)
                     : (const void *)dy;
    }
};

// weight operand of LoadTConvP: rows t = (tap, o) of the CTA's parity class
struct LoadWeightTP {
    static constexpr bool U8 = false, TABLE = false;
    const bf16 *w;
    int O, KS, C, tpc;
    FastDiv f_o;
    int cls;  // parity class of the current tile (bound by at_tile)
    PQ_DEV void at_tile(int m0) { cls = (m0 >> 7) / tpc; }
    struct Row {
        int off;
        bool ok;
    };
    struct Col {
        int c;
        bool ok;
    };
    PQ_DEV Row row(int t) const {
        if (t >= 4 * O) return {0, false};
        int py = cls >> 1, px = cls & 1;
        int tap = f_o.div(t), o = t - tap * O;
        int kh = py + 2 * (tap >> 1), kw = px + 2 * (tap & 1);
        return {o * (KS * KS * C) + (kh * KS + kw) * C, true};
    }
    PQ_DEV Col col(int c) const { return {c, c < C}; }
    PQ_DEV const void *addr(const Row &R, const Col &Cc, int &bytes, const LoadCtx &) const {
        bytes = (R.ok && Cc.ok) ? 16 : 0;
        return bytes ? (const void *)(w + R.off + Cc.c) : (const void *)w;
    }
};

// loader factories (host or device: the multiply-shift divisors are computed here)
#define PQ_HD __host__ __device__ inline
PQ_HD LoadIm2col im2col(const bf16 *x, int n, int H, int W, int C, int KS, int S, int OH, int OW) {
    LoadIm2col l{x, n, H, W, C, KS, S, OH, OW};
    l.f_npix = FastDiv(OH * OW), l.f_ow = FastDiv(OW), l.f_kc = FastDiv(KS * C), l.f_c = FastDiv(C);
    return l;
}
PQ_HD LoadTConv tconv(const bf16 *dy, int n, int H, int W, int OH, int OW, int O, int KS) {
    LoadTConv l{dy, n, H, W, OH, OW, O, KS};
    l.f_npix = FastDiv(H * W), l.f_w = FastDiv(W), l.f_ko = FastDiv(KS * O), l.f_o = FastDiv(O);
    return l;
}
PQ_HD LoadWeightT weight_t(const bf16 *w, int O, int KS, int C) {
    LoadWeightT l{w, O, KS, C};
    l.f_ko = FastDiv(KS * O), l.f_o = FastDiv(O);
    return l;
}
PQ_HD LoadTConvP tconv_p(const bf16 *dy, int n, int H2, int W2, int OH, int OW, int O, int tpc) {
    LoadTConvP l{dy, n, H2, W2, OH, OW, O, tpc};
    l.f_per = FastDiv(tpc * 128), l.f_npix = FastDiv(H2 * W2), l.f_w2 = FastDiv(W2), l.f_o = FastDiv(O);
    return l;
}
PQ_HD LoadWeightTP weight_tp(const bf16 *w, int O, int KS, int C, int tpc) {
    LoadWeightTP l{w, O, KS, C, tpc};
    l.f_o = FastDiv(O);
    l.cls = 0;
    return l;
}
PQ_HD LoadFrames frames(const uint8_t *ring, const int32_t *refs, const int64_t *map,
                        const int32_t *counter, int map_stride, int n, int ref_stride, int ref_off) {
    LoadFrames l;
    l.ring = ring, l.refs = refs, l.map = map, l.counter = counter, l.counter_add = 0, l.map_stride = map_stride;
    l.n = n, l.ref_stride = ref_stride, l.ref_off = ref_off;
    l.f400 = FastDiv(400), l.f20 = FastDiv(20);
    return l;
}

// Patch gather from an activation tile held in SHARED memory (one sample, NHWC
// [H][W][C] bf16, C = 32 or 64): row m = output pixel (oy, ox) of an OH x OW grid,
// col k = (tap t = (kh, kw), channel c); the input pixel is (oy*S + kh*D - pad,
// ox*S + kw*D - pad) (D = +1 convolution, D = -1 transposed-convolution window);
// out-of-range pixels and rows >= rows read zero.  gemm_tile copies such operands
// with plain 16-byte shared loads / stores instead of cp.async.
struct LoadSmemConv {
    static constexpr bool U8 = false, TABLE = false, SMEM = true;
    const bf16 *src;  // generic pointer into shared memory
    int H, W, C, KW, S, D, pad, OW, rows;
    int ty0, tx0;  // tap origin (parity classes: the class's first tap)
    PQ_DEV void at_tile(int) {}
    struct Row {
        int oy, ox;
        bool ok;
    };
    struct Col {
        int kh, kw, c;
    };
    PQ_DEV Row row(int m) const {
        if (m >= rows) return {0, 0, false};
        const int oy = m / OW;
        return {oy, m - oy * OW, true};
    }
    PQ_DEV Col col(int k) const {
        const int t = k / C, c = k - t * C, kh = t / KW;
        return {kh, t - kh * KW, c};
    }
    PQ_DEV const bf16 *at(const Row &R, const Col &c) const {
        if (!R.ok) return nullptr;
        const int iy = R.oy * S + (ty0 + c.kh) * D - pad, ix = R.ox * S + (tx0 + c.kw) * D - pad;
        if (iy < 0 || iy >= H || ix < 0 || ix >= W) return nullptr;
        return src + (iy * W + ix) * C + c.c;
    }
    // unused by the shared-memory path; present for the generic loader interface
    PQ_DEV const void *addr(const Row &, const Col &, int &bytes, const LoadCtx &) const {
        bytes = 0;
        return src;
    }
};

template <class L, class = void>
struct is_smem_src {
    static constexpr bool value = false;
};
template <class L>
struct is_smem_src<L, decltype((void)L::SMEM)> {
    static constexpr bool value = L::SMEM;
};

// ------------------------------------------------------------------------ epilogues
// apply(m, n0, v, cnt, split): tile row m (global), columns n0 .. n0+cnt-1

// conv forward: bf16 NHWC out = relu(acc * scale + bias)
struct EpiBiasRelu {
    bf16 *out;
    const float *bias;
    int M, N, ld;
    float scale;
    // all 32 columns of row m (n0 = 0, N >= 32) to out[m] and to dst2 as well
    PQ_DEV void apply_dual(int m, const float *v, bf16 *dst2) const {
        bf16 *dst = out + (size_t)m * ld;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            float y[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float t = v[j + e] * scale + __ldg(bias + j + e);
                y[e] = t > 0.f ? t : 0.f;
            }
            const uint4 pk = make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]), pack_bf16(y[4], y[5]),
                                        pack_bf16(y[6], y[7]));
            *reinterpret_cast<uint4 *>(dst + j) = pk;
            *reinterpret_cast<uint4 *>(dst2 + j) = pk;
        }
    }
    PQ_DEV void apply(int m, int n0, const float *v, int cnt, int) const {
        float bv[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) bv[e] = (e < cnt && n0 + e < N) ? __ldg(bias + n0 + e) : 0.f;
        if (m >= M) return;
        bf16 *dst = out + (size_t)m * ld;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            const int n = n0 + j;
            if (j >= cnt || n >= N) break;
            float y[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float t = v[j + e] * scale + bv[j + e];
                y[e] = t > 0.f ? t : 0.f;
            }
            *reinterpret_cast<uint4 *>(dst + n) = make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]),
                                                           pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7]));
        }
    }
};

// fp32 store of D transposed: out[split][n][m] (ld = row length m-extent)
struct EpiF32T {
    float *out;
    int M, N, ld;
    size_t split_stride;
    PQ_DEV void apply(int m, int n0, const float *v, int cnt, int split) const {
        if (m >= M) return;
        float *base = out + split * split_stride + m;
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) base[(size_t)n * ld] = v[j];
        }
    }
};

// fp32 row store: out[split][m][n]
struct EpiF32 {
    float *out;
    int M, N, ld;
    size_t split_stride;
    PQ_DEV void apply(int m, int n0, const float *v, int cnt, int split) const {
        if (m >= M) return;
        float *dst = out + split * split_stride + (size_t)m * ld;
        if (n0 + cnt <= N && (ld & 3) == 0) {
            for (int j = 0; j < cnt; j += 4)
                *reinterpret_cast<float4 *>(dst + n0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            return;
        }
        for (int j = 0; j < cnt; ++j)
            if (n0 + j < N) dst[n0 + j] = v[j];
    }
};

// masked bf16 store of up to 32 values (4 x 8) at dst; all mask loads are issued
// before any store (mask = forward activation at the same place)
PQ_DEV void store_masked32(bf16 *dst, const bf16 *mask, const float *v, int nvalid) {
    uint4 mk[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
        mk[c] = c * 8 < nvalid ? __ldg(reinterpret_cast<const uint4 *>(mask + c * 8)) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        if (c * 8 >= nvalid) break;
        const uint32_t mw[4] = {mk[c].x, mk[c].y, mk[c].z, mk[c].w};
        float y[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            y[2 * e] = bf16_lo(mw[e]) > 0.f ? v[c * 8 + 2 * e] : 0.f;
            y[2 * e + 1] = bf16_hi(mw[e]) > 0.f ? v[c * 8 + 2 * e + 1] : 0.f;
        }
        *reinterpret_cast<uint4 *>(dst + c * 8) = make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]),
                                                           pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7]));
    }
}

// A 64-channel row of a data gradient, the mask (forward activation) loaded ahead of the
// accumulator (a TMA kernel's epilogue issues it before waiting for the MMAs), the masked
// bf16 row computed once and stored to every layout the consumers want.
struct MaskRow64 {
    uint4 w[8];
    PQ_DEV void load(const bf16 *mask) {
#pragma unroll
        for (int c = 0; c < 8; ++c) w[c] = __ldg(reinterpret_cast<const uint4 *>(mask) + c);
    }
    // w <- bf16(v * (mask > 0)) in place
    PQ_DEV void apply(const float *v) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t mw[4] = {w[c].x, w[c].y, w[c].z, w[c].w};
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                o[e] = pack_bf16(bf16_lo(mw[e]) > 0.f ? v[c * 8 + 2 * e] : 0.f,
                                 bf16_hi(mw[e]) > 0.f ? v[c * 8 + 2 * e + 1] : 0.f);
            w[c] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
    PQ_DEV void store(bf16 *dst) const {
#pragma unroll
        for (int c = 0; c < 8; ++c) reinterpret_cast<uint4 *>(dst)[c] = w[c];
    }
};

// 32 channels of the same (for conv2's data gradient: one parity class of an s2d pixel)
struct MaskRow32 {
    uint4 w[4];
    PQ_DEV void load(const bf16 *mask) {
#pragma unroll
        for (int c = 0; c < 4; ++c) w[c] = __ldg(reinterpret_cast<const uint4 *>(mask) + c);
    }
    PQ_DEV void apply_store(bf16 *dst, const float *v) const {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t mw[4] = {w[c].x, w[c].y, w[c].z, w[c].w};
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                o[e] = pack_bf16(bf16_lo(mw[e]) > 0.f ? v[c * 8 + 2 * e] : 0.f,
                                 bf16_hi(mw[e]) > 0.f ? v[c * 8 + 2 * e + 1] : 0.f);
            reinterpret_cast<uint4 *>(dst)[c] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
};

// data gradient: bf16 out[m][n] = acc * (mask[m][n] > 0), mask = forward activation
struct EpiMask {
    bf16 *out;
    const bf16 *mask;
    int M, N, ld;
    PQ_DEV void apply(int m, int n0, const float *v, int cnt, int) const {
        if (m >= M || n0 >= N) return;
        const int nv = min(cnt, N - n0);
        store_masked32(out + (size_t)m * ld + n0, mask + (size_t)m * ld + n0, v, nv);
    }
    // 32-column prefetch (the cp.async engine requests it before its dependency wait:
    // the mask is a forward activation of the step, written two or more launches back)
    using Pre = MaskRow32;
    PQ_DEV bool pre_ok(int m, int n0) const { return m < M && n0 + 32 <= N; }
    PQ_DEV void prefetch(Pre &p, int m, int n0) const {
        if (pre_ok(m, n0)) p.load(mask + (size_t)m * ld + n0);
    }
    PQ_DEV void apply_pre(const Pre &p, int m, int n0, const float *v) const {
        if (pre_ok(m, n0)) p.apply_store(out + (size_t)m * ld + n0, v);
        else apply(m, n0, v, 32, 0);
    }
};

// EpiMask that also writes the masked rows of a 9 x 9 map onto a zero-padded 11 x 11
// grid at (y + 1, x + 1) (conv3's data gradient for k_conv2_dgrad_shift)
// fc1's data gradient [b][(y*7 + x)*64 + c] also onto a zero-padded 11 x 11 grid at
// (y + 2, x + 2) (k_conv3_dgrad_shift's operand); rows = samples, columns = (pixel, channel)
struct EpiMaskPad7 {
    EpiMask e;
    bf16 *out_pad;
    PQ_DEV void apply(int m, int n0, const float *v, int cnt, int sp) const {
        e.apply(m, n0, v, cnt, sp);
        if (m >= e.M || n0 >= e.N) return;
        const int p = n0 >> 6, y = p / 7, x = p - y * 7;
        const size_t oo = ((size_t)(m * 11 + y + 2) * 11 + x + 2) * 64 + (n0 & 63);
        store_masked32(out_pad + oo, e.mask + (size_t)m * e.ld + n0, v, min(cnt, e.N - n0));
    }
};

// (and, if out10 is set, onto a 10 x 10 grid at (y, x): k_conv2_wgrad_shift's operand)
struct EpiMaskPad {
    EpiMask e;
    bf16 *out_pad;
    FastDiv f81, f9;
    bf16 *out10;
    PQ_DEV void apply(int m, int n0, const float *v, int cnt, int sp) const {
        e.apply(m, n0, v, cnt, sp);
        if (m >= e.M || n0 >= e.N) return;
        const int s = f81.div(m), q = m - s * 81, y = f9.div(q), x = q - y * 9;
        const size_t oo = ((size_t)(s * 11 + y + 1) * 11 + x + 1) * e.ld + n0;
        store_masked32(out_pad + oo, e.mask + (size_t)m * e.ld + n0, v, min(cnt, e.N - n0));
        if (out10)
            store_masked32(out10 + ((size_t)(s * 10 + y) * 10 + x) * e.ld + n0, e.mask + (size_t)m * e.ld + n0, v,
                           min(cnt, e.N - n0));
    }
};

// EpiMask for LoadTConvP rows (class-major) -> NHWC position of the H x W input
struct EpiMaskP {
    bf16 *out;
    const bf16 *mask;
    int n, H2, W2, C, tpc;
    FastDiv f_per, f_npix, f_w2;
    int pad;  // out on the (2 H2 + 1) x (2 W2 + 1) grid of the space-to-depth conv1 (k_conv1_wgrad_shift)
    PQ_DEV void apply(int m, int n0, const float *v, int cnt, int) const {
        int cls = f_per.div(m), loc = m - cls * tpc * 128;
        int npix = H2 * W2;
        if (loc >= n * npix || n0 >= C) return;
        int b = f_npix.div(loc), rem = loc - b * npix;
        int ry = f_w2.div(rem);
        int iy = 2 * ry + (cls >> 1), ix = 2 * (rem - ry * W2) + (cls & 1);
        size_t o = ((size_t)(b * 2 * H2 + iy) * (2 * W2) + ix) * C + n0;
        size_t oo = pad ? ((size_t)(b * (2 * H2 + 1) + iy) * (2 * W2 + 1) + ix) * C + n0 : o;
        store_masked32(out + oo, mask + o, v, min(cnt, C - n0));
    }
    // prefetch (see EpiMask): the mask offset and the output offset of row m
    struct Pre {
        MaskRow32 mk;
        int64_t o, oo;  // -1: not a live row / not a full 32-column chunk
    };
    PQ_DEV void prefetch(Pre &p, int m, int n0) const {
        p.o = p.oo = -1;
        int cls = f_per.div(m), loc = m - cls * tpc * 128;
        int npix = H2 * W2;
        if (loc >= n * npix || n0 + 32 > C) return;
        int b = f_npix.div(loc), rem = loc - b * npix;
        int ry = f_w2.div(rem);
        int iy = 2 * ry + (cls >> 1), ix = 2 * (rem - ry * W2) + (cls & 1);
        p.o = ((int64_t)(b * 2 * H2 + iy) * (2 * W2) + ix) * C + n0;
        p.oo = pad ? ((int64_t)(b * (2 * H2 + 1) + iy) * (2 * W2 + 1) + ix) * C + n0 : p.o;
        p.mk.load(mask + p.o);
    }
    PQ_DEV void apply_pre(const Pre &p, int m, int n0, const float *v) const {
        if (p.o >= 0) p.mk.apply_store(out + p.oo, v);
        else apply(m, n0, v, 32, 0);
    }
};
PQ_HD EpiMaskP epi_mask_p(bf16 *out, const bf16 *mask, int n, int H2, int W2, int C, int tpc, int pad = 0) {
    EpiMaskP e{out, mask, n, H2, W2, C, tpc};
    e.f_per = FastDiv(tpc * 128), e.f_npix = FastDiv(H2 * W2), e.f_w2 = FastDiv(W2);
    e.pad = pad;
    return e;
}

// data gradient of a swapped GEMM (D[feature][sample]): out[n][m] = acc * (mask[n][m] > 0)
struct EpiMaskT {
    bf16 *out;
    const bf16 *mask;
    int M, N, ld;
    // optional: fc1's data gradient also onto the zero-padded 11 x 11 grid of the shifted
    // conv3 data gradient, out_pad[((b * 11 + y + 2) * 11 + x + 2) * 64 + c] for feature
    // m = (y * 7 + x) * 64 + c of sample b
    bf16 *out_pad;
    PQ_DEV void store_pad(int m, int b, bf16 val) const {
        const int p = m >> 6, y = p / 7, x = p - y * 7;
        out_pad[((size_t)(b * 11 + y + 2) * 11 + x + 2) * 64 + (m & 63)] = val;
    }
    // prefetch (see EpiMask): the 32 samples' mask values of feature m
    struct Pre {
        bf16 mk[32];
    };
    PQ_DEV void prefetch(Pre &p, int m, int n0) const {
        if (m >= M) return;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            p.mk[j] = n0 + j < N ? mask[(size_t)(n0 + j) * ld + m] : __float2bfloat16_rn(0.f);
    }
    PQ_DEV void apply_pre(const Pre &p, int m, int n0, const float *v) const {
        if (m >= M) return;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (n0 + j >= N) break;
            const bf16 val = __float2bfloat16_rn(__bfloat162float(p.mk[j]) > 0.f ? v[j] : 0.f);
            out[(size_t)(n0 + j) * ld + m] = val;
            if (out_pad) store_pad(m, n0 + j, val);
        }
    }
    PQ_DEV void apply(int m, int n0, const float *v, int cnt, int) const {
        if (m >= M) return;
        bf16 mk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
            mk[j] = (j < cnt && n0 + j < N) ? mask[(size_t)(n0 + j) * ld + m] : __float2bfloat16_rn(0.f);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j >= cnt || n0 + j >= N) break;
            const bf16 val = __float2bfloat16_rn(__bfloat162float(mk[j]) > 0.f ? v[j] : 0.f);
            out[(size_t)(n0 + j) * ld + m] = val;
            if (out_pad) store_pad(m, n0 + j, val);
        }
    }
};

// fc1 weight gradient fused with its centered RMSProp update (the contraction over the
// batch is complete in one CTA): D[j][k] = dW4[j][k]; parameter i = base + j*N + k.
// STAGED: the kernel parks the fp32 accumulator tile in shared memory so the update
// walks rows with lanes over consecutive parameters (coalesced p / m / v traffic).
struct EpiRms {
    static constexpr bool STAGED = true;
    const float *p, *m, *v;
    float *p2, *m2, *v2;
    bf16 *shadow;
    float *grad_out;
    int32_t *flag;
    const int32_t *counter;
    float lr, rho, kappa;
    int M, N;
    int64_t pbase, sbase;
    int upd;  // update id reported on a non-finite gradient when counter is NULL
    PQ_DEV void apply(int, int, const float *, int, int) const {}
    // tile: [128][ld] fp32, rows m0.., cols n0.. (width BN).  Rows are walked by warps,
    // lanes cover consecutive parameters (coalesced); 32 / NW rows per round keep
    // 3 x (32 / NW) x BN/32 loads in flight per thread.
    template <int BN>
    PQ_DEV void apply_tile(const float *tile, int ld, int m0, int n0) const {
        apply_tile_w<BN, 8>(tile, ld, m0, n0, threadIdx.x >> 5);
    }
    // the same walk by NW warps (warp = 0..NW-1 of the participating warps)
    template <int BN, int NW, int Q = 8>
    PQ_DEV void apply_tile_w(const float *tile, int ld, int m0, int n0, int warp) const {
        if (BN >= 16 && ((N | pbase | sbase) & 3) == 0) {
            apply_tile_v<BN, NW, Q>(tile, ld, m0, n0, warp);
            return;
        }
        const int lane = threadIdx.x & 31;
        constexpr int U = BN / 32, RR = 32 / NW;
        const float one_m_rho = 1.0f - rho;
        bool bad = false;
        for (int r0 = warp; r0 < 128; r0 += NW * RR) {
            float mm[RR][U], vv[RR][U], pp[RR][U];
            int off[RR][U];
#pragma unroll
            for (int rr = 0; rr < RR; ++rr) {
                const int r = r0 + rr * NW;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int col = lane + 32 * u;
                    const bool ok = m0 + r < M && n0 + col < N;
                    off[rr][u] = ok ? (m0 + r) * N + n0 + col : -1;  // < 2^31 for fc1
                    mm[rr][u] = ok ? __ldcg(m + pbase + off[rr][u]) : 0.f;
                    vv[rr][u] = ok ? __ldcg(v + pbase + off[rr][u]) : 0.f;
                    pp[rr][u] = ok ? __ldcg(p + pbase + off[rr][u]) : 0.f;
                }
            }
#pragma unroll
            for (int rr = 0; rr < RR; ++rr) {
                const int r = r0 + rr * NW;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int o = off[rr][u];
                    if (o < 0) continue;
                    const float g = tile[r * ld + lane + 32 * u];
                    bad |= !isfinite(g);
                    const float mi = rho * mm[rr][u] + one_m_rho * g;
                    const float vi = rho * vv[rr][u] + one_m_rho * g * g;
                    const float pi = pp[rr][u] - lr * g * rsqrtf(vi - mi * mi + kappa);
                    m2[pbase + o] = mi;
                    v2[pbase + o] = vi;
                    p2[pbase + o] = pi;
                    shadow[sbase + o] = __float2bfloat16_rn(pi);
                    if (grad_out) grad_out[pbase + o] = g;
                }
            }
        }
        if (bad) atomicMin(flag, counter ? *counter : upd);
    }
    // float4 walk (N, pbase, sbase multiples of 4): a lane owns 4 consecutive parameters,
    // BN/4 lanes span a tile row, and every thread keeps Q rows x 3 float4 loads in flight
    // (4x the bytes in flight of the scalar walk: the epilogue is L2/HBM-latency bound)
    template <int BN, int NW, int Q>
    PQ_DEV void apply_tile_v(const float *tile, int ld, int m0, int n0, int warp) const {
        constexpr int LPR = BN / 4, RPW = 32 / LPR;
        const int lane = threadIdx.x & 31;
        const int c = (lane % LPR) * 4, rsub = lane / LPR;
        const float one_m_rho = 1.0f - rho;
        bool bad = false;
        for (int r0 = warp * RPW + rsub; r0 < 128; r0 += NW * RPW * Q) {
            float4 mm[Q], vv[Q], pp[Q];
            int off[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int r = r0 + q * NW * RPW;
                const bool ok = r < 128 && m0 + r < M && n0 + c < N;
                off[q] = ok ? (m0 + r) * N + n0 + c : -1;
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                mm[q] = ok ? __ldcg(reinterpret_cast<const float4 *>(m + pbase + off[q])) : z;
                vv[q] = ok ? __ldcg(reinterpret_cast<const float4 *>(v + pbase + off[q])) : z;
                pp[q] = ok ? __ldcg(reinterpret_cast<const float4 *>(p + pbase + off[q])) : z;
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int o = off[q];
                if (o < 0) continue;
                const float *t = tile + (r0 + q * NW * RPW) * ld + c;
                const float g[4] = {t[0], t[1], t[2], t[3]};
                const float ma[4] = {mm[q].x, mm[q].y, mm[q].z, mm[q].w};
                const float va[4] = {vv[q].x, vv[q].y, vv[q].z, vv[q].w};
                const float pa[4] = {pp[q].x, pp[q].y, pp[q].z, pp[q].w};
                float mi[4], vi[4], pi[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    bad |= !isfinite(g[e]);
                    mi[e] = rho * ma[e] + one_m_rho * g[e];
                    vi[e] = rho * va[e] + one_m_rho * g[e] * g[e];
                    pi[e] = pa[e] - lr * g[e] * rsqrtf(vi[e] - mi[e] * mi[e] + kappa);
                }
                *reinterpret_cast<float4 *>(m2 + pbase + o) = make_float4(mi[0], mi[1], mi[2], mi[3]);
                *reinterpret_cast<float4 *>(v2 + pbase + o) = make_float4(vi[0], vi[1], vi[2], vi[3]);
                *reinterpret_cast<float4 *>(p2 + pbase + o) = make_float4(pi[0], pi[1], pi[2], pi[3]);
                __nv_bfloat162 s01 = __floats2bfloat162_rn(pi[0], pi[1]);
                __nv_bfloat162 s23 = __floats2bfloat162_rn(pi[2], pi[3]);
                uint2 sv;
                sv.x = *reinterpret_cast<uint32_t *>(&s01);
                sv.y = *reinterpret_cast<uint32_t *>(&s23);
                *reinterpret_cast<uint2 *>(shadow + sbase + o) = sv;
                if (grad_out)
                    *reinterpret_cast<float4 *>(grad_out + pbase + o) = make_float4(g[0], g[1], g[2], g[3]);
            }
        }
        if (bad) atomicMin(flag, counter ? *counter : upd);
    }
};

// EpiRms for a tile that starts before the launch it follows has finished (GemmOp with
// TriggerHook): its operands (dh1 from the head, act3 from conv3) and p / m / v are older
// than that launch, whose only overlap with this tile is a READ of the W4 bf16 shadow (the
// fc1 data gradient).  So the update runs at once and writes p / m / v, and the tile's new
// shadow values wait in registers for griddepcontrol.wait before they are stored.
struct EpiRms4Late : EpiRms {
    template <int BN>
    PQ_DEV void apply_tile(const float *tile, int ld, int m0, int n0) const {
        constexpr int NW = 8, Q = 4, LPR = BN / 4, RPW = 32 / LPR, STEP = NW * RPW * Q;
        static_assert(BN >= 16 && 128 % STEP == 0, "late RMSProp walk");
        constexpr int IT = 128 / STEP;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int c = (lane % LPR) * 4, rsub = lane / LPR;
        const float one_m_rho = 1.0f - rho;
        bool bad = false;
        uint2 sv[IT][Q];
        int off[IT][Q];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int r0 = warp * RPW + rsub + it * STEP;
            float4 mm[Q], vv[Q], pp[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int r = r0 + q * NW * RPW;
                const bool ok = m0 + r < M && n0 + c < N;
                off[it][q] = ok ? (m0 + r) * N + n0 + c : -1;
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                mm[q] = ok ? __ldcg(reinterpret_cast<const float4 *>(m + pbase + off[it][q])) : z;
                vv[q] = ok ? __ldcg(reinterpret_cast<const float4 *>(v + pbase + off[it][q])) : z;
                pp[q] = ok ? __ldcg(reinterpret_cast<const float4 *>(p + pbase + off[it][q])) : z;
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int o = off[it][q];
                const float *t = tile + (r0 + q * NW * RPW) * ld + c;
                const float g[4] = {t[0], t[1], t[2], t[3]};
                const float ma[4] = {mm[q].x, mm[q].y, mm[q].z, mm[q].w};
                const float va[4] = {vv[q].x, vv[q].y, vv[q].z, vv[q].w};
                const float pa[4] = {pp[q].x, pp[q].y, pp[q].z, pp[q].w};
                float mi[4], vi[4], pi[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    mi[e] = rho * ma[e] + one_m_rho * g[e];
                    vi[e] = rho * va[e] + one_m_rho * g[e] * g[e];
                    pi[e] = pa[e] - lr * g[e] * rsqrtf(vi[e] - mi[e] * mi[e] + kappa);
                }
                __nv_bfloat162 s01 = __floats2bfloat162_rn(pi[0], pi[1]);
                __nv_bfloat162 s23 = __floats2bfloat162_rn(pi[2], pi[3]);
                sv[it][q].x = *reinterpret_cast<uint32_t *>(&s01);
                sv[it][q].y = *reinterpret_cast<uint32_t *>(&s23);
                if (o < 0) continue;
#pragma unroll
                for (int e = 0; e < 4; ++e) bad |= !isfinite(g[e]);
                *reinterpret_cast<float4 *>(m2 + pbase + o) = make_float4(mi[0], mi[1], mi[2], mi[3]);
                *reinterpret_cast<float4 *>(v2 + pbase + o) = make_float4(vi[0], vi[1], vi[2], vi[3]);
                *reinterpret_cast<float4 *>(p2 + pbase + o) = make_float4(pi[0], pi[1], pi[2], pi[3]);
                if (grad_out)
                    *reinterpret_cast<float4 *>(grad_out + pbase + o) = make_float4(g[0], g[1], g[2], g[3]);
            }
        }
        if (bad) atomicMin(flag, counter ? *counter : upd);
        griddep_wait();  // the fc1 data gradient has read the old shadow
#pragma unroll
        for (int it = 0; it < IT; ++it)
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (off[it][q] >= 0) *reinterpret_cast<uint2 *>(shadow + sbase + off[it][q]) = sv[it][q];
    }
};

// epilogues that can request their per-row inputs before the dependency wait
template <class EP, class = void>
struct has_pre {
    static constexpr bool value = false;
    struct Pre {};
};
template <class EP>
struct has_pre<EP, decltype((void)sizeof(typename EP::Pre))> {
    static constexpr bool value = true;
    using Pre = typename EP::Pre;
};

template <class EP, class = void>
struct is_staged {
    static constexpr bool value = false;
};
template <class EP>
struct is_staged<EP, decltype((void)EP::STAGED)> {
    static constexpr bool value = EP::STAGED;
};

// ------------------------------------------------------------------------ kernel
template <class LA, class LB, class EP>
struct GemmArgs {
    LA a[2];
    LB b[2];
    EP e[2];
    int M, N, K;
    int kc_per_split;  // 64-wide K chunks per split
    int splits;
    int ones_at;      // MN-major A: this MN index reads 1.0 (bias-gradient row), -1 = off
    int ones_extent;  // ... for contraction indices < ones_extent
};

constexpr int GEMM_THREADS = 256;
constexpr int GEMM_A_BYTES = 128 * 64 * 2;
constexpr int TABLE_SAMPLES = 64;

template <int BN, bool U8A, int ST = 0>
struct GemmCfg {
    static constexpr int B_BYTES = BN * 128;
    static constexpr int U8_BYTES = U8A ? 128 * 64 : 0;  // raw uint8 staging of the A tile
    static constexpr int STAGE = GEMM_A_BYTES + B_BYTES + U8_BYTES;
#ifndef PQ_MAX_STAGES
#define PQ_MAX_STAGES 4
#endif
    static constexpr int AUTO = (200 * 1024 / STAGE) < PQ_MAX_STAGES ? (200 * 1024 / STAGE) : PQ_MAX_STAGES;
    static constexpr int STAGES = ST > 0 ? ST : AUTO;
    static constexpr int SMEM = STAGES * STAGE + 1024;
};

// Pipeline state a CTA carries from tile to tile: the operand ring (STAGES slots of
// SLOT bytes at a 1024-aligned base), one MMA-completion mbarrier per slot and the
// running K-chunk sequence number (chunk q lives in slot q % STAGES; its slot was last
// used by chunk q - STAGES, whose barrier phase is (q / STAGES - 1) & 1).  A one-shot
// kernel starts at seq 0; the persistent learner keeps counting across tiles, phases
// and updates, so barriers are initialised once per launch.
struct TileRing {
    uint8_t *smem;
    uint32_t smem_s;
    uint64_t *bars;
    uint32_t seq;
    const uint32_t *tmem_s;  // TMEM accumulator base (shared memory, valid after a CTA sync)
    int32_t *table;          // frame-slot table (LoadFrames operands)
};

struct NoHook {
    PQ_DEV void operator()() const {}
};

// One 128 x BN output tile over K-chunks [kb0, kb1): operand gathers into the ring,
// tcgen05.mma into TMEM, fused epilogue.  PF: operand whose data never comes from the
// immediately preceding producer (weights), issued before hook() -- the one-shot
// kernel's griddepcontrol.wait -- so it lands while the predecessor drains
// (0 = none, 1 = A, 2 = B).  All 256 threads enter; returns with TMEM and the ring free.
template <int BN, bool AMN, bool BMN, int STAGES, int SLOT, int PF, class LA, class LB, class EP,
          class Hook, bool FRESH = false>
PQ_DEV void gemm_tile(const LA &la_in, const LB &lb_in, const EP &ep, int kb0, int kb1, int m0, int n0,
                      int split, int ones_at, int ones_extent, TileRing &R, const Hook &hook) {
    static_assert(BN == 16 || BN == 32 || BN == 64 || BN == 128 || BN == 256, "BN");
    static_assert(!BMN || BN >= 64, "MN-major B needs 64-wide swizzle atoms");
    static_assert(!LB::TABLE, "frame tables are A-operand only");
    static_assert(STAGES >= 2, "stages");
    static_assert(GEMM_A_BYTES + BN * 128 + (LA::U8 ? 128 * 64 : 0) <= SLOT, "slot size");
    constexpr int B_BYTES = BN * 128;
    // chunks in flight ahead of the MMA; refilling the slot of chunk i-2 (not i-1)
    // gives each MMA a full iteration to retire before its slot is reused.  Deep rings
    // (>= 8 slots: the small-batch critical-path GEMMs, whose whole K range fits) put
    // every chunk but at most one in flight before the first MMA.
    constexpr int PRE = STAGES >= 8 ? STAGES - 1 : STAGES >= 4 ? STAGES - 2 : STAGES - 1;
    constexpr uint32_t IDESC = idesc_bf16(BN, AMN, BMN);
    constexpr int NA = 1024 / GEMM_THREADS;                   // A chunks per thread (4)
    constexpr int BCH = BN * 8;                               // B chunks per stage
    constexpr int NB = BCH >= GEMM_THREADS ? BCH / GEMM_THREADS : 1;
    constexpr int CPR = BN / 8;                               // MN-major B chunks per K row
    constexpr int BSTEP = BMN ? GEMM_THREADS / CPR : GEMM_THREADS / 8;  // K (resp. MN) rows per i

    LA la = la_in;
    LB lb = lb_in;
    la.at_tile(m0);
    lb.at_tile(m0);
    uint8_t *smem = R.smem;
    const uint32_t smem_s = R.smem_s;
    const uint32_t seq0 = FRESH ? 0u : R.seq;  // FRESH: a one-shot kernel's first tile
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool tl = kProbes && g_tl.on && tl_cta0() && tid == 0;
    int tl_i = 0;
    unsigned long long tl_t[12];
    if (tl) tl_t[tl_i++] = gtime();
    const int nk = kb1 > kb0 ? kb1 - kb0 : 0;
    LoadCtx cx{R.table, 0};

    // fixed per-thread operand contexts
    const int a_c8 = AMN ? (tid & 15) : (tid & 7);      // fixed inner chunk
    const int a_r0 = AMN ? (tid >> 4) : (tid >> 3);     // first outer row
    const int a_rs = AMN ? 16 : 32;                     // outer step per i
    const int b_c8 = BMN ? (tid % CPR) : (tid & 7);
    const int b_r0 = BMN ? (tid / CPR) : (tid >> 3);
    typename LA::Row ra[NA];
    typename LA::Col ca{};
    typename LB::Row rb[NB];
    typename LB::Col cb{};
    if (!AMN) {
#pragma unroll
        for (int i = 0; i < NA; ++i) ra[i] = la.row(m0 + a_r0 + i * a_rs);
    } else {
        ca = la.col(m0 + a_c8 * 8);
    }
    const bool b_live = BCH >= GEMM_THREADS || tid < BCH;
    if (!BMN) {
#pragma unroll
        for (int i = 0; i < NB; ++i) rb[i] = lb.row(n0 + b_r0 + i * BSTEP);
    } else {
        cb = lb.col(n0 + b_c8 * 8);
    }
    const bool has_ones = AMN && ones_at >= m0 + a_c8 * 8 && ones_at < m0 + a_c8 * 8 + 8;

    // slot of local chunk i; before reuse, wait for the MMA of its previous occupant
    auto slot_of = [&](int i) -> int { return (int)((seq0 + (uint32_t)i) % STAGES); };
    auto slot_free = [&](int i) {
        const uint32_t q = seq0 + (uint32_t)i;
        if (q >= STAGES) mbar_wait(&R.bars[q % STAGES], ((q / STAGES) - 1) & 1);
    };
    // issue the cp.async copies of K-chunk kb into ring slot s (A / B separately)
    auto issue_a = [&](int kb, int s) {
        const int k0 = kb * 64;
        const uint32_t a_s = smem_s + s * SLOT;
        const uint32_t u_s = a_s + GEMM_A_BYTES + B_BYTES;
        typename LA::Col cak = AMN ? ca : la.col(k0 + a_c8 * 8);
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int r = a_r0 + i * a_rs;  // outer row within the tile
            const int q = AMN ? (r * 16 + a_c8) : (r * 8 + a_c8);
            typename LA::Row rr = AMN ? la.row(k0 + r) : ra[i];
            if constexpr (is_smem_src<LA>::value) {  // synchronous 16-byte shared copy
                const bf16 *p = la.at(rr, cak);
                const uint4 v = p ? *reinterpret_cast<const uint4 *>(p) : make_uint4(0, 0, 0, 0);
                const uint32_t off = AMN ? mnmaj_off(r, a_c8) : kmaj_off(r, a_c8);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a_s + off), "r"(v.x), "r"(v.y),
                             "r"(v.z), "r"(v.w)
                             : "memory");
                continue;
            }
            int bytes;
            const void *src = la.addr(rr, cak, bytes, cx);
            if constexpr (LA::U8) {
                const uint8_t *p = static_cast<const uint8_t *>(src);
                cp_async4(u_s + q * 8, p, bytes > 0 ? 4 : 0);
                cp_async4(u_s + q * 8 + 4, bytes > 0 ? p + LA::HALF2 : p, bytes > 0 ? 4 : 0);
            } else {
                const uint32_t off = AMN ? mnmaj_off(r, a_c8) : kmaj_off(r, a_c8);
                cp_async16(a_s + off, src, bytes);
            }
        }
    };
    auto issue_b = [&](int kb, int s) {
        if (!b_live) return;
        const int k0 = kb * 64;
        const uint32_t b_s = smem_s + s * SLOT + GEMM_A_BYTES;
        typename LB::Col cbk = BMN ? cb : lb.col(k0 + b_c8 * 8);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int r = b_r0 + i * BSTEP;
            typename LB::Row rr = BMN ? lb.row(k0 + r) : rb[i];
            int bytes;
            const void *src = lb.addr(rr, cbk, bytes, cx);
            const uint32_t off = BMN ? mnmaj_off(r, b_c8) : kmaj_off(r, b_c8);
            cp_async16(b_s + off, src, bytes);
        }
    };
    // after this thread's copies of chunk kb landed: widen its own uint8 chunks to
    // bf16 and write the bias-gradient "ones" element into its own chunk (if any)
    auto post = [&](int kb, int s) {
        if (!LA::U8 && !has_ones) return;
        uint8_t *a_p = smem + s * SLOT;
        const uint8_t *u_p = a_p + GEMM_A_BYTES + B_BYTES;
        const int k0 = kb * 64;
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int r = a_r0 + i * a_rs;
            const int q = AMN ? (r * 16 + a_c8) : (r * 8 + a_c8);
            const uint32_t off = AMN ? mnmaj_off(r, a_c8) : kmaj_off(r, a_c8);
            if (LA::U8) {
                uint2 raw = *reinterpret_cast<const uint2 *>(u_p + q * 8);
                *reinterpret_cast<uint4 *>(a_p + off) = u8x8_to_bf16(raw.x, raw.y);
            }
            if (has_ones && k0 + r < ones_extent)
                *reinterpret_cast<uint16_t *>(a_p + off + (ones_at - m0 - a_c8 * 8) * 2) = 0x3F80;
        }
    };

    // frame-table operands: the sample window of the rows this CTA reads -- MN rows
    // (K-major) or the split's contraction range (MN-major)
    auto fill_table = [&] {
        if constexpr (LA::TABLE) {
            const int lo = AMN ? kb0 * 64 : m0;
            const int hi = AMN ? max(lo, kb1 * 64 - 1) : m0 + 127;
            cx.tb = lo / 400;
            int last = min(hi / 400, cx.tb + TABLE_SAMPLES - 1);
            la.fill(cx.tb, last, R.table);
        }
    };
    // PF == 1 with a frame table (the learner's conv1 forward): the replay frames and
    // records are not written by the predecessor either, so the table is built and the
    // first A chunks requested before the dependency wait
    constexpr bool EARLY_TABLE = LA::TABLE && PF == 1;
    if constexpr (EARLY_TABLE) {
        fill_table();
        __syncthreads();
    }
    // weights (never written by the previous producer) go out before the dependency wait
#pragma unroll
    for (int s = 0; s < PRE; ++s) {
        if (s < nk && PF != 0) {
            slot_free(s);
            if (PF == 1) issue_a(kb0 + s, slot_of(s));
            if (PF == 2) issue_b(kb0 + s, slot_of(s));
        }
    }
    // the epilogue's per-row inputs (data gradients' ReLU masks: forward activations of
    // the step, written two or more launches back) also go out before the wait; each
    // thread owns exactly one 32-column chunk of the tile (BN <= 64)
    constexpr bool EPRE = has_pre<EP>::value && BN <= 64 && BN >= 32 && !is_staged<EP>::value;
    typename has_pre<EP>::Pre epre{};
    const int e_wq = warp & 3, e_half = warp >> 2;
    const int e_row = m0 + e_wq * 32 + lane, e_c0 = BN >= 64 ? e_half * (BN / 2) : 0;
    if constexpr (EPRE)
        if (BN >= 64 || e_half == 0) ep.prefetch(epre, e_row, n0 + e_c0);
    hook();
    ct_mark(1);
    if (tl) tl_t[tl_i++] = gtime();  // 1: predecessor done
    if constexpr (LA::TABLE && !EARLY_TABLE) fill_table();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *R.tmem_s;

    if (tl) tl_t[tl_i++] = gtime();  // 2: contexts ready
#pragma unroll
    for (int s = 0; s < PRE; ++s) {
        if (s < nk) {
            if (PF == 0) slot_free(s);
            if (PF != 1) issue_a(kb0 + s, slot_of(s));
            if (PF != 2) issue_b(kb0 + s, slot_of(s));
        }
        cp_async_commit();
    }
    if (tl) tl_t[tl_i++] = gtime();  // 3: prologue issued
    for (int i = 0; i < nk; ++i) {
        const int s = slot_of(i);
        cp_async_wait<PRE - 1>();
        post(kb0 + i, s);
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t a_addr = smem_s + s * SLOT;
            const uint32_t b_addr = a_addr + GEMM_A_BYTES;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint64_t ad = AMN ? desc_sw128(a_addr + j * 2048, 8192) : desc_sw128(a_addr + j * 32, 0);
                uint64_t bd = BMN ? desc_sw128(b_addr + j * 2048, 8192) : desc_sw128(b_addr + j * 32, 0);
                umma_bf16(tmem, ad, bd, IDESC, (i > 0 || j > 0) ? 1u : 0u);
            }
            umma_commit(&R.bars[s]);
            if (tl && (i == 0 || i == nk - 1)) tl_t[tl_i++] = gtime();  // 4, 5: first / last MMA issued
        }
        const int jn = i + PRE;
        if (jn < nk) {
            const int sl = slot_of(jn);
            slot_free(jn);
            issue_a(kb0 + jn, sl);
            issue_b(kb0 + jn, sl);
        }
        cp_async_commit();
    }
    if (nk > 0) {
        const uint32_t q = seq0 + (uint32_t)(nk - 1);
        mbar_wait(&R.bars[q % STAGES], (q / STAGES) & 1);
    }
    R.seq = seq0 + (uint32_t)nk;
    tc_fence_after();
    ct_mark(2);
    if (tl) tl_t[tl_i++] = gtime();  // 6: accumulator ready

    // epilogue: warp w reads TMEM lanes 32*(w%4).. (tile rows); the two warpgroups
    // split the columns
    const int wq = warp & 3, half = warp >> 2;
    const int row = m0 + wq * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
    constexpr int CW = BN >= 64 ? BN / 2 : BN;  // columns per warpgroup
    if constexpr (is_staged<EP>::value) {
        // park the accumulator tile in the (now idle) operand ring, then let the
        // epilogue walk it row-wise; row stride BN+1 keeps both passes conflict-free
        static_assert(128 * (BN + 1) * 4 <= STAGES * SLOT, "staging tile");
        float *tile = reinterpret_cast<float *>(smem);
        if (BN >= 64 || half == 0) {
            const int cbeg = BN >= 64 ? half * CW : 0;
            for (int c0 = cbeg; c0 < cbeg + CW; c0 += 32) {
                float v[32];
                if (nk > 0) {
                    tmem_ld32(trow + c0, v);
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                }
#pragma unroll
                for (int e = 0; e < 32; ++e) tile[(wq * 32 + lane) * (BN + 1) + c0 + e] = v[e];
            }
        }
        __syncthreads();
        ep.template apply_tile<BN>(tile, BN + 1, m0, n0);
    } else if constexpr (EPRE) {
        if (BN >= 64 || half == 0) {
            float v[32];
            if (nk > 0) {
                tmem_ld32(trow + e_c0, v);
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0.f;
            }
            ep.apply_pre(epre, row, n0 + e_c0, v);
        }
    } else if (BN >= 64 || half == 0) {
        const int cbeg = BN >= 64 ? half * CW : 0;
#pragma unroll 1
        for (int c0 = cbeg; c0 < cbeg + CW; c0 += 32) {
            float v[32];
            if (nk > 0) {
                if (BN >= 32)
                    tmem_ld32(trow + c0, v);
                else
                    tmem_ld16(trow + c0, v);
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0.f;
            }
            ep.apply(row, n0 + c0, v, BN < 32 ? BN : 32, split);
        }
    }
    // TMEM reads and ring reads are complete before anyone starts the next tile
    tc_fence_before();
    __syncthreads();
    if (tl) {
        tl_t[tl_i++] = gtime();  // 7: epilogue done
        const int slot = atomicAdd(&g_tl.n, 1);
        if (slot < 256) {
            for (int k = 0; k < 8; ++k) g_tl.t[slot][k] = k < tl_i ? tl_t[k] : 0ull;
            tl_ident(slot, 'G');
        }
    }
}

struct GridDepHook {
    PQ_DEV void operator()() const {
        griddep_wait();
        griddep_launch();
    }
};
// a tile whose inputs are all older than the launch before (see EpiRms4Late): no wait
struct TriggerHook {
    PQ_DEV void operator()() const { griddep_launch(); }
};

// One-shot kernel: one tile per CTA (grid x = M tiles, y = N tiles, z = group x split).
template <int BN, bool AMN, bool BMN, int ST, int PF, class LA, class LB, class EP>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm(const __grid_constant__ GemmArgs<LA, LB, EP> g) {
    ct_begin();
    using Cfg = GemmCfg<BN, LA::U8, ST>;
    constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[Cfg::STAGES];
    __shared__ uint32_t tmem_base_s;
    __shared__ int32_t table[LA::TABLE ? TABLE_SAMPLES * 4 : 1];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int grp = blockIdx.z / g.splits, split = blockIdx.z - grp * g.splits;
    const int nk_total = (g.K + 63) >> 6;
    const int kb0 = split * g.kc_per_split;
    const int kb1 = min(nk_total, kb0 + g.kc_per_split);
    if (threadIdx.x == 0) {
        for (int s = 0; s < Cfg::STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    if ((threadIdx.x >> 5) == 0) tmem_alloc<TMEM_COLS>(&tmem_base_s);
    TileRing R{smem, smem_u32(smem), bars, 0u, &tmem_base_s, table};
    gemm_tile<BN, AMN, BMN, Cfg::STAGES, Cfg::STAGE, PF, LA, LB, EP, GridDepHook, true>(
        g.a[grp], g.b[grp], g.e[grp], kb0, kb1, blockIdx.x * 128, blockIdx.y * BN, split, g.ones_at,
        g.ones_extent, R, GridDepHook{});
    if ((threadIdx.x >> 5) == 0) tmem_dealloc<TMEM_COLS>(tmem_base_s);
    tl_cta_end('G');
    ct_end('G');
}

template <int BN, bool AMN, bool BMN, int ST = 0, int PF = 0, class LA, class LB, class EP>
cudaError_t launch_gemm(const GemmArgs<LA, LB, EP> &g, int groups, cudaStream_t st, int grid_x = 0) {
    auto kern = k_gemm<BN, AMN, BMN, ST, PF, LA, LB, EP>;
    constexpr int smem = GemmCfg<BN, LA::U8, ST>::SMEM;
    static bool configured = false;  // per instantiation
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid(grid_x ? grid_x : (g.M + 127) / 128, (g.N + BN - 1) / BN, groups * g.splits);
    return launch_k(kern, grid, dim3(GEMM_THREADS), smem, st, g);
}

// ------------------------------------------------------------ fused heterogeneous launches
// Independent GEMMs (and other 256-thread work) of one learner stage share ONE grid:
// CTAs [0, n0) run part 0, [n0, n0 + n1) part 1, ...  On one stream every launch then
// chains to the next by programmatic dependent launch, with no cross-stream joins (a
// joined graph node only starts once all its predecessors have completed), and the
// side work fills SMs next to the critical-path tiles (two CTAs per SM).
template <int BN_, bool AMN_, bool BMN_, int ST_, int PF_, class LA_, class LB_, class EP_,
          class HK_ = GridDepHook>
struct GemmOp {
    using Args = GemmArgs<LA_, LB_, EP_>;
    using Cfg = GemmCfg<BN_, LA_::U8, ST_>;
    static constexpr bool GEMM = true, TABLE = LA_::TABLE;
    static constexpr int SMEM = Cfg::SMEM, STAGES = Cfg::STAGES;
    static constexpr uint32_t TMEM_COLS = BN_ < 32 ? 32 : BN_;
    struct Launch {
        Args g;
        int gx, gy;
    };
    static Launch make(const Args &g) { return Launch{g, (g.M + 127) / 128, (g.N + BN_ - 1) / BN_}; }
    static int ctas(const Launch &l, int groups) { return l.gx * l.gy * groups * l.g.splits; }
    PQ_DEV static void run(const Launch &l, int lin, TileRing &R) {
        const Args &g = l.g;
        const int x = lin % l.gx, y = (lin / l.gx) % l.gy, z = lin / (l.gx * l.gy);
        const int grp = z / g.splits, split = z - grp * g.splits;
        const int nk_total = (g.K + 63) >> 6;
        const int kb0 = split * g.kc_per_split, kb1 = min(nk_total, kb0 + g.kc_per_split);
        gemm_tile<BN_, AMN_, BMN_, STAGES, Cfg::STAGE, PF_, LA_, LB_, EP_, HK_, true>(
            g.a[grp], g.b[grp], g.e[grp], kb0, kb1, x * 128, y * BN_, split, g.ones_at, g.ones_extent, R,
            HK_{});
    }
};
// conv3 data gradient at small batches as a k_fused part, by row-shifted descriptors (the
// cp.async twin of learner.cu k_conv3_dgrad_shift): dY3 on the zero-padded 11 x 11 grid
// (dY3p, written by fc1's data gradient) -- GEMM row r = (s, y, x) of that grid reads row
// r + 11 (2 - kh) + (2 - kw) for tap (kh, kw), so ONE block of 152 rows x 64 channels
// (19 KB) feeds all 9 taps through UMMA descriptors (the SW128 swizzle is a function of
// the shared-memory address) instead of nine 16 KB im2col gathers; W3 as 9 MN-major
// tiles, requested before the dependency wait with each row's ReLU mask.  Same MMA order
// (tap, 16-channel step) as the im2col kernel, so dY2 is bit-identical.
struct Dg3Args {
    const bf16 *dy3p;  // [n * 121][64]
    const bf16 *w3;    // bf16 shadow of W3 [o][kh][kw][c]
    const bf16 *act2;  // ReLU mask [n * 81][64]
    bf16 *dy2;         // [n * 81][64]
    int n;
};
struct Dg3ShiftOp {
    static constexpr bool GEMM = true, TABLE = false;
    static constexpr int ROWS = 152, A_BYTES = 20 * 1024, W_TILE = 8192;
    static constexpr int SMEM = 1024 + 9 * W_TILE + A_BYTES, STAGES = 1;
    static constexpr uint32_t TMEM_COLS = 64;
    struct Launch {
        Dg3Args a;
        int tiles;
    };
    static Launch make(const Dg3Args &a) { return Launch{a, (a.n * 121 + 127) / 128}; }
    static int ctas(const Launch &l, int) { return l.tiles; }
    PQ_DEV static void run(const Launch &l, int t, TileRing &R) {
        const Dg3Args &g = l.a;
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        const uint32_t w_s = R.smem_s, a_s = w_s + 9 * W_TILE;
        // W3: tap tile (kh, kw) = K rows o (64) x N = c (64), MN-major SW128
        for (int i = tid; i < 9 * 64 * 8; i += blockDim.x) {
            const int c8 = i & 7, o = (i >> 3) & 63, tap = i >> 9;
            cp_async16(w_s + tap * W_TILE + mnmaj_off(o, c8), g.w3 + (size_t)o * 576 + tap * 64 + c8 * 8, 16);
        }
        cp_async_commit();
        // this thread's epilogue row and column half, and its ReLU mask
        const int q = warp & 3, h = warp >> 2;
        const int r = t * 128 + q * 32 + lane, smp = r / 121, p = r - smp * 121, y = p / 11, x = p - y * 11;
        const bool live = smp < g.n && y < 9 && x < 9;
        const int m = smp * 81 + y * 9 + x;
        MaskRow32 mk;
        if (live) mk.load(g.act2 + (size_t)m * 64 + h * 32);
        griddep_wait();
        griddep_launch();
        // the 152 padded-grid rows of this tile (zeros past the end), K-major SW128
        const int rows_total = g.n * 121;
        for (int i = tid; i < ROWS * 8; i += blockDim.x) {
            const int c8 = i & 7, rr = i >> 3, row = t * 128 + rr;
            const bool ok = row < rows_total;
            cp_async16(a_s + kmaj_off(rr, c8), ok ? (const void *)(g.dy3p + (size_t)row * 64 + c8 * 8) : (const void *)g.dy3p,
                       ok ? 16 : 0);
        }
        cp_async_commit();
        cp_async_wait<0>();
        fence_proxy_async_smem();
        __syncthreads();
        const uint32_t tmem = *R.tmem_s;
        if (tid == 0) {
            tc_fence_after();
            constexpr uint32_t IDESC = idesc_bf16(64, false, true);
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
                const uint32_t shift = (uint32_t)((2 - tap / 3) * 11 + (2 - tap % 3)) * 128;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    umma_bf16(tmem, desc_sw128(a_s + shift + j * 32, 0), desc_sw128(w_s + tap * W_TILE + j * 2048, 8192),
                              IDESC, (tap > 0 || j > 0) ? 1u : 0u);
            }
            umma_commit(&R.bars[0]);
        }
        mbar_wait(&R.bars[0], 0);
        tc_fence_after();
        float v[32];
        tmem_ld32(tmem + h * 32 + ((uint32_t)(q * 32) << 16), v);
        if (live) mk.apply_store(g.dy2 + (size_t)m * 64 + h * 32, v);
        tc_fence_before();
        __syncthreads();
    }
};

struct NoOp {
    static constexpr bool GEMM = false, TABLE = false;
    static constexpr int SMEM = 0, STAGES = 1;
    static constexpr uint32_t TMEM_COLS = 32;
    struct Launch {};
    PQ_DEV static void run(const Launch &, int, TileRing &) {}
};

template <class P0, class P1, class P2>
struct FusedArgs {
    typename P0::Launch p0;
    typename P1::Launch p1;
    typename P2::Launch p2;
    int n0, n1;  // CTAs of parts 0 and 1
    // optional: CTA 0 copies *stash_src to *stash_dst (a step's update id for launches
    // that must not read the live counter before their dependency wait)
    const int32_t *stash_src;
    int32_t *stash_dst;
    // optional: CTA 0 sets *bump_dst = *bump_src + 1 after its part (i.e. after its
    // dependency wait) -- the pipelined step advances the update counter here instead of
    // in the head, whose CTAs then need no fence + atomic last-block election
    const int32_t *bump_src;
    int32_t *bump_dst;
};

PQ_HD constexpr int cmax(int a, int b) { return a > b ? a : b; }

template <class P0, class P1, class P2>
__global__ void __launch_bounds__(GEMM_THREADS, 2) k_fused(const __grid_constant__ FusedArgs<P0, P1, P2> f) {
    ct_begin();
    constexpr int STAGES = cmax(P0::STAGES, cmax(P1::STAGES, P2::STAGES));
    constexpr uint32_t COLS = (uint32_t)cmax(P0::TMEM_COLS, cmax(P1::TMEM_COLS, P2::TMEM_COLS));
    constexpr bool TABLE = P0::TABLE || P1::TABLE || P2::TABLE;
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[STAGES];
    __shared__ uint32_t tmem_base_s;
    __shared__ int32_t table[TABLE ? TABLE_SAMPLES * 4 : 1];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int lin = blockIdx.x;
    const int part = lin < f.n0 ? 0 : lin < f.n0 + f.n1 ? 1 : 2;
    if (f.stash_dst && lin == 0 && threadIdx.x == 0) *f.stash_dst = *f.stash_src;
    const bool gemm = part == 0 ? P0::GEMM : part == 1 ? P1::GEMM : P2::GEMM;
    if (gemm) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
            fence_mbar_init();
        }
        if ((threadIdx.x >> 5) == 0) tmem_alloc<COLS>(&tmem_base_s);
    }
    TileRing R{smem, smem_u32(smem), bars, 0u, &tmem_base_s, table};
    if (part == 0)
        P0::run(f.p0, lin, R);
    else if (part == 1)
        P1::run(f.p1, lin - f.n0, R);
    else
        P2::run(f.p2, lin - f.n0 - f.n1, R);
    if (f.bump_dst && lin == 0 && threadIdx.x == 0) *f.bump_dst = *f.bump_src + 1;
    if (gemm && (threadIdx.x >> 5) == 0) tmem_dealloc<COLS>(tmem_base_s);
    tl_cta_end('F');
    ct_end('F', part);
}

template <class P0, class P1, class P2>
cudaError_t launch_fused(const FusedArgs<P0, P1, P2> &f, int n2, cudaStream_t st) {
    auto kern = k_fused<P0, P1, P2>;
    constexpr int smem = cmax(P0::SMEM, cmax(P1::SMEM, P2::SMEM));
    static bool configured = false;  // per instantiation
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    return launch_k(kern, dim3(f.n0 + f.n1 + n2), dim3(GEMM_THREADS), smem, st, f);
}

}  // namespace pq
