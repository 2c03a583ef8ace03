// fp64 kernel module on the B200 -- the reference's plugin API (backend.py:18-34,
// _kernels_numba.py:19-111) with bit-identical results.
//
// numba compiles the reference kernels without fastmath and never contracts to FMA
// (SURVEY.md fact 6); every reduction below keeps the reference's per-element order
// and uses explicitly rounded __dmul_rn / __dadd_rn, so each output equals the numba
// value bit for bit.  One thread per output element; the work is tiny (the dense MLP
// of the reference), the point is exact parity at the plugin boundary.
#include "../../include/paraq_b200.h"
#include "common.cuh"

namespace pq {
int cuda_err(cudaError_t e, const char *where);

// _kernels_numba.py:19-31
__global__ void k64_affine_rows(const double *w, const double *b, const double *x, int64_t n,
                                int64_t o, int64_t d, double *out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * o) return;
    const int64_t r = t / o, i = t - r * o;
    const double *wi = w + i * d, *xr = x + r * d;
    double acc = b[i];
    for (int64_t j = 0; j < d; ++j) acc = __dadd_rn(acc, __dmul_rn(wi[j], xr[j]));
    out[t] = acc;
}

// _kernels_numba.py:34-42
__global__ void k64_relu(const double *x, int64_t count, double *out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < count) out[t] = x[t] > 0.0 ? x[t] : 0.0;
}

// _kernels_numba.py:45-52 (delta pre-zeroed by the caller)
__global__ void k64_output_delta(const double *q, const int64_t *actions, const double *targets,
                                 int64_t n, int64_t o, double *delta) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t a = actions[r];
    delta[r * o + a] = __ddiv_rn(q[r * o + a] - targets[r], (double)n);
}

// _kernels_numba.py:55-67: dw[i,j] accumulates over r ascending, skipping dv == 0
__global__ void k64_weight_grad(const double *delta, const double *acts, int64_t n, int64_t o,
                                int64_t d, double *dw) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= o * d) return;
    const int64_t i = t / d, j = t - i * d;
    double acc = 0.0;
    for (int64_t r = 0; r < n; ++r) {
        const double dv = delta[r * o + i];
        if (dv != 0.0) acc = __dadd_rn(acc, __dmul_rn(dv, acts[r * d + j]));
    }
    dw[t] = acc;
}

// _kernels_numba.py:70-77
__global__ void k64_bias_grad(const double *delta, int64_t n, int64_t o, double *db) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= o) return;
    double acc = 0.0;
    for (int64_t r = 0; r < n; ++r) acc = __dadd_rn(acc, delta[r * o + i]);
    db[i] = acc;
}

// _kernels_numba.py:80-95
__global__ void k64_hidden_delta(const double *delta, const double *w, const double *pre,
                                 int64_t n, int64_t o, int64_t d, double *out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * d) return;
    const int64_t r = t / d, j = t - r * d;
    double acc = 0.0;
    if (pre[t] > 0.0) {
        for (int64_t i = 0; i < o; ++i) acc = __dadd_rn(acc, __dmul_rn(delta[r * o + i], w[i * d + j]));
    }
    out[t] = acc;
}

// _kernels_numba.py:98-111
__global__ void k64_rmsprop(const double *p, const double *g, const double *m, const double *v,
                            int64_t count, double lr, double rho, double kappa, double *p2,
                            double *m2, double *v2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double gi = g[i];
    const double one_m_rho = __dsub_rn(1.0, rho);
    const double mi = __dadd_rn(__dmul_rn(rho, m[i]), __dmul_rn(one_m_rho, gi));
    const double vi = __dadd_rn(__dmul_rn(rho, v[i]), __dmul_rn(__dmul_rn(one_m_rho, gi), gi));
    m2[i] = mi;
    v2[i] = vi;
    const double den = __dsqrt_rn(__dadd_rn(__dsub_rn(vi, __dmul_rn(mi, mi)), kappa));
    p2[i] = __dsub_rn(p[i], __ddiv_rn(__dmul_rn(lr, gi), den));
}

static unsigned blocks(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace pq

using namespace pq;

extern "C" {

int pq64_affine_rows(const double *w, const double *b, const double *x, int64_t n, int64_t o,
                     int64_t d, double *out, void *stream) {
    if (n * o == 0) return 0;
    k64_affine_rows<<<blocks(n * o), 256, 0, (cudaStream_t)stream>>>(w, b, x, n, o, d, out);
    return cuda_err(cudaGetLastError(), "affine_rows");
}
int pq64_relu(const double *x, int64_t count, double *out, void *stream) {
    if (count == 0) return 0;
    k64_relu<<<blocks(count), 256, 0, (cudaStream_t)stream>>>(x, count, out);
    return cuda_err(cudaGetLastError(), "relu");
}
int pq64_output_delta(const double *q, const int64_t *actions, const double *targets, int64_t n,
                      int64_t o, double *delta, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int rc = cuda_err(cudaMemsetAsync(delta, 0, sizeof(double) * n * o, st), "output_delta zero");
    if (rc || n == 0) return rc;
    k64_output_delta<<<blocks(n), 256, 0, st>>>(q, actions, targets, n, o, delta);
    return cuda_err(cudaGetLastError(), "output_delta");
}
int pq64_weight_grad(const double *delta, const double *acts, int64_t n, int64_t o, int64_t d,
                     double *dw, void *stream) {
    if (o * d == 0) return 0;
    k64_weight_grad<<<blocks(o * d), 256, 0, (cudaStream_t)stream>>>(delta, acts, n, o, d, dw);
    return cuda_err(cudaGetLastError(), "weight_grad");
}
int pq64_bias_grad(const double *delta, int64_t n, int64_t o, double *db, void *stream) {
    if (o == 0) return 0;
    k64_bias_grad<<<blocks(o), 256, 0, (cudaStream_t)stream>>>(delta, n, o, db);
    return cuda_err(cudaGetLastError(), "bias_grad");
}
int pq64_hidden_delta(const double *delta, const double *w, const double *pre, int64_t n,
                      int64_t o, int64_t d, double *out, void *stream) {
    if (n * d == 0) return 0;
    k64_hidden_delta<<<blocks(n * d), 256, 0, (cudaStream_t)stream>>>(delta, w, pre, n, o, d, out);
    return cuda_err(cudaGetLastError(), "hidden_delta");
}
int pq64_rmsprop_flat(const double *p, const double *g, const double *m, const double *v,
                      int64_t count, double lr, double rho, double kappa, double *p2, double *m2,
                      double *v2, void *stream) {
    if (count == 0) return 0;
    k64_rmsprop<<<blocks(count), 256, 0, (cudaStream_t)stream>>>(p, g, m, v, count, lr, rho,
                                                                  kappa, p2, m2, v2);
    return cuda_err(cudaGetLastError(), "rmsprop_flat");
}

}  // extern "C"
