// FP64 reference computations of the reference API, on the device:
//   cgemm_oracle             cgemm.cpp:62-74   (gemm_rows_f64 per plane, f64 combine)
//   cgemm_f64 / contract_pair_oracle / contract_network_oracle
//                            network.cpp:87-110, 141-145, 179-186 (gemm_rows_dd)
//   statevector_oracle       qcircuit.cpp:197-225
// These are the reference's f64 "truth" functions (what its own tests and
// experiments measure errors against).  They follow the reference's
// accumulation order exactly: every output is a sequential ascending-k chain
// starting at +0.0 with separate RN multiply and add (the reference is built
// with -ffp-contract=off), so the results are bit-identical to it.  Nothing in
// the TCEC path calls them.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tcec_b200.h"
#include "tcec_handle.h"

namespace tcec {
namespace {

template <typename T>
TCEC_DEV double2 load_c128(const T* p, int64_t i);
template <>
TCEC_DEV double2 load_c128<float2>(const float2* p, int64_t i) {
    const float2 v = p[i];
    return make_double2(v.x, v.y);
}
template <>
TCEC_DEV double2 load_c128<double2>(const double2* p, int64_t i) {
    return p[i];
}

// C (m x n, complex128) = A (m x k) B (k x n): P1 = sum Re Re, P2 = Im Im,
// P3 = Re Im, P4 = Im Re (each an ascending-k RN chain), C = (P1 - P2, P3 + P4).
// 16 x 16 outputs per block, 16-deep k tiles staged in shared memory.
template <typename T>
__global__ void __launch_bounds__(256) cgemm_c128_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                         double2* __restrict__ c, int64_t m, int64_t n,
                                                         int64_t k) {
    __shared__ double2 sa[16][17], sb[16][17];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t tiles_n = (n + 15) / 16;
    const int64_t i0 = (int64_t(blockIdx.x) / tiles_n) * 16, j0 = (int64_t(blockIdx.x) % tiles_n) * 16;
    const int64_t i = i0 + ty, j = j0 + tx;
    double p1 = 0.0, p2 = 0.0, p3 = 0.0, p4 = 0.0;
    for (int64_t k0 = 0; k0 < k; k0 += 16) {
        const int64_t ka = k0 + tx, kb = k0 + ty;
        sa[ty][tx] = (i < m && ka < k) ? load_c128(a, i * k + ka) : make_double2(0.0, 0.0);
        sb[ty][tx] = (kb < k && j < n) ? load_c128(b, kb * n + j) : make_double2(0.0, 0.0);
        __syncthreads();
        const int kend = int(k - k0 < 16 ? k - k0 : 16);
        for (int kk = 0; kk < kend; ++kk) {
            const double2 va = sa[ty][kk], vb = sb[kk][tx];
            p1 = __dadd_rn(p1, __dmul_rn(va.x, vb.x));
            p2 = __dadd_rn(p2, __dmul_rn(va.y, vb.y));
            p3 = __dadd_rn(p3, __dmul_rn(va.x, vb.y));
            p4 = __dadd_rn(p4, __dmul_rn(va.y, vb.x));
        }
        __syncthreads();
    }
    if (i < m && j < n) c[i * n + j] = make_double2(__dsub_rn(p1, p2), __dadd_rn(p3, p4));
}

struct PermDesc {
    int rank;
    int64_t out_dims[kMaxRank];
    int64_t in_stride[kMaxRank];  // input stride of output axis a
};

// permute (tensor.hpp:56-105) of complex128 elements: one thread per output
// element, gather from the input (a pure data movement, bit-exact by construction)
__global__ void permute_c128_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                                    int64_t total, PermDesc d) {
    for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total;
         o += int64_t(gridDim.x) * blockDim.x) {
        int64_t rem = o, in = 0;
        for (int a = d.rank - 1; a >= 0; --a) {
            const int64_t q = rem / d.out_dims[a];
            in += (rem - q * d.out_dims[a]) * d.in_stride[a];
            rem = q;
        }
        dst[o] = src[in];
    }
}

__global__ void widen_kernel(const float2* __restrict__ src, double2* __restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const float2 v = src[i];
        dst[i] = make_double2(v.x, v.y);
    }
}

// complex<double> product as GCC evaluates it for finite operands under
// -ffp-contract=off: (ac - bd, ad + bc)
TCEC_DEV double2 cmul(double2 u, double2 v) {
    return make_double2(__dsub_rn(__dmul_rn(u.x, v.x), __dmul_rn(u.y, v.y)),
                        __dadd_rn(__dmul_rn(u.x, v.y), __dmul_rn(u.y, v.x)));
}
TCEC_DEV double2 cadd(double2 u, double2 v) { return make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y)); }

struct GateU {
    double2 u[4];
};

// one single-qubit gate: every pair (i, i | mq) with bit q clear
__global__ void sv_gate1_kernel(double2* __restrict__ st, int64_t half, int q, GateU g) {
    const int64_t mq = int64_t(1) << q;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < half;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = ((t >> q) << (q + 1)) | (t & (mq - 1));
        const double2 a0 = st[i], a1 = st[i | mq];
        st[i] = cadd(cmul(g.u[0], a0), cmul(g.u[1], a1));
        st[i | mq] = cadd(cmul(g.u[2], a0), cmul(g.u[3], a1));
    }
}

// CZ: negate the amplitudes with both bits set (negation is exact)
__global__ void sv_cz_kernel(double2* __restrict__ st, int64_t dim, int qa, int qb) {
    const int64_t ma = int64_t(1) << qa, mb = int64_t(1) << qb;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < dim;
         i += int64_t(gridDim.x) * blockDim.x)
        if ((i & ma) && (i & mb)) st[i] = make_double2(-st[i].x, -st[i].y);
}

inline unsigned blocks_for(int64_t n, int per = 256) {
    int64_t g = (n + per - 1) / per;
    if (g < 1) g = 1;
    if (g > 148 * 32) g = 148 * 32;
    return unsigned(g);
}

}  // namespace

void launch_cgemm_c128(const void* a, bool a_f32, const void* b, bool b_f32, double2* c, int64_t m,
                       int64_t n, int64_t k, cudaStream_t s) {
    if (m <= 0 || n <= 0) return;
    const int64_t blocks = ((m + 15) / 16) * ((n + 15) / 16);
    // mixed inputs do not occur: both complex64 (cgemm_oracle) or both complex128
    if (a_f32 && b_f32)
        cgemm_c128_kernel<float2><<<unsigned(blocks), 256, 0, s>>>(
            static_cast<const float2*>(a), static_cast<const float2*>(b), c, m, n, k);
    else
        cgemm_c128_kernel<double2><<<unsigned(blocks), 256, 0, s>>>(
            static_cast<const double2*>(a), static_cast<const double2*>(b), c, m, n, k);
}

void launch_permute_c128(const double2* src, double2* dst, int rank, const int64_t* old_dims,
                         const int* axis_of, cudaStream_t s) {
    PermDesc d{};
    d.rank = rank;
    int64_t stride[kMaxRank];
    int64_t total = 1;
    for (int a = rank - 1; a >= 0; --a) {
        stride[a] = total;
        total *= old_dims[a];
    }
    for (int a = 0; a < rank; ++a) {
        d.out_dims[a] = old_dims[axis_of[a]];
        d.in_stride[a] = stride[axis_of[a]];
    }
    if (total <= 0) return;
    permute_c128_kernel<<<blocks_for(total), 256, 0, s>>>(src, dst, total, d);
}

void launch_widen(const float2* src, double2* dst, int64_t n, cudaStream_t s) {
    if (n > 0) widen_kernel<<<blocks_for(n), 256, 0, s>>>(src, dst, n);
}

}  // namespace tcec

using namespace tcec;

#define F64_HANDLE(h)                                                         \
    do {                                                                      \
        if (!(h)) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null handle"); \
        cudaSetDevice((h)->device);                                           \
    } while (0)

extern "C" {

int tcec_cgemm_oracle(tcec_handle h, const void* a, const void* b, void* c, int64_t m, int64_t n,
                      int64_t k) {
    F64_HANDLE(h);
    if (m < 0 || n < 0 || k < 0) return set_error(TCEC_ERR_SHAPE_MISMATCH, "cgemm_oracle: negative extent");
    launch_cgemm_c128(a, true, b, true, static_cast<double2*>(c), m, n, k, h->stream);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TCEC_OK : cuda_error(e, "cgemm_oracle");
}

int tcec_cgemm_c128(tcec_handle h, const void* a, const void* b, void* c, int64_t m, int64_t n,
                    int64_t k) {
    F64_HANDLE(h);
    if (m < 0 || n < 0 || k < 0) return set_error(TCEC_ERR_SHAPE_MISMATCH, "cgemm_f64: negative extent");
    launch_cgemm_c128(a, false, b, false, static_cast<double2*>(c), m, n, k, h->stream);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TCEC_OK : cuda_error(e, "cgemm_f64");
}

int tcec_permute_c128(tcec_handle h, const void* src, void* dst, int rank, const int64_t* old_dims,
                      const int* axis_of) {
    F64_HANDLE(h);
    if (rank < 0 || rank > kMaxRank)
        return set_error(TCEC_ERR_INVALID_PERMUTATION, "permutation has wrong length");
    bool used[kMaxRank] = {false};
    for (int a = 0; a < rank; ++a) {
        const int o = axis_of[a];
        if (o < 0 || o >= rank || used[o])
            return set_error(TCEC_ERR_INVALID_PERMUTATION, "label not in tensor: axis " + std::to_string(o));
        used[o] = true;
        if (old_dims[a] < 1) return set_error(TCEC_ERR_SHAPE_MISMATCH, "tensor extents must be >= 1");
    }
    if (rank == 0) {
        const cudaError_t e = cudaMemcpyAsync(dst, src, 16, cudaMemcpyDeviceToDevice, h->stream);
        return e == cudaSuccess ? TCEC_OK : cuda_error(e, "permute_c128");
    }
    launch_permute_c128(static_cast<const double2*>(src), static_cast<double2*>(dst), rank, old_dims,
                        axis_of, h->stream);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TCEC_OK : cuda_error(e, "permute_c128");
}

int tcec_statevector_f64(tcec_handle h, int n_qubits, int n_gates, const int* qa, const int* qb,
                         const double* u, void* state) {
    F64_HANDLE(h);
    if (n_qubits < 0 || n_qubits > 30) return set_error(TCEC_ERR_TOO_MANY_QUBITS, "state vector too large");
    const int64_t dim = int64_t(1) << n_qubits;
    double2* st = static_cast<double2*>(state);
    cudaStream_t s = h->stream;
    cudaError_t e = cudaMemsetAsync(st, 0, size_t(dim) * sizeof(double2), s);
    const double one[2] = {1.0, 0.0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(st, one, sizeof(one), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_error(e, "statevector init");
    for (int g = 0; g < n_gates; ++g) {
        if (qa[g] < 0 || qa[g] >= n_qubits || (qb[g] >= n_qubits))
            return set_error(TCEC_ERR_SHAPE_MISMATCH, "qubit index out of range");
        if (qb[g] >= 0) {
            sv_cz_kernel<<<blocks_for(dim), 256, 0, s>>>(st, dim, qa[g], qb[g]);
        } else {
            GateU gu;
            for (int i = 0; i < 4; ++i) gu.u[i] = make_double2(u[8 * g + 2 * i], u[8 * g + 2 * i + 1]);
            sv_gate1_kernel<<<blocks_for(dim / 2), 256, 0, s>>>(st, dim / 2, qa[g], gu);
        }
    }
    e = cudaGetLastError();
    return e == cudaSuccess ? TCEC_OK : cuda_error(e, "statevector");
}

}  // extern "C"
