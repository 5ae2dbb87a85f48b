// Does ptxas keep mul.rn.f32x2 + add.rn.f32x2 as two roundings?  Compares the
// packed chain with the scalar __fmul_rn/__fadd_rn chain bit for bit.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__global__ void k(const float* x, const float* y, int n, float* o_pack, float* o_ref) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    float r0 = 0.f, r1 = 0.f;
    for (int i = 0; i < n; ++i) {
        const float a0 = x[(t * n + i) * 2], a1 = x[(t * n + i) * 2 + 1];
        const float b0 = y[(t * n + i) * 2], b1 = y[(t * n + i) * 2 + 1];
        float2 fa = make_float2(a0, a1), fb = make_float2(b0, b1);
        acc = add2(acc, mul2(*reinterpret_cast<uint64_t*>(&fa), *reinterpret_cast<uint64_t*>(&fb)));
        r0 = __fadd_rn(r0, __fmul_rn(a0, b0));
        r1 = __fadd_rn(r1, __fmul_rn(a1, b1));
    }
    float2 v = *reinterpret_cast<float2*>(&acc);
    o_pack[2 * t] = v.x; o_pack[2 * t + 1] = v.y;
    o_ref[2 * t] = r0; o_ref[2 * t + 1] = r1;
}
int main() {
    const int T = 4096, n = 256;
    size_t N = size_t(T) * n * 2;
    float *x, *y, *op, *orf;
    cudaMallocManaged(&x, N * 4); cudaMallocManaged(&y, N * 4);
    cudaMallocManaged(&op, T * 8); cudaMallocManaged(&orf, T * 8);
    srand(1);
    for (size_t i = 0; i < N; ++i) { x[i] = rand() / float(RAND_MAX) * 2 - 1; y[i] = rand() / float(RAND_MAX) * 2 - 1; }
    k<<<T / 128, 128>>>(x, y, n, op, orf);
    cudaDeviceSynchronize();
    int diff = 0;
    for (int i = 0; i < 2 * T; ++i) diff += (*reinterpret_cast<uint32_t*>(&op[i]) != *reinterpret_cast<uint32_t*>(&orf[i]));
    printf("f32x2 chain vs scalar chain: %d of %d outputs differ\n", diff, 2 * T);
    return 0;
}
