// Microbenchmarks that separate the three feeds of the TCEC GEMM on one B200:
//   mma  : tcgen05.mma issue rate from resident shared memory (no TMA), for the
//          UMMA shapes the kernel can use (cta_group::1 M=128 N=128/256 and
//          cta_group::2 M=256 N=128/256), in the TCEC pattern (1 main + 2 corr
//          products per K step, 2 accumulators)
//   tma  : TMA (L2 -> smem) feed rate of the GEMM's tile pattern with an
//          instantly-releasing consumer (no MMA)
//   ldtm : TMEM -> register read rate (tcgen05.ld 32x32b.x32) per SM
// Timing: one CTA (or CTA pair) per SM, clock64 cycles inside the kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2303_08989_b200/csrc \
//        tools/mma_probe.cu -o tools/mma_probe
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tcec_common.cuh"

using namespace tcec;

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                   \
            std::exit(1);                                                            \
        }                                                                            \
    } while (0)

// ---------------------------------------------------------------- MMA rate
// smem: 4 stages x (A 16 KB + B N*128 B)
template <int N>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    constexpr int kA = 128 * 128, kB = N * 128, kStage = kA + kB;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 4 * kStage / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    constexpr uint32_t idesc = umma_idesc<kFp16, 128, N>();
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it & 3;
            const uint64_t da = umma_desc_k_sw128(smem + s * kStage);
            const uint64_t db = umma_desc_k_sw128(smem + s * kStage + kA);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t adv = uint64_t((ks * 32) >> 4);
                mma_f16(tmem, da + adv, db + adv, idesc, it | ks);
                mma_f16(tmem + 256, da + adv, db + adv, idesc, it | ks);
                mma_f16(tmem + 256, da + adv, db + adv, idesc, 1u);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// cta_group::2: each CTA holds A 128 rows and B N/2 rows; the leader issues
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_rate(int iters, long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    constexpr int kA = 128 * 128, kB = (N / 2) * 128, kStage = kA + kB;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 4 * kStage / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc_pair<512>(&tbase);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tbase;
    constexpr uint32_t idesc = umma_idesc<kFp16, 256, N>();
    if (threadIdx.x == 0 && rank == 0) {
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it & 3;
            const uint64_t da = umma_desc_k_sw128(smem + s * kStage);
            const uint64_t db = umma_desc_k_sw128(smem + s * kStage + kA);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t adv = uint64_t((ks * 32) >> 4);
                mma2_f16(tmem, da + adv, db + adv, idesc, it | ks);
                mma2_f16(tmem + 256, da + adv, db + adv, idesc, it | ks);
                mma2_f16(tmem + 256, da + adv, db + adv, idesc, 1u);
            }
        }
        mma_commit_pair(&bar, 1);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x >> 1] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem);
    }
}

// ---------------------------------------------------------------- TMA rate
// producer: per k-block A hi/lo (128 rows) + B hi/lo (bn rows) into 3 stages;
// consumer thread releases each stage as soon as it lands
__global__ void __launch_bounds__(64, 1) tma_rate(const __grid_constant__ CUtensorMap ma,
                                                   const __grid_constant__ CUtensorMap mb, int tiles_m,
                                                   int tiles_n, int bn, int nkb, long long* cyc) {
    // hi rows [0, m) / [0, n2), lo rows [m, 2m) / [n2, 2 n2)
    const int m_rows = tiles_m * 128, n_rows = tiles_n * bn;
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = 2 * 16384 + 2 * bn * 128;
    __shared__ uint64_t full[3], empty[3];
    if (threadIdx.x == 0) {
        for (int s = 0; s < 3; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    // grouped rasterization as the GEMM (kGroupM = 16)
    const int id = blockIdx.x;
    const int group = 16 * tiles_n;
    const int first_m = (id / group) * 16;
    const int gsize = min(tiles_m - first_m, 16);
    const int m0 = (first_m + (id % group) % gsize) * 128;
    const int n0 = ((id % group) / gsize) * bn;
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % 3;
            mbar_wait(&empty[s], ((kb / 3) & 1) ^ 1);
            mbar_expect_tx(&full[s], stage_bytes);
            uint8_t* st = smem + s * stage_bytes;
            const int kx = kb * 64;
            tma_load_2d(st, &ma, &full[s], kx, m0);
            tma_load_2d(st + 16384, &ma, &full[s], kx, m_rows + m0);
            for (int r = 0; r < bn; r += 128) {
                tma_load_2d(st + 32768 + r * 128, &mb, &full[s], kx, n0 + r);
                tma_load_2d(st + 32768 + bn * 128 + r * 128, &mb, &full[s], kx, n_rows + n0 + r);
            }
        }
    } else if (threadIdx.x == 32) {
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % 3;
            mbar_wait(&full[s], (kb / 3) & 1);
            mbar_arrive(&empty[s]);
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
}

// --------------------------------------------------- TMA + MMA (no epilogue)
// the GEMM main loop without the epilogue: PRODUCTS = 1 (plain) or 3 (TCEC)
template <int PRODUCTS>
__global__ void __launch_bounds__(64, 1) pipe_rate(const __grid_constant__ CUtensorMap ma,
                                                    const __grid_constant__ CUtensorMap mb, int tiles_m,
                                                    int tiles_n, int nkb, long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    constexpr int kTiles = PRODUCTS == 1 ? 2 : 4;
    constexpr int stage_bytes = kTiles * 16384;
    __shared__ uint64_t full[3], empty[3], done;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 3; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(&tbase);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const int m_rows = tiles_m * 128, n_rows = tiles_n * 128;
    const int id = blockIdx.x;
    const int group = 16 * tiles_n;
    const int first_m = (id / group) * 16;
    const int gsize = min(tiles_m - first_m, 16);
    const int m0 = (first_m + (id % group) % gsize) * 128;
    const int n0 = ((id % group) / gsize) * 128;
    if (warp == 0) {
        if (threadIdx.x == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % 3;
                mbar_wait(&empty[s], ((kb / 3) & 1) ^ 1);
                mbar_expect_tx(&full[s], stage_bytes);
                uint8_t* st = smem + s * stage_bytes;
                const int kx = kb * 64;
                tma_load_2d(st, &ma, &full[s], kx, m0);
                tma_load_2d(st + 16384, &mb, &full[s], kx, n0);
                if (PRODUCTS == 3) {
                    tma_load_2d(st + 32768, &ma, &full[s], kx, m_rows + m0);
                    tma_load_2d(st + 49152, &mb, &full[s], kx, n_rows + n0);
                }
            }
        }
    } else {
        constexpr uint32_t idesc = umma_idesc<kFp16, 128, 128>();
        const long long t0 = clock64();
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % 3;
            mbar_wait(&full[s], (kb / 3) & 1);
            tc_fence_after();
            uint8_t* st = smem + s * stage_bytes;
            const uint64_t dah = umma_desc_k_sw128(st), dbh = umma_desc_k_sw128(st + 16384);
            const uint64_t dal = umma_desc_k_sw128(st + 32768), dbl = umma_desc_k_sw128(st + 49152);
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t adv = uint64_t(2 * ks);
                    mma_f16(tmem, dah + adv, dbh + adv, idesc, (kb | ks) ? 1u : 0u);
                    if (PRODUCTS == 3) {
                        mma_f16(tmem + 384, dal + adv, dbh + adv, idesc, (kb | ks) ? 1u : 0u);
                        mma_f16(tmem + 384, dah + adv, dbl + adv, idesc, 1u);
                    }
                }
                mma_commit(&empty[s]);
                if (kb == nkb - 1) mma_commit(&done);
            }
            __syncwarp();
        }
        mbar_wait(&done, 0);
        if (threadIdx.x == 32) cyc[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ---------------------------------------------------------------- TMEM read
__global__ void __launch_bounds__(256, 1) ldtm_rate(int iters, long long* cyc, float* sink) {
    __shared__ uint32_t tbase;
    if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const int warp = threadIdx.x >> 5;
    const uint32_t base = tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(256 * (warp >> 2));
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        float v[64];
        tmem_ld64(base + uint32_t((it & 3) * 64), v);
#pragma unroll
        for (int i = 0; i < 64; ++i) acc += v[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    if (acc == 12345.f) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 g_enc;

static CUtensorMap make_map(void* base, long long rows, long long kp) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(kp), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(kp) * 2};
    cuuint32_t box[2] = {64u, 128u};
    cuuint32_t estr[2] = {1u, 1u};
    g_enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
}

static double median(std::vector<long long> v) {
    std::sort(v.begin(), v.end());
    return double(v[v.size() / 2]);
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    long long* d_cyc;
    CK(cudaMalloc(&d_cyc, 8192 * sizeof(long long)));
    std::vector<long long> h(8192);
    const int iters = 4096;  // k-blocks of 12 MMAs
    auto run1 = [&](auto kern, int n, size_t smem) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<sms, 128, smem>>>(iters, d_cyc);
        CK(cudaDeviceSynchronize());
        kern<<<sms, 128, smem>>>(iters, d_cyc);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h.data(), d_cyc, sms * 8, cudaMemcpyDeviceToHost));
        const double c = median(std::vector<long long>(h.begin(), h.begin() + sms));
        const double per = c / (iters * 12.0);
        const double ideal = 128.0 * n / 256.0;
        std::printf("mma cta1 M=128 N=%d: %.1f cyc/MMA (floor %.0f) -> %.0f%% of tensor peak\n", n, per, ideal,
                    100.0 * ideal / per);
    };
    run1(mma_rate<128>, 128, 1024 + 4 * (16384 + 128 * 128));
    run1(mma_rate<256>, 256, 1024 + 4 * (16384 + 256 * 128));
    auto run2 = [&](auto kern, int n, size_t smem) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<sms - (sms & 1), 128, smem>>>(iters, d_cyc);
        CK(cudaDeviceSynchronize());
        kern<<<sms - (sms & 1), 128, smem>>>(iters, d_cyc);
        CK(cudaDeviceSynchronize());
        const int np = sms / 2;
        CK(cudaMemcpy(h.data(), d_cyc, np * 8, cudaMemcpyDeviceToHost));
        const double c = median(std::vector<long long>(h.begin(), h.begin() + np));
        const double per = c / (iters * 12.0);
        const double ideal = 256.0 * n / 512.0;
        std::printf("mma cta2 M=256 N=%d: %.1f cyc/MMA (floor %.0f) -> %.0f%% of tensor peak\n", n, per, ideal,
                    100.0 * ideal / per);
    };
    run2(mma2_rate<128>, 128, 1024 + 4 * (16384 + 64 * 128));
    run2(mma2_rate<256>, 256, 1024 + 4 * (16384 + 128 * 128));

    // TMA feed
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    for (int nsz : {4096, 16384}) {
        const long long m = nsz, n2 = 2LL * nsz, kp = 2LL * nsz;
        void *a, *b;
        CK(cudaMalloc(&a, size_t(2 * m * kp * 2)));
        CK(cudaMalloc(&b, size_t(2 * n2 * kp * 2)));
        CK(cudaMemset(a, 0, size_t(2 * m * kp * 2)));
        CK(cudaMemset(b, 0, size_t(2 * n2 * kp * 2)));
        CUtensorMap ma = make_map(a, 2 * m, kp), mb = make_map(b, 2 * n2, kp);
        for (int bn : {128}) {
            const int tiles_m = int(m / 128), tiles_n = int(n2 / bn);
            const int nkb = int(kp / 64);
            const size_t smem = 1024 + 3 * size_t(2 * 16384 + 2 * bn * 128);
            CK(cudaFuncSetAttribute(tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            const int grid = std::min(tiles_m * tiles_n, 4 * sms);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            tma_rate<<<grid, 64, smem>>>(ma, mb, tiles_m, tiles_n, bn, nkb, d_cyc);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            tma_rate<<<grid, 64, smem>>>(ma, mb, tiles_m, tiles_n, bn, nkb, d_cyc);
            cudaEventRecord(e1);
            CK(cudaDeviceSynchronize());
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            CK(cudaMemcpy(h.data(), d_cyc, grid * 8, cudaMemcpyDeviceToHost));
            const double c = median(std::vector<long long>(h.begin(), h.begin() + grid));
            const double stage = 2 * 16384.0 + 2 * bn * 128.0;
            const double bytes = stage * nkb * grid;
            std::printf("tma n=%d tile 128x%d: %.0f cyc/k-block per CTA (%.1f B/cyc/SM), %.2f TB/s L2->SM (%d CTAs)\n",
                        nsz, bn, c / nkb, stage * nkb / c, bytes / (ms * 1e-3) / 1e12, grid);
        }
        // main loop = TMA + MMA, no epilogue
        auto pipe = [&](auto kern, int products) {
            const int tiles_m = int(m / 128), tiles_n = int(n2 / 128), nkb = int(kp / 64);
            const size_t smem = 1024 + 3 * size_t(products == 1 ? 2 : 4) * 16384;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            const int grid = std::min(tiles_m * tiles_n, 4 * sms);
            kern<<<grid, 64, smem>>>(ma, mb, tiles_m, tiles_n, nkb, d_cyc);
            CK(cudaDeviceSynchronize());
            kern<<<grid, 64, smem>>>(ma, mb, tiles_m, tiles_n, nkb, d_cyc);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h.data(), d_cyc, grid * 8, cudaMemcpyDeviceToHost));
            const double c = median(std::vector<long long>(h.begin(), h.begin() + grid));
            const double ideal = 4.0 * products * 64.0;
            std::printf("pipe n=%d products=%d: %.0f cyc/k-block (MMA floor %.0f -> %.0f%%)\n", nsz, products,
                        c / nkb, ideal, 100.0 * ideal / (c / nkb));
        };
        pipe(pipe_rate<1>, 1);
        pipe(pipe_rate<3>, 3);
        cudaFree(a);
        cudaFree(b);
    }
    // TMEM read
    float* sink;
    CK(cudaMalloc(&sink, 4));
    for (int w : {4, 8}) {
        ldtm_rate<<<sms, 32 * w>>>(4096, d_cyc, sink);
        CK(cudaDeviceSynchronize());
        ldtm_rate<<<sms, 32 * w>>>(4096, d_cyc, sink);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h.data(), d_cyc, sms * 8, cudaMemcpyDeviceToHost));
        const double c = median(std::vector<long long>(h.begin(), h.begin() + sms));
        const double bytes = 4096.0 * w * 32 * 64 * 4;
        std::printf("ldtm %d warps: %.1f B/cyc/SM (64 KB main partial drains in %.0f cyc)\n", w, bytes / c,
                    65536.0 / (bytes / c));
    }
    return 0;
}
