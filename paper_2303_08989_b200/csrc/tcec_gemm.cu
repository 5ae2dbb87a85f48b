// TCEC complex GEMM on sm_100a tensor cores (tcgen05 + TMA + TMEM).
//
// The complex product C = A B (A m x k, B k x n, interleaved c32) runs as ONE
// real GEMM C' = A' B' with A' = A viewed as m x 2k (interleaved (re, im)
// columns) and B' the 2k x 2n block expansion of B (prepared K-major by
// prep_b_kernel), so C' is exactly the interleaved C.  Each real operand is
// split into (hi, lo) in FP16 or TF32 (reference lowprec.hpp:84-88) and the
// error-corrected product (reference gemm.cpp:92-106, kernels_scalar.cpp:102-135,
// PAPER.md Eq. 2) is
//
//     C' = RN( main + corr * 2^-11 ),  main = Ah Bh,  corr = Al Bh + Ah Bl
//
// main and corr accumulate in separate TMEM accumulators.  Following the
// paper's rounding-mode care ("FP32 SIMT cores for addition with
// RN ... to avoid the RZ rounding inside Tensor Cores"), the main term can be
// flushed every `flush_kblocks` k-blocks: the MMA warp rotates the main
// accumulator over three TMEM buffers and the epilogue warps fold each
// finished partial into a register accumulator with __fadd_rn while the tensor
// core fills the other buffer.  The correction term stays in TMEM for the whole
// K (its error is scaled by 2^-11).  The epilogue applies the FP16TCEC_SCALED
// descale 2^-(sa+sb) (precsel.cpp:171-174) and stores C.
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// MMA issuer (the whole warp runs the loop, one elected lane issues), warps
// 2..9 = epilogue (TMEM lane quadrant warp%4, two 64-column halves).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "tcec_common.cuh"
#include "tcec_internal.h"

namespace tcec {

namespace {

constexpr int BM = 128;           // rows of C' per CTA (UMMA M)
constexpr int BN = 128;           // columns of C' per CTA (UMMA N)
constexpr int kStages = 3;
constexpr int kTileBytes = 128 * 128;  // one operand tile: 128 rows x 128 B (swizzle-128B)
constexpr int kEpiWarps = 8;      // 2 warps per TMEM lane quadrant, 64 columns each
constexpr int kThreadsGemm = 64 + 32 * kEpiWarps;
constexpr int kGroupM = 16;       // rasterization: CTAs of a wave share A/B panels in L2
constexpr int kWideGroupM = 4;    // the same for the 256 x 256 pair tiles (swept: 4 minimises DRAM re-reads)
constexpr uint32_t kTmemCols = 512;
constexpr int kMainBufs = 3;      // ping-pong-pong main partials: cols 0, 128, 256
constexpr uint32_t kColCorr = 384;
constexpr int kCStride = BN + 4;  // padded smem row (floats) of the staged C tile

template <int FMT>
struct Traits {
    static constexpr int kElem = FMT == kFp16 ? 2 : 4;
    static constexpr int kBK = 128 / kElem;              // elements per 128-B row
    static constexpr int kUK = FMT == kFp16 ? 16 : 8;    // K per tcgen05.mma
    static constexpr int kKSteps = kBK / kUK;            // 4
    static constexpr uint32_t kIdesc = umma_idesc<FMT, BM, BN>();
};

template <int kS>
struct alignas(8) SmemTailT {
    uint64_t full[kS];
    uint64_t empty[kS];
    uint64_t tfull[kMainBufs];
    uint64_t tempty[kMainBufs];
    uint32_t tmem_base;
};
using GemmSmemTail = SmemTailT<kStages>;

constexpr size_t kSmemBytes = 1024 /*align slack*/ + size_t(kStages) * 4 * kTileBytes +
                              sizeof(GemmSmemTail);
static_assert(size_t(BM) * kCStride * 4 <= size_t(kStages) * 4 * kTileBytes,
              "C staging tile must fit in the operand stages");

TCEC_DEV void epi_bar_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
}

// A-expanded layout store: one C row from the staged Re row `s0` and the Im
// row s0 + cs (COLS columns, `valid` of them inside C): each lane interleaves
// 4 columns at a time into two 16-B stores, a warp writes 1 KB contiguous
template <int COLS>
TCEC_DEV void store_xa_row(float* __restrict__ dst, const float* s0, int cs, int valid, bool full, int lane) {
    const float* s1 = s0 + cs;
    if (full) {
#pragma unroll
        for (int j = 4 * lane; j < COLS; j += 128) {
            const float4 re = *reinterpret_cast<const float4*>(s0 + j);
            const float4 im = *reinterpret_cast<const float4*>(s1 + j);
            float4* d4 = reinterpret_cast<float4*>(dst + 2 * j);
            __stcs(d4, make_float4(re.x, im.x, re.y, im.y));
            __stcs(d4 + 1, make_float4(re.z, im.z, re.w, im.w));
        }
    } else {
        for (int j = lane; j < COLS && j < valid; j += 32) {
            dst[2 * j] = s0[j];
            dst[2 * j + 1] = s1[j];
        }
    }
}

template <int FMT>
__global__ void __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_kernel(const __grid_constant__ CUtensorMap map_ahi,
                     const __grid_constant__ CUtensorMap map_alo,
                     const __grid_constant__ CUtensorMap map_bhi,
                     const __grid_constant__ CUtensorMap map_blo, float* __restrict__ c,
                     int m, int n2, int kp, const DevDecision* __restrict__ dec, int kind_fixed,
                     int corrected, int flush_kblocks, float* __restrict__ partial, int kb_per, int xa) {
    using T = Traits<FMT>;
    // device-side mode selection: the kernel of the unselected format exits
    // (the paper's "both kernels launched, one exits early")
    const int kind = kind_fixed >= 0 ? kind_fixed : dec->kind;
    const bool mine = FMT == kTf32 ? kind == kKindTf32 : (kind == kKindFp16 || kind == kKindFp16Scaled);
    if (!mine) return;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    GemmSmemTail* tail = reinterpret_cast<GemmSmemTail*>(smem + size_t(kStages) * 4 * kTileBytes);
    auto tile = [&](int stage, int which) -> uint8_t* {
        return smem + (size_t(stage) * 4 + which) * kTileBytes;
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // grouped rasterization over (m_blk, n_blk)
    const int tiles_m = (m + BM - 1) / BM, tiles_n = (n2 + BN - 1) / BN;
    const int id = blockIdx.x;
    const int group = kGroupM * tiles_n;
    const int first_m = (id / group) * kGroupM;
    const int gsize = min(tiles_m - first_m, kGroupM);
    const int m_blk = first_m + (id % group) % gsize;
    const int n_blk = (id % group) / gsize;
    const int m0 = m_blk * BM, n0 = n_blk * BN;

    // split-K (gridDim.y > 1, few tiles and long K): this CTA chains k-blocks
    // [kb_base, kb_base + nkb) and writes an un-descaled fp32 partial that
    // split_reduce_kernel sums in split order
    const int nkb_all = kp / T::kBK;
    const int per = FMT == kTf32 ? 2 * kb_per : kb_per;  // kb_per counts 64-element f16 blocks
    const int kb_base = partial ? int(blockIdx.y) * per : 0;
    const int nkb = partial ? min(per, nkb_all - kb_base) : nkb_all;
    const int F = flush_of(flush_kblocks, FMT) > 0 ? flush_of(flush_kblocks, FMT) : (nkb > 0 ? nkb : 1);
    const int nchunks = (nkb + F - 1) / F;
    const uint32_t stage_bytes = uint32_t(corrected ? 4 : 2) * kTileBytes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&tail->full[s], 1);
            mbar_init(&tail->empty[s], 1);
        }
        for (int b = 0; b < kMainBufs; ++b) {
            mbar_init(&tail->tfull[b], 1);
            mbar_init(&tail->tempty[b], kEpiWarps);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&map_ahi);
        tma_prefetch(&map_bhi);
        if (corrected) {
            tma_prefetch(&map_alo);
            tma_prefetch(&map_blo);
        }
    }
    if (warp == 1) tmem_alloc<kTmemCols>(&tail->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tail->tmem_base;

    if (warp == 0) {
        // ---------------------------------------------------- TMA producer
        if (lane == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kStages;
                const uint32_t ph = (kb / kStages) & 1;
                mbar_wait(&tail->empty[s], ph ^ 1);
                mbar_expect_tx(&tail->full[s], stage_bytes);
                const int kx = (kb_base + kb) * T::kBK;
                tma_load_2d(tile(s, 0), &map_ahi, &tail->full[s], kx, m0);
                tma_load_2d(tile(s, 2), &map_bhi, &tail->full[s], kx, n0);
                if (corrected) {
                    tma_load_2d(tile(s, 1), &map_alo, &tail->full[s], kx, m0);
                    tma_load_2d(tile(s, 3), &map_blo, &tail->full[s], kx, n0);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        // The whole warp runs the loop (waits and operand math stay
        // warp-uniform, in uniform registers); one elected lane issues.
        for (int kb = 0; kb < nkb; ++kb) {
            const int chunk = kb / F;
            const int buf = chunk % kMainBufs;
            const bool chunk_start = (kb % F) == 0;
            if (chunk_start) {
                mbar_wait(&tail->tempty[buf], ((chunk / kMainBufs) & 1) ^ 1);
                tc_fence_after();
            }
            const int s = kb % kStages;
            mbar_wait(&tail->full[s], (kb / kStages) & 1);
            tc_fence_after();
            const uint64_t dah = umma_desc_k_sw128(tile(s, 0));
            const uint64_t dal = umma_desc_k_sw128(tile(s, 1));
            const uint64_t dbh = umma_desc_k_sw128(tile(s, 2));
            const uint64_t dbl = umma_desc_k_sw128(tile(s, 3));
            const uint32_t d_main = tmem + uint32_t(buf * BN);
            const uint32_t d_corr = tmem + kColCorr;
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < T::kKSteps; ++ks) {
                    const uint64_t adv = uint64_t((ks * T::kUK * T::kElem) >> 4);
                    const uint32_t acc_main = (!chunk_start || ks > 0) ? 1u : 0u;
                    const uint32_t acc_corr = (kb > 0 || ks > 0) ? 1u : 0u;
                    if (FMT == kFp16) {
                        mma_f16(d_main, dah + adv, dbh + adv, T::kIdesc, acc_main);
                        if (corrected) {
                            mma_f16(d_corr, dal + adv, dbh + adv, T::kIdesc, acc_corr);
                            mma_f16(d_corr, dah + adv, dbl + adv, T::kIdesc, 1u);
                        }
                    } else {
                        mma_tf32(d_main, dah + adv, dbh + adv, T::kIdesc, acc_main);
                        if (corrected) {
                            mma_tf32(d_corr, dal + adv, dbh + adv, T::kIdesc, acc_corr);
                            mma_tf32(d_corr, dah + adv, dbl + adv, T::kIdesc, 1u);
                        }
                    }
                }
                mma_commit(&tail->empty[s]);
                if ((kb % F) == F - 1 || kb == nkb - 1) mma_commit(&tail->tfull[buf]);
            }
            __syncwarp();
        }
    } else {
        // -------------------------------------------------------- epilogue
        // warp w owns TMEM lanes 32*(w%4).. (the hardware quadrant rule) and
        // the 64-column half (w-2)/4 of the tile
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const int rloc = 32 * q + lane;
        const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16) + uint32_t(64 * half);
        constexpr int kCols = BN / 2;
        // -0 is the identity of RN addition (-0 + x == x for every x, zeros
        // included), so every partial folds in with one FADD
        float acc[kCols];
#pragma unroll
        for (int i = 0; i < kCols; ++i) acc[i] = -0.0f;
        for (int ch = 0; ch < nchunks; ++ch) {
            const int buf = ch % kMainBufs;
            mbar_wait(&tail->tfull[buf], (ch / kMainBufs) & 1);
            tc_fence_after();
            float v[kCols];
            tmem_ld64(lane_base + uint32_t(buf * BN), v);
            // the partial is in registers: hand the TMEM buffer back first
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tail->tempty[buf]);
#pragma unroll
            for (int i = 0; i < kCols; ++i) acc[i] = __fadd_rn(acc[i], v[i]);
        }
        if (corrected && nkb > 0) {
#pragma unroll
            for (int cb = 0; cb < kCols / 32; ++cb) {
                float v[32];
                tmem_ld32(lane_base + kColCorr + uint32_t(32 * cb), v);
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    acc[32 * cb + i] = __fadd_rn(acc[32 * cb + i], __fmul_rn(v[i], 0x1.0p-11f));
            }
        }
        const bool scaled = !partial && kind == kKindFp16Scaled && (dec->scale_a + dec->scale_b) != 0;
        if (scaled) {
            const double f = ldexp(1.0, -(dec->scale_a + dec->scale_b));
#pragma unroll
            for (int i = 0; i < kCols; ++i) acc[i] = scale_pow2(acc[i], f);
        }
        if (partial) c = partial + size_t(blockIdx.y) * size_t(m) * size_t(n2);
        // stage the tile in the (now idle) operand smem, then store coalesced rows
        float* ctile = reinterpret_cast<float*>(smem);
        float* myrow = ctile + size_t(rloc) * kCStride + kCols * half;
#pragma unroll
        for (int i = 0; i < kCols; i += 4)
            *reinterpret_cast<float4*>(myrow + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
        epi_bar_sync();
        const int ew = warp - 2;
        const bool full_cols = n0 + BN <= n2 && (n2 & 3) == 0;
        if (xa && !partial) {
            // A-expanded layout: tile rows 2i / 2i+1 = Re / Im of C row m0/2 + i
            for (int r = ew; r < BM / 2; r += kEpiWarps) {
                if (m0 + 2 * r >= m) break;
                store_xa_row<BN>(c + size_t(m0 / 2 + r) * (2 * size_t(n2)) + 2 * size_t(n0),
                                 ctile + size_t(2 * r) * kCStride, kCStride, n2 - n0, full_cols, lane);
            }
        } else
        for (int r = ew; r < BM; r += kEpiWarps) {
            const int grow = m0 + r;
            if (grow >= m) break;
            float* dst = c + size_t(grow) * n2 + n0;
            const float* srow = ctile + size_t(r) * kCStride;
            if (full_cols) {
                reinterpret_cast<float4*>(dst)[lane] = reinterpret_cast<const float4*>(srow)[lane];
            } else {
                for (int i = lane; i < BN; i += 32)
                    if (n0 + i < n2) dst[i] = srow[i];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

// split-K epilogue: C = descale(sum of the partials in split order), RN
// (A-expanded layout: output float o = (i, j, e) of C reads GEMM row 2i + e, column j)
__global__ void __launch_bounds__(256) split_reduce_kernel(const float* __restrict__ partial,
                                                           float* __restrict__ c, int64_t count,
                                                           int splits, const DevDecision* __restrict__ dec,
                                                           int kind_fixed, int64_t xa_cols) {
    const int kind = kind_fixed >= 0 ? kind_fixed : dec->kind;
    const bool scaled = kind == kKindFp16Scaled && (dec->scale_a + dec->scale_b) != 0;
    const double f = scaled ? ldexp(1.0, -(dec->scale_a + dec->scale_b)) : 1.0;
    for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < count;
         o += int64_t(gridDim.x) * blockDim.x) {
        int64_t i = o;
        if (xa_cols > 0) {
            const int64_t row = o / (2 * xa_cols), rem = o - row * 2 * xa_cols;
            i = (2 * row + (rem & 1)) * xa_cols + (rem >> 1);
        }
        float s = partial[i];
        for (int y = 1; y < splits; ++y) s = __fadd_rn(s, partial[size_t(y) * size_t(count) + size_t(i)]);
        c[o] = scaled ? scale_pow2(s, f) : s;
    }
}

// ===================================================================== CTA pair
// cta_group::2 variant: a cluster of 2 CTAs computes a 256 x 128 tile of C'
// with UMMA M = 256.  Each CTA stages its own 128 rows of A and 64 of the 128
// B rows (48 KB per k-block instead of 64 KB for the same MACs per SM), the
// leader issues the MMAs for both and multicasts its commits; each CTA drains
// its own 128 TMEM lanes.  4 smem stages.
constexpr int kPairStages = 4;
constexpr int kPairATile = 128 * 128;   // 128 rows x 128 B
constexpr int kPairBTile = 64 * 128;    // 64 rows x 128 B
constexpr int kPairStageBytes = 2 * kPairATile + 2 * kPairBTile;  // per CTA, corrected
using PairSmemTail = SmemTailT<kPairStages>;
constexpr size_t kPairSmemBytes = 1024 + size_t(kPairStages) * kPairStageBytes + sizeof(PairSmemTail);
static_assert(size_t(BM) * kCStride * 4 <= size_t(kPairStages) * kPairStageBytes,
              "C staging tile must fit in the operand stages");

template <int FMT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_pair_kernel(const __grid_constant__ CUtensorMap map_ahi,
                          const __grid_constant__ CUtensorMap map_alo,
                          const __grid_constant__ CUtensorMap map_bhi,
                          const __grid_constant__ CUtensorMap map_blo, float* __restrict__ c,
                          int m, int n2, int kp, const DevDecision* __restrict__ dec, int kind_fixed,
                          int corrected, int flush_kblocks) {
    using T = Traits<FMT>;
    constexpr uint32_t kIdesc2 = umma_idesc<FMT, 2 * BM, BN>();
    const int kind = kind_fixed >= 0 ? kind_fixed : dec->kind;
    const bool mine = FMT == kTf32 ? kind == kKindTf32 : (kind == kKindFp16 || kind == kKindFp16Scaled);
    if (!mine) return;  // both CTAs of the pair read the same decision

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    PairSmemTail* tail =
        reinterpret_cast<PairSmemTail*>(smem + size_t(kPairStages) * kPairStageBytes);
    // stage layout: A_hi | A_lo | B_hi | B_lo
    auto a_tile = [&](int s, int lo) -> uint8_t* {
        return smem + size_t(s) * kPairStageBytes + size_t(lo) * kPairATile;
    };
    auto b_tile = [&](int s, int lo) -> uint8_t* {
        return smem + size_t(s) * kPairStageBytes + 2 * kPairATile + size_t(lo) * kPairBTile;
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    const int tiles_m = (m + 2 * BM - 1) / (2 * BM), tiles_n = (n2 + BN - 1) / BN;
    const int id = blockIdx.x >> 1;
    const int group = kGroupM * tiles_n;
    const int first_m = (id / group) * kGroupM;
    const int gsize = min(tiles_m - first_m, kGroupM);
    const int m_blk = first_m + (id % group) % gsize;
    const int n_blk = (id % group) / gsize;
    const int m0 = m_blk * 2 * BM + int(rank) * BM;  // this CTA's 128 rows
    const int n0 = n_blk * BN;                       // the pair's 128 columns

    const int nkb = kp / T::kBK;
    const int F = flush_of(flush_kblocks, FMT) > 0 ? flush_of(flush_kblocks, FMT) : (nkb > 0 ? nkb : 1);
    const int nchunks = (nkb + F - 1) / F;
    const uint32_t cta_bytes = corrected ? uint32_t(kPairStageBytes)
                                         : uint32_t(kPairATile + kPairBTile);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPairStages; ++s) {
            mbar_init(&tail->full[s], 1);
            mbar_init(&tail->empty[s], 1);
        }
        for (int b = 0; b < kMainBufs; ++b) {
            mbar_init(&tail->tfull[b], 1);
            mbar_init(&tail->tempty[b], 2 * kEpiWarps);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&map_ahi);
        tma_prefetch(&map_bhi);
        if (corrected) {
            tma_prefetch(&map_alo);
            tma_prefetch(&map_blo);
        }
    }
    if (warp == 1) tmem_alloc_pair<kTmemCols>(&tail->tmem_base);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tail->tmem_base;

    if (warp == 0) {
        // -------------------------------------------- TMA producer (both CTAs)
        if (lane == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kPairStages;
                mbar_wait(&tail->empty[s], ((kb / kPairStages) & 1) ^ 1);
                if (leader) mbar_expect_tx(&tail->full[s], 2 * cta_bytes);
                const int kx = kb * T::kBK;
                tma_load_2d_pair(a_tile(s, 0), &map_ahi, &tail->full[s], kx, m0);
                tma_load_2d_pair(b_tile(s, 0), &map_bhi, &tail->full[s], kx, n0 + 64 * int(rank));
                if (corrected) {
                    tma_load_2d_pair(a_tile(s, 1), &map_alo, &tail->full[s], kx, m0);
                    tma_load_2d_pair(b_tile(s, 1), &map_blo, &tail->full[s], kx, n0 + 64 * int(rank));
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------- MMA issuer (pair leader only)
        if (leader) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int chunk = kb / F;
                const int buf = chunk % kMainBufs;
                const bool chunk_start = (kb % F) == 0;
                if (chunk_start) {
                    mbar_wait(&tail->tempty[buf], ((chunk / kMainBufs) & 1) ^ 1);
                    tc_fence_after();
                }
                const int s = kb % kPairStages;
                mbar_wait(&tail->full[s], (kb / kPairStages) & 1);
                tc_fence_after();
                const uint64_t dah = umma_desc_k_sw128(a_tile(s, 0));
                const uint64_t dal = umma_desc_k_sw128(a_tile(s, 1));
                const uint64_t dbh = umma_desc_k_sw128(b_tile(s, 0));
                const uint64_t dbl = umma_desc_k_sw128(b_tile(s, 1));
                const uint32_t d_main = tmem + uint32_t(buf * BN);
                const uint32_t d_corr = tmem + kColCorr;
                if (elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < T::kKSteps; ++ks) {
                        const uint64_t adv = uint64_t((ks * T::kUK * T::kElem) >> 4);
                        const uint32_t acc_main = (!chunk_start || ks > 0) ? 1u : 0u;
                        const uint32_t acc_corr = (kb > 0 || ks > 0) ? 1u : 0u;
                        if (FMT == kFp16) {
                            mma2_f16(d_main, dah + adv, dbh + adv, kIdesc2, acc_main);
                            if (corrected) {
                                mma2_f16(d_corr, dal + adv, dbh + adv, kIdesc2, acc_corr);
                                mma2_f16(d_corr, dah + adv, dbl + adv, kIdesc2, 1u);
                            }
                        } else {
                            mma2_tf32(d_main, dah + adv, dbh + adv, kIdesc2, acc_main);
                            if (corrected) {
                                mma2_tf32(d_corr, dal + adv, dbh + adv, kIdesc2, acc_corr);
                                mma2_tf32(d_corr, dah + adv, dbl + adv, kIdesc2, 1u);
                            }
                        }
                    }
                    mma_commit_pair(&tail->empty[s], 0x3);
                    if ((kb % F) == F - 1 || kb == nkb - 1) mma_commit_pair(&tail->tfull[buf], 0x3);
                }
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------ epilogue (both CTAs)
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const int rloc = 32 * q + lane;
        const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16) + uint32_t(64 * half);
        constexpr int kCols = BN / 2;
        const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tail->tempty[0]), 0);
        float acc[kCols];
#pragma unroll
        for (int i = 0; i < kCols; ++i) acc[i] = -0.0f;  // RN identity
        for (int ch = 0; ch < nchunks; ++ch) {
            const int buf = ch % kMainBufs;
            mbar_wait(&tail->tfull[buf], (ch / kMainBufs) & 1);
            tc_fence_after();
            float v[kCols];
            tmem_ld64(lane_base + uint32_t(buf * BN), v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader0 + uint32_t(buf * sizeof(uint64_t)));
#pragma unroll
            for (int i = 0; i < kCols; ++i) acc[i] = __fadd_rn(acc[i], v[i]);
        }
        if (corrected && nkb > 0) {
#pragma unroll
            for (int cb = 0; cb < kCols / 32; ++cb) {
                float v[32];
                tmem_ld32(lane_base + kColCorr + uint32_t(32 * cb), v);
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    acc[32 * cb + i] = __fadd_rn(acc[32 * cb + i], __fmul_rn(v[i], 0x1.0p-11f));
            }
        }
        const bool scaled = kind == kKindFp16Scaled && (dec->scale_a + dec->scale_b) != 0;
        if (scaled) {
            const double f = ldexp(1.0, -(dec->scale_a + dec->scale_b));
#pragma unroll
            for (int i = 0; i < kCols; ++i) acc[i] = scale_pow2(acc[i], f);
        }
        float* ctile = reinterpret_cast<float*>(smem);
        float* myrow = ctile + size_t(rloc) * kCStride + kCols * half;
#pragma unroll
        for (int i = 0; i < kCols; i += 4)
            *reinterpret_cast<float4*>(myrow + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
        epi_bar_sync();
        const int ew = warp - 2;
        const bool full_cols = n0 + BN <= n2 && (n2 & 3) == 0;
        for (int r = ew; r < BM; r += kEpiWarps) {
            const int grow = m0 + r;
            if (grow >= m) break;
            float* dst = c + size_t(grow) * n2 + n0;
            const float* srow = ctile + size_t(r) * kCStride;
            if (full_cols) {
                reinterpret_cast<float4*>(dst)[lane] = reinterpret_cast<const float4*>(srow)[lane];
            } else {
                for (int i = lane; i < BN; i += 32)
                    if (n0 + i < n2) dst[i] = srow[i];
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<kTmemCols>(tmem);
    }
}

// ================================================== wide pair, persistent
// Persistent cta_group::2 kernel (variant 4; measured on par with the
// one-tile-per-cluster kernel below, which is the default "wide") with a 256 x 256 tile of C' per CTA pair
// (128 x 256 per CTA), one pair per two SMs looping over a static tile
// schedule.  Per k-block each CTA stages A_hi/A_lo (its 128 rows) and
// B_hi/B_lo (its 128 of the pair's 256 columns): 64 KB for 3 x 128x256x64
// MACs, half the operand bytes per MAC of the 128 x 128 kernel, so neither the
// L2->SM feed nor shared-memory bandwidth paces the tensor pipe.
//
// TMEM (512 columns per CTA): main partial as two 128-column halves (cols
// 0..127 and 128..255), correction accumulator cols 256..511.  The main term
// is issued per half (N = 128 MMAs) and committed per half, so the epilogue
// drains half h while the tensor core runs the other half and the correction
// products (5/6 of a k-block of slack); the correction MMAs run at N = 256.
// Column maps (CTA r of the pair holds B rows n0 + 128 r + [0,128)):
//   main half h, TMEM col j:  j < 64 -> n0 + 64h + j,  j >= 64 -> n0 + 128 + 64h + (j-64)
//   corr, TMEM col 256 + j:   n0 + j
// Across tiles: the smem ring and the main-half barriers run on continuous
// counters, so the producer prefetches the next tile during the epilogue and
// the next tile's main products start as soon as their halves are drained; the
// next tile's correction products wait only for the epilogue's read of the
// correction accumulator (cempty).  The epilogue stores C straight from
// registers (each thread owns one row x 2 x 64 contiguous columns).
constexpr int kWideStages = 3;
constexpr int kWideBN = 256;
constexpr int kWideStageBytes = 4 * kTileBytes;  // A_hi | A_lo | B_hi | B_lo, 16 KB each
struct alignas(8) WideSmemTail {
    uint64_t full[kWideStages];
    uint64_t empty[kWideStages];
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint64_t cfull;
    uint64_t cempty;
    uint32_t tmem_base;
};
// C staging: 32 rows (one TMEM lane quadrant) x 256 columns, padded rows
constexpr int kWideCStride = kWideBN + 4;
constexpr size_t kWideStageCBytes = size_t(32) * kWideCStride * 4;
constexpr size_t kWideSmemBytes =
    1024 + size_t(kWideStages) * kWideStageBytes + kWideStageCBytes + sizeof(WideSmemTail);
static_assert(kWideSmemBytes <= 232448, "exceeds the 227 KB dynamic shared memory of sm_100");

struct WideMaps {
    CUtensorMap ahi, alo, bhi, blo;
    CUtensorMap bhi_h, blo_h;  // 64-row boxes: the halves a pair multicasts (clusters of 2 pairs)
};

template <int FMT>
__device__ __forceinline__ void widep_body(const WideMaps& mp, float* __restrict__ c, int m, int n2,
                                          int kp, const DevDecision* __restrict__ dec, int kind,
                                          int corrected, int flush_kblocks, int xa) {
    using T = Traits<FMT>;
    constexpr uint32_t kIdescHalf = umma_idesc<FMT, 2 * BM, 128>();
    constexpr uint32_t kIdescFull = umma_idesc<FMT, 2 * BM, kWideBN>();

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    float* cstage = reinterpret_cast<float*>(smem + size_t(kWideStages) * kWideStageBytes);
    WideSmemTail* tail = reinterpret_cast<WideSmemTail*>(smem + size_t(kWideStages) * kWideStageBytes +
                                                         kWideStageCBytes);
    auto tile = [&](int s, int which) -> uint8_t* {
        return smem + size_t(s) * kWideStageBytes + size_t(which) * kTileBytes;
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    const int tiles_m = (m + 2 * BM - 1) / (2 * BM), tiles_n = (n2 + kWideBN - 1) / kWideBN;
    const int ntiles = tiles_m * tiles_n;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int group = kGroupM * tiles_n;
    auto tile_coords = [&](int t, int& m_blk, int& n_blk) {
        const int first_m = (t / group) * kGroupM;
        const int gsize = min(tiles_m - first_m, kGroupM);
        m_blk = first_m + (t % group) % gsize;
        n_blk = (t % group) / gsize;
    };

    const int nkb = kp / T::kBK;
    const int F = flush_of(flush_kblocks, FMT) > 0 ? flush_of(flush_kblocks, FMT) : nkb;
    const int nchunks = (nkb + F - 1) / F;
    const uint32_t cta_bytes = uint32_t(corrected ? 4 : 2) * kTileBytes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kWideStages; ++s) {
            mbar_init(&tail->full[s], 1);
            mbar_init(&tail->empty[s], 1);
        }
        for (int h = 0; h < 2; ++h) {
            mbar_init(&tail->tfull[h], 1);
            mbar_init(&tail->tempty[h], kEpiWarps);  // 4 warps per CTA drain a half, 2 CTAs
        }
        mbar_init(&tail->cfull, 1);
        mbar_init(&tail->cempty, 2 * kEpiWarps);
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&mp.ahi);
        tma_prefetch(&mp.bhi);
        if (corrected) {
            tma_prefetch(&mp.alo);
            tma_prefetch(&mp.blo);
        }
    }
    if (warp == 1) tmem_alloc_pair<kTmemCols>(&tail->tmem_base);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tail->tmem_base;

    if (warp == 0) {
        // -------------------------------------------- TMA producer (both CTAs)
        if (lane == 0) {
            int it = 0;
            for (int t = pair; t < ntiles; t += npairs) {
                int m_blk, n_blk;
                tile_coords(t, m_blk, n_blk);
                const int m0 = m_blk * 2 * BM + int(rank) * BM;
                const int nb0 = n_blk * kWideBN + 128 * int(rank);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % kWideStages;
                    mbar_wait(&tail->empty[s], ((it / kWideStages) & 1) ^ 1);
                    if (leader) mbar_expect_tx(&tail->full[s], 2 * cta_bytes);
                    const int kx = kb * T::kBK;
                    tma_load_2d_pair(tile(s, 0), &mp.ahi, &tail->full[s], kx, m0);
                    tma_load_2d_pair(tile(s, 2), &mp.bhi, &tail->full[s], kx, nb0);
                    if (corrected) {
                        tma_load_2d_pair(tile(s, 1), &mp.alo, &tail->full[s], kx, m0);
                        tma_load_2d_pair(tile(s, 3), &mp.blo, &tail->full[s], kx, nb0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------- MMA issuer (pair leader only)
        if (leader) {
            int it = 0, gc = 0, lt = 0;
            for (int t = pair; t < ntiles; t += npairs, ++lt) {
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const bool chunk_start = (kb % F) == 0;
                    const bool chunk_end = (kb % F) == F - 1 || kb == nkb - 1;
                    const int s = it % kWideStages;
                    mbar_wait(&tail->full[s], (it / kWideStages) & 1);
                    tc_fence_after();
                    const uint64_t dah = umma_desc_k_sw128(tile(s, 0));
                    const uint64_t dal = umma_desc_k_sw128(tile(s, 1));
                    const uint64_t dbh = umma_desc_k_sw128(tile(s, 2));
                    const uint64_t dbl = umma_desc_k_sw128(tile(s, 3));
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (chunk_start && gc > 0) {
                            mbar_wait(&tail->tempty[h], (gc - 1) & 1);
                            tc_fence_after();
                        }
                        // B rows 64h.. of each CTA's tile: 64 rows x 128 B = 8 KB (>> 4 = 512)
                        const uint64_t dbh_h = dbh + uint64_t(512 * h);
                        if (elect_one()) {
#pragma unroll
                            for (int ks = 0; ks < T::kKSteps; ++ks) {
                                const uint64_t adv = uint64_t((ks * T::kUK * T::kElem) >> 4);
                                const uint32_t acc = (!chunk_start || ks > 0) ? 1u : 0u;
                                if (FMT == kFp16)
                                    mma2_f16(tmem + uint32_t(128 * h), dah + adv, dbh_h + adv, kIdescHalf, acc);
                                else
                                    mma2_tf32(tmem + uint32_t(128 * h), dah + adv, dbh_h + adv, kIdescHalf, acc);
                            }
                            if (chunk_end) mma_commit_pair(&tail->tfull[h], 0x3);
                        }
                        __syncwarp();
                    }
                    if (chunk_end) ++gc;
                    if (corrected && kb == 0 && lt > 0) {
                        // the epilogue has read the previous tile's correction accumulator
                        mbar_wait(&tail->cempty, (lt - 1) & 1);
                        tc_fence_after();
                    }
                    if (elect_one()) {
                        if (corrected) {
#pragma unroll
                            for (int ks = 0; ks < T::kKSteps; ++ks) {
                                const uint64_t adv = uint64_t((ks * T::kUK * T::kElem) >> 4);
                                const uint32_t acc = (kb > 0 || ks > 0) ? 1u : 0u;
                                if (FMT == kFp16) {
                                    mma2_f16(tmem + 256u, dal + adv, dbh + adv, kIdescFull, acc);
                                    mma2_f16(tmem + 256u, dah + adv, dbl + adv, kIdescFull, 1u);
                                } else {
                                    mma2_tf32(tmem + 256u, dal + adv, dbh + adv, kIdescFull, acc);
                                    mma2_tf32(tmem + 256u, dah + adv, dbl + adv, kIdescFull, 1u);
                                }
                            }
                        }
                        mma_commit_pair(&tail->empty[s], 0x3);
                        if (kb == nkb - 1) mma_commit_pair(&tail->cfull, 0x3);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (both CTAs)
        // warp w: TMEM lane quadrant q = w % 4, main half p; it owns C' columns
        // n0 + 64p + [0,64) (acc[0..63]) and n0 + 128 + 64p + [0,64) (acc[64..127])
        const int q = warp & 3;
        const int p = (warp - 2) >> 2;
        const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
        const uint32_t tempty_leader = mapa_shared(smem_u32(&tail->tempty[p]), 0);
        const uint32_t cempty_leader = mapa_shared(smem_u32(&tail->cempty), 0);
        const bool scaled = kind == kKindFp16Scaled && (dec->scale_a + dec->scale_b) != 0;
        const double f = scaled ? ldexp(1.0, -(dec->scale_a + dec->scale_b)) : 1.0;
        int gc = 0, lt = 0;
        for (int t = pair; t < ntiles; t += npairs, ++lt) {
            int m_blk, n_blk;
            tile_coords(t, m_blk, n_blk);
            float acc[128];
#pragma unroll
            for (int i = 0; i < 128; ++i) acc[i] = -0.0f;  // RN identity
            for (int ch = 0; ch < nchunks; ++ch, ++gc) {
                mbar_wait(&tail->tfull[p], gc & 1);
                tc_fence_after();
#pragma unroll
                for (int cb = 0; cb < 8; ++cb) {
                    float v[16];
                    tmem_ld16(lane_base + uint32_t(128 * p + 16 * cb), v);
                    if (cb == 7) {
                        // the partial is in registers: hand the TMEM half back
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(tempty_leader);
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i) acc[16 * cb + i] = __fadd_rn(acc[16 * cb + i], v[i]);
                }
            }
            mbar_wait(&tail->cfull, lt & 1);
            tc_fence_after();
            if (corrected) {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
                    for (int cb = 0; cb < 4; ++cb) {
                        float v[16];
                        tmem_ld16(lane_base + 256u + uint32_t(128 * hh + 64 * p + 16 * cb), v);
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            float& a = acc[64 * hh + 16 * cb + i];
                            a = __fadd_rn(a, __fmul_rn(v[i], 0x1.0p-11f));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(cempty_leader);
            if (scaled) {
#pragma unroll
                for (int i = 0; i < 128; ++i) acc[i] = scale_pow2(acc[i], f);
            }
            // store through a 32-row smem stage, one lane quadrant at a time:
            // the quadrant's two warps write their rows, then all eight warps
            // store 4 rows each as coalesced 1 KB rows
            const int m0 = m_blk * 2 * BM + int(rank) * BM;
            const int n0 = n_blk * kWideBN;
            const int ew = warp - 2;
            const bool full_cols = n0 + kWideBN <= n2 && (n2 & 3) == 0;
#pragma unroll 1
            for (int qq = 0; qq < 4; ++qq) {
                if (q == qq) {
                    float* myrow = cstage + size_t(lane) * kWideCStride;
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                        for (int i = 0; i < 64; i += 4)
                            *reinterpret_cast<float4*>(myrow + 128 * hh + 64 * p + i) =
                                make_float4(acc[64 * hh + i], acc[64 * hh + i + 1], acc[64 * hh + i + 2],
                                            acc[64 * hh + i + 3]);
                }
                epi_bar_sync();
                if (xa) {
                    // A-expanded layout: 16 C rows per quadrant, 2 per warp
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
                        const int r = 2 * ew + rr;  // C row within the quadrant's 16
                        const int grow2 = m0 + 32 * qq + 2 * r;
                        if (grow2 < m)
                            store_xa_row<kWideBN>(c + size_t(grow2 / 2) * (2 * size_t(n2)) + 2 * size_t(n0),
                                                  cstage + size_t(2 * r) * kWideCStride, kWideCStride, n2 - n0,
                                                  full_cols, lane);
                    }
                } else
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    const int r = 4 * ew + rr;
                    const int grow = m0 + 32 * qq + r;
                    if (grow < m) {
                        float* dst = c + size_t(grow) * n2 + n0;
                        const float* srow = cstage + size_t(r) * kWideCStride;
                        if (full_cols) {
                            __stcs(reinterpret_cast<float4*>(dst) + lane, reinterpret_cast<const float4*>(srow)[lane]);
                            __stcs(reinterpret_cast<float4*>(dst) + lane + 32,
                                   reinterpret_cast<const float4*>(srow)[lane + 32]);
                        } else {
                            for (int i = lane; i < kWideBN; i += 32)
                                if (n0 + i < n2) dst[i] = srow[i];
                        }
                    }
                }
                epi_bar_sync();
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<kTmemCols>(tmem);
    }
}

// host-known format
template <int FMT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_widep_kernel(const __grid_constant__ WideMaps maps, float* __restrict__ c, int m,
                          int n2, int kp, const DevDecision* __restrict__ dec, int kind_fixed,
                          int corrected, int flush_kblocks, int xa) {
    const int kind = kind_fixed >= 0 ? kind_fixed : dec->kind;
    const bool mine = FMT == kTf32 ? kind == kKindTf32 : (kind == kKindFp16 || kind == kKindFp16Scaled);
    if (!mine) return;
    widep_body<FMT>(maps, c, m, n2, kp, dec, kind, corrected, flush_kblocks, xa);
}

// format decided on the device (AUTO): one launch that runs the selected
// format (instead of launching both and letting one exit)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_widep_auto_kernel(const __grid_constant__ WideMaps maps16,
                               const __grid_constant__ WideMaps maps32, float* __restrict__ c,
                               int m, int n2, int kp, const DevDecision* __restrict__ dec,
                               int corrected, int flush_kblocks, int xa) {
    const int kind = dec->kind;
    if (kind == kKindTf32)
        widep_body<kTf32>(maps32, c, m, n2, kp, dec, kind, corrected, flush_kblocks, xa);
    else if (kind == kKindFp16 || kind == kKindFp16Scaled)
        widep_body<kFp16>(maps16, c, m, n2, kp, dec, kind, corrected, flush_kblocks, xa);
}

// ===================================================================== wide pair
// cta_group::2 kernel with a 256 x 256 tile of C' per CTA pair (128 x 256 per
// CTA), one tile per cluster (variant 3, the default for large shapes).  Per
// k-block each CTA stages A_hi/A_lo (its 128 rows) and B_hi/B_lo (its 128 of
// the pair's 256 columns): 64 KB for 3 x 128x256x64 MACs, half the operand
// bytes per MAC of the 128 x 128 kernel, so neither the L2->SM feed nor
// shared-memory bandwidth paces the tensor pipe.  TMEM: main partial as two
// 128-column halves (issued and committed per half, N = 128 MMAs, drained by
// the epilogue while the tensor core runs the other half and the N = 256
// correction products), correction accumulator in cols 256..511.
// Column maps (CTA r of the pair holds B rows n0 + 128 r + [0,128)):
//   main half h, TMEM col j:  j < 64 -> n0 + 64h + j,  j >= 64 -> n0 + 128 + 64h + (j-64)
//   corr, TMEM col 256 + j:   n0 + j
constexpr int kNpStages = 3;
constexpr int kNpBN = 256;
constexpr int kNpStageBytes = 4 * kTileBytes;  // A_hi | A_lo | B_hi | B_lo, 16 KB each
constexpr int kNpCStride = kNpBN + 4;
struct alignas(8) NpSmemTail {
    uint64_t full[kNpStages];
    uint64_t empty[kNpStages];
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint64_t cfull;
    uint32_t tmem_base;
};
constexpr size_t kNpSmemBytes = 1024 + size_t(kNpStages) * kNpStageBytes + sizeof(NpSmemTail);
static_assert(size_t(BM) * kNpCStride * 4 <= size_t(kNpStages) * kNpStageBytes,
              "C staging tile must fit in the operand stages");

// CL = CTA pairs per cluster.  CL = 2: two pairs on vertically adjacent
// 256-row tiles of the same 256 B' columns share each B' tile -- CTA r of pair
// p loads rows [64p, 64p + 64) of its 128-row B' tile and multicasts them to
// CTA r of both pairs -- which halves the B' traffic from L2 to the SMs and
// keeps the two pairs' B' reads in k-lockstep (one DRAM read per cluster).
// A stage is refilled only when BOTH pairs' MMAs released it (empty barriers
// count one commit per pair; the commits multicast to all four CTAs).
template <int FMT, int CL>
__device__ __forceinline__ void wide_body(const WideMaps& mp, float* __restrict__ c, int m, int n2,
                                          int kp, const DevDecision* __restrict__ dec, int kind,
                                          int corrected, int flush_kblocks, int group_m,
                                          int a_row_off, int ldc, float* __restrict__ partial,
                                          int kb_per, int xa) {
    using T = Traits<FMT>;
    constexpr uint32_t kIdescHalf = umma_idesc<FMT, 2 * BM, 128>();
    constexpr uint32_t kIdescFull = umma_idesc<FMT, 2 * BM, kNpBN>();

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    NpSmemTail* tail =
        reinterpret_cast<NpSmemTail*>(smem + size_t(kNpStages) * kNpStageBytes);
    auto tile = [&](int s, int which) -> uint8_t* {
        return smem + size_t(s) * kNpStageBytes + size_t(which) * kTileBytes;
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_ctarank();
    const uint32_t rank = CL == 2 ? (crank & 1u) : crank;  // CTA within its pair
    const int pr = CL == 2 ? int(crank >> 1) : 0;            // pair within the cluster
    const bool leader = rank == 0;
    const uint16_t pair_mask = CL == 2 ? uint16_t(0x3u << (2 * pr)) : uint16_t(0x3);  // this pair's CTAs
    const uint16_t all_mask = CL == 2 ? uint16_t(0xF) : uint16_t(0x3);

    // raster over cluster tiles (CL vertically adjacent pair tiles), groups of
    // group_m of them share B' panels in L2
    const int tiles_m = (m + 2 * BM - 1) / (2 * BM), tiles_n = (n2 + kNpBN - 1) / kNpBN;
    const int tiles_mc = CL == 2 ? (tiles_m + 1) >> 1 : tiles_m;
    const int id = CL == 2 ? int(blockIdx.x >> 2) : int(blockIdx.x >> 1);
    const int group = group_m * tiles_n;
    const int first_m = (id / group) * group_m;
    const int gsize = min(tiles_mc - first_m, group_m);
    const int m_blk = CL == 2 ? 2 * (first_m + (id % group) % gsize) + pr : first_m + (id % group) % gsize;
    const int n_blk = (id % group) / gsize;
    const int m0 = m_blk * 2 * BM + int(rank) * BM;  // this CTA's 128 rows
    const int n0 = n_blk * kNpBN;                  // the pair's 256 columns

    // split-K (gridDim.y > 1): k-blocks [kb_base, kb_base + nkb), un-descaled
    // fp32 partial per split (summed in split order by split_reduce_kernel)
    const int nkb_all = kp / T::kBK;
    const int per = FMT == kTf32 ? 2 * kb_per : kb_per;  // kb_per counts 64-element f16 blocks
    const int kb_base = partial ? int(blockIdx.y) * per : 0;
    const int nkb = partial ? min(per, nkb_all - kb_base) : nkb_all;
    const int F = flush_of(flush_kblocks, FMT) > 0 ? flush_of(flush_kblocks, FMT) : (nkb > 0 ? nkb : 1);
    const int nchunks = (nkb + F - 1) / F;
    const uint32_t cta_bytes = uint32_t(corrected ? 4 : 2) * kTileBytes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kNpStages; ++s) {
            mbar_init(&tail->full[s], 1);
            mbar_init(&tail->empty[s], CL);  // one MMA commit per pair of the cluster
        }
        for (int h = 0; h < 2; ++h) {
            mbar_init(&tail->tfull[h], 1);
            mbar_init(&tail->tempty[h], 2 * kEpiWarps / 2);  // 4 warps per CTA drain a half
        }
        mbar_init(&tail->cfull, 1);
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&mp.ahi);
        tma_prefetch(CL == 2 ? &mp.bhi_h : &mp.bhi);
        if (corrected) {
            tma_prefetch(&mp.alo);
            tma_prefetch(CL == 2 ? &mp.blo_h : &mp.blo);
        }
    }
    if (warp == 1) tmem_alloc_pair<kTmemCols>(&tail->tmem_base);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tail->tmem_base;

    if (warp == 0) {
        // -------------------------------------------- TMA producer (both CTAs)
        if (lane == 0) {
            const int nb0 = n0 + 128 * int(rank);
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kNpStages;
                mbar_wait(&tail->empty[s], ((kb / kNpStages) & 1) ^ 1);
                if (leader) mbar_expect_tx(&tail->full[s], 2 * cta_bytes);
                const int kx = (kb_base + kb) * T::kBK;
                tma_load_2d_pair(tile(s, 0), &mp.ahi, &tail->full[s], kx, m0 + a_row_off);
                if (corrected) tma_load_2d_pair(tile(s, 1), &mp.alo, &tail->full[s], kx, m0 + a_row_off);
                if constexpr (CL == 2) {
                    // B' rows [64 pr, 64 pr + 64) of this CTA's tile, to CTA `rank` of both pairs
                    const uint16_t mc = uint16_t((1u << rank) | (1u << (2 + rank)));
                    const int off = pr * 64 * 128;
                    tma_load_2d_pair_mc(tile(s, 2) + off, &mp.bhi_h, &tail->full[s], kx, nb0 + 64 * pr, mc);
                    if (corrected)
                        tma_load_2d_pair_mc(tile(s, 3) + off, &mp.blo_h, &tail->full[s], kx, nb0 + 64 * pr, mc);
                } else {
                    tma_load_2d_pair(tile(s, 2), &mp.bhi, &tail->full[s], kx, nb0);
                    if (corrected) tma_load_2d_pair(tile(s, 3), &mp.blo, &tail->full[s], kx, nb0);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------- MMA issuer (pair leader only)
        if (leader) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int chunk = kb / F;
                const bool chunk_start = (kb % F) == 0;
                const bool chunk_end = (kb % F) == F - 1 || kb == nkb - 1;
                const int s = kb % kNpStages;
                mbar_wait(&tail->full[s], (kb / kNpStages) & 1);
                tc_fence_after();
                const uint64_t dah = umma_desc_k_sw128(tile(s, 0));
                const uint64_t dal = umma_desc_k_sw128(tile(s, 1));
                const uint64_t dbh = umma_desc_k_sw128(tile(s, 2));
                const uint64_t dbl = umma_desc_k_sw128(tile(s, 3));
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (chunk_start && chunk > 0) {
                        mbar_wait(&tail->tempty[h], (chunk - 1) & 1);
                        tc_fence_after();
                    }
                    // B rows 64h.. of each CTA's tile: 64 rows x 128 B = 8 KB (>> 4 = 512)
                    const uint64_t dbh_h = dbh + uint64_t(512 * h);
                    if (elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < T::kKSteps; ++ks) {
                            const uint64_t adv = uint64_t((ks * T::kUK * T::kElem) >> 4);
                            const uint32_t acc = (!chunk_start || ks > 0) ? 1u : 0u;
                            if (FMT == kFp16)
                                mma2_f16(tmem + uint32_t(128 * h), dah + adv, dbh_h + adv, kIdescHalf, acc);
                            else
                                mma2_tf32(tmem + uint32_t(128 * h), dah + adv, dbh_h + adv, kIdescHalf, acc);
                        }
                        if (chunk_end) mma_commit_pair(&tail->tfull[h], pair_mask);
                    }
                    __syncwarp();
                }
                if (elect_one()) {
                    if (corrected) {
#pragma unroll
                        for (int ks = 0; ks < T::kKSteps; ++ks) {
                            const uint64_t adv = uint64_t((ks * T::kUK * T::kElem) >> 4);
                            const uint32_t acc = (kb > 0 || ks > 0) ? 1u : 0u;
                            if (FMT == kFp16) {
                                mma2_f16(tmem + 256u, dal + adv, dbh + adv, kIdescFull, acc);
                                mma2_f16(tmem + 256u, dah + adv, dbl + adv, kIdescFull, 1u);
                            } else {
                                mma2_tf32(tmem + 256u, dal + adv, dbh + adv, kIdescFull, acc);
                                mma2_tf32(tmem + 256u, dah + adv, dbl + adv, kIdescFull, 1u);
                            }
                        }
                    }
                    mma_commit_pair(&tail->empty[s], all_mask);
                    if (kb == nkb - 1) mma_commit_pair(&tail->cfull, pair_mask);
                }
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------ epilogue (both CTAs)
        // warp w: TMEM lane quadrant q = w % 4, main half p; it owns C' columns
        // n0 + 64p + [0,64) (acc[0..63]) and n0 + 128 + 64p + [0,64) (acc[64..127])
        const int q = warp & 3;
        const int p = (warp - 2) >> 2;
        const int rloc = 32 * q + lane;
        const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
        const uint32_t tempty_leader = mapa_shared(smem_u32(&tail->tempty[p]), CL == 2 ? (crank & ~1u) : 0u);
        float acc[128];
#pragma unroll
        for (int i = 0; i < 128; ++i) acc[i] = -0.0f;  // RN identity
        for (int ch = 0; ch < nchunks; ++ch) {
            mbar_wait(&tail->tfull[p], ch & 1);
            tc_fence_after();
#pragma unroll
            for (int cb = 0; cb < 8; ++cb) {
                float v[16];
                tmem_ld16(lane_base + uint32_t(128 * p + 16 * cb), v);
                if (cb == 7) {
                    // the partial is in registers: hand the TMEM half back
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_leader);
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[16 * cb + i] = __fadd_rn(acc[16 * cb + i], v[i]);
            }
        }
        if (nkb > 0) {
            mbar_wait(&tail->cfull, 0);
            tc_fence_after();
        }
        if (corrected && nkb > 0) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
                for (int cb = 0; cb < 2; ++cb) {
                    float v[32];
                    tmem_ld32(lane_base + 256u + uint32_t(128 * hh + 64 * p + 32 * cb), v);
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        float& a = acc[64 * hh + 32 * cb + i];
                        a = __fadd_rn(a, __fmul_rn(v[i], 0x1.0p-11f));
                    }
                }
            }
        }
        const bool scaled = !partial && kind == kKindFp16Scaled && (dec->scale_a + dec->scale_b) != 0;
        if (partial) c = partial + size_t(blockIdx.y) * size_t(m) * size_t(n2);
        if (scaled) {
            const double f = ldexp(1.0, -(dec->scale_a + dec->scale_b));
#pragma unroll
            for (int i = 0; i < 128; ++i) acc[i] = scale_pow2(acc[i], f);
        }
        // stage the 128 x 256 tile in the idle operand smem, then store rows
        float* ctile = reinterpret_cast<float*>(smem);
        float* myrow = ctile + size_t(rloc) * kNpCStride;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int i = 0; i < 64; i += 4)
                *reinterpret_cast<float4*>(myrow + 128 * hh + 64 * p + i) =
                    make_float4(acc[64 * hh + i], acc[64 * hh + i + 1], acc[64 * hh + i + 2],
                                acc[64 * hh + i + 3]);
        epi_bar_sync();
        const int ew = warp - 2;
        const int ld = partial ? n2 : ldc;  // C may be a column block of a wider matrix
        const bool full_cols = n0 + kNpBN <= n2 && (ld & 3) == 0;
        if (xa && !partial) {
            // A-expanded layout: tile rows 2i / 2i+1 = Re / Im of C row m0/2 + i
            // (ldc = floats per C row)
            for (int r = ew; r < BM / 2; r += kEpiWarps) {
                if (m0 + 2 * r >= m) break;
                store_xa_row<kNpBN>(c + size_t(m0 / 2 + r) * size_t(ld) + 2 * size_t(n0),
                                    ctile + size_t(2 * r) * kNpCStride, kNpCStride, n2 - n0, full_cols, lane);
            }
        } else
        for (int r = ew; r < BM; r += kEpiWarps) {
            const int grow = m0 + r;
            if (grow >= m) break;
            float* dst = c + size_t(grow) * ld + n0;
            const float* srow = ctile + size_t(r) * kNpCStride;
            if (full_cols) {
                reinterpret_cast<float4*>(dst)[lane] = reinterpret_cast<const float4*>(srow)[lane];
                reinterpret_cast<float4*>(dst)[lane + 32] =
                    reinterpret_cast<const float4*>(srow)[lane + 32];
            } else {
                for (int i = lane; i < kNpBN; i += 32)
                    if (n0 + i < n2) dst[i] = srow[i];
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<kTmemCols>(tmem);
    }
}

// host-known format
template <int FMT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_wide_kernel(const __grid_constant__ WideMaps maps, float* __restrict__ c, int m,
                          int n2, int kp, const DevDecision* __restrict__ dec, int kind_fixed,
                          int corrected, int flush_kblocks, int group_m, int a_row_off, int ldc,
                          float* __restrict__ partial, int kb_per, int xa) {
    const int kind = kind_fixed >= 0 ? kind_fixed : dec->kind;
    const bool mine = FMT == kTf32 ? kind == kKindTf32 : (kind == kKindFp16 || kind == kKindFp16Scaled);
    if (!mine) return;  // both CTAs of the pair read the same decision
    wide_body<FMT, 1>(maps, c, m, n2, kp, dec, kind, corrected, flush_kblocks, group_m, a_row_off, ldc,
                      partial, kb_per, xa);
}

// clusters of two CTA pairs sharing B' tiles by TMA multicast
template <int FMT>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_widemc_kernel(const __grid_constant__ WideMaps maps, float* __restrict__ c, int m,
                            int n2, int kp, const DevDecision* __restrict__ dec, int kind_fixed,
                            int corrected, int flush_kblocks, int group_m, int a_row_off, int ldc,
                            float* __restrict__ partial, int kb_per, int xa) {
    const int kind = kind_fixed >= 0 ? kind_fixed : dec->kind;
    const bool mine = FMT == kTf32 ? kind == kKindTf32 : (kind == kKindFp16 || kind == kKindFp16Scaled);
    if (!mine) return;  // all four CTAs read the same decision
    wide_body<FMT, 2>(maps, c, m, n2, kp, dec, kind, corrected, flush_kblocks, group_m, a_row_off, ldc,
                      partial, kb_per, xa);
}

// format decided on the device (AUTO): one launch that runs the selected
// format instead of launching both and letting one exit
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_wide_auto_kernel(const __grid_constant__ WideMaps maps16,
                               const __grid_constant__ WideMaps maps32, float* __restrict__ c,
                               int m, int n2, int kp, const DevDecision* __restrict__ dec,
                               int corrected, int flush_kblocks, int group_m, int a_row_off,
                               int ldc, float* __restrict__ partial, int kb_per, int xa) {
    const int kind = dec->kind;
    if (kind == kKindTf32)
        wide_body<kTf32, 1>(maps32, c, m, n2, kp, dec, kind, corrected, flush_kblocks, group_m, a_row_off,
                            ldc, partial, kb_per, xa);
    else if (kind == kKindFp16 || kind == kKindFp16Scaled)
        wide_body<kFp16, 1>(maps16, c, m, n2, kp, dec, kind, corrected, flush_kblocks, group_m, a_row_off,
                            ldc, partial, kb_per, xa);
}

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_widemc_auto_kernel(const __grid_constant__ WideMaps maps16,
                                 const __grid_constant__ WideMaps maps32, float* __restrict__ c,
                                 int m, int n2, int kp, const DevDecision* __restrict__ dec,
                                 int corrected, int flush_kblocks, int group_m, int a_row_off,
                                 int ldc, float* __restrict__ partial, int kb_per, int xa) {
    const int kind = dec->kind;
    if (kind == kKindTf32)
        wide_body<kTf32, 2>(maps32, c, m, n2, kp, dec, kind, corrected, flush_kblocks, group_m, a_row_off,
                            ldc, partial, kb_per, xa);
    else if (kind == kKindFp16 || kind == kKindFp16Scaled)
        wide_body<kFp16, 2>(maps16, c, m, n2, kp, dec, kind, corrected, flush_kblocks, group_m, a_row_off,
                            ldc, partial, kb_per, xa);
}

// ============================================ pair tiles, persistent, 2 buffers
// Persistent cta_group::2 kernel on 256 x 128 tiles (variant 6) whose two
// tiles in flight each own half of TMEM: buffer b = main partial (cols 256b +
// [0,128)) + correction accumulator (256b + 128 + [0,128)).  The epilogue
// warps form two sets, set b drains and stores the tiles of buffer b, so one
// tile's correction drain and C store overlap the next tile's MMAs -- with the
// 256 x 256 tile the whole of TMEM holds one tile and the next tile's main
// products wait for the store (tensor pipe ~30 % busy at 4 k-blocks per tile,
// ~77 % at 32).  The main term is drained (RN-added) every flush interval as
// in the other kernels, while the tensor core runs the correction products of
// the same k-block.  Each warp stores its 32 x 128 block through a private
// 32 x 64 smem stage (two halves), no barrier across warps.
constexpr int kP2Stages = 3;
constexpr int kP2BN = 128;
constexpr int kP2ATile = 128 * 128;  // 128 rows x 128 B
constexpr int kP2BTile = 64 * 128;   // 64 rows x 128 B (this CTA's half of the pair's 128 B' rows)
constexpr int kP2StageBytes = 2 * kP2ATile + 2 * kP2BTile;
constexpr int kP2CStride = 68;       // padded staging row (floats): 64 columns
constexpr size_t kP2WarpStage = size_t(32) * kP2CStride * 4;
struct alignas(8) P2SmemTail {
    uint64_t full[kP2Stages];
    uint64_t empty[kP2Stages];
    uint64_t tfull[2], tempty[2], cfull[2], cempty[2];
    uint32_t tmem_base;
};
constexpr size_t kP2SmemBytes =
    1024 + size_t(kP2Stages) * kP2StageBytes + size_t(kEpiWarps) * kP2WarpStage + sizeof(P2SmemTail);
static_assert(kP2SmemBytes <= 232448, "exceeds the 227 KB dynamic shared memory of sm_100");

template <int FMT>
__device__ __forceinline__ void pairp_body(const WideMaps& mp, float* __restrict__ c, int m, int n2, int kp,
                                           const DevDecision* __restrict__ dec, int kind, int corrected,
                                           int flush_kblocks, int xa) {
    using T = Traits<FMT>;
    constexpr uint32_t kIdesc = umma_idesc<FMT, 2 * BM, kP2BN>();

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    float* cstage = reinterpret_cast<float*>(smem + size_t(kP2Stages) * kP2StageBytes);
    P2SmemTail* tail = reinterpret_cast<P2SmemTail*>(smem + size_t(kP2Stages) * kP2StageBytes +
                                                     size_t(kEpiWarps) * kP2WarpStage);
    auto a_tile = [&](int st, int lo) -> uint8_t* {
        return smem + size_t(st) * kP2StageBytes + size_t(lo) * kP2ATile;
    };
    auto b_tile = [&](int st, int lo) -> uint8_t* {
        return smem + size_t(st) * kP2StageBytes + 2 * kP2ATile + size_t(lo) * kP2BTile;
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    const int tiles_m = (m + 2 * BM - 1) / (2 * BM), tiles_n = (n2 + kP2BN - 1) / kP2BN;
    const int ntiles = tiles_m * tiles_n;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int group = kWideGroupM * tiles_n;
    auto tile_coords = [&](int t, int& m_blk, int& n_blk) {
        const int first_m = (t / group) * kWideGroupM;
        const int gsize = min(tiles_m - first_m, kWideGroupM);
        m_blk = first_m + (t % group) % gsize;
        n_blk = (t % group) / gsize;
    };

    const int nkb = kp / T::kBK;
    const int F = flush_of(flush_kblocks, FMT) > 0 ? flush_of(flush_kblocks, FMT) : nkb;
    const int nchunks = (nkb + F - 1) / F;
    const uint32_t cta_bytes = corrected ? uint32_t(kP2StageBytes) : uint32_t(kP2ATile + kP2BTile);

    if (threadIdx.x == 0) {
        for (int st = 0; st < kP2Stages; ++st) {
            mbar_init(&tail->full[st], 1);
            mbar_init(&tail->empty[st], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tail->tfull[b], 1);
            mbar_init(&tail->tempty[b], 2 * (kEpiWarps / 2));  // one set: 4 warps in each CTA
            mbar_init(&tail->cfull[b], 1);
            mbar_init(&tail->cempty[b], 2 * (kEpiWarps / 2));
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&mp.ahi);
        tma_prefetch(&mp.bhi_h);
        if (corrected) {
            tma_prefetch(&mp.alo);
            tma_prefetch(&mp.blo_h);
        }
    }
    if (warp == 1) tmem_alloc_pair<kTmemCols>(&tail->tmem_base);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tail->tmem_base;

    if (warp == 0) {
        // -------------------------------------------- TMA producer (both CTAs)
        if (lane == 0) {
            int it = 0;
            for (int t = pair; t < ntiles; t += npairs) {
                int m_blk, n_blk;
                tile_coords(t, m_blk, n_blk);
                const int m0 = m_blk * 2 * BM + int(rank) * BM;
                const int nb0 = n_blk * kP2BN + 64 * int(rank);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int st = it % kP2Stages;
                    mbar_wait(&tail->empty[st], ((it / kP2Stages) & 1) ^ 1);
                    if (leader) mbar_expect_tx(&tail->full[st], 2 * cta_bytes);
                    const int kx = kb * T::kBK;
                    tma_load_2d_pair(a_tile(st, 0), &mp.ahi, &tail->full[st], kx, m0);
                    tma_load_2d_pair(b_tile(st, 0), &mp.bhi_h, &tail->full[st], kx, nb0);
                    if (corrected) {
                        tma_load_2d_pair(a_tile(st, 1), &mp.alo, &tail->full[st], kx, m0);
                        tma_load_2d_pair(b_tile(st, 1), &mp.blo_h, &tail->full[st], kx, nb0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------- MMA issuer (pair leader only)
        if (leader) {
            int it = 0, lt = 0;
            int mcount[2] = {0, 0}, ccount[2] = {0, 0};  // main chunks / tiles issued per buffer
            for (int t = pair; t < ntiles; t += npairs, ++lt) {
                const int b = lt & 1;
                const uint32_t d_main = tmem + uint32_t(256 * b);
                const uint32_t d_corr = d_main + 128u;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const bool chunk_start = (kb % F) == 0;
                    const bool chunk_end = (kb % F) == F - 1 || kb == nkb - 1;
                    const int st = it % kP2Stages;
                    mbar_wait(&tail->full[st], (it / kP2Stages) & 1);
                    tc_fence_after();
                    if (chunk_start && mcount[b] > 0) {  // the previous partial of this buffer was drained
                        mbar_wait(&tail->tempty[b], (mcount[b] - 1) & 1);
                        tc_fence_after();
                    }
                    const uint64_t dah = umma_desc_k_sw128(a_tile(st, 0));
                    const uint64_t dal = umma_desc_k_sw128(a_tile(st, 1));
                    const uint64_t dbh = umma_desc_k_sw128(b_tile(st, 0));
                    const uint64_t dbl = umma_desc_k_sw128(b_tile(st, 1));
                    if (elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < T::kKSteps; ++ks) {
                            const uint64_t adv = uint64_t((ks * T::kUK * T::kElem) >> 4);
                            const uint32_t acc = (!chunk_start || ks > 0) ? 1u : 0u;
                            if (FMT == kFp16)
                                mma2_f16(d_main, dah + adv, dbh + adv, kIdesc, acc);
                            else
                                mma2_tf32(d_main, dah + adv, dbh + adv, kIdesc, acc);
                        }
                        if (chunk_end) mma_commit_pair(&tail->tfull[b], 0x3);
                    }
                    __syncwarp();
                    if (chunk_end) ++mcount[b];
                    if (kb == 0 && ccount[b] > 0) {  // this buffer's previous correction was read
                        mbar_wait(&tail->cempty[b], (ccount[b] - 1) & 1);
                        tc_fence_after();
                    }
                    if (elect_one()) {
                        if (corrected) {
#pragma unroll
                            for (int ks = 0; ks < T::kKSteps; ++ks) {
                                const uint64_t adv = uint64_t((ks * T::kUK * T::kElem) >> 4);
                                const uint32_t acc = (kb > 0 || ks > 0) ? 1u : 0u;
                                if (FMT == kFp16) {
                                    mma2_f16(d_corr, dal + adv, dbh + adv, kIdesc, acc);
                                    mma2_f16(d_corr, dah + adv, dbl + adv, kIdesc, 1u);
                                } else {
                                    mma2_tf32(d_corr, dal + adv, dbh + adv, kIdesc, acc);
                                    mma2_tf32(d_corr, dah + adv, dbl + adv, kIdesc, 1u);
                                }
                            }
                        }
                        mma_commit_pair(&tail->empty[st], 0x3);
                        if (kb == nkb - 1) mma_commit_pair(&tail->cfull[b], 0x3);
                    }
                    __syncwarp();
                }
                ++ccount[b];
            }
        }
    } else {
        // -------------------------------- epilogue: set e = (warp - 2) / 4 (both CTAs)
        const int q = warp & 3;
        const int e = (warp - 2) >> 2;
        const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16) + uint32_t(256 * e);
        const uint32_t tempty_leader = mapa_shared(smem_u32(&tail->tempty[e]), 0);
        const uint32_t cempty_leader = mapa_shared(smem_u32(&tail->cempty[e]), 0);
        const bool scaled = kind == kKindFp16Scaled && (dec->scale_a + dec->scale_b) != 0;
        const double f = scaled ? ldexp(1.0, -(dec->scale_a + dec->scale_b)) : 1.0;
        float* wst = cstage + size_t(warp - 2) * (kP2WarpStage / 4);  // this warp's private stage
        int mc = 0, cc = 0, lt = e;
        for (int t = pair + e * npairs; t < ntiles; t += 2 * npairs, lt += 2) {
            int m_blk, n_blk;
            tile_coords(t, m_blk, n_blk);
            float acc[128];
#pragma unroll
            for (int i = 0; i < 128; ++i) acc[i] = -0.0f;  // RN identity
            for (int ch = 0; ch < nchunks; ++ch, ++mc) {
                mbar_wait(&tail->tfull[e], mc & 1);
                tc_fence_after();
#pragma unroll
                for (int cb = 0; cb < 8; ++cb) {
                    float v[16];
                    tmem_ld16(lane_base + uint32_t(16 * cb), v);
                    if (cb == 7) {  // the partial is in registers: hand the buffer back
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(tempty_leader);
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i) acc[16 * cb + i] = __fadd_rn(acc[16 * cb + i], v[i]);
                }
            }
            mbar_wait(&tail->cfull[e], cc & 1);
            ++cc;
            tc_fence_after();
            if (corrected) {
#pragma unroll
                for (int cb = 0; cb < 8; ++cb) {
                    float v[16];
                    tmem_ld16(lane_base + 128u + uint32_t(16 * cb), v);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        float& a = acc[16 * cb + i];
                        a = __fadd_rn(a, __fmul_rn(v[i], 0x1.0p-11f));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(cempty_leader);
            if (scaled) {
#pragma unroll
                for (int i = 0; i < 128; ++i) acc[i] = scale_pow2(acc[i], f);
            }
            // store this warp's 32 rows x 128 columns, 64 columns at a time
            const int r0 = m_blk * 2 * BM + int(rank) * BM + 32 * q;  // first GEMM row of the warp
            const int n0 = n_blk * kP2BN;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int c0 = n0 + 64 * hh;
                const bool full_cols = c0 + 64 <= n2 && (n2 & 3) == 0;
#pragma unroll
                for (int i = 0; i < 64; i += 4)
                    *reinterpret_cast<float4*>(wst + size_t(lane) * kP2CStride + i) =
                        make_float4(acc[64 * hh + i], acc[64 * hh + i + 1], acc[64 * hh + i + 2],
                                    acc[64 * hh + i + 3]);
                __syncwarp();
                if (xa) {
                    // A-expanded layout: stage rows 2i / 2i+1 = Re / Im of C row (r0 + 2i) / 2; two C rows
                    // per instruction (lanes 0-15 / 16-31), each lane interleaves 4 columns into 32 B
                    const int rsub = lane >> 4, cl = 4 * (lane & 15);
                    for (int i = 0; i < 16; i += 2) {
                        const int ii = i + rsub;
                        if (r0 + 2 * ii >= m) continue;
                        float* dst = c + size_t((r0 + 2 * ii) / 2) * (2 * size_t(n2)) + 2 * size_t(c0);
                        const float* s0 = wst + size_t(2 * ii) * kP2CStride;
                        const float* s1 = s0 + kP2CStride;
                        if (full_cols) {
                            const float4 re = *reinterpret_cast<const float4*>(s0 + cl);
                            const float4 im = *reinterpret_cast<const float4*>(s1 + cl);
                            float4* d4 = reinterpret_cast<float4*>(dst + 2 * cl);
                            __stcs(d4, make_float4(re.x, im.x, re.y, im.y));
                            __stcs(d4 + 1, make_float4(re.z, im.z, re.w, im.w));
                        } else {
                            for (int j = cl; j < cl + 4; ++j)
                                if (c0 + j < n2) {
                                    dst[2 * j] = s0[j];
                                    dst[2 * j + 1] = s1[j];
                                }
                        }
                    }
                } else {
                    // two rows per instruction: lanes 0-15 row 2i, 16-31 row 2i+1, 16 B each
                    const int rsub = lane >> 4, cl = 4 * (lane & 15);
                    for (int i = 0; i < 16; ++i) {
                        const int r = 2 * i + rsub;
                        if (r0 + r >= m) continue;
                        float* dst = c + size_t(r0 + r) * n2 + c0;
                        const float* srow = wst + size_t(r) * kP2CStride;
                        if (full_cols) {
                            __stcs(reinterpret_cast<float4*>(dst + cl), *reinterpret_cast<const float4*>(srow + cl));
                        } else {
                            for (int j = cl; j < cl + 4; ++j)
                                if (c0 + j < n2) dst[j] = srow[j];
                        }
                    }
                }
                __syncwarp();
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<kTmemCols>(tmem);
    }
}

template <int FMT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_pairp_kernel(const __grid_constant__ WideMaps maps, float* __restrict__ c, int m, int n2, int kp,
                           const DevDecision* __restrict__ dec, int kind_fixed, int corrected,
                           int flush_kblocks, int xa) {
    const int kind = kind_fixed >= 0 ? kind_fixed : dec->kind;
    const bool mine = FMT == kTf32 ? kind == kKindTf32 : (kind == kKindFp16 || kind == kKindFp16Scaled);
    if (!mine) return;
    pairp_body<FMT>(maps, c, m, n2, kp, dec, kind, corrected, flush_kblocks, xa);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsGemm, 1)
    tcec_gemm_pairp_auto_kernel(const __grid_constant__ WideMaps maps16, const __grid_constant__ WideMaps maps32,
                                float* __restrict__ c, int m, int n2, int kp, const DevDecision* __restrict__ dec,
                                int corrected, int flush_kblocks, int xa) {
    const int kind = dec->kind;
    if (kind == kKindTf32)
        pairp_body<kTf32>(maps32, c, m, n2, kp, dec, kind, corrected, flush_kblocks, xa);
    else if (kind == kKindFp16 || kind == kKindFp16Scaled)
        pairp_body<kFp16>(maps16, c, m, n2, kp, dec, kind, corrected, flush_kblocks, xa);
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encode() {
    std::call_once(g_encode_once, [] {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    return g_encode != nullptr;
}

// 2-D K-major operand: rows x kp elements, box = 128 rows x 128 B, swizzle 128B
bool make_map(CUtensorMap* map, const void* base, int fmt, int64_t rows, int64_t kp,
              uint32_t box_rows) {
    const int elem = fmt == kFp16 ? 2 : 4;
    cuuint64_t dims[2] = {cuuint64_t(kp), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(kp) * elem};
    cuuint32_t box[2] = {cuuint32_t(128 / elem), box_rows};
    cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = g_encode(
        map, fmt == kFp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_wide_maps(WideMaps* w, const TcecGemmArgs& g, int fmt) {
    const void* alo = g.corrected ? g.a_lo : g.a_hi;
    const void* blo = g.corrected ? g.b_lo : g.b_hi;
    const int64_t arows = g.a_rows > 0 ? g.a_rows : g.m;  // the whole A' (row chunks index into it)
    // a column block of B: its n2 rows of B' start b_row_off rows in (the byte
    // offset depends on the format, so each format's map gets its own base)
    const size_t boff = size_t(g.b_row_off) * size_t(g.kp) * (fmt == kFp16 ? 2 : 4);
    const void* bhi = static_cast<const uint8_t*>(g.b_hi) + boff;
    blo = static_cast<const uint8_t*>(blo) + boff;
    return make_map(&w->ahi, g.a_hi, fmt, arows, g.kp, 128u) && make_map(&w->alo, alo, fmt, arows, g.kp, 128u) &&
           make_map(&w->bhi, bhi, fmt, g.n2, g.kp, 128u) && make_map(&w->blo, blo, fmt, g.n2, g.kp, 128u) &&
           make_map(&w->bhi_h, bhi, fmt, g.n2, g.kp, 64u) && make_map(&w->blo_h, blo, fmt, g.n2, g.kp, 64u);
}

// rasterization group (M tiles per group) of the wide kernel; TCEC_GROUP_M
// overrides it for tuning
int wide_group_m() {
    static const int g = [] {
        const char* e = std::getenv("TCEC_GROUP_M");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? v : kWideGroupM;
    }();
    return g;
}

// floats per row of C (A-expanded layout: one C row per GEMM row pair)
int64_t ldc_of(const TcecGemmArgs& g) { return g.ldc > 0 ? g.ldc : (g.xa ? 2 * g.n2 : g.n2); }

// one cluster per 256 x 256 tile
unsigned wide_tiles_grid(const TcecGemmArgs& g) {
    return unsigned(2 * ((g.m + 2 * BM - 1) / (2 * BM)) * ((g.n2 + kWideBN - 1) / kWideBN));
}

// persistent grid: one CTA pair per two SMs, never more pairs than tiles
unsigned wide_grid(const TcecGemmArgs& g) {
    const int64_t tiles = ((g.m + 2 * BM - 1) / (2 * BM)) * ((g.n2 + kWideBN - 1) / kWideBN);
    const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(tiles, (g.sms > 1 ? g.sms : 148) / 2));
    return unsigned(2 * pairs);
}

// persistent 256 x 128 pairs: one pair per two SMs, never more pairs than tiles
unsigned pairp_grid(const TcecGemmArgs& g) {
    const int64_t tiles = ((g.m + 2 * BM - 1) / (2 * BM)) * ((g.n2 + kP2BN - 1) / kP2BN);
    const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(tiles, (g.sms > 1 ? g.sms : 148) / 2));
    return unsigned(2 * pairs);
}

template <int FMT>
int launch_fmt(const TcecGemmArgs& g, cudaStream_t s) {
    static std::atomic<uint64_t> attr_set{0};
    const cudaError_t ea = ensure_smem_attr(attr_set, [] {
        cudaError_t e = cudaFuncSetAttribute(tcec_gemm_kernel<FMT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(kSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tcec_gemm_pair_kernel<FMT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPairSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tcec_gemm_wide_kernel<FMT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(kNpSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tcec_gemm_widep_kernel<FMT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWideSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tcec_gemm_widemc_kernel<FMT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(kNpSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tcec_gemm_pairp_kernel<FMT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(kP2SmemBytes));
        return e;
    });
    if (ea != cudaSuccess) return int(ea);
    if (g.pair == kVariantPairPersistent) {
        WideMaps w;
        if (!make_wide_maps(&w, g, FMT)) return int(cudaErrorInvalidValue);
        tcec_gemm_pairp_kernel<FMT><<<pairp_grid(g), kThreadsGemm, kP2SmemBytes, s>>>(
            w, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.kind_fixed, g.corrected, g.flush_kblocks, g.xa);
        return int(cudaGetLastError());
    }
    if (g.pair == kVariantWide || g.pair == kVariantWidePersistent || g.pair == kVariantWideMc) {
        WideMaps w;
        if (!make_wide_maps(&w, g, FMT)) return int(cudaErrorInvalidValue);
        if (g.pair == kVariantWideMc)
            tcec_gemm_widemc_kernel<FMT><<<dim3(wide_tiles_grid(g), unsigned(g.partial ? g.splits : 1)),
                                           kThreadsGemm, kNpSmemBytes, s>>>(
                w, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.kind_fixed, g.corrected, g.flush_kblocks,
                wide_group_m(), int(g.a_row_off), int(ldc_of(g)), g.partial, g.kb_per, g.xa);
        else if (g.pair == kVariantWide)
            tcec_gemm_wide_kernel<FMT><<<dim3(wide_tiles_grid(g), unsigned(g.partial ? g.splits : 1)),
                                         kThreadsGemm, kNpSmemBytes, s>>>(
                w, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.kind_fixed, g.corrected, g.flush_kblocks,
                wide_group_m(), int(g.a_row_off), int(ldc_of(g)), g.partial, g.kb_per, g.xa);
        else
            tcec_gemm_widep_kernel<FMT><<<wide_grid(g), kThreadsGemm, kWideSmemBytes, s>>>(
                w, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.kind_fixed, g.corrected, g.flush_kblocks, g.xa);
        return int(cudaGetLastError());
    }
    CUtensorMap mah, mal, mbh, mbl;
    const void* alo = g.corrected ? g.a_lo : g.a_hi;
    const void* blo = g.corrected ? g.b_lo : g.b_hi;
    const uint32_t b_box = g.pair == kVariantPair ? 64u : 128u;
    if (!make_map(&mah, g.a_hi, FMT, g.m, g.kp, 128u) || !make_map(&mal, alo, FMT, g.m, g.kp, 128u) ||
        !make_map(&mbh, g.b_hi, FMT, g.n2, g.kp, b_box) ||
        !make_map(&mbl, blo, FMT, g.n2, g.kp, b_box))
        return int(cudaErrorInvalidValue);
    if (g.pair == kVariantPair) {
        const int64_t tiles = ((g.m + 2 * BM - 1) / (2 * BM)) * ((g.n2 + BN - 1) / BN);
        tcec_gemm_pair_kernel<FMT><<<unsigned(2 * tiles), kThreadsGemm, kPairSmemBytes, s>>>(
            mah, mal, mbh, mbl, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.kind_fixed,
            g.corrected, g.flush_kblocks);
    } else {
        const int64_t tiles = ((g.m + BM - 1) / BM) * ((g.n2 + BN - 1) / BN);
        const dim3 grid(unsigned(tiles), unsigned(g.partial ? g.splits : 1));
        tcec_gemm_kernel<FMT><<<grid, kThreadsGemm, kSmemBytes, s>>>(
            mah, mal, mbh, mbl, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.kind_fixed,
            g.corrected, g.flush_kblocks, g.partial, g.kb_per, g.xa);
    }
    return int(cudaGetLastError());
}

// format decided on the device: one wide launch that runs the selected format
int launch_wide_auto(const TcecGemmArgs& g, cudaStream_t s) {
    static std::atomic<uint64_t> attr_set{0};
    const cudaError_t ea = ensure_smem_attr(attr_set, [] {
        cudaError_t e = cudaFuncSetAttribute(tcec_gemm_wide_auto_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(kNpSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tcec_gemm_widep_auto_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWideSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tcec_gemm_widemc_auto_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(kNpSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tcec_gemm_pairp_auto_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(kP2SmemBytes));
        return e;
    });
    if (ea != cudaSuccess) return int(ea);
    WideMaps w16, w32;
    if (!make_wide_maps(&w16, g, kFp16) || !make_wide_maps(&w32, g, kTf32))
        return int(cudaErrorInvalidValue);
    if (g.pair == kVariantPairPersistent)
        tcec_gemm_pairp_auto_kernel<<<pairp_grid(g), kThreadsGemm, kP2SmemBytes, s>>>(
            w16, w32, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.corrected, g.flush_kblocks, g.xa);
    else if (g.pair == kVariantWideMc)
        tcec_gemm_widemc_auto_kernel<<<dim3(wide_tiles_grid(g), unsigned(g.partial ? g.splits : 1)),
                                       kThreadsGemm, kNpSmemBytes, s>>>(
            w16, w32, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.corrected, g.flush_kblocks,
            wide_group_m(), int(g.a_row_off), int(ldc_of(g)), g.partial, g.kb_per, g.xa);
    else if (g.pair == kVariantWide)
        tcec_gemm_wide_auto_kernel<<<dim3(wide_tiles_grid(g), unsigned(g.partial ? g.splits : 1)),
                                     kThreadsGemm, kNpSmemBytes, s>>>(
            w16, w32, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.corrected, g.flush_kblocks,
            wide_group_m(), int(g.a_row_off), int(ldc_of(g)), g.partial, g.kb_per, g.xa);
    else
        tcec_gemm_widep_auto_kernel<<<wide_grid(g), kThreadsGemm, kWideSmemBytes, s>>>(
            w16, w32, g.c, int(g.m), int(g.n2), int(g.kp), g.d, g.corrected, g.flush_kblocks, g.xa);
    return int(cudaGetLastError());
}

}  // namespace

int resolve_gemm_variant(int requested, int64_t m, int64_t n2, int64_t kp, int sm_count, bool allow_pair,
                         bool allow_pairp) {
    if (requested != kVariantAuto) return requested;
    const int64_t wide_ctas = 2 * ((m + 2 * BM - 1) / (2 * BM)) * ((n2 + kWideBN - 1) / kWideBN);
    // too few 256 x 256 tiles and a K too short to split: the 256 x 128 pair
    // tiles double the CTAs at ~0.9 of the wide tile's MMA efficiency --
    // 1024^3 TF32TCEC 58 (single) -> 42 us, 768^3 46 -> 34 us
    if (allow_pair && wide_ctas < sm_count && kp / 64 < 64) return kVariantPair;
    // the 256 x 256 tiles fill the SMs and K is short (<= 512 K' elements):
    // persistent 256 x 128 pairs with two tiles' accumulators in TMEM, so one
    // tile's epilogue overlaps the next tile's MMAs ((2048, 16384, 64) TF32
    // 0.164 -> 0.126 ms, (2048, 4096, 32) 0.045 -> 0.035); also up to 1024 K'
    // when the 256 x 256 tiles come in few waves ((512, 16384, 512) TF32 0.159
    // -> 0.147, FP16 0.102 -> 0.085) -- with longer K or many tiles the wide
    // tile's lower operand traffic per MAC wins (profiles/r02_pairp_ab.log)
    const int64_t half_sms = std::max(1, sm_count / 2);
    if (allow_pairp && wide_ctas >= sm_count && (kp / 64 <= 8 || (kp / 64 <= 16 && wide_ctas / 2 < 8 * half_sms)))
        return kVariantPairPersistent;
    if (wide_ctas >= sm_count && kp / 64 <= 8) return kVariantWidePersistent;
    return (wide_ctas >= sm_count || kp / 64 >= 256) ? kVariantWide : kVariantSingle;
}

static int launch_formats(const TcecGemmArgs& g, cudaStream_t s);

int launch_tcec_gemm(const TcecGemmArgs& g_in, cudaStream_t s) {
    if (!get_encode()) return int(cudaErrorNotSupported);
    if (g_in.m <= 0 || g_in.n2 <= 0) return 0;
    TcecGemmArgs g = g_in;
    g.partial = nullptr;
    g.splits = 1;
    g.kb_per = 0;
    // clusters of two pairs need an even number of 256-row tiles
    if (g.pair == kVariantWideMc && ((g.m + 2 * BM - 1) / (2 * BM)) % 2 != 0) g.pair = kVariantWide;
    // the 256 x 128 pair kernel has no A-expanded store
    if (g.xa && g.pair == kVariantPair) g.pair = kVariantWide;
    if (g.ldc > 0 && g.ldc != g.n2) g.no_split = 1;  // partials and their reduction assume ldc = n2
    if (!g.no_split && (g.pair == kVariantSingle || g.pair == kVariantWide || g.pair == kVariantWideMc)) {
        // few tiles and a long K (e.g. (512, 512, 2^19) contraction steps):
        // split K so the grid covers the SMs several times
        const int64_t tiles = g.pair != kVariantSingle
                                  ? int64_t(wide_tiles_grid(g))
                                  : ((g.m + BM - 1) / BM) * ((g.n2 + BN - 1) / BN);
        const int bk = (g.fmt == kTf32 || g.fmt < 0) ? 32 : 64;  // the finer format decides
        const int64_t nkb = g.kp / bk;
        const int sms = g.sms > 1 ? g.sms : 148;
        auto split_with = [&](int64_t want) {
            if (want < 2) return;
            // k-blocks per split in units of the f16 block (2 tf32 blocks), so
            // both format kernels cut K at the same element
            const int64_t nkb16 = g.kp / 64;
            const int64_t per16 = (nkb16 + want - 1) / want;
            const int splits = int((nkb16 + per16 - 1) / per16);
            if (splits < 2) return;
            const size_t bytes = size_t(splits) * size_t(g.m) * size_t(g.n2) * 4;
            if (cudaMallocAsync(reinterpret_cast<void**>(&g.partial), bytes, s) == cudaSuccess) {
                g.splits = splits;
                g.kb_per = int(per16);  // f16 units; the tf32 kernel doubles it
            } else {
                cudaGetLastError();
                g.partial = nullptr;
            }
        };
        // minimum f16 k-blocks (64 K' elements each) per split; TCEC_SPLIT_MINKB overrides
        static const int min_kb = [] {
            const char* e = std::getenv("TCEC_SPLIT_MINKB");
            const int v = e ? std::atoi(e) : 0;
            return v > 0 ? v : 32;
        }();
        if (tiles < sms && nkb >= 16) {
            static const int waves = [] {
                const char* e = std::getenv("TCEC_SPLIT_WAVES");  // tuning override
                const int v = e ? std::atoi(e) : 0;
                return v > 0 ? v : 8;  // swept 1/2/4/8: more waves balance best
            }();
            // every split keeps >= 32 f16 k-blocks (2048 K' elements) so the
            // partial round trip stays small against its MMA time
            int64_t want = std::min<int64_t>((waves * sms + tiles - 1) / tiles, (g.kp / 64) / min_kb);
            split_with(want);
        } else if (tiles < 8 * sms && g.pair != kVariantSingle && (g.kp / 64) / min_kb >= 2) {
            // a few waves of long tiles: split K just enough that the last wave
            // is nearly full (e.g. 512 CTAs = 3.46 waves -> 2 splits = 6.92
            // waves: (4096, 2048, 65536) TF32 steps of the Sycamore slices)
            const double w1 = double(tiles) / sms;
            int best = 1;
            double best_eff = w1 / std::ceil(w1);
            for (int sp = 2; sp <= 4 && sp <= (g.kp / 64) / min_kb; ++sp) {
                const double w = w1 * sp;
                const double eff = w / std::ceil(w);
                if (best_eff < 0.95 && eff > best_eff + 0.02) {
                    best = sp;
                    best_eff = eff;
                }
            }
            if (best >= 2) split_with(best);
        }
    }
    int e = launch_formats(g, s);
    if (!e && g.partial) {
        const int64_t count = g.m * g.n2;
        const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 16);
        split_reduce_kernel<<<unsigned(blocks), 256, 0, s>>>(g.partial, g.c, count, g.splits, g.d,
                                                            g.kind_fixed, g.xa ? g.n2 : 0);
        e = int(cudaGetLastError());
    }
    if (g.partial) cudaFreeAsync(g.partial, s);
    return e;
}

static int launch_formats(const TcecGemmArgs& g, cudaStream_t s) {
    if (g.fmt < 0) {
        // device-decided format: the wide kernel branches on the decision; the
        // other variants launch both formats and the unselected one exits
        if (g.pair == kVariantWide || g.pair == kVariantWidePersistent || g.pair == kVariantWideMc ||
            g.pair == kVariantPairPersistent)
            return launch_wide_auto(g, s);
        const int e = launch_fmt<kFp16>(g, s);
        return e ? e : launch_fmt<kTf32>(g, s);
    }
    return g.fmt == kFp16 ? launch_fmt<kFp16>(g, s) : launch_fmt<kTf32>(g, s);
}

}  // namespace tcec
