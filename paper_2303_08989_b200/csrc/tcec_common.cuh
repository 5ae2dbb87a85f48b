// Shared device helpers for the sm_100a TCEC path: bit-exact format emulation
// (mirrors reference lowprec.hpp:44-101), PTX wrappers for mbarrier / TMA /
// tcgen05, and small utilities.  Compiled for -gencode arch=compute_100a only;
// no fast-math anywhere on this path (RN/RZ semantics are part of the contract).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per device for a group
// of kernels (the attribute is per device context); `done` holds one bit per
// device, so concurrent callers and several devices in one process are safe
// (setting it twice is harmless).
template <typename F>
inline cudaError_t ensure_smem_attr(std::atomic<uint64_t>& done, F&& set_all) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    const cudaError_t e = set_all();
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

#define TCEC_DEV __device__ __forceinline__

namespace tcec {

// ------------------------------------------------------------------ formats
enum Fmt : int { kFp16 = 0, kTf32 = 1 };

// (2 - 2^-10) * 2^15 and (2 - 2^-10) * 2^127, lowprec.hpp:28-33
constexpr float kFp16Max = 65504.0f;
constexpr float kTf32Max = 0x1.ffcp127f;

// floor(log2|x|) from the bits of a nonzero magnitude (lowprec.hpp:44-51)
TCEC_DEV int exponent_of_bits(uint32_t b) {
    const int raw = int(b >> 23);
    return raw ? raw - 127 : -149 + (31 - __clz(b));
}
inline int exponent_of_bits_host(uint32_t b) {
    const int raw = int(b >> 23);
    return raw ? raw - 127 : -149 + (31 - __builtin_clz(b));
}

// quantize to FP16 (values kept in f32), lowprec.hpp:58-74.  cvt.rn/rz.f16.f32
// are IEEE conversions that produce FP16 subnormals, which is exactly
// nearbyint/trunc(x * 2^-q) * 2^q with q = max(e - 10, -24); saturation above
// 65504 is explicit because the hardware conversion would produce infinity.
TCEC_DEV float quantize_fp16(float x, bool rz, unsigned& ovf) {
    if (x == 0.0f) return x;
    if (fabsf(x) > kFp16Max) {
        ovf = 1u;
        return copysignf(kFp16Max, x);
    }
    return __half2float(rz ? __float2half_rz(x) : __float2half_rn(x));
}

// quantize to TF32: q = e - 10 for every finite f32 (TF32 keeps the f32
// exponent range), so rounding is an integer RNE/RZ at bit 13 of the pattern
// (the same trick as reference kernels_avx2.cpp:62-81, equal to lowprec.hpp).
TCEC_DEV float quantize_tf32(float x, bool rz, unsigned& ovf) {
    if (x == 0.0f) return x;
    if (fabsf(x) > kTf32Max) {
        ovf = 1u;
        return copysignf(kTf32Max, x);
    }
    uint32_t b = __float_as_uint(x);
    if ((b & 0x7FFFFFFFu) > 0x7F800000u) return x;  // NaN passes through
    if (!rz) b += 0xFFFu + ((b >> 13) & 1u);
    return __uint_as_float(b & ~0x1FFFu);
}

TCEC_DEV float quantize(float x, int fmt, bool rz, unsigned& ovf) {
    return fmt == kFp16 ? quantize_fp16(x, rz, ovf) : quantize_tf32(x, rz, ovf);
}

// residual split, lowprec.hpp:84-88: hi = RN(x), lo = RN((x - hi) * 2^11)
template <int FMT>
TCEC_DEV void split(float x, float& hi, float& lo, unsigned& ovf) {
    if (FMT == kFp16) {
        hi = quantize_fp16(x, false, ovf);
        lo = quantize_fp16(__fmul_rn(__fsub_rn(x, hi), 2048.0f), false, ovf);
    } else {
        hi = quantize_tf32(x, false, ovf);
        lo = quantize_tf32(__fmul_rn(__fsub_rn(x, hi), 2048.0f), false, ovf);
    }
}

// dst = float(double(x) * 2^s): one rounding of the exact product, with the
// factor formed in double exactly as reference kernels_scalar.cpp:34-40
TCEC_DEV float scale_pow2(float x, double factor) {
    return __double2float_rn(__dmul_rn(double(x), factor));
}

// f32 add rounded toward zero (lowprec.hpp:94-101): the native RZ add
TCEC_DEV float add_rz(float a, float b) { return __fadd_rz(a, b); }

// ----------------------------------------------------------------- mbarrier
TCEC_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

TCEC_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

TCEC_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

TCEC_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

TCEC_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

TCEC_DEV void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

TCEC_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------------- TMA
TCEC_DEV void tma_prefetch(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

TCEC_DEV void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// ------------------------------------------------------------------ tcgen05
TCEC_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
TCEC_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <uint32_t kCols>
TCEC_DEV void tmem_alloc(uint32_t* smem_slot) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
TCEC_DEV void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

// one lane of a converged warp (elect.sync); lets the whole warp run the MMA
// issue loop so its operands stay in uniform registers
TCEC_DEV bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred P;\n"
        "elect.sync _|P, 0xffffffff;\n"
        "selp.b32 %0, 1, 0, P;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

// D[tmem] (+)= A[smem] * B[smem]; idesc selects kind/shape/majors
TCEC_DEV void mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                      uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

TCEC_DEV void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                       uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// arrive on an mbarrier once every previously issued tcgen05 op of this
// thread has completed (implicitly fence::before_thread_sync)
TCEC_DEV void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// RN flush interval of the TCEC main term in the kernel's own k-blocks:
// `packed` carries the FP16 interval (k-blocks of 64 elements) in its low 16
// bits and, when non-zero, the TF32 interval (k-blocks of 32) in its high 16
TCEC_DEV int flush_of(int packed, int fmt) {
    const int tf = (packed >> 16) & 0xFFFF;
    return (fmt == 1 && tf > 0) ? tf : (packed & 0xFFFF);
}

// ---------------------------------------------------- CTA pair (cta_group::2)
TCEC_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

TCEC_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// address of the same shared-memory object in CTA `rank` of the cluster
TCEC_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

// arrive on an mbarrier of another CTA of the cluster.  Default semantics
// (release at CTA scope, as cute's ClusterBarrier::arrive): the arrivals only
// hand TMEM buffers back, which tcgen05.fence::before_thread_sync orders; an
// explicit .release.cluster costs a GPU-scope MEMBAR per arrive (measured:
// ~15 % of the warp stall samples of a small-k wide GEMM)
TCEC_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// TMA into this CTA's smem whose transaction bytes land on the pair leader's
// mbarrier (peer bit cleared, cute SM100_TMA_2SM_LOAD_2D)
TCEC_DEV void tma_load_2d_pair(void* smem_dst, const void* tmap, uint64_t* bar, int x, int y) {
    const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(mbar), "r"(x), "r"(y)
        : "memory");
}

// the same load multicast to the CTAs of `mask` (same smem offset in each);
// every destination's bytes land on the leader of the destination's pair
// (cute SM100_TMA_2SM_LOAD_MULTICAST)
TCEC_DEV void tma_load_2d_pair_mc(void* smem_dst, const void* tmap, uint64_t* bar, int x, int y,
                                  uint16_t mask) {
    const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(mbar), "r"(x), "r"(y), "h"(mask)
        : "memory");
}

template <uint32_t kCols>
TCEC_DEV void tmem_alloc_pair(uint32_t* smem_slot) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
TCEC_DEV void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

TCEC_DEV void mma2_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                       uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

TCEC_DEV void mma2_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                        uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// commit of the pair leader's MMAs, arriving on the barrier at the same smem
// offset in every CTA of `mask`
TCEC_DEV void mma_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns; thread t of the warp receives
// lane (32*(warp%4) + t), columns [col, col+32)
TCEC_DEV void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 16 consecutive 32-bit columns
TCEC_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// two 32-column loads issued back to back with one wait (64 columns)
TCEC_DEV void tmem_ld64(uint32_t taddr, float (&v)[64]) {
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]),
          "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]),
          "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),
          "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]),
          "=r"(r[62]), "=r"(r[63])
        : "r"(taddr + 32u));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory matrix descriptor for a K-major, 128-byte-swizzled tile
// whose rows are 128 B and whose 8-row core groups are 1024 B apart
// (cute/arch/mma_sm100_desc.hpp SmemDescriptor: start>>4 @0, LBO>>4 @16,
// SBO>>4 @32, version 1 @46, layout SWIZZLE_128B = 2 @61)
TCEC_DEV uint64_t umma_desc_k_sw128(const void* smem_tile) {
    const uint64_t start = (smem_u32(smem_tile) & 0x3FFFFu) >> 4;
    const uint64_t sbo = 1024u >> 4;
    return start | (sbo << 32) | (1ull << 46) | (2ull << 61);
}

// instruction descriptor (mma_sm100_desc.hpp InstrDescriptor): D f32 @4,
// A/B format @7/@10 (F16 = 0, TF32 = 2), K-major A/B, N>>3 @17, M>>4 @24
template <int FMT, int M, int N>
__host__ __device__ constexpr uint32_t umma_idesc() {
    constexpr uint32_t ab = FMT == kFp16 ? 0u : 2u;
    return (1u << 4) | (ab << 7) | (ab << 10) | (uint32_t(N >> 3) << 17) |
           (uint32_t(M >> 4) << 24);
}

}  // namespace tcec
