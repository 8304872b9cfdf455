// First-layer distances on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// dots_h[q, t] = sum_u q_h[u] * c_h[t][u] for both halves (coarse_scan's
// sgemv pair, multi_index.py:283-288) as a bf16 GEMM whose products are
// exact: every f32 operand is split into three bf16 limbs (hi + mid + lo ==
// x exactly, 3 x 8 mantissa bits), each limb product is exact in the f32
// accumulator, and the six products above 2^-24 relative
// (AlBh, AmBm, AmBh, AhBl, AhBm, AhBh) are accumulated in TMEM.  Query rows
// whose mid / lo limbs are all zero -- the integer-valued queries of
// BASELINE configs 0, 1, 2 and 4 -- skip those products, so the common case
// is three MMAs per K step.  The result differs from a correctly rounded f32
// dot product by accumulation rounding only (the FFMA kernel and OpenBLAS
// differ the same way; SURVEY §7.3.4 / §8c(ii) classify the near-ties).
//
// One CTA = 128 queries (UMMA M, TMEM lanes) x one half x a range of
// 128-codeword tiles (UMMA N).  A (the queries' limbs) is converted once into
// 128-byte-swizzled K-major shared tiles; the centroid limbs are pre-swizzled
// at index creation (coarse_limb_image_kernel) so each B tile is a single
// 48 KB TMA bulk copy.  Two B stages and two TMEM accumulators let the MMAs
// of tile n + 1 run under the epilogue of tile n (tcgen05.ld -> f32 rows ->
// 16-byte global stores).  Valid for dh = 64 (one swizzle atom of K).
#include <cuda_bf16.h>

#include <algorithm>

#include "bpq_internal.cuh"

namespace bpq {

namespace {

constexpr int TC_M = 128;                 // queries per CTA (UMMA M = TMEM lanes)
constexpr int TC_N = 128;                 // codewords per tile (UMMA N)
constexpr int TC_K = 64;                  // dh: one 128-byte swizzle atom of bf16
constexpr int TC_UK = 16;                 // K per tcgen05.mma (kind::f16)
constexpr int TC_THREADS = 128;
constexpr int kLimbs = 3;
constexpr int A_LIMB_BYTES = TC_M * TC_K * 2;         // 16 KB
constexpr int B_LIMB_BYTES = TC_N * TC_K * 2;         // 16 KB
constexpr int B_TILE_BYTES = kLimbs * B_LIMB_BYTES;   // 48 KB (one bulk copy)
constexpr int kStages = 2;
constexpr int TC_SMEM = kLimbs * A_LIMB_BYTES + kStages * B_TILE_BYTES + 1024;  // + alignment slack
constexpr int kTmemCols = 2 * TC_N;                    // two f32 accumulators

// byte offset of bf16 element (row r, k) in a K-major tile with the 128-byte
// swizzle (16-byte chunk c of row r stored at chunk c ^ (r % 8))
__host__ __device__ __forceinline__ uint32_t sw128(int r, int k) {
    return (uint32_t)(r * 128 + (((k >> 3) ^ (r & 7)) << 4) + ((k & 7) << 1));
}

__device__ __forceinline__ void split3(float x, __nv_bfloat16 &h, __nv_bfloat16 &m, __nv_bfloat16 &l) {
    h = __float2bfloat16_rn(x);
    const float r1 = __fsub_rn(x, __bfloat162float(h));
    m = __float2bfloat16_rn(r1);
    const float r2 = __fsub_rn(r1, __bfloat162float(m));
    l = __float2bfloat16_rn(r2);
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;             // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;   // stride byte offset
    d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;             // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major, M x N
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                            ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void bar_init(uint64_t *bar, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *bar, unsigned parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(su32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// Centroid limb image: [tile][limb][128 rows][64 bf16] with the 128-byte
// swizzle, rows t >= T zero.  One thread per (row, k).
__global__ void coarse_limb_image_kernel(const float *__restrict__ C, int T, int ntiles, uint8_t *__restrict__ img) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)ntiles * TC_N * TC_K) return;
    const int t = (int)(idx / TC_K), k = (int)(idx % TC_K);
    const int tile = t / TC_N, r = t % TC_N;
    const float x = t < T ? C[(int64_t)t * TC_K + k] : 0.f;
    __nv_bfloat16 h, m, l;
    split3(x, h, m, l);
    uint8_t *base = img + (size_t)tile * B_TILE_BYTES + sw128(r, k);
    *reinterpret_cast<__nv_bfloat16 *>(base) = h;
    *reinterpret_cast<__nv_bfloat16 *>(base + B_LIMB_BYTES) = m;
    *reinterpret_cast<__nv_bfloat16 *>(base + 2 * B_LIMB_BYTES) = l;
}

// grid (query blocks of 128, 2 halves, tile splits); 128 threads
__global__ void __launch_bounds__(TC_THREADS, 1)
    coarse_dots_tc_kernel(const float *__restrict__ Q, int64_t nq, int D, const uint8_t *__restrict__ img1,
                          const uint8_t *__restrict__ img2, int T, int ntiles, int tiles_per_cta,
                          float *__restrict__ dots1, float *__restrict__ dots2) {
    extern __shared__ uint8_t tc_smem_raw[];
    __shared__ __align__(8) uint64_t bar_full[kStages];
    __shared__ __align__(8) uint64_t bar_mma[2];
    __shared__ uint32_t tmem_base_sh;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;                              // [3 limbs][128][64] bf16, swizzled
    uint8_t *sB = smem + kLimbs * A_LIMB_BYTES;      // [2 stages][3 limbs][128][64]
    const int h = blockIdx.y;
    const int64_t q0 = (int64_t)blockIdx.x * TC_M;
    const int tile0 = blockIdx.z * tiles_per_cta;
    const int ntl = min(tiles_per_cta, ntiles - tile0);
    if (ntl <= 0) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint8_t *img = h ? img2 : img1;
    float *out = h ? dots2 : dots1;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base_sh)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; s++) bar_init(&bar_full[s], 1);
        for (int s = 0; s < 2; s++) bar_init(&bar_mma[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // B prologue: the first two tiles stream in while A is converted
    if (tid == 0) {
        for (int j = 0; j < min(kStages, ntl); j++) {
            bar_expect_tx(&bar_full[j], B_TILE_BYTES);
            bulk_load(sB + (size_t)j * B_TILE_BYTES, img + (size_t)(tile0 + j) * B_TILE_BYTES, B_TILE_BYTES,
                      &bar_full[j]);
        }
    }
    // A: thread = query row, 64 floats of its half -> 3 swizzled bf16 limbs
    bool need_m = false, need_l = false;
    {
        const int64_t q = q0 + tid;
        const float *src = Q + q * D + (int64_t)h * TC_K;
#pragma unroll 4
        for (int k = 0; k < TC_K; k += 4) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (q < nq) {
                if ((D & 3) == 0) {
                    v = __ldg(reinterpret_cast<const float4 *>(src + k));
                } else {
                    v = make_float4(__ldg(src + k), __ldg(src + k + 1), __ldg(src + k + 2), __ldg(src + k + 3));
                }
            }
            const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int z = 0; z < 4; z++) {
                __nv_bfloat16 bh, bm, bl;
                split3(x[z], bh, bm, bl);
                need_m |= __bfloat162float(bm) != 0.f;
                need_l |= __bfloat162float(bl) != 0.f;
                uint8_t *dst = sA + sw128(tid, k + z);
                *reinterpret_cast<__nv_bfloat16 *>(dst) = bh;
                *reinterpret_cast<__nv_bfloat16 *>(dst + A_LIMB_BYTES) = bm;
                *reinterpret_cast<__nv_bfloat16 *>(dst + 2 * A_LIMB_BYTES) = bl;
            }
        }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic stores -> tensor-core reads
    need_m = __syncthreads_or(need_m);
    need_l = __syncthreads_or(need_l);
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    // the limb products, smallest first: (A limb, B limb)
    auto issue_tile = [&](int j) {
        const int s = j % kStages;
        bar_wait(&bar_full[s], (uint32_t)(j / kStages) & 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)((j & 1) * TC_N);
        const uint32_t a0 = su32(sA), b0 = su32(sB + (size_t)s * B_TILE_BYTES);
        const int pa[6] = {2, 1, 1, 0, 0, 0};
        const int pb[6] = {0, 1, 0, 2, 1, 0};
        uint32_t acc = 0;
#pragma unroll
        for (int p = 0; p < 6; p++) {
            if ((pa[p] == 2 && !need_l) || (pa[p] == 1 && !need_m)) continue;
#pragma unroll
            for (int ks = 0; ks < TC_K / TC_UK; ks++) {
                const uint32_t koff = (uint32_t)(ks * TC_UK * 2);
                mma_bf16(d, umma_desc(a0 + pa[p] * A_LIMB_BYTES + koff), umma_desc(b0 + pb[p] * B_LIMB_BYTES + koff),
                         acc);
                acc = 1;
            }
        }
        mma_commit(&bar_mma[j & 1]);
    };
    if (tid == 0) issue_tile(0);
    for (int n = 0; n < ntl; n++) {
        if (tid == 0 && n + 1 < ntl) issue_tile(n + 1);
        bar_wait(&bar_mma[n & 1], (uint32_t)(n >> 1) & 1u);
        tc_fence_after();
        // tile n's MMAs are done, so its B stage is free: stream tile n + 2 into it
        if (tid == 0 && n + kStages < ntl) {
            const int s = n % kStages;
            bar_expect_tx(&bar_full[s], B_TILE_BYTES);
            bulk_load(sB + (size_t)s * B_TILE_BYTES, img + (size_t)(tile0 + n + kStages) * B_TILE_BYTES,
                      B_TILE_BYTES, &bar_full[s]);
        }
        // epilogue: warp w owns TMEM lanes 32w..32w+31 = query rows
        const int64_t q = q0 + warp * 32 + lane;
        const int tbase = (tile0 + n) * TC_N;
#pragma unroll 1
        for (int c = 0; c < TC_N / 32; c++) {
            uint32_t v[32];
            tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((n & 1) * TC_N + c * 32), v);
            const int t0 = tbase + c * 32;
            if (q < nq && t0 < T) {
                float *row = out + q * (int64_t)T + t0;
                if ((T & 3) == 0 && t0 + 32 <= T) {
#pragma unroll
                    for (int z = 0; z < 32; z += 4)
                        *reinterpret_cast<float4 *>(row + z) = make_float4(
                            __uint_as_float(v[z]), __uint_as_float(v[z + 1]), __uint_as_float(v[z + 2]),
                            __uint_as_float(v[z + 3]));
                } else {
                    for (int z = 0; z < 32 && t0 + z < T; z++) row[z] = __uint_as_float(v[z]);
                }
            }
        }
        tc_fence_before();
        __syncthreads();  // accumulator (n & 1) drained before tile n + 2's MMAs reuse it
    }
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
    }
}

// nearest_centroids (quantizer.py:109-130) for d = 64 on the tensor cores:
// score = |c|^2 - 2 x.c with the exact-limb GEMM, argmin (first minimum ->
// lowest id) fused into the TMEM epilogue, d2 = max(score + |x|^2, 0).  One
// CTA = 128 rows x all centroid tiles (the same two-stage B ring and two
// TMEM accumulators as coarse_dots_tc_kernel).
__global__ void __launch_bounds__(TC_THREADS, 1)
    nearest_tc_kernel(const float *__restrict__ X, int64_t n, int64_t ldx, const uint8_t *__restrict__ img,
                      const float *__restrict__ cn, int nc, int ntiles, int64_t *__restrict__ out_ids,
                      float *__restrict__ out_d2, uint8_t *__restrict__ out_code, int64_t code_stride) {
    extern __shared__ uint8_t tc_smem_raw[];
    __shared__ __align__(8) uint64_t bar_full[kStages];
    __shared__ __align__(8) uint64_t bar_mma[2];
    __shared__ uint32_t tmem_base_sh;
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;
    uint8_t *sB = smem + kLimbs * A_LIMB_BYTES;
    const int64_t r0 = (int64_t)blockIdx.x * TC_M;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntl = ntiles;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base_sh)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; s++) bar_init(&bar_full[s], 1);
        for (int s = 0; s < 2; s++) bar_init(&bar_mma[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        for (int j = 0; j < min(kStages, ntl); j++) {
            bar_expect_tx(&bar_full[j], B_TILE_BYTES);
            bulk_load(sB + (size_t)j * B_TILE_BYTES, img + (size_t)j * B_TILE_BYTES, B_TILE_BYTES, &bar_full[j]);
        }
    }
    // A: thread = data row; |x|^2 as the FFMA encoder computes it (ascending fmaf chain)
    bool need_m = false, need_l = false;
    float xn = 0.f;
    {
        const int64_t r = r0 + tid;
        const float *src = X + r * ldx;
#pragma unroll 4
        for (int k = 0; k < TC_K; k++) {
            const float x = r < n ? __ldg(src + k) : 0.f;
            xn = fmaf(x, x, xn);
            __nv_bfloat16 bh, bm, bl;
            split3(x, bh, bm, bl);
            need_m |= __bfloat162float(bm) != 0.f;
            need_l |= __bfloat162float(bl) != 0.f;
            uint8_t *dst = sA + sw128(tid, k);
            *reinterpret_cast<__nv_bfloat16 *>(dst) = bh;
            *reinterpret_cast<__nv_bfloat16 *>(dst + A_LIMB_BYTES) = bm;
            *reinterpret_cast<__nv_bfloat16 *>(dst + 2 * A_LIMB_BYTES) = bl;
        }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    need_m = __syncthreads_or(need_m);
    need_l = __syncthreads_or(need_l);
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    auto issue_tile = [&](int j) {
        const int s = j % kStages;
        bar_wait(&bar_full[s], (uint32_t)(j / kStages) & 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)((j & 1) * TC_N);
        const uint32_t a0 = su32(sA), b0 = su32(sB + (size_t)s * B_TILE_BYTES);
        const int pa[6] = {2, 1, 1, 0, 0, 0};
        const int pb[6] = {0, 1, 0, 2, 1, 0};
        uint32_t acc = 0;
#pragma unroll
        for (int p = 0; p < 6; p++) {
            if ((pa[p] == 2 && !need_l) || (pa[p] == 1 && !need_m)) continue;
#pragma unroll
            for (int ks = 0; ks < TC_K / TC_UK; ks++) {
                const uint32_t koff = (uint32_t)(ks * TC_UK * 2);
                mma_bf16(d, umma_desc(a0 + pa[p] * A_LIMB_BYTES + koff), umma_desc(b0 + pb[p] * B_LIMB_BYTES + koff),
                         acc);
                acc = 1;
            }
        }
        mma_commit(&bar_mma[j & 1]);
    };
    float best = INFINITY;
    int bidx = 0x7fffffff;
    if (tid == 0) issue_tile(0);
    for (int t = 0; t < ntl; t++) {
        if (tid == 0 && t + 1 < ntl) issue_tile(t + 1);
        bar_wait(&bar_mma[t & 1], (uint32_t)(t >> 1) & 1u);
        tc_fence_after();
        if (tid == 0 && t + kStages < ntl) {
            const int s = t % kStages;
            bar_expect_tx(&bar_full[s], B_TILE_BYTES);
            bulk_load(sB + (size_t)s * B_TILE_BYTES, img + (size_t)(t + kStages) * B_TILE_BYTES, B_TILE_BYTES,
                      &bar_full[s]);
        }
#pragma unroll 1
        for (int c = 0; c < TC_N / 32; c++) {
            uint32_t v[32];
            tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((t & 1) * TC_N + c * 32), v);
            const int c0 = t * TC_N + c * 32;
#pragma unroll
            for (int z = 0; z < 32; z++) {
                const int ci = c0 + z;
                if (ci < nc) {
                    const float sc = __fsub_rn(__ldg(cn + ci), __fmul_rn(2.f, __uint_as_float(v[z])));
                    if (sc < best) {
                        best = sc;
                        bidx = ci;
                    }
                }
            }
        }
        tc_fence_before();
        __syncthreads();
    }
    {
        const int64_t r = r0 + warp * 32 + lane;
        // the epilogue row of thread tid is TMEM lane tid = A row tid: the same row
        if (r < n) {
            const int id = bidx == 0x7fffffff ? 0 : bidx;
            if (out_ids) out_ids[r] = id;
            if (out_code) out_code[r * code_stride] = (uint8_t)id;
            if (out_d2) {
                const float v = __fadd_rn(best, xn);
                out_d2[r] = v > 0.f ? v : 0.f;
            }
        }
    }
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
    }
}

}  // namespace

size_t coarse_limb_image_bytes(int32_t T) {
    return (size_t)((T + TC_N - 1) / TC_N) * B_TILE_BYTES;
}

int launch_coarse_limb_image(const float *C, int32_t T, uint8_t *img, cudaStream_t s) {
    const int ntiles = (T + TC_N - 1) / TC_N;
    const int64_t n = (int64_t)ntiles * TC_N * TC_K;
    coarse_limb_image_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(C, T, ntiles, img);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

int launch_nearest_tc(const float *xs, int64_t n, int64_t ld_x, const uint8_t *img, const float *cn, int32_t nc,
                      int64_t *out_ids, float *out_d2, uint8_t *out_code, int64_t code_stride, cudaStream_t s) {
    if (n <= 0) return BPQ_OK;
    static bool attr = false;
    if (!attr) {
        BPQ_CUDA_TRY(cudaFuncSetAttribute(nearest_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM));
        attr = true;
    }
    const int ntiles = (nc + TC_N - 1) / TC_N;
    const int64_t blocks = (n + TC_M - 1) / TC_M;
    BPQ_CHECK(blocks <= 0x7FFFFFFF, BPQ_ERR_UNSUPPORTED, "too many rows for one nearest_centroids call");
    nearest_tc_kernel<<<(unsigned)blocks, TC_THREADS, TC_SMEM, s>>>(xs, n, ld_x, img, cn, nc, ntiles, out_ids,
                                                                      out_d2, out_code, code_stride);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

int launch_coarse_dots_tc(const float *queries, int64_t nq, int32_t D, const uint8_t *img1, const uint8_t *img2,
                          int32_t T, float *dots1, float *dots2, cudaStream_t s) {
    BPQ_CHECK(D == 2 * TC_K, BPQ_ERR_UNSUPPORTED, "tensor-core first layer needs D = 128");
    if (nq <= 0) return BPQ_OK;
    static bool attr = false;
    if (!attr) {
        BPQ_CUDA_TRY(cudaFuncSetAttribute(coarse_dots_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM));
        attr = true;
    }
    const int ntiles = (T + TC_N - 1) / TC_N;
    const int qblocks = (int)((nq + TC_M - 1) / TC_M);
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // about four CTAs per SM over the launch (one resident at a time)
    int splits = (4 * sms + 2 * qblocks - 1) / (2 * qblocks);
    splits = std::max(1, std::min(splits, ntiles));
    const int per = (ntiles + splits - 1) / splits;
    splits = (ntiles + per - 1) / per;
    dim3 grid((unsigned)qblocks, 2, (unsigned)splits);
    coarse_dots_tc_kernel<<<grid, TC_THREADS, TC_SMEM, s>>>(queries, nq, D, img1, img2, T, ntiles, per, dots1, dots2);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

}  // namespace bpq
