// msd_lmhead.cu -- SURVEY 8(f) NEXT-2: the lm_head GEMM fused with the row normaliser.
//
// logits = H W^T (Eq. 1's h_t W) for M rows of hidden states H [M][D] and a vocabulary
// projection W [V][D] (bf16, the nn.Linear weight layout), reduced on the fly to the Eq. 1
// normaliser LSE_r = log sum_v exp(z_rv) and the logit of a candidate token per row -- the
// B x R x V logit tensor is never written.
//
// tcgen05 GEMM: one CTA per (128-row M tile, vocabulary part); the CTA walks the 256-column N
// tiles of its part.  Warp roles: warp 0 TMA producer (A 128x64 and B 256x64 bf16 boxes, 128-byte
// swizzle, 4-stage ring), warp 1 MMA issuer (one elected lane: tcgen05.mma.cta_group::1.kind::f16,
// M = 128, N = 256, K = 16, fp32 accumulator in TMEM, double-buffered: 2 x 256 columns), warps
// 2..5 epilogue (thread = accumulator row = TMEM lane; tcgen05.ld 32 columns at a time, online
// (max, sum) in fp32 per 32 columns and float64 across them).  A second small kernel combines the
// per-part records of a row in a fixed order.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <mutex>

#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int LM_BM = 128, LM_BN = 256, LM_BK = 64, LM_STAGES = 4;
constexpr int LM_THREADS = 6 * 32;
constexpr uint32_t LM_A_BYTES = LM_BM * LM_BK * 2, LM_B_BYTES = LM_BN * LM_BK * 2;

struct LmPart {             // per (row, vocabulary part)
    float m;                // max logit of the part (-inf: none)
    int32_t has_cand;       // the candidate's logit is in this part
    double s;               // sum exp(z - m) over the part
    float zc;               // candidate logit
    float pad;
};

__device__ __forceinline__ void lm_mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle (8-row x 128-byte atoms, SBO = 1024 B)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);          // start address [0,14)
    d |= (uint64_t)0 << 16;                            // LBO (unused for K-major swizzled)
    d |= (uint64_t)(1024u >> 4) << 32;                 // SBO [32,46)
    d |= (uint64_t)1 << 46;                            // version = 1 (sm100)
    d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
    return d;
}

// instruction descriptor: bf16 x bf16 -> f32, both K-major, M = 128, N = 256
constexpr uint32_t LM_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(LM_BN >> 3) << 17) |
                              ((uint32_t)(LM_BM >> 4) << 24);

__global__ void __launch_bounds__(LM_THREADS, 1)
lmhead_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int32_t M,
              int32_t D, int64_t V, int32_t parts, const int32_t* cand, LmPart* out,
              __nv_bfloat16* logits, int64_t ldz) {
    extern __shared__ __align__(1024) unsigned char lm_smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(lm_smem_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char* sA = smem;
    unsigned char* sB = smem + LM_STAGES * LM_A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + LM_STAGES * LM_B_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + LM_STAGES;
    uint64_t* tfull = bars + 2 * LM_STAGES;
    uint64_t* tempty = bars + 2 * LM_STAGES + 2;
    uint32_t* taddr_s = reinterpret_cast<uint32_t*>(bars + 2 * LM_STAGES + 4);
    // per epilogue warp: a 32-row x 32-column bf16 chunk (rows padded to 17 words) staged so the
    // logit stores go out as whole 64-byte row segments
    uint32_t* zstage = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(bars) + 256);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x / parts, part = blockIdx.x % parts;
    const int m0 = mt * LM_BM;
    const int ntiles = (int)((V + LM_BN - 1) / LM_BN);
    const int t0 = (int)((int64_t)ntiles * part / parts), t1 = (int)((int64_t)ntiles * (part + 1) / parts);
    const int nk = D / LM_BK;

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < LM_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
            for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
        }
        __syncwarp();
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *taddr_s;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            for (int t = t0; t < t1; ++t) {
                for (int kb = 0; kb < nk; ++kb) {
                    lm_mbar_wait(&empty[st], ph ^ 1);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])),
                                 "r"(LM_A_BYTES + LM_B_BYTES) : "memory");
                    tma_load_2d(sA + st * LM_A_BYTES, &mapA, &full[st], kb * LM_BK, m0);
                    tma_load_2d(sB + st * LM_B_BYTES, &mapB, &full[st], kb * LM_BK, t * LM_BN);
                    if (++st == LM_STAGES) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        int st = 0;
        uint32_t ph = 0;
        int acc = 0;
        uint32_t aph = 0;
        for (int t = t0; t < t1; ++t) {
            lm_mbar_wait(&tempty[acc], aph ^ 1);          // the epilogue drained this accumulator
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dcol = tbase + (uint32_t)(acc * LM_BN);
            for (int kb = 0; kb < nk; ++kb) {
                lm_mbar_wait(&full[st], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(sA + st * LM_A_BYTES), b0 = smem_u32(sB + st * LM_B_BYTES);
#pragma unroll
                    for (int k = 0; k < LM_BK / 16; ++k) {
                        const uint64_t da = umma_desc_sw128(a0 + k * 32), db = umma_desc_sw128(b0 + k * 32);
                        const uint32_t accum = (kb | k) ? 1u : 0u;
                        asm volatile(
                            "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                            ::"r"(dcol), "l"(da), "l"(db), "r"(LM_IDESC), "r"(accum)
                            : "memory");
                    }
                    // the stage's operands are consumed once these MMAs complete
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 ::"r"(smem_u32(&empty[st])) : "memory");
                    if (kb == nk - 1)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                     ::"r"(smem_u32(&tfull[acc])) : "memory");
                }
                __syncwarp();
                if (++st == LM_STAGES) { st = 0; ph ^= 1; }
            }
            if (++acc == 2) { acc = 0; aph ^= 1; }
        }
    } else {
        // ---------------------------------------------------------------- epilogue (warps 2..5)
        const int q = warp & 3;                 // TMEM lane quadrant of this warp
        const int row = q * 32 + lane;          // accumulator row = TMEM lane
        const int r = m0 + row;
        const int32_t c = (cand && r < M) ? cand[r] : -1;
        float m = -INFINITY, zc = 0.f;
        int has = 0;
        double s = 0.0;
        int acc = 0;
        uint32_t aph = 0;
        for (int t = t0; t < t1; ++t) {
            lm_mbar_wait(&tfull[acc], aph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t n0 = (int64_t)t * LM_BN;
#pragma unroll 1
            for (int ch = 0; ch < LM_BN / 32; ++ch) {
                float v[32];
                const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * LM_BN + ch * 32);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                      "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]),
                      "=f"(v[15]), "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]),
                      "=f"(v[22]), "=f"(v[23]), "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]),
                      "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
                    : "r"(ta));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int64_t c0 = n0 + ch * 32;
                // columns past the vocabulary (TMA zero fill of the last tile) do not count
                const int nv = (int)max((int64_t)0, min((int64_t)32, V - c0));
                if (logits) {
                    // the logits are emitted in bf16 and everything below (maximum, normaliser,
                    // candidate) is computed from the emitted values, so the LSE is that of the
                    // tensor the verify reads
                    uint32_t w[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w[k]) : "f"(v[2 * k + 1]), "f"(v[2 * k]));
                        v[2 * k] = __uint_as_float(w[k] << 16);
                        v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
                    }
                    if (nv == 32) {
                        uint32_t* st = zstage + (warp - 2) * (32 * 17);
#pragma unroll
                        for (int k = 0; k < 16; ++k) st[lane * 17 + k] = w[k];
                        __syncwarp();
                        // 8 rows per store instruction: lane -> (row 8 q + lane / 4, 16-byte part lane % 4)
#pragma unroll
                        for (int qq = 0; qq < 4; ++qq) {
                            const int rl = qq * 8 + (lane >> 2), part = lane & 3;
                            const int rg = m0 + q * 32 + rl;
                            const uint32_t* sr = st + rl * 17 + part * 4;
                            if (rg < M)
                                *reinterpret_cast<uint4*>(logits + (int64_t)rg * ldz + c0 + part * 8) =
                                    make_uint4(sr[0], sr[1], sr[2], sr[3]);
                        }
                        __syncwarp();
                    } else if (r < M) {
                        __nv_bfloat16* dst = logits + (int64_t)r * ldz + c0;
                        for (int k = 0; k < nv; ++k)
                            dst[k] = __ushort_as_bfloat16((unsigned short)(k & 1 ? w[k / 2] >> 16 : w[k / 2] & 0xffffu));
                    }
                }
                float cm = -INFINITY;
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (k < nv) cm = fmaxf(cm, v[k]);
                if (c >= c0 && c < c0 + nv) {
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        if (c == c0 + k) zc = v[k];
                    has = 1;
                }
                if (nv > 0) {
                    if (cm > m) {                      // new running maximum: rescale the sum
                        s *= (m == -INFINITY) ? 0.0 : exp((double)m - (double)cm);
                        m = cm;
                    }
                    float cs = 0.f;
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        if (k < nv) cs += ex2f((v[k] - m) * LOG2E);
                    s += (double)cs;
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[acc])) : "memory");
            if (++acc == 2) { acc = 0; aph ^= 1; }
        }
        if (r < M) {
            LmPart o;
            o.m = m; o.has_cand = has; o.s = s; o.zc = zc; o.pad = 0.f;
            out[(size_t)r * parts + part] = o;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

// row normaliser and candidate logit from the parts (fixed order, float64)
__global__ void lmhead_combine(const LmPart* in, int32_t M, int32_t parts, float* lse, float* zc, double* lse64) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= M) return;
    float m = -INFINITY;
    for (int p = 0; p < parts; ++p) m = fmaxf(m, in[(size_t)r * parts + p].m);
    double s = 0.0;
    float z = NAN;
    for (int p = 0; p < parts; ++p) {
        const LmPart q = in[(size_t)r * parts + p];
        if (q.m > -INFINITY) s += q.s * exp((double)q.m - (double)m);
        if (q.has_cand) z = q.zc;
    }
    const double l = (double)m + log(s);
    if (lse) lse[r] = (float)l;
    if (lse64) lse64[r] = l;
    if (zc) zc[r] = z;
}

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, []() {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}
bool make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_outer) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * 2};
    const cuuint32_t box[2] = {(cuuint32_t)LM_BK, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

size_t lmhead_workspace(int32_t M, int64_t V, int nsm) {
    const int mtiles = (M + LM_BM - 1) / LM_BM;
    const int ntiles = (int)((V + LM_BN - 1) / LM_BN);
    int parts = std::max(1, nsm / std::max(1, mtiles));
    parts = std::min(parts, ntiles);
    return (size_t)M * parts * sizeof(LmPart);
}

cudaError_t launch_lmhead(const LmHeadParams& p, cudaStream_t s) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int mtiles = (p.M + LM_BM - 1) / LM_BM;
    const int ntiles = (int)((p.V + LM_BN - 1) / LM_BN);
    int parts = std::max(1, nsm / std::max(1, mtiles));
    parts = std::min(parts, ntiles);
    if ((size_t)p.M * parts * sizeof(LmPart) > p.ws_bytes) return cudaErrorInvalidValue;
    CUtensorMap ma, mb;
    if (!make_map(&ma, p.H, (uint64_t)p.D, (uint64_t)p.M, LM_BM) ||
        !make_map(&mb, p.W, (uint64_t)p.D, (uint64_t)p.V, LM_BN))
        return cudaErrorInvalidValue;
    const size_t smem = 1024 + LM_STAGES * (LM_A_BYTES + LM_B_BYTES) + 256 + 4 * 32 * 17 * 4;
    cudaError_t e = cudaFuncSetAttribute(lmhead_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    LmPart* parts_buf = reinterpret_cast<LmPart*>(p.ws);
    lmhead_kernel<<<mtiles * parts, LM_THREADS, smem, s>>>(ma, mb, p.M, p.D, p.V, parts, p.cand, parts_buf,
                                                           reinterpret_cast<__nv_bfloat16*>(p.logits), p.ldz);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    lmhead_combine<<<(p.M + 255) / 256, 256, 0, s>>>(parts_buf, p.M, parts, p.lse, p.z_cand, p.lse64);
    return cudaGetLastError();
}

}  // namespace msd
