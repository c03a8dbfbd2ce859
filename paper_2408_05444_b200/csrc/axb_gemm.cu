// axb_gemm.cu — K1: FP64 dense contraction on the DMMA tensor pipe.
//
// Replaces the reference's sequential ikj matmul (matrix.hpp:325-338) where the
// solver forms the residual R = C − (A·X)·B: at construction (solver.hpp:173),
// at every drift checkpoint (:420, :427-436) and at every exact-metric confirm
// (:412-419), plus G = A·Aᵀ (gram_mmt, matrix.hpp:481-494) when the Gram
// columns are cached.  sm_100a has no tcgen05 f64 kind, so the FP64 tensor path
// is `mma.sync.m8n8k4.f64` (SASS DMMA.8x8x4); operands are staged global→shared
// with cp.async in a 3-stage ring.
//
// CTA tile 64×128×16, 4 warps (2×2), warp tile 32×64 = 4×8 DMMA tiles, two CTAs
// per SM (≤ 256 registers, 92 KB smem each).  Measured against the 128×128
// one-CTA-per-SM tile (tools/gemm_variants.cu, config-3 / config-5 shapes):
// 34.2 / 35.0 vs 31.5 / 32.2 TFLOP/s; cuBLAS DGEMM 35.8 / 36.0.
// Epilogue fuses the "C −" subtraction, the Σ D² partials (‖R‖²) and the
// Σ (R_old − D)² partials (the drift guard), so a checkpoint is one pass.
#include <cmath>

#include "axb_device.cuh"

namespace axb_dev {

namespace {

constexpr int BM = 64, BN = 128, BK = 16, PAD = 4, STAGES = 3, THREADS = 128;
constexpr int WARPS_N = 2, FM = 4, FN = 8;  // warp grid 2×2, warp tile (FM·8)×(FN·8)
static_assert(BK == 16 && BN == 128, "load_stage's index math assumes BK = 16, BN = 128");
static_assert(WARPS_N * FN * 8 == BN && (THREADS / 32 / WARPS_N) * FM * 8 == BM, "warp grid");
constexpr int A_LD = BK + PAD;       // A tile: BM × (BK+PAD), k contiguous
constexpr int BN_LD = BN + PAD;      // B tile (K×N source): BK × (BN+PAD)
constexpr int BT_LD = BK + PAD;      // B tile (N×K source): BN × (BK+PAD)
constexpr int A_STAGE = BM * A_LD;
constexpr int B_STAGE = (BN * BT_LD > BK * BN_LD) ? BN * BT_LD : BK * BN_LD;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    const int src = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int src_bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// stage loader: tile k-range [k0, k0+BK)
template <bool BTRANS, bool V16>
__device__ __forceinline__ void load_stage(const GemmArgs& g, double* As, double* Bs, long long m0,
                                           long long n0, long long k0) {
    const int tid = threadIdx.x;
    if (V16) {
        // A: 128 rows × 8 double2
#pragma unroll
        for (int it = 0; it < (BM * BK / 2) / THREADS; ++it) {
            const int e = tid + it * THREADS;
            const int r = e >> 3, c2 = (e & 7) * 2;
            const long long gr = m0 + r, gc = k0 + c2;
            const bool ok = gr < g.M && gc < g.K;
            const int bytes = ok ? (gc + 1 < g.K ? 16 : 8) : 0;
            cp_async16(As + r * A_LD + c2, ok ? g.A + gr * g.lda + gc : g.A, bytes);
        }
        if (!BTRANS) {
            // B: 16 rows × 64 double2
#pragma unroll
            for (int it = 0; it < (BK * BN / 2) / THREADS; ++it) {
                const int e = tid + it * THREADS;
                const int r = e >> 6, c2 = (e & 63) * 2;
                const long long gr = k0 + r, gc = n0 + c2;
                const bool ok = gr < g.K && gc < g.N;
                const int bytes = ok ? (gc + 1 < g.N ? 16 : 8) : 0;
                cp_async16(Bs + r * BN_LD + c2, ok ? g.B + gr * g.ldb + gc : g.B, bytes);
            }
        } else {
#pragma unroll
            for (int it = 0; it < (BN * BK / 2) / THREADS; ++it) {
                const int e = tid + it * THREADS;
                const int r = e >> 3, c2 = (e & 7) * 2;
                const long long gr = n0 + r, gc = k0 + c2;
                const bool ok = gr < g.N && gc < g.K;
                const int bytes = ok ? (gc + 1 < g.K ? 16 : 8) : 0;
                cp_async16(Bs + r * BT_LD + c2, ok ? g.B + gr * g.ldb + gc : g.B, bytes);
            }
        }
    } else {
#pragma unroll
        for (int it = 0; it < (BM * BK) / THREADS; ++it) {
            const int e = tid + it * THREADS;
            const int r = e >> 4, c = e & 15;
            const long long gr = m0 + r, gc = k0 + c;
            const bool ok = gr < g.M && gc < g.K;
            cp_async8(As + r * A_LD + c, ok ? g.A + gr * g.lda + gc : g.A, ok);
        }
        if (!BTRANS) {
#pragma unroll
            for (int it = 0; it < (BK * BN) / THREADS; ++it) {
                const int e = tid + it * THREADS;
                const int r = e >> 7, c = e & 127;
                const long long gr = k0 + r, gc = n0 + c;
                const bool ok = gr < g.K && gc < g.N;
                cp_async8(Bs + r * BN_LD + c, ok ? g.B + gr * g.ldb + gc : g.B, ok);
            }
        } else {
#pragma unroll
            for (int it = 0; it < (BN * BK) / THREADS; ++it) {
                const int e = tid + it * THREADS;
                const int r = e >> 4, c = e & 15;
                const long long gr = n0 + r, gc = k0 + c;
                const bool ok = gr < g.N && gc < g.K;
                cp_async8(Bs + r * BT_LD + c, ok ? g.B + gr * g.ldb + gc : g.B, ok);
            }
        }
    }
}

template <bool BTRANS, bool V16>
__global__ void __launch_bounds__(THREADS, 2) k_dgemm(GemmArgs g) {
    extern __shared__ __align__(16) double sm[];
    double* As = sm;
    double* Bs = sm + STAGES * A_STAGE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WARPS_N, wn = warp % WARPS_N;
    const int gq = lane >> 2, tq = lane & 3;
    const long long m0 = (long long)blockIdx.y * BM, n0 = (long long)blockIdx.x * BN;
    if (g.sym && n0 + BN <= m0) return;  // strictly below the diagonal: mirrored later
    const long long KT = (g.K + BK - 1) / BK;

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < KT) load_stage<BTRANS, V16>(g, As + s * A_STAGE, Bs + s * B_STAGE, m0, n0, s * BK);
        cp_commit();
    }
    for (long long kt = 0; kt < KT; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const long long nk = kt + STAGES - 1;
        if (nk < KT) {
            const int st = (int)(nk % STAGES);
            load_stage<BTRANS, V16>(g, As + st * A_STAGE, Bs + st * B_STAGE, m0, n0, nk * BK);
        }
        cp_commit();
        const int cs = (int)(kt % STAGES);
        const double* a_s = As + cs * A_STAGE + (wm * FM * 8 + gq) * A_LD + tq;
        const double* b_s = Bs + cs * B_STAGE;
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
            double af[FM], bf[FN];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) af[mi] = a_s[mi * 8 * A_LD + kk * 4];
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) {
                const int col = wn * FN * 8 + ni * 8 + gq;
                bf[ni] = BTRANS ? b_s[col * BT_LD + kk * 4 + tq] : b_s[(kk * 4 + tq) * BN_LD + col];
            }
#pragma unroll
            for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
    }
    cp_wait<0>();

    // ---- fused epilogue ----
    double sq = 0.0, df = 0.0;
    const bool v2 = ((g.ldd | g.ldc | g.ldr) & 1) == 0;
#pragma unroll
    for (int mi = 0; mi < FM; ++mi) {
        const long long r = m0 + wm * FM * 8 + mi * 8 + gq;
        if (r >= g.M) continue;
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) {
            const long long c = n0 + wn * FN * 8 + ni * 8 + 2 * tq;
            if (c >= g.N) continue;
            const bool two = c + 1 < g.N;
            double o0 = acc[mi][ni][0], o1 = acc[mi][ni][1];
            if (g.Cin) {
                if (two && v2) {
                    const double2 cc = *reinterpret_cast<const double2*>(g.Cin + r * g.ldc + c);
                    o0 = cc.x - o0;
                    o1 = cc.y - o1;
                } else {
                    o0 = g.Cin[r * g.ldc + c] - o0;
                    if (two) o1 = g.Cin[r * g.ldc + c + 1] - o1;
                }
            }
            sq += o0 * o0 + (two ? o1 * o1 : 0.0);
            if (g.Rold) {
                const double d0 = g.Rold[r * g.ldr + c] - o0;
                const double d1 = two ? g.Rold[r * g.ldr + c + 1] - o1 : 0.0;
                df += d0 * d0 + d1 * d1;
            }
            if (g.store) {
                if (two && v2) {
                    *reinterpret_cast<double2*>(g.D + r * g.ldd + c) = make_double2(o0, o1);
                } else {
                    g.D[r * g.ldd + c] = o0;
                    if (two) g.D[r * g.ldd + c + 1] = o1;
                }
            }
        }
    }
    if (g.sq_part || g.diff_part) {
        __shared__ double red[2][THREADS / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sq += __shfl_xor_sync(0xffffffffu, sq, o);
            df += __shfl_xor_sync(0xffffffffu, df, o);
        }
        if (lane == 0) {
            red[0][warp] = sq;
            red[1][warp] = df;
        }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, b = 0.0;
            for (int w = 0; w < THREADS / 32; ++w) {
                a += red[0][w];
                b += red[1][w];
            }
            const long long bid = (long long)blockIdx.y * gridDim.x + blockIdx.x;
            if (g.sq_part) g.sq_part[bid] = a;
            if (g.diff_part) g.diff_part[bid] = b;
        }
    }
}

__global__ void __launch_bounds__(1024) k_reduce_parts(const double* part, long long n,
                                                       double* out) {
    __shared__ double red[32];
    double s = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = red[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) *out = t;
    }
}

// lower 32×32 blocks ← transposed upper blocks (gram_mmt's mirror, matrix.hpp:489-490)
__global__ void k_mirror_lower(double* D, long long nn, long long ld) {
    __shared__ double t[32][33];
    const long long bi = blockIdx.y, bj = blockIdx.x;  // destination block (bi, bj), bj < bi
    if (bj >= bi) return;
    const long long r0 = bj * 32, c0 = bi * 32;  // source block (bj, bi) in the upper part
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const long long r = r0 + j, c = c0 + threadIdx.x;
        if (r < nn && c < nn) t[j][threadIdx.x] = D[r * ld + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const long long r = c0 + j, c = r0 + threadIdx.x;  // D[c0+j][r0+x] = D[r0+x][c0+j]
        if (r < nn && c < nn) D[r * ld + c] = t[threadIdx.x][j];
    }
}

template <bool BT, bool V>
void launch_t(const GemmArgs& g, cudaStream_t s) {
    const size_t smem = sizeof(double) * (size_t)STAGES * (A_STAGE + B_STAGE);
    static bool attr[64] = {};  // the attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaFuncSetAttribute(k_dgemm<BT, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM));
    k_dgemm<BT, V><<<grid, THREADS, smem, s>>>(g);
}

}  // namespace

int gemm_num_ctas(long long M, long long N) {
    return (int)(((N + BN - 1) / BN) * ((M + BM - 1) / BM));
}

void launch_gemm(const GemmArgs& g, cudaStream_t s) {
    if (g.M <= 0 || g.N <= 0) return;
    const bool v16 = ((g.lda | g.ldb) & 1) == 0 && ((reinterpret_cast<uintptr_t>(g.A) |
                                                       reinterpret_cast<uintptr_t>(g.B)) & 15) == 0;
    if (g.b_trans) {
        if (v16) launch_t<true, true>(g, s);
        else launch_t<true, false>(g, s);
    } else {
        if (v16) launch_t<false, true>(g, s);
        else launch_t<false, false>(g, s);
    }
}

void launch_mirror_lower(double* D, long long nn, long long ld, cudaStream_t s) {
    const unsigned nb = (unsigned)((nn + 31) / 32);
    k_mirror_lower<<<dim3(nb, nb), dim3(32, 8), 0, s>>>(D, nn, ld);
}

void launch_reduce_parts(const double* part, long long n, double* out, cudaStream_t s) {
    k_reduce_parts<<<1, 1024, 0, s>>>(part, n, out);
}

}  // namespace axb_dev
