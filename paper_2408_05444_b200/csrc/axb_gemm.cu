// axb_gemm.cu — K1: FP64 dense contraction on the DMMA tensor pipe.
//
// Replaces the reference's sequential ikj matmul (matrix.hpp:325-338) where the
// solver forms the residual R = C − (A·X)·B: at construction (solver.hpp:173),
// at every drift checkpoint (:420, :427-436) and at every exact-metric confirm
// (:412-419), plus G = A·Aᵀ (gram_mmt, matrix.hpp:481-494) when the Gram
// columns are cached.  sm_100a has no tcgen05 f64 kind, so the FP64 tensor path
// is `mma.sync.m8n8k4.f64` (SASS DMMA.8x8x4).
//
// Two kernels share one tile — CTA 64×128×16, 4 compute warps (2×2), warp tile
// 32×64 = 4×8 DMMA tiles, two CTAs per SM — and one fused epilogue (the "C −"
// subtraction, the Σ D² partials for ‖R‖² and the Σ (R_old − D)² partials of the
// drift guard, so a checkpoint is one pass):
//   * k_dgemm_tma (below, the production path): operands arrive as TMA tensor
//     boxes issued by a fifth, producer warp into a 4-stage mbarrier ring; the C
//     tile of the epilogue follows the k-tiles through the same ring.
//     36.3 TFLOP/s at the config-5 shape (cuBLAS DGEMM 35.7, measured DMMA peak
//     36.99), 34.8–35.0 at the config-3 shapes (cuBLAS 33.5–35.0).
//   * k_dgemm (round 1; operands whose rows are not 16-byte aligned): cp.async
//     into a 3-stage ring of padded tiles, 33.4 / 31.3–31.5 TFLOP/s.
// Every output element accumulates over k in the same order in both, so they
// agree bitwise (tests/test_gpu_gemm.py).
#include <cuda.h>  // CUtensorMap (types only: the encoder is fetched through cudart)

#include <cmath>
#include <cstdlib>

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

// ------------------------------------------------------------------------
// k_dgemm_tma — the same 64×128×16 tile fed by TMA instead of cp.async.
//
// One producer warp (its lane 0) issues `cp.async.bulk.tensor.2d` (SASS UTMALDG)
// box loads into a 4-stage ring guarded by full/empty mbarriers; the four
// consumer warps only wait on a barrier, read DMMA fragments from shared memory
// and issue `mma.sync.m8n8k4.f64` — no address arithmetic, no cp.async issue
// slots and no CTA-wide barrier in the main loop.  Out-of-range rows, columns
// and k are zero-filled by the tensor map's bounds, so there are no predicates.
//
// Shared-memory layout: every box row is 16 doubles = 128 B under
// CU_TENSOR_MAP_SWIZZLE_128B (16-byte chunk c of row r sits at chunk c ^ (r&7)).
// A dense 128-byte pitch puts every row on bank 0, so which tile row / column a
// DMMA lane takes is permuted to make each half-warp's 16 fragment loads hit 16
// distinct 8-byte slots:
//   * k-contiguous tiles (A; B when b_trans): the lane of fragment row gq reads
//     tile row 8·i + π(gq), π(g) = 2·(g&3) + (g>>2), so a half-warp's rows have
//     distinct (r&7)>>1 and its two k-chunks land on 8 distinct swizzled chunks;
//   * n-contiguous tiles (B as K×N): eight 16×16 boxes side by side; fragment
//     column j of the 8-wide DMMA tile `ni` reads box ni>>1, column
//     8·((j>>1)&1) + (j&1) + 2·(j>>2) + 4·(ni&1).
// The epilogue applies the same permutations to the global row / column of each
// accumulator, so results are those of the plain mapping.
constexpr int T_STAGES = 4, T_CONS_WARPS = 4, T_THREADS = (T_CONS_WARPS + 1) * 32;
constexpr int T_A_BYTES = BM * BK * 8;  // 8 KB
constexpr int T_B_BYTES = BK * BN * 8;  // 16 KB
constexpr int T_STAGE_BYTES = T_A_BYTES + T_B_BYTES;
constexpr int T_C_STAGES = 3;  // epilogue stages holding the Cin tile (3 + 3 + 2 boxes of 8 KB)
static_assert(3 * T_A_BYTES == T_STAGE_BYTES && T_C_STAGES * 3 >= BN / 16 && T_C_STAGES <= T_STAGES, "Cin staging");
constexpr size_t T_SMEM = (size_t)T_STAGES * T_STAGE_BYTES + 1024 /*alignment slack*/ + 128;

__device__ __forceinline__ unsigned g_smem_u32(const void* ptr) {
    return (unsigned)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void g_mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void g_mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void g_mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void g_mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar) : "memory");
}

__device__ __forceinline__ void l2_prefetch_bulk(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool getenv_no_prefetch(const GemmArgs& g) { return g.no_pf != 0; }

template <bool BTRANS>
__global__ void __launch_bounds__(T_THREADS, 2)
k_dgemm_tma(GemmArgs g, const __grid_constant__ CUtensorMap mapA,
            const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapC,
            int c_tma) {
    extern __shared__ unsigned char t_dsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m0 = (long long)blockIdx.y * BM, n0 = (long long)blockIdx.x * BN;
    if (g.sym && n0 + BN <= m0) return;  // strictly below the diagonal: mirrored later
    const int KT = (int)((g.K + BK - 1) / BK);
    const unsigned base = (g_smem_u32(t_dsm) + 1023u) & ~1023u;
    const unsigned char* sbase = t_dsm + (base - g_smem_u32(t_dsm));  // the ring, generic view
    const unsigned bars = base + T_STAGES * T_STAGE_BYTES;  // full[S], empty[S]
    if (tid == 0) {
        for (int i = 0; i < T_STAGES; ++i) {
            g_mbar_init(bars + 8 * i, 1);
            g_mbar_init(bars + 8 * (T_STAGES + i), T_CONS_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int wm = warp / WARPS_N, wn = warp % WARPS_N;
    const int gq = lane >> 2, tq = lane & 3;
    const int pg = 2 * (gq & 3) + (gq >> 2);  // π(gq)

    if (warp == T_CONS_WARPS) {
        if (lane != 0) {
            // idle producer lanes: bulk-prefetch the tile's epilogue operands (Cin,
            // Rold) into L2 so the epilogue's loads are L2 hits
            const bool pf_c = !c_tma && g.Cin && (g.ldc & 1) == 0 &&
                              (reinterpret_cast<uintptr_t>(g.Cin) & 15) == 0;
            const bool pf_r = g.Rold && (g.ldr & 1) == 0 && (reinterpret_cast<uintptr_t>(g.Rold) & 15) == 0;
            const long long w = (g.N - n0 < BN ? g.N - n0 : BN) & ~1ll;
            if (w > 0 && (pf_c || pf_r) && !getenv_no_prefetch(g))
                for (int r = lane - 1; r < BM && m0 + r < g.M; r += 31) {
                    if (pf_c) l2_prefetch_bulk(g.Cin + (m0 + r) * g.ldc + n0, (unsigned)(w * 8));
                    if (pf_r) l2_prefetch_bulk(g.Rold + (m0 + r) * g.ldr + n0, (unsigned)(w * 8));
                }
        } else {
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % T_STAGES;
                if (kt >= T_STAGES) g_mbar_wait(bars + 8 * (T_STAGES + s), ((kt / T_STAGES) - 1) & 1);
                const unsigned full = bars + 8 * s;
                const unsigned a_s = base + s * T_STAGE_BYTES, b_s = a_s + T_A_BYTES;
                g_mbar_expect_tx(full, T_STAGE_BYTES);
                tma_load_2d(a_s, &mapA, kt * BK, (int)m0, full);
                if (BTRANS) {
                    tma_load_2d(b_s, &mapB, kt * BK, (int)n0, full);
                } else {
#pragma unroll
                    for (int b = 0; b < BN / 16; ++b)
                        tma_load_2d(b_s + b * (BK * 128), &mapB, (int)n0 + b * 16, kt * BK, full);
                }
            }
            if (c_tma) {
                // the Cin tile follows the k-tiles through the ring: eight 64×16 boxes
                // (the A-tile geometry), three per stage, in flight while the
                // consumers finish the last k-tiles
#pragma unroll
                for (int u = 0; u < T_C_STAGES; ++u) {
                    const int j = KT + u, s = j % T_STAGES;
                    if (j >= T_STAGES) g_mbar_wait(bars + 8 * (T_STAGES + s), ((j / T_STAGES) - 1) & 1);
                    const unsigned full = bars + 8 * s;
                    const int nb = (BN / 16 - 3 * u) < 3 ? (BN / 16 - 3 * u) : 3;
                    g_mbar_expect_tx(full, nb * T_A_BYTES);
                    for (int b = 0; b < nb; ++b)
                        tma_load_2d(base + s * T_STAGE_BYTES + b * T_A_BYTES, &mapC,
                                    (int)n0 + (3 * u + b) * 16, (int)m0, full);
                }
            }
        }
    } else {
        // per-lane fragment offsets (bytes) inside a stage
        unsigned offA[BK / 4];  // k-contiguous tile, row 8·i + π(gq)
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk)
            offA[kk] = pg * 128 + (((2 * kk + (tq >> 1)) ^ pg) << 4) + (tq & 1) * 8;
        // n-contiguous boxes: k row 4kk+tq, chunk cj ^ 2e ^ (4(kk&1)+tq), half j&1
        const int cj = 4 * ((gq >> 1) & 1) + (gq >> 2);
        unsigned offB[2][2];  // [kk&1][e]
#pragma unroll
        for (int k1 = 0; k1 < 2; ++k1)
#pragma unroll
            for (int e = 0; e < 2; ++e)
                offB[k1][e] = tq * 128 + (((cj ^ (2 * e) ^ (4 * k1 + tq)) & 7) << 4) + (gq & 1) * 8;
        for (int kt = 0; kt < KT; ++kt) {
            const int s = kt % T_STAGES;
            g_mbar_wait(bars + 8 * s, (kt / T_STAGES) & 1);
            const unsigned char* a_s = sbase + s * T_STAGE_BYTES + wm * (FM * 8 * 128);
            const unsigned char* b_s = sbase + s * T_STAGE_BYTES + T_A_BYTES;
            auto lds64 = [](const unsigned char* p) { return *reinterpret_cast<const double*>(p); };
#pragma unroll
            for (int kk = 0; kk < BK / 4; ++kk) {
                double af[FM], bf[FN];
#pragma unroll
                for (int mi = 0; mi < FM; ++mi) af[mi] = lds64(a_s + mi * 1024 + offA[kk]);
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) {
                    if (BTRANS)
                        bf[ni] = lds64(b_s + (wn * FN + ni) * 1024 + offA[kk]);
                    else
                        bf[ni] = lds64(b_s + (wn * (FN / 2) + (ni >> 1)) * (BK * 128) + kk * 512 +
                                       offB[kk & 1][ni & 1]);
                }
#pragma unroll
                for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                    for (int ni = 0; ni < FN; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
            }
            __syncwarp();
            if (lane == 0) g_mbar_arrive(bars + 8 * (T_STAGES + s));
        }
    }

    // ---- fused epilogue (consumer warps hold the accumulators) ----
    double sq = 0.0, df = 0.0;
    if (warp < T_CONS_WARPS) {
        const bool v2 = !BTRANS && ((g.ldd | g.ldc | g.ldr) & 1) == 0;
        if (c_tma) {
#pragma unroll
            for (int u = 0; u < T_C_STAGES; ++u) {
                const int j = KT + u;
                g_mbar_wait(bars + 8 * (j % T_STAGES), (j / T_STAGES) & 1);
            }
        }
#pragma unroll
        for (int mi = 0; mi < FM; ++mi) {
            const long long r = m0 + wm * FM * 8 + mi * 8 + pg;
            if (r >= g.M) continue;
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) {
                long long c, c1;
                if (BTRANS) {
                    const int j0 = 2 * tq, j1 = 2 * tq + 1;
                    c = n0 + (wn * FN + ni) * 8 + 2 * (j0 & 3) + (j0 >> 2);
                    c1 = n0 + (wn * FN + ni) * 8 + 2 * (j1 & 3) + (j1 >> 2);
                } else {
                    c = n0 + (wn * (FN / 2) + (ni >> 1)) * 16 + 8 * (tq & 1) + 2 * (tq >> 1) +
                        4 * (ni & 1);
                    c1 = c + 1;
                }
                const bool one = c < g.N, two = c1 < g.N;
                if (!one && !two) continue;
                double o0 = acc[mi][ni][0], o1 = acc[mi][ni][1];
                if (g.Cin) {
                    if (!BTRANS && c_tma) {
                        // box b of the Cin tile, row 8·i + π(gq), 16-byte chunk under the 128 B swizzle
                        const int b = wn * (FN / 2) + (ni >> 1), j = KT + b / 3;
                        const int rl = wm * FM * 8 + mi * 8 + pg;
                        const int ch = 4 * (tq & 1) + (tq >> 1) + 2 * (ni & 1);
                        const double2 cc = *reinterpret_cast<const double2*>(
                            sbase + (j % T_STAGES) * T_STAGE_BYTES + (b % 3) * T_A_BYTES + rl * 128 +
                            ((ch ^ pg) << 4));
                        o0 = cc.x - o0;
                        o1 = cc.y - o1;
                    } else if (one && two && v2) {
                        const double2 cc = *reinterpret_cast<const double2*>(g.Cin + r * g.ldc + c);
                        o0 = cc.x - o0;
                        o1 = cc.y - o1;
                    } else {
                        if (one) o0 = g.Cin[r * g.ldc + c] - o0;
                        if (two) o1 = g.Cin[r * g.ldc + c1] - o1;
                    }
                }
                sq += (one ? o0 * o0 : 0.0) + (two ? o1 * o1 : 0.0);
                if (g.Rold) {
                    const double d0 = one ? g.Rold[r * g.ldr + c] - o0 : 0.0;
                    const double d1 = two ? g.Rold[r * g.ldr + c1] - o1 : 0.0;
                    df += d0 * d0 + d1 * d1;
                }
                if (g.store) {
                    if (one && two && v2) {
                        *reinterpret_cast<double2*>(g.D + r * g.ldd + c) = make_double2(o0, o1);
                    } else {
                        if (one) g.D[r * g.ldd + c] = o0;
                        if (two) g.D[r * g.ldd + c1] = o1;
                    }
                }
            }
        }
    }
    if (g.sq_part || g.diff_part) {
        __shared__ double red[2][T_CONS_WARPS];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sq += __shfl_xor_sync(0xffffffffu, sq, o);
            df += __shfl_xor_sync(0xffffffffu, df, o);
        }
        if (lane == 0 && warp < T_CONS_WARPS) {
            red[0][warp] = sq;
            red[1][warp] = df;
        }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, b = 0.0;
            for (int w = 0; w < T_CONS_WARPS; ++w) {
                a += red[0][w];
                b += red[1][w];
            }
            const long long bid = (long long)blockIdx.y * gridDim.x + blockIdx.x;
            if (g.sq_part) g.sq_part[bid] = a;
            if (g.diff_part) g.diff_part[bid] = b;
        }
    }
}

// cuTensorMapEncodeTiled, fetched through the runtime (no libcuda link dependency)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// row-major FP64 matrix rows×cols (leading dimension ld) as a 2-D map with a
// box of box_rows × 16 columns (128 B), 128-byte swizzle, zero fill out of range
bool make_map(CUtensorMap* map, const double* ptr, long long rows, long long cols, long long ld,
              unsigned box_rows) {
    EncodeTiledFn enc = encode_tiled_fn();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {16, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA needs 16-byte aligned bases and row pitches and 32-bit box coordinates
bool tma_eligible(const GemmArgs& g) {
    const char* e = getenv("AXB_GEMM_TMA");  // read per launch: tests toggle it
    if (e && atoi(e) == 0) return false;
    const long long lim = 1ll << 31;
    return ((g.lda | g.ldb) & 1) == 0 &&
           ((reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B)) & 15) == 0 &&
           g.M + BM < lim && g.N + BN < lim && g.K + BK < lim;
}

template <bool BT>
bool launch_tma(const GemmArgs& g0, cudaStream_t s) {
    GemmArgs g = g0;
    if (const char* e = getenv("AXB_GEMM_PF")) g.no_pf = atoi(e) == 0;
    CUtensorMap mapA, mapB, mapC;
    if (!make_map(&mapA, g.A, g.M, g.K, g.lda, BM)) return false;
    // Cin through the ring when its rows are 16-byte aligned (else global loads)
    int c_tma = !BT && g.Cin && (g.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(g.Cin) & 15) == 0;
    if (const char* e = getenv("AXB_GEMM_CTMA")) c_tma = c_tma && atoi(e) != 0;
    if (c_tma) {
        if (!make_map(&mapC, g.Cin, g.M, g.N, g.ldc, BM)) return false;
    } else {
        mapC = mapA;
    }
    if (BT) {
        if (!make_map(&mapB, g.B, g.N, g.K, g.ldb, BN)) return false;
    } else {
        if (!make_map(&mapB, g.B, g.K, g.N, g.ldb, BK)) return false;
    }
    static bool attr[64] = {};  // the attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaFuncSetAttribute(k_dgemm_tma<BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T_SMEM);
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM));
    k_dgemm_tma<BT><<<grid, T_THREADS, T_SMEM, s>>>(g, mapA, mapB, mapC, c_tma);
    return true;
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
    if (tma_eligible(g) && (g.b_trans ? launch_tma<true>(g, s) : launch_tma<false>(g, s))) return;
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
