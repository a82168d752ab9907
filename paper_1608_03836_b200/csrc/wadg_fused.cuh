// Fused LSRK45 stage for tetrahedra, strong-weak form (the configs' hot path):
//
//   rhs   = Mhat^-1 [volume + surface](Q_in)          solver.py:241-265, 207-238
//   res   = a res + dt * Pq diag(w) Vq rhs             solver.py:290-301, 348-363
//   Q_out = Q_in + b res
//
// in ONE kernel per stage.  Q is ping-ponged (Q_in is read-only for the whole
// stage, so neighbour face traces need no grid-wide barrier), which brings the
// HBM traffic per element down to the fused lower bound of SURVEY.md §8(d):
// own fields, neighbour face nodes, geometric factors, face factors, WADG
// weights, res read/write and Q_out write.
//
// Each CTA owns KB elements.  All dense operator applications are CTA-level
// register-tiled GEMMs on CUDA cores (elements = M, quadrature points / nodes
// = N, nodes / quadrature points = K): a thread accumulates a TE x TQ (or
// TE2 x TJ) tile, loading TE element values and TQ operator values per k-step
// as 16-byte vectors, so each shared-memory load feeds several FMAs.  The
// operator matrices are repacked on the host into quadrature-chunk-contiguous
// tiles and staged into shared memory by TMA bulk copies
// (cp.async.bulk + mbarrier).  The volume and update reference operators are
// dense (Nq x Np with Nq = (N+1)^3 > Np); fp64 runs on the DFMA pipe, fp32 on
// the FFMA pipe (see DESIGN.md for why no tensor-core path here).

#pragma once

// unroll factor of the GEMM k-loops (compile-time trip counts)
#ifndef WADG_KUNROLL_N
#define WADG_KUNROLL_N 8
#endif
#define WADG_PRAGMA(x) _Pragma(#x)
#define WADG_KUNROLL_I(n) WADG_PRAGMA(unroll n)
#define WADG_KUNROLL WADG_KUNROLL_I(WADG_KUNROLL_N)

namespace wadg {
namespace fused {

__host__ __device__ constexpr int np_tet(int N) { return (N + 1) * (N + 2) * (N + 3) / 6; }
__host__ __device__ constexpr int nfp_tri(int N) { return (N + 1) * (N + 2) / 2; }
__host__ __device__ constexpr int rup(int a, int b) { return ((a + b - 1) / b) * b; }
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ constexpr size_t maxz(size_t a, size_t b) { return a > b ? a : b; }

constexpr int NTF = 256;   // threads per CTA

// compile-time configuration per (real type, order)
template <typename T, int N>
struct Cfg {
    static constexpr bool F32 = sizeof(T) == 4;
    static constexpr int NP = np_tet(N);
    static constexpr int NPP = rup(NP, 4);
    static constexpr int NQ = (N + 1) * (N + 1) * (N + 1);
    static constexpr int NFP = nfp_tri(N);
    static constexpr int NFQ = (N + 1) * (N + 1);
    static constexpr int NF = 4, FLD = 4;
    static constexpr int KB = F32 ? (N <= 4 ? 64 : 32) : (N == 1 ? 64 : (N <= 5 ? 32 : 16));
    static constexpr int QC0 = F32 ? (N <= 4 ? 64 : 32) : (N <= 2 ? 64 : (N <= 5 ? 32 : 16));
    static constexpr int QC = QC0 < rup(NQ, 8) ? QC0 : rup(NQ, 8);   // never wider than Nq
    static constexpr int MINB = N == 1 ? 3 : (((!F32 && (N == 2 || N == 3)) || (F32 && N == 5)) ? 2 : 1);   // low order: several CTAs / SM
    static constexpr int NCH = cdiv(NQ, QC);
    // phase A (interp-to-quadrature GEMMs): TE elements x TQ quad points
    // low orders use 1-element tiles so that every phase keeps most of the 256
    // threads busy (at N = 1 a CTA has only 64 x 4 nodes / quadrature points)
    static constexpr int TE = (N == 1 || (F32 && N == 5)) ? 1 : (F32 ? (QC == 64 ? 4 : 2) : 2);
    static constexpr int TQ = N == 1 ? 2 : (F32 ? 4 : (QC == 64 ? 4 : (QC == 32 ? 2 : 1)));
    static constexpr int TILES_A = (KB / TE) * (QC / TQ);
    // phase B (projection GEMMs): TE2 elements x TJ nodes, all 4 fields
    // (TE2, TJ) chosen per order so that most of the 256 threads own a tile
    static constexpr int TE2 = N == 1 ? 1 : (F32 ? ((N == 2 || N == 3 || N == 5) ? 2 : 4) : (N == 2 ? 1 : 2));
    static constexpr int TJ = N == 1 ? 1 : ((N == 4 || N == 6) ? 3 : ((N == 2 || (!F32 && N == 3)) ? 2 : 4));
    static constexpr int EG2 = KB / TE2;
    static constexpr int TILES_B = EG2 * (NPP / TJ);
    static constexpr int SLOTS = cdiv(TILES_B, NTF);
    // face-trace interpolation tiles: TFQ face points x TEF elements
    static constexpr int TFQ = N == 1 ? 1 : 2;
    static constexpr int TEF = N == 1 ? 1 : (F32 ? (N == 5 ? 2 : 4) : ((N == 2 || N == 3) ? 1 : 2));
    static constexpr int NFQP = rup(NFQ, TFQ);
    static constexpr int TILES_F = (KB / TEF) * (NFQP / TFQ);
    static constexpr int SLOTS_F = cdiv(TILES_F, NTF);
    // shared memory (bytes)
    static constexpr size_t SQ = (size_t)FLD * NPP * KB * sizeof(T);
    static constexpr size_t S_OPA = (size_t)NPP * QC * 4 * sizeof(T);
    static constexpr size_t S_OPB = (size_t)QC * NPP * 4 * sizeof(T);
    static constexpr size_t S_W = (size_t)6 * QC * KB * sizeof(T);
    static constexpr size_t PH_V = S_OPA + S_OPB + S_W;
    // surface: exterior face nodes of one face, double buffered (cp.async)
    static constexpr size_t S_P1 = (size_t)FLD * NFP * KB * sizeof(T);
    static constexpr size_t S_P = 2 * S_P1;
    static constexpr size_t S_G = (size_t)FLD * NFQ * KB * sizeof(T);
    static constexpr size_t S_LIFT = (size_t)NFQ * NPP * sizeof(T);
    static constexpr size_t S_VFI = (size_t)rup(NFP * NFQP, 4) * sizeof(T);   // transposed [i][fq]
    static constexpr size_t S_TAB = (size_t)rup(2 * NF * KB + NF * NFP + NF * 6 * NFP + 6 * NFP, 4) * 4;
    static constexpr size_t PH_S = S_P + S_G + S_LIFT + S_VFI + S_TAB;
    static constexpr int FPT = cdiv(NFQ * KB, NTF);   // flux points per thread
    static constexpr size_t S_R = (size_t)FLD * NPP * KB * sizeof(T);
    static constexpr size_t S_U1 = (size_t)NPP * QC * sizeof(T);
    static constexpr size_t S_U2 = (size_t)QC * NPP * sizeof(T);
    static constexpr size_t S_W2 = (size_t)FLD * QC * KB * sizeof(T);
    static constexpr size_t PH_U = S_R + S_U1 + S_U2 + S_W2;
    static constexpr size_t PH = PH_V > PH_S ? (PH_V > PH_U ? PH_V : PH_U) : (PH_S > PH_U ? PH_S : PH_U);
    static constexpr size_t SMEM = 16 + SQ + PH;   // 16 B: mbarrier
};

template <typename T, int V> struct Vec;
template <> struct Vec<float, 4> { using type = float4; };
template <> struct Vec<float, 2> { using type = float2; };
template <> struct Vec<float, 1> { using type = float; };
template <> struct Vec<double, 2> { using type = double2; };
template <> struct Vec<double, 1> { using type = double; };

// load / store V contiguous reals (16 B aligned where V*sizeof(T) == 16)
template <typename T, int V>
__device__ __forceinline__ void ldv(T (&d)[V], const T *p) {
    if constexpr (V * sizeof(T) == 16 || V * sizeof(T) == 8) {
        using VT = typename Vec<T, V>::type;
        const VT v = *reinterpret_cast<const VT *>(p);
        const T *s = reinterpret_cast<const T *>(&v);
#pragma unroll
        for (int i = 0; i < V; ++i) d[i] = s[i];
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) d[i] = p[i];
    }
}

template <typename T, int V>
__device__ __forceinline__ void stv(T *p, const T (&d)[V]) {
    if constexpr (V * sizeof(T) == 16 || V * sizeof(T) == 8) {
        using VT = typename Vec<T, V>::type;
        VT v;
        T *s = reinterpret_cast<T *>(&v);
#pragma unroll
        for (int i = 0; i < V; ++i) s[i] = d[i];
        *reinterpret_cast<VT *>(p) = v;
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) p[i] = d[i];
    }
}

template <typename T, int V>
__device__ __forceinline__ void ldg_v(T (&d)[V], const T *p) {
    if constexpr (V * sizeof(T) == 16 || V * sizeof(T) == 8) {
        using VT = typename Vec<T, V>::type;
        const VT v = __ldg(reinterpret_cast<const VT *>(p));
        const T *s = reinterpret_cast<const T *>(&v);
#pragma unroll
        for (int i = 0; i < V; ++i) d[i] = s[i];
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) d[i] = __ldg(p + i);
    }
}

// ---- TMA bulk copy (global -> shared) with an mbarrier -----------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%1], %0;\n" ::"r"(count), "r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %0;\n" ::"r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <typename T>
__device__ __forceinline__ void cp_async_elem(T *dst, const T *src) {
    if constexpr (sizeof(T) == 4) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    }
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(PENDING) : "memory"); }

// Copy `n` byte segments to shared memory through the barrier (thread 0 issues).
struct BulkLoader {
    uint64_t *bar;
    uint32_t phase;
    __device__ void load2(void *d0, const void *s0, uint32_t b0, void *d1, const void *s1, uint32_t b1) {
        __syncthreads();                 // previous readers of the destination are done
        if (threadIdx.x == 0) {
            fence_proxy_async();
            mbar_expect_tx(bar, b0 + b1);
            bulk_g2s(d0, s0, b0, bar);
            if (b1) bulk_g2s(d1, s1, b1, bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
    }
};

template <typename T>
struct FProb {
    int K, Kpad;
    const T *opVA, *opVB, *opU1, *opU2, *liftT, *Vfi;
    const int32_t *fmask, *ext_node, *fperm;
    const T *geo, *fgeo, *wu, *wp;
    T c2;
    const int32_t *nbr, *ncode;
    const T *halo;
    int nor;
    long long *prof;   // optional: per-CTA clock64 at phase boundaries (debug)
    const T *geo_il, *fgeo_il, *wu_il, *wp_il;   // block-interleaved copies (tcgen05 stage)
    const T *wbar;                               // tcgen05 stage: [2][Kpad] mean update weights (or NULL)
};

#define WADG_PROF_MARK(slot)                                                          \
    do {                                                                              \
        if (P.prof && threadIdx.x == 0) P.prof[(size_t)blockIdx.x * 8 + (slot)] = clock64(); \
    } while (0)

template <typename T, int N>
__global__ void __launch_bounds__(NTF, (Cfg<T, N>::MINB))
k_stage_fused(const FProb<T> P, const T *__restrict__ Qin, T *__restrict__ Qout, T *__restrict__ res,
              T tau_p, T tau_u, T a_rk, T b_rk, T dt, int block0) {
    using C = Cfg<T, N>;
    constexpr int NP = C::NP, NPP = C::NPP, NQ = C::NQ, NFP = C::NFP, NFQ = C::NFQ, NF = C::NF;
    constexpr int KB = C::KB, QC = C::QC, TE = C::TE, TQ = C::TQ, TE2 = C::TE2, TJ = C::TJ;
    constexpr int FLD = 4;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
    T *sQ = reinterpret_cast<T *>(smem_raw + 16);
    unsigned char *ph = smem_raw + 16 + C::SQ;
    // phase V
    T *sOpA = reinterpret_cast<T *>(ph);
    T *sOpB = reinterpret_cast<T *>(ph + C::S_OPA);
    T *sW = reinterpret_cast<T *>(ph + C::S_OPA + C::S_OPB);
    // phase S
    T *sP = reinterpret_cast<T *>(ph);
    T *sG = reinterpret_cast<T *>(ph + C::S_P);
    T *sLift = reinterpret_cast<T *>(ph + C::S_P + C::S_G);
    T *sVfi = reinterpret_cast<T *>(ph + C::S_P + C::S_G + C::S_LIFT);
    int32_t *sNbr = reinterpret_cast<int32_t *>(ph + C::S_P + C::S_G + C::S_LIFT + C::S_VFI);
    int32_t *sCode = sNbr + NF * KB;
    int32_t *sFmask = sCode + NF * KB;
    int32_t *sExt = sFmask + NF * NFP;
    int32_t *sPerm = sExt + NF * 6 * NFP;
    // phase U
    T *sR = reinterpret_cast<T *>(ph);
    T *sU1 = reinterpret_cast<T *>(ph + C::S_R);
    T *sU2 = reinterpret_cast<T *>(ph + C::S_R + C::S_U1);
    T *sW2 = reinterpret_cast<T *>(ph + C::S_R + C::S_U1 + C::S_U2);

    const int tid = threadIdx.x;
    const size_t S = P.Kpad;
    const size_t kblk = (size_t)(block0 + blockIdx.x) * KB;

    WADG_PROF_MARK(0);
    if (tid == 0) mbar_init(bar, 1);
    // stage the element fields with 16-byte cp.async (rows >= NP zero)
    for (int r = tid; r < FLD * NPP * (KB * (int)sizeof(T) / 16); r += NTF) {
        constexpr int PER = 16 / sizeof(T);
        const int e4 = (r % (KB / PER)) * PER, row = r / (KB / PER);
        const int c = row / NPP, j = row % NPP;
        T *dst = sQ + row * KB + e4;
        if (j < NP) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)),
                         "l"(Qin + (size_t)(c * NP + j) * S + kblk + e4) : "memory");
        } else {
#pragma unroll
            for (int t = 0; t < PER; ++t) dst[t] = T(0);
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
    BulkLoader ld{bar, 0u};

    // phase-B tile ownership (persistent accumulators)
    T acc[C::SLOTS][FLD][TE2][TJ];
#pragma unroll
    for (int s = 0; s < C::SLOTS; ++s)
#pragma unroll
        for (int c = 0; c < FLD; ++c)
#pragma unroll
            for (int t = 0; t < TE2; ++t)
#pragma unroll
                for (int u = 0; u < TJ; ++u) acc[s][c][t][u] = T(0);

    __syncthreads();
    WADG_PROF_MARK(1);
    // ======================= volume =======================================
    for (int ch = 0; ch < C::NCH; ++ch) {
        ld.load2(sOpA, P.opVA + (size_t)ch * NPP * QC * 4, (uint32_t)C::S_OPA,
                 sOpB, P.opVB + (size_t)ch * QC * NPP * 4, (uint32_t)C::S_OPB);
        // A: D_a p and V u_i at the chunk's quadrature points, then geometric factors
        for (int tile = tid; tile < C::TILES_A; tile += NTF) {
            const int te = tile % (KB / TE), tq = tile / (KB / TE);
            const int e0 = te * TE, q0 = tq * TQ;
            T av[6][TE][TQ];
#pragma unroll
            for (int m = 0; m < 6; ++m)
#pragma unroll
                for (int t = 0; t < TE; ++t)
#pragma unroll
                    for (int s = 0; s < TQ; ++s) av[m][t][s] = T(0);
WADG_KUNROLL
            for (int j = 0; j < NPP; ++j) {
                T x[4][TE];
#pragma unroll
                for (int c = 0; c < 4; ++c) ldv<T, TE>(x[c], sQ + (c * NPP + j) * KB + e0);
                T o[TQ][4];
#pragma unroll
                for (int s = 0; s < TQ; ++s) ldv<T, 4>(o[s], sOpA + (j * QC + q0 + s) * 4);
#pragma unroll
                for (int t = 0; t < TE; ++t)
#pragma unroll
                    for (int s = 0; s < TQ; ++s) {
#pragma unroll
                        for (int a = 0; a < 3; ++a) av[a][t][s] = fma(o[s][a], x[0][t], av[a][t][s]);
#pragma unroll
                        for (int i = 0; i < 3; ++i) av[3 + i][t][s] = fma(o[s][3], x[1 + i][t], av[3 + i][t][s]);
                    }
            }
#pragma unroll
            for (int s = 0; s < TQ; ++s) {
                const int q = ch * QC + q0 + s;
                T gp[3][TE], F[3][TE];
                if (q < NQ) {
                    T G[9][TE];
#pragma unroll
                    for (int r = 0; r < 9; ++r) ldg_v<T, TE>(G[r], P.geo + (size_t)(r * NQ + q) * S + kblk + e0);
#pragma unroll
                    for (int t = 0; t < TE; ++t) {
#pragma unroll
                        for (int i = 0; i < 3; ++i) {
                            gp[i][t] = G[0 * 3 + i][t] * av[0][t][s] + G[1 * 3 + i][t] * av[1][t][s] +
                                       G[2 * 3 + i][t] * av[2][t][s];
                        }
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            F[a][t] = G[a * 3 + 0][t] * av[3][t][s] + G[a * 3 + 1][t] * av[4][t][s] +
                                      G[a * 3 + 2][t] * av[5][t][s];
                        }
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < TE; ++t)
#pragma unroll
                        for (int i = 0; i < 3; ++i) { gp[i][t] = T(0); F[i][t] = T(0); }
                }
#pragma unroll
                for (int i = 0; i < 3; ++i) stv<T, TE>(sW + (i * QC + q0 + s) * KB + e0, gp[i]);
#pragma unroll
                for (int a = 0; a < 3; ++a) stv<T, TE>(sW + ((3 + a) * QC + q0 + s) * KB + e0, F[a]);
            }
        }
        __syncthreads();
        // B: project back to nodes: r_p += sum_a DTW_a F_a ; r_u_i -= Pq gp_i
#pragma unroll
        for (int sl = 0; sl < C::SLOTS; ++sl) {
            const int tile = tid + sl * NTF;
            if (tile < C::TILES_B) {
                const int e0 = (tile % C::EG2) * TE2, j0 = (tile / C::EG2) * TJ;
WADG_KUNROLL
                for (int qq = 0; qq < QC; ++qq) {
                    T w[6][TE2];
#pragma unroll
                    for (int m = 0; m < 6; ++m) ldv<T, TE2>(w[m], sW + (m * QC + qq) * KB + e0);
                    T o[TJ][4];
#pragma unroll
                    for (int u = 0; u < TJ; ++u) ldv<T, 4>(o[u], sOpB + (qq * NPP + j0 + u) * 4);
#pragma unroll
                    for (int t = 0; t < TE2; ++t)
#pragma unroll
                        for (int u = 0; u < TJ; ++u) {
                            T s0 = acc[sl][0][t][u];
                            s0 = fma(o[u][0], w[3][t], s0);
                            s0 = fma(o[u][1], w[4][t], s0);
                            s0 = fma(o[u][2], w[5][t], s0);
                            acc[sl][0][t][u] = s0;
#pragma unroll
                            for (int i = 0; i < 3; ++i) acc[sl][1 + i][t][u] = fma(-o[u][3], w[i][t], acc[sl][1 + i][t][u]);
                        }
                }
            }
        }
    }

    // ======================= surface ======================================
    const int NFQT = NF * NFQ;
    __syncthreads();
    WADG_PROF_MARK(2);
    // connectivity tables and the face interpolation matrix into shared memory
    for (int r = tid; r < NF * KB; r += NTF) {
        const int f = r / KB, e = r % KB;
        sNbr[r] = P.nbr[(size_t)f * S + kblk + e];
        sCode[r] = P.ncode[(size_t)f * S + kblk + e];
    }
    for (int r = tid; r < NF * NFP; r += NTF) sFmask[r] = __ldg(P.fmask + r);
    for (int r = tid; r < NF * 6 * NFP; r += NTF) sExt[r] = __ldg(P.ext_node + r);
    for (int r = tid; r < 6 * NFP; r += NTF) sPerm[r] = __ldg(P.fperm + r);
    for (int r = tid; r < NFP * C::NFQP; r += NTF) {
        const int i = r / C::NFQP, fq = r % C::NFQP;
        sVfi[r] = fq < NFQ ? __ldg(P.Vfi + fq * NFP + i) : T(0);
    }
    __syncthreads();
    // exterior face-node values of face f into buffer `buf`: neighbours and halo
    // slots by cp.async (all loads in flight at once), Dirichlet mirror from sQ
    auto gather = [&](int f, T *buf) {
        for (int r = tid; r < FLD * NFP * KB; r += NTF) {
            const int e = r % KB, rest = r / KB;
            const int i = rest % NFP, c = rest / NFP;
            const int nb = sNbr[f * KB + e];
            const int code = sCode[f * KB + e];
            T *dst = buf + (c * NFP + i) * KB + e;
            if (nb >= 0) {
                cp_async_elem(dst, Qin + (size_t)(c * NP + sExt[code * NFP + i]) * S + nb);
            } else if (nb == -1) {
                const T m = sQ[(c * NPP + sFmask[f * NFP + i]) * KB + e];
                *dst = (c == 0) ? -m : m;
            } else {
                cp_async_elem(dst, P.halo + ((size_t)(-nb - 2) * FLD + c) * NFP + sPerm[(code % P.nor) * NFP + i]);
            }
        }
        cp_async_commit();
    };
    gather(0, sP);
    for (int f = 0; f < NF; ++f) {
        T *cur = sP + (f & 1) * (FLD * NFP * KB);
        if (f + 1 < NF) {
            gather(f + 1, sP + ((f + 1) & 1) * (FLD * NFP * KB));
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        // lift rows of this face (TMA bulk copy, lands while the flux is computed)
        if (tid == 0) {
            fence_proxy_async();
            mbar_expect_tx(bar, (uint32_t)C::S_LIFT);
            bulk_g2s(sLift, P.liftT + (size_t)f * NFQ * NPP, (uint32_t)C::S_LIFT, bar);
        }
        __syncthreads();
        if (f == 0) WADG_PROF_MARK(3);
        // traces at face quadrature points: register-tiled interpolation of the
        // interior (sQ via fmask) and exterior (cur) face nodes, then the flux
        constexpr int TFQ = C::TFQ, TEF = C::TEF;
#pragma unroll
        for (int sl = 0; sl < C::SLOTS_F; ++sl) {
            const int tile = tid + sl * NTF;
            if (tile < C::TILES_F) {
                const int e0 = (tile % (KB / TEF)) * TEF, fq0 = (tile / (KB / TEF)) * TFQ;
                T fg[TFQ][4][TEF];
#pragma unroll
                for (int s2 = 0; s2 < TFQ; ++s2) {
                    const int fq = min(fq0 + s2, NFQ - 1);
#pragma unroll
                    for (int d = 0; d < 4; ++d)
                        ldg_v<T, TEF>(fg[s2][d], P.fgeo + (size_t)(d * NFQT + f * NFQ + fq) * S + kblk + e0);
                }
                T mM[TFQ][FLD][TEF], mP[TFQ][FLD][TEF];
#pragma unroll
                for (int s2 = 0; s2 < TFQ; ++s2)
#pragma unroll
                    for (int c = 0; c < FLD; ++c)
#pragma unroll
                        for (int t = 0; t < TEF; ++t) { mM[s2][c][t] = T(0); mP[s2][c][t] = T(0); }
#pragma unroll 3
                for (int i = 0; i < NFP; ++i) {
                    T v[TFQ];
                    ldv<T, TFQ>(v, sVfi + i * C::NFQP + fq0);
                    const int node = sFmask[f * NFP + i];
#pragma unroll
                    for (int c = 0; c < FLD; ++c) {
                        T xm[TEF], xp[TEF];
                        ldv<T, TEF>(xm, sQ + (c * NPP + node) * KB + e0);
                        ldv<T, TEF>(xp, cur + (c * NFP + i) * KB + e0);
#pragma unroll
                        for (int s2 = 0; s2 < TFQ; ++s2)
#pragma unroll
                            for (int t = 0; t < TEF; ++t) {
                                mM[s2][c][t] = fma(v[s2], xm[t], mM[s2][c][t]);
                                mP[s2][c][t] = fma(v[s2], xp[t], mP[s2][c][t]);
                            }
                    }
                }
#pragma unroll
                for (int s2 = 0; s2 < TFQ; ++s2) {
                    const int fq = fq0 + s2;
                    if (fq < NFQ) {
                        T g[FLD][TEF];
#pragma unroll
                        for (int t = 0; t < TEF; ++t) {
                            const T n0 = fg[s2][0][t], n1 = fg[s2][1][t], n2 = fg[s2][2][t], sJh = fg[s2][3][t];
                            const T dp = mP[s2][0][t] - mM[s2][0][t];
                            const T dUn = (mP[s2][1][t] - mM[s2][1][t]) * n0 + (mP[s2][2][t] - mM[s2][2][t]) * n1 +
                                          (mP[s2][3][t] - mM[s2][3][t]) * n2;
                            const T avg = (mP[s2][1][t] + mM[s2][1][t]) * n0 + (mP[s2][2][t] + mM[s2][2][t]) * n1 +
                                          (mP[s2][3][t] + mM[s2][3][t]) * n2;
                            const T fp = avg - tau_p * dp;
                            const T fu = dp - tau_u * dUn;
                            g[0][t] = fp * sJh;
                            g[1][t] = fu * (sJh * n0);
                            g[2][t] = fu * (sJh * n1);
                            g[3][t] = fu * (sJh * n2);
                        }
#pragma unroll
                        for (int c = 0; c < FLD; ++c) stv<T, TEF>(sG + (c * NFQ + fq) * KB + e0, g[c]);
                    }
                }
            }
        }
        __syncthreads();
        mbar_wait(bar, ld.phase);
        ld.phase ^= 1u;
        // lift: r_c -= Pf_f g_c
#pragma unroll
        for (int sl = 0; sl < C::SLOTS; ++sl) {
            const int tile = tid + sl * NTF;
            if (tile < C::TILES_B) {
                const int e0 = (tile % C::EG2) * TE2, j0 = (tile / C::EG2) * TJ;
WADG_KUNROLL
                for (int fq = 0; fq < NFQ; ++fq) {
                    T L[TJ];
                    ldv<T, TJ>(L, sLift + fq * NPP + j0);
#pragma unroll
                    for (int c = 0; c < FLD; ++c) {
                        T g[TE2];
                        ldv<T, TE2>(g, sG + (c * NFQ + fq) * KB + e0);
#pragma unroll
                        for (int t = 0; t < TE2; ++t)
#pragma unroll
                            for (int u = 0; u < TJ; ++u) acc[sl][c][t][u] = fma(-L[u], g[t], acc[sl][c][t][u]);
                    }
                }
            }
        }
        __syncthreads();
    }

    // ======================= WADG update + LSRK ===========================
    __syncthreads();
    WADG_PROF_MARK(4);
#pragma unroll
    for (int sl = 0; sl < C::SLOTS; ++sl) {
        const int tile = tid + sl * NTF;
        if (tile < C::TILES_B) {
            const int e0 = (tile % C::EG2) * TE2, j0 = (tile / C::EG2) * TJ;
#pragma unroll
            for (int c = 0; c < FLD; ++c)
#pragma unroll
                for (int u = 0; u < TJ; ++u) {
                    T v[TE2];
#pragma unroll
                    for (int t = 0; t < TE2; ++t) { v[t] = acc[sl][c][t][u]; acc[sl][c][t][u] = T(0); }
                    stv<T, TE2>(sR + (c * NPP + j0 + u) * KB + e0, v);
                }
        }
    }
    for (int ch = 0; ch < C::NCH; ++ch) {
        ld.load2(sU1, P.opU1 + (size_t)ch * NPP * QC, (uint32_t)C::S_U1,
                 sU2, P.opU2 + (size_t)ch * QC * NPP, (uint32_t)C::S_U2);
        for (int tile = tid; tile < C::TILES_A; tile += NTF) {
            const int te = tile % (KB / TE), tq = tile / (KB / TE);
            const int e0 = te * TE, q0 = tq * TQ;
            T z[FLD][TE][TQ];
#pragma unroll
            for (int c = 0; c < FLD; ++c)
#pragma unroll
                for (int t = 0; t < TE; ++t)
#pragma unroll
                    for (int s = 0; s < TQ; ++s) z[c][t][s] = T(0);
WADG_KUNROLL
            for (int j = 0; j < NPP; ++j) {
                T o[TQ];
                ldv<T, TQ>(o, sU1 + j * QC + q0);
#pragma unroll
                for (int c = 0; c < FLD; ++c) {
                    T x[TE];
                    ldv<T, TE>(x, sR + (c * NPP + j) * KB + e0);
#pragma unroll
                    for (int t = 0; t < TE; ++t)
#pragma unroll
                        for (int s = 0; s < TQ; ++s) z[c][t][s] = fma(o[s], x[t], z[c][t][s]);
                }
            }
#pragma unroll
            for (int s = 0; s < TQ; ++s) {
                const int q = ch * QC + q0 + s;
                T wu[TE], wpv[TE];
                if (q < NQ) {
                    ldg_v<T, TE>(wu, P.wu + (size_t)q * S + kblk + e0);
                    if (P.wp) {
                        ldg_v<T, TE>(wpv, P.wp + (size_t)q * S + kblk + e0);
                    } else {
#pragma unroll
                        for (int t = 0; t < TE; ++t) wpv[t] = P.c2 * wu[t];
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < TE; ++t) { wu[t] = T(0); wpv[t] = T(0); }
                }
                T v[TE];
#pragma unroll
                for (int t = 0; t < TE; ++t) v[t] = wpv[t] * z[0][t][s];
                stv<T, TE>(sW2 + (0 * QC + q0 + s) * KB + e0, v);
#pragma unroll
                for (int c = 1; c < FLD; ++c) {
#pragma unroll
                    for (int t = 0; t < TE; ++t) v[t] = wu[t] * z[c][t][s];
                    stv<T, TE>(sW2 + (c * QC + q0 + s) * KB + e0, v);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int sl = 0; sl < C::SLOTS; ++sl) {
            const int tile = tid + sl * NTF;
            if (tile < C::TILES_B) {
                const int e0 = (tile % C::EG2) * TE2, j0 = (tile / C::EG2) * TJ;
WADG_KUNROLL
                for (int qq = 0; qq < QC; ++qq) {
                    T o[TJ];
                    ldv<T, TJ>(o, sU2 + qq * NPP + j0);
#pragma unroll
                    for (int c = 0; c < FLD; ++c) {
                        T w[TE2];
                        ldv<T, TE2>(w, sW2 + (c * QC + qq) * KB + e0);
#pragma unroll
                        for (int t = 0; t < TE2; ++t)
#pragma unroll
                            for (int u = 0; u < TJ; ++u) acc[sl][c][t][u] = fma(o[u], w[t], acc[sl][c][t][u]);
                    }
                }
            }
        }
    }
    __syncthreads();
    WADG_PROF_MARK(5);
    // res = a res + dt Minv(rhs); Q_out = Q_in + b res
#pragma unroll
    for (int sl = 0; sl < C::SLOTS; ++sl) {
        const int tile = tid + sl * NTF;
        if (tile < C::TILES_B) {
            const int e0 = (tile % C::EG2) * TE2, j0 = (tile / C::EG2) * TJ;
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                // the field's old res values are all loaded before its first store
                T rold[TJ][TE2];
#pragma unroll
                for (int u = 0; u < TJ; ++u) {
                    const int j = j0 + u;
#pragma unroll
                    for (int t = 0; t < TE2; ++t)
                        rold[u][t] = (a_rk != T(0) && j < NP) ? __ldg(res + (size_t)(c * NP + j) * S + kblk + e0 + t)
                                                             : T(0);
                }
#pragma unroll
                for (int u = 0; u < TJ; ++u) {
                    const int j = j0 + u;
                    if (j < NP) {
                        const size_t o = (size_t)(c * NP + j) * S + kblk + e0;
                        T r[TE2], q[TE2], qi[TE2];
#pragma unroll
                        for (int t = 0; t < TE2; ++t) r[t] = a_rk * rold[u][t] + dt * acc[sl][c][t][u];
                        ldv<T, TE2>(qi, sQ + (c * NPP + j) * KB + e0);
#pragma unroll
                        for (int t = 0; t < TE2; ++t) q[t] = qi[t] + b_rk * r[t];
                        stv<T, TE2>(res + o, r);
                        stv<T, TE2>(Qout + o, q);
                    }
                }
            }
        }
    }
    __syncthreads();
    WADG_PROF_MARK(6);
}

}  // namespace fused
}  // namespace wadg
