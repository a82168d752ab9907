// Fused LSRK45 stage for tetrahedra at N = 1, one thread per element, the
// whole stage in registers.  Same algebra as k_stage_fused (strong-weak
// volume, upwind/penalty surface, WADG update and LSRK axpy of
// R/pkg/src/wadg/solver.py:207-301, 348-363; one kernel per stage, Q
// ping-ponged).
//
// At N = 1 an element has 4 nodes, 8 volume and 4 x 4 face quadrature points:
// about 1.7k FMAs against ~0.9 KB (fp32) of HBM traffic, so the stage is
// HBM-bound and the tiled CTA-wide GEMMs of the other stages only add shared-
// memory staging and barriers.  Here every thread owns one element: its
// fields, the exterior face-node values and the right-hand side stay in
// registers, every per-element array is read once with coalesced loads
// (element-fastest layout), and the reference operators (464 values,
// device.n1_operator_image) sit in shared memory, read with warp-uniform
// addresses (broadcast, compile-time offsets).
#pragma once

namespace wadg {
namespace n1 {

constexpr int NP = 4, NQ = 8, NF = 4, NFP = 3, NFQ = 4, NQU = 8, FLD = 4;
constexpr int KB = 128;                                  // elements (threads) per CTA
// operator image offsets (values), device.n1_operator_image
constexpr int O_D = 0;                                   // D_a  [a][q][j]
constexpr int O_VQ = O_D + 3 * NQ * NP;                  // Vq   [q][j]
constexpr int O_DTW = O_VQ + NQ * NP;                    // DTW_a^T [q][a][j]
constexpr int O_PQ = O_DTW + NQ * 3 * NP;                // Pq^T [q][j]
constexpr int O_VF = O_PQ + NQ * NP;                     // own-trace interpolation [f][fq][j]
constexpr int O_VFI = O_VF + NF * NFQ * NP;              // Vfi  [fq][i] (16 slots)
constexpr int O_L = O_VFI + 16;                          // Pf^T [f][fq][j]
constexpr int O_VU = O_L + NF * NFQ * NP;                // Vu   [q][j] (update rule)
constexpr int O_PU = O_VU + NQU * NP;                    // Pu^T [q][j]
constexpr int OP_TOTAL = O_PU + NQU * NP;                // 464

template <typename T>
__global__ void __launch_bounds__(KB, sizeof(T) == 4 ? 4 : 3)
k_stage_n1(const fused::FProb<T> P, const T *__restrict__ Qin, T *__restrict__ Qout, T *__restrict__ res,
           T tau_p, T tau_u, T a_rk, T b_rk, T dt, int block0) {
    __shared__ __align__(16) T sOp[OP_TOTAL];
    __shared__ int32_t sExt[NF * 6 * NFP], sPerm[6 * NFP];
    const int tid = threadIdx.x;
    for (int r = tid; r < OP_TOTAL; r += KB) sOp[r] = __ldg(P.opVA + r);
    for (int r = tid; r < NF * 6 * NFP; r += KB) sExt[r] = __ldg(P.ext_node + r);
    for (int r = tid; r < 6 * NFP; r += KB) sPerm[r] = __ldg(P.fperm + r);
    const size_t S = P.Kpad;
    const size_t k = (size_t)(block0 + blockIdx.x) * KB + tid;
    // the element's fields
    T q[FLD][NP];
#pragma unroll
    for (int c = 0; c < FLD; ++c)
#pragma unroll
        for (int j = 0; j < NP; ++j) q[c][j] = __ldg(Qin + (size_t)(c * NP + j) * S + k);
    // L2 prefetch of every per-element row the stage reads after the fields
    // (factors, face factors, weights, neighbour tables, old res): fire-and-
    // forget, so the whole element's traffic is in flight without registers.
    // fp32 / fp64 at K = 1.57M +19 / +6.5 %; prefetching the neighbours' face
    // nodes as well, which needs the neighbour table first, was 8 % slower.
    {
        // the warp's rows are spread over its lanes: lane l prefetches rows
        // l, l + 32, ... (one 128-byte line per row and 32 elements, two in fp64)
        const int lane = tid & 31;
        const size_t kw = k - lane;
        constexpr int NR = 9 * NQ + 4 * NF * NFQ + 2 * NQU + 2 * NF + FLD * NP;
#pragma unroll 1
        for (int r = lane; r < NR; r += 32) {
            const void *p;
            int t = r;
            if (t < 9 * NQ) p = P.geo + (size_t)t * S + kw;
            else if ((t -= 9 * NQ) < 4 * NF * NFQ) p = P.fgeo + (size_t)t * S + kw;
            else if ((t -= 4 * NF * NFQ) < NQU) p = P.wu + (size_t)t * S + kw;
            else if ((t -= NQU) < NQU) p = P.wp ? P.wp + (size_t)t * S + kw : nullptr;
            else if ((t -= NQU) < NF) p = P.nbr + (size_t)t * S + kw;
            else if ((t -= NF) < NF) p = P.ncode + (size_t)t * S + kw;
            else p = a_rk != T(0) ? res + (size_t)(t - NF) * S + kw : nullptr;
            if (p) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
                if (sizeof(T) == 8) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char *)p + 128));
            }
        }
    }
    __syncthreads();
    T R[FLD][NP];
#pragma unroll
    for (int c = 0; c < FLD; ++c)
#pragma unroll
        for (int j = 0; j < NP; ++j) R[c][j] = T(0);

    // ---- volume: dp_a = D_a p, U_i = Vq u_i; gp_i = sum_a G_ai dp_a,
    // F_a = sum_i G_ai U_i; R_p += sum_a DTW_a F_a, R_u_i -= Pq gp_i
    // (R/pkg/src/wadg/solver.py:241-265, strong-weak).  One point per
    // iteration with the next point's factors in flight (a fully unrolled loop
    // hoists all 72 factor loads and spills). ----
    T G[9], Gn[9];
    auto load_G = [&](T (&g)[9], int qq) {
#pragma unroll
        for (int r = 0; r < 9; ++r) g[r] = __ldg(P.geo + (size_t)(r * NQ + qq) * S + k);
    };
    load_G(G, 0);
#pragma unroll 1
    for (int qq = 0; qq < NQ; ++qq) {
        if (qq + 1 < NQ) load_G(Gn, qq + 1);
        const T *D = sOp + O_D + qq * NP, *Vq = sOp + O_VQ + qq * NP;
        const T *DTW = sOp + O_DTW + qq * 3 * NP, *Pq = sOp + O_PQ + qq * NP;
        T dp[3], U[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            T s = T(0);
#pragma unroll
            for (int j = 0; j < NP; ++j) s = fma(D[a * NQ * NP + j], q[0][j], s);
            dp[a] = s;
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            T s = T(0);
#pragma unroll
            for (int j = 0; j < NP; ++j) s = fma(Vq[j], q[1 + i][j], s);
            U[i] = s;
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const T F = G[a * 3 + 0] * U[0] + G[a * 3 + 1] * U[1] + G[a * 3 + 2] * U[2];
#pragma unroll
            for (int j = 0; j < NP; ++j) R[0][j] = fma(DTW[a * NP + j], F, R[0][j]);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const T gp = G[0 * 3 + i] * dp[0] + G[1 * 3 + i] * dp[1] + G[2 * 3 + i] * dp[2];
#pragma unroll
            for (int j = 0; j < NP; ++j) R[1 + i][j] = fma(-Pq[j], gp, R[1 + i][j]);
        }
#pragma unroll
        for (int r = 0; r < 9; ++r) G[r] = Gn[r];
    }

    // ---- surface: traces at the face points, upwind / penalty flux times
    // sJ/2 (and n_i), lift R_c -= Pf g_c (R/pkg/src/wadg/solver.py:195-238).
    // Per face: the exterior face-node values (neighbour, or halo slot; the
    // mirror BC p+ = -p-, u+ = u- of solver.py:214-217 is applied to the
    // traces) and the face factors, all in flight together ----
    const int NFQT = NF * NFQ;
#pragma unroll 1
    for (int f = 0; f < NF; ++f) {
        const int nb = __ldg(P.nbr + (size_t)f * S + k);
        const int code = __ldg(P.ncode + (size_t)f * S + k);
        T xp[FLD][NFP];
#pragma unroll
        for (int i = 0; i < NFP; ++i)
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                T v = T(0);
                if (nb >= 0)
                    v = __ldg(Qin + (size_t)(c * NP + sExt[code * NFP + i]) * S + nb);
                else if (nb <= -2)
                    v = __ldg(P.halo + ((size_t)(-nb - 2) * FLD + c) * NFP + sPerm[(code % P.nor) * NFP + i]);
                xp[c][i] = v;
            }
        T fg[NFQ][4];
#pragma unroll
        for (int fq = 0; fq < NFQ; ++fq)
#pragma unroll
            for (int d = 0; d < 4; ++d) fg[fq][d] = __ldg(P.fgeo + (size_t)(d * NFQT + f * NFQ + fq) * S + k);
        const bool mirror = nb == -1;
        const T *VF = sOp + O_VF + f * NFQ * NP, *L = sOp + O_L + f * NFQ * NP;
#pragma unroll
        for (int fq = 0; fq < NFQ; ++fq) {
            T m[FLD], x[FLD];
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                T sm = T(0), sx = T(0);
#pragma unroll
                for (int j = 0; j < NP; ++j) sm = fma(VF[fq * NP + j], q[c][j], sm);
#pragma unroll
                for (int i = 0; i < NFP; ++i) sx = fma(sOp[O_VFI + fq * NFP + i], xp[c][i], sx);
                m[c] = sm;
                x[c] = mirror ? (c == 0 ? -sm : sm) : sx;
            }
            const T n0 = fg[fq][0], n1 = fg[fq][1], n2 = fg[fq][2], sJh = fg[fq][3];
            const T djp = x[0] - m[0];
            const T dUn = (x[1] - m[1]) * n0 + (x[2] - m[2]) * n1 + (x[3] - m[3]) * n2;
            const T avg = (x[1] + m[1]) * n0 + (x[2] + m[2]) * n1 + (x[3] + m[3]) * n2;
            const T fpp = avg - tau_p * djp;
            const T fuu = djp - tau_u * dUn;
            const T g[FLD] = {fpp * sJh, fuu * (sJh * n0), fuu * (sJh * n1), fuu * (sJh * n2)};
#pragma unroll
            for (int c = 0; c < FLD; ++c)
#pragma unroll
                for (int j = 0; j < NP; ++j) R[c][j] = fma(-L[fq * NP + j], g[c], R[c][j]);
        }
    }

    // ---- WADG update: R'_c = Pu (omega Vu R_c), omega = c^2/J (p) or 1/J (u)
    // (R/pkg/src/wadg/operators.py:45-61), then the LSRK axpy ----
    T Rn[FLD][NP];
#pragma unroll
    for (int c = 0; c < FLD; ++c)
#pragma unroll
        for (int j = 0; j < NP; ++j) Rn[c][j] = T(0);
    T wun = __ldg(P.wu + k), wpn = P.wp ? __ldg(P.wp + k) : T(0);
#pragma unroll 2
    for (int qq = 0; qq < NQU; ++qq) {
        const T wu = wun, wp = P.wp ? wpn : P.c2 * wu;
        if (qq + 1 < NQU) {
            wun = __ldg(P.wu + (size_t)(qq + 1) * S + k);
            if (P.wp) wpn = __ldg(P.wp + (size_t)(qq + 1) * S + k);
        }
#pragma unroll
        for (int c = 0; c < FLD; ++c) {
            T z = T(0);
#pragma unroll
            for (int j = 0; j < NP; ++j) z = fma(sOp[O_VU + qq * NP + j], R[c][j], z);
            z *= (c == 0 ? wp : wu);
#pragma unroll
            for (int j = 0; j < NP; ++j) Rn[c][j] = fma(sOp[O_PU + qq * NP + j], z, Rn[c][j]);
        }
    }
#pragma unroll
    for (int c = 0; c < FLD; ++c)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const size_t o = (size_t)(c * NP + j) * S + k;
            const T rold = a_rk != T(0) ? __ldg(res + o) : T(0);
            const T r = a_rk * rold + dt * Rn[c][j];
            res[o] = r;
            Qout[o] = q[c][j] + b_rk * r;
        }
}

}  // namespace n1
}  // namespace wadg
