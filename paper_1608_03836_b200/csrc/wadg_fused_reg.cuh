// Fused LSRK45 stage for tetrahedra at low order (the default at N = 1; N = 2
// compiles and is parity-tested, but is slower than the tensor-core stages
// there), one thread per element, the whole stage in registers.  Same algebra as k_stage_fused (strong-weak
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
// device.reg_operator_image) sit in shared memory, read with warp-uniform
// addresses (broadcast, compile-time offsets).
#pragma once

namespace wadg {
namespace rk {

// per-order extents (tetrahedra, strong-weak rules: (N+1)^3 volume and update
// points, (N+1)^2 points per face) and operator image offsets (values; rows
// over nodes padded to NPS = rup(Np, 4) so that 4 consecutive operator values
// are one aligned vector load), device.reg_operator_image
// SW: strong-weak form; otherwise the strong form with the sufficiency rules
// at N_geo = N ((2N-1)^3 volume, (2N)^2 face points; R/PAPER.md:288,294), the
// update on the 2N+1 rule either way
template <int N, bool SW = true>
struct CfgR {
    static constexpr int NP = (N + 1) * (N + 2) * (N + 3) / 6, NPS = fused::rup(NP, 4);
    // strong form: (2N-1)^3 points, but the volume rule is floored at degree 2N
    // (refelem.build_reference_element), which at N = 1 is the 2^3 rule
    static constexpr int NQS1 = N == 1 ? 2 : 2 * N - 1;
    static constexpr int NQ = SW ? (N + 1) * (N + 1) * (N + 1) : NQS1 * NQS1 * NQS1;
    static constexpr int NQU = (N + 1) * (N + 1) * (N + 1);
    static constexpr int NF = 4, NFP = (N + 1) * (N + 2) / 2, NFPS = fused::rup(NFP, 4);
    static constexpr int NFQ = SW ? (N + 1) * (N + 1) : 4 * N * N;
    static constexpr int FLD = 4;
    static constexpr int O_D = 0;                                   // D_a  [a][q][j]
    static constexpr int O_VQ = O_D + 3 * NQ * NPS;                 // Vq   [q][j]
    static constexpr int O_DTW = O_VQ + NQ * NPS;                   // DTW_a^T [q][a][j]
    static constexpr int O_PQ = O_DTW + NQ * 3 * NPS;               // Pq^T [q][j]
    static constexpr int O_VF = O_PQ + NQ * NPS;                    // own-trace interpolation [f][fq][j]
    static constexpr int O_VFI = O_VF + NF * NFQ * NPS;             // Vfi  [fq][i]
    static constexpr int O_L = O_VFI + NFQ * NFPS;                  // Pf^T [f][fq][j]
    static constexpr int O_VU = O_L + NF * NFQ * NPS;               // Vu   [q][j] (update rule)
    static constexpr int O_PU = O_VU + NQU * NPS;                   // Pu^T [q][j]
    static constexpr int OP_TOTAL = O_PU + NQU * NPS;               // 464 at N = 1
};
constexpr int KB = 128;                                  // elements (threads) per CTA
// registers: fp32 N = 1 128 (four CTAs per SM), fp32 N = 2 and fp64 N = 1 168
// (three), fp64 N = 2 255 (two).  At N = 1, five CTAs per SM (96 registers)
// or the field-by-field update of N = 2 were within +-2 % in fp32 and up to
// 12 % slower in fp64 (spills)
template <typename T, int N>
constexpr int minb() { return N == 1 ? (sizeof(T) == 4 ? 4 : 3) : (sizeof(T) == 4 ? 3 : 2); }

template <typename T, int N, bool SW = true>
__global__ void __launch_bounds__(KB, (minb<T, N>()))
k_stage_reg(const fused::FProb<T> P, const T *__restrict__ Qin, T *__restrict__ Qout, T *__restrict__ res,
            T tau_p, T tau_u, T a_rk, T b_rk, T dt, int block0) {
    using C = CfgR<N, SW>;
    constexpr int NP = C::NP, NPS = C::NPS, NQ = C::NQ, NQU = C::NQU, NF = C::NF, NFP = C::NFP, NFPS = C::NFPS;
    constexpr int NFQ = C::NFQ, FLD = C::FLD;
    constexpr int O_D = C::O_D, O_VQ = C::O_VQ, O_DTW = C::O_DTW, O_PQ = C::O_PQ, O_VF = C::O_VF, O_VFI = C::O_VFI;
    constexpr int O_L = C::O_L, O_VU = C::O_VU, O_PU = C::O_PU, OP_TOTAL = C::OP_TOTAL;
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
        const T *D = sOp + O_D + qq * NPS, *Vq = sOp + O_VQ + qq * NPS;
        const T *DTW = sOp + O_DTW + qq * 3 * NPS, *Pq = sOp + O_PQ + qq * NPS;
        if constexpr (!SW) {
            // strong form: du_a,c = D_a Q_c; gp_i = sum_a G_ai du_a,0, div =
            // sum_i sum_a G_ai du_a,i; R_p -= Pq div, R_u_i -= Pq gp_i
            // (R/pkg/src/wadg/solver.py:259-264)
            T du[3][FLD];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int c = 0; c < FLD; ++c) {
                    T s = T(0);
#pragma unroll
                    for (int j = 0; j < NP; ++j) s = fma(D[a * NQ * NPS + j], q[c][j], s);
                    du[a][c] = s;
                }
            T div = T(0);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const T gp = G[0 * 3 + i] * du[0][0] + G[1 * 3 + i] * du[1][0] + G[2 * 3 + i] * du[2][0];
                div += G[0 * 3 + i] * du[0][1 + i] + G[1 * 3 + i] * du[1][1 + i] + G[2 * 3 + i] * du[2][1 + i];
#pragma unroll
                for (int j = 0; j < NP; ++j) R[1 + i][j] = fma(-Pq[j], gp, R[1 + i][j]);
            }
#pragma unroll
            for (int j = 0; j < NP; ++j) R[0][j] = fma(-Pq[j], div, R[0][j]);
        } else {
            T dp[3], U[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                T s = T(0);
#pragma unroll
                for (int j = 0; j < NP; ++j) s = fma(D[a * NQ * NPS + j], q[0][j], s);
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
                for (int j = 0; j < NP; ++j) R[0][j] = fma(DTW[a * NPS + j], F, R[0][j]);
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const T gp = G[0 * 3 + i] * dp[0] + G[1 * 3 + i] * dp[1] + G[2 * 3 + i] * dp[2];
#pragma unroll
                for (int j = 0; j < NP; ++j) R[1 + i][j] = fma(-Pq[j], gp, R[1 + i][j]);
            }
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
        const bool mirror = nb == -1;
        const T *VF = sOp + O_VF + f * NFQ * NPS, *L = sOp + O_L + f * NFQ * NPS;
#pragma unroll (N == 1 ? NFQ : 1)
        for (int fq = 0; fq < NFQ; ++fq) {
            T fg[4];
#pragma unroll
            for (int d = 0; d < 4; ++d) fg[d] = __ldg(P.fgeo + (size_t)(d * NFQT + f * NFQ + fq) * S + k);
            T m[FLD], x[FLD];
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                T sm = T(0), sx = T(0);
#pragma unroll
                for (int j = 0; j < NP; ++j) sm = fma(VF[fq * NPS + j], q[c][j], sm);
#pragma unroll
                for (int i = 0; i < NFP; ++i) sx = fma(sOp[O_VFI + fq * NFPS + i], xp[c][i], sx);
                m[c] = sm;
                x[c] = mirror ? (c == 0 ? -sm : sm) : sx;
            }
            const T n0 = fg[0], n1 = fg[1], n2 = fg[2], sJh = fg[3];
            const T djp = x[0] - m[0];
            const T dUn = (x[1] - m[1]) * n0 + (x[2] - m[2]) * n1 + (x[3] - m[3]) * n2;
            const T avg = (x[1] + m[1]) * n0 + (x[2] + m[2]) * n1 + (x[3] + m[3]) * n2;
            const T fpp = (SW ? avg : dUn) - tau_p * djp;   // strong: [u.n] (solver.py:220-232)
            const T fuu = djp - tau_u * dUn;
            const T g[FLD] = {fpp * sJh, fuu * (sJh * n0), fuu * (sJh * n1), fuu * (sJh * n2)};
#pragma unroll
            for (int c = 0; c < FLD; ++c)
#pragma unroll
                for (int j = 0; j < NP; ++j) R[c][j] = fma(-L[fq * NPS + j], g[c], R[c][j]);
        }
    }

    // ---- WADG update: R'_c = Pu (omega Vu R_c), omega = c^2/J (p) or 1/J (u)
    // (R/pkg/src/wadg/operators.py:45-61), then the LSRK axpy ----
    if constexpr (N == 1) {
        // all fields per point, the next point's weights in flight
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
                for (int j = 0; j < NP; ++j) z = fma(sOp[O_VU + qq * NPS + j], R[c][j], z);
                z *= (c == 0 ? wp : wu);
#pragma unroll
                for (int j = 0; j < NP; ++j) Rn[c][j] = fma(sOp[O_PU + qq * NPS + j], z, Rn[c][j]);
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
    } else {
    // N = 2, field by field: z = Vu R_c at each point, times the weight,
    // projected with Pu into R'_c (only one field's R' live), then the field's
    // LSRK write.  The weight rows are L1 hits after the first field.
#pragma unroll
    for (int c = 0; c < FLD; ++c) {
        const T *wrow = (c == 0 && P.wp) ? P.wp : P.wu;
        const T wsc = (c == 0 && !P.wp) ? P.c2 : T(1);
        T Rn[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) Rn[j] = T(0);
        T wn = __ldg(wrow + k);
#pragma unroll (N == 1 ? 2 : 1)
        for (int qq = 0; qq < NQU; ++qq) {
            const T w = wn * wsc;
            if (qq + 1 < NQU) wn = __ldg(wrow + (size_t)(qq + 1) * S + k);
            T z = T(0);
#pragma unroll
            for (int j = 0; j < NP; ++j) z = fma(sOp[O_VU + qq * NPS + j], R[c][j], z);
            z *= w;
#pragma unroll
            for (int j = 0; j < NP; ++j) Rn[j] = fma(sOp[O_PU + qq * NPS + j], z, Rn[j]);
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const size_t o = (size_t)(c * NP + j) * S + k;
            const T rold = a_rk != T(0) ? __ldg(res + o) : T(0);
            const T r = a_rk * rold + dt * Rn[j];
            res[o] = r;
            Qout[o] = q[c][j] + b_rk * r;
        }
    }
    }
}

}  // namespace rk
}  // namespace wadg
