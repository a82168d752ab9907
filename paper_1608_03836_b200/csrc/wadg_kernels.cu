// B200 (sm_100a) kernels for the WADG right-hand side and LSRK45 stage.
//
// Execution model (all kernels): one CTA owns KB = 32 consecutive elements;
// lane e of every warp is element e of the block, warp g walks operator rows
// g, g+NG, ...  Per-element arrays are stored element-fastest, so each warp
// access to a per-element row is one coalesced 128 B (fp32) / 256 B (fp64)
// transaction, and every operator entry a warp needs is warp-uniform (one
// broadcast through L1).  Element fields are staged once in shared memory;
// quadrature-point intermediates go through a chunked shared-memory scratch
// so any N (1..7) fits.  Register accumulators hold each thread's output rows.
//
// Reference counterparts (R/pkg/src/wadg/):
//   k_volume  <- solver._volume_terms      solver.py:241-265
//   k_surface <- solver._surface_terms     solver.py:207-238 (+ face_traces :195-201)
//   k_update  <- solver.apply_mass_inverse / operators.apply_weight_adjusted_inverse
//                fused with the lsrk_step axpy (solver.py:290-301, 348-363)
//   k_energy  <- solver.energy             solver.py:314-321

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "wadg_b200.h"

namespace wadg {
}
#include "wadg_fused.cuh"
#include "wadg_umma.cuh"
#include "wadg_fused_umma.cuh"
#include "wadg_fused_dmma.cuh"
#include "wadg_fused_tmma.cuh"
#include "wadg_fused_reg.cuh"

namespace wadg {

constexpr int KB = WADG_ELEMS_PER_BLOCK;
constexpr int NT = 256;
constexpr int NG = NT / KB;

template <typename T>
struct Prob {
    int K, Kpad, Np, Nq, Nqu, Nf, Nfp, Nfq, nor;
    const T *Vq, *Dq, *Pq, *DTW, *Vu, *Pu, *Vfi, *Pf;
    const int32_t *fmask, *ext_node, *fperm;
    const T *geo, *fgeo, *wu, *wp;
    T c2;
    const int32_t *nbr, *ncode;
    const T *halo;
    int n_halo;
    int Ne;
    const T *Ve, *we, *ewp, *ewu;
    int e_recip;
};

template <typename T>
Prob<T> make_prob(const wadg_problem &p) {
    Prob<T> q;
    q.K = p.K; q.Kpad = p.Kpad; q.Np = p.Np; q.Nq = p.Nq; q.Nqu = p.Nqu;
    q.Nf = p.Nf; q.Nfp = p.Nfp; q.Nfq = p.Nfq; q.nor = p.n_orient;
    q.Vq = (const T *)p.Vq; q.Dq = (const T *)p.Dq; q.Pq = (const T *)p.Pq;
    q.DTW = (const T *)p.DTW; q.Vu = (const T *)p.Vu; q.Pu = (const T *)p.Pu;
    q.Vfi = (const T *)p.Vfi; q.Pf = (const T *)p.Pf;
    q.fmask = p.fmask; q.ext_node = p.ext_node; q.fperm = p.fperm;
    q.geo = (const T *)p.geo; q.fgeo = (const T *)p.fgeo;
    q.wu = (const T *)p.wu; q.wp = (const T *)p.wp; q.c2 = (T)p.c2;
    q.nbr = p.nbr; q.ncode = p.ncode;
    q.halo = (const T *)p.halo; q.n_halo = p.n_halo;
    q.Ne = p.Ne; q.Ve = (const T *)p.Ve; q.we = (const T *)p.we;
    q.ewp = (const T *)p.ewp; q.ewu = (const T *)p.ewu; q.e_recip = p.e_recip;
    return q;
}

// ---------------------------------------------------------------------------
// Volume term.  Strong-weak (SW): r_u_i = -Pq (sum_a G_ai D_a p),
// r_p = sum_a DTW_a (sum_i G_ai Vq u_i).  Strong: r_p = -Pq (sum_ia G_ai D_a u_i).
template <typename T, int DIM, int RJ, bool SW>
__global__ void __launch_bounds__(NT)
k_volume(const Prob<T> P, const T *__restrict__ Q, T *__restrict__ rhs, int QC) {
    constexpr int FLD = DIM + 1;
    constexpr int NW = SW ? 2 * DIM : DIM + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *sQ = reinterpret_cast<T *>(smem_raw);
    T *sW = sQ + FLD * P.Np * KB;
    const int e = threadIdx.x % KB, g = threadIdx.x / KB;
    const size_t S = P.Kpad;
    const size_t k = (size_t)blockIdx.x * KB + e;
    const int Np = P.Np, Nq = P.Nq;

    for (int r = g; r < FLD * Np; r += NG) sQ[r * KB + e] = Q[(size_t)r * S + k];
    __syncthreads();

    T acc[FLD][RJ];
#pragma unroll
    for (int f = 0; f < FLD; ++f)
#pragma unroll
        for (int r = 0; r < RJ; ++r) acc[f][r] = T(0);

    for (int q0 = 0; q0 < Nq; q0 += QC) {
        const int qn = min(QC, Nq - q0);
        for (int qq = g; qq < qn; qq += NG) {
            const int q = q0 + qq;
            T G[DIM][DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a)
#pragma unroll
                for (int i = 0; i < DIM; ++i)
                    G[a][i] = P.geo[(size_t)((a * DIM + i) * Nq + q) * S + k];
            if (SW) {
                T d[DIM], U[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) { d[a] = T(0); U[a] = T(0); }
                const T *Vrow = P.Vq + (size_t)q * Np;
                const T *Drow = P.Dq + (size_t)q * Np;
#pragma unroll 4
                for (int j = 0; j < Np; ++j) {
                    const T pj = sQ[j * KB + e];
#pragma unroll
                    for (int a = 0; a < DIM; ++a)
                        d[a] = fma(__ldg(Drow + (size_t)a * Nq * Np + j), pj, d[a]);
                    const T vj = __ldg(Vrow + j);
#pragma unroll
                    for (int i = 0; i < DIM; ++i)
                        U[i] = fma(vj, sQ[((1 + i) * Np + j) * KB + e], U[i]);
                }
#pragma unroll
                for (int i = 0; i < DIM; ++i) {
                    T s = T(0);
#pragma unroll
                    for (int a = 0; a < DIM; ++a) s = fma(G[a][i], d[a], s);
                    sW[(i * QC + qq) * KB + e] = s;
                }
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    T s = T(0);
#pragma unroll
                    for (int i = 0; i < DIM; ++i) s = fma(G[a][i], U[i], s);
                    sW[((DIM + a) * QC + qq) * KB + e] = s;
                }
            } else {
                T d[FLD][DIM];
#pragma unroll
                for (int f = 0; f < FLD; ++f)
#pragma unroll
                    for (int a = 0; a < DIM; ++a) d[f][a] = T(0);
                const T *Drow = P.Dq + (size_t)q * Np;
#pragma unroll 2
                for (int j = 0; j < Np; ++j) {
                    T x[FLD];
#pragma unroll
                    for (int f = 0; f < FLD; ++f) x[f] = sQ[(f * Np + j) * KB + e];
#pragma unroll
                    for (int a = 0; a < DIM; ++a) {
                        const T D = __ldg(Drow + (size_t)a * Nq * Np + j);
#pragma unroll
                        for (int f = 0; f < FLD; ++f) d[f][a] = fma(D, x[f], d[f][a]);
                    }
                }
                T div = T(0);
#pragma unroll
                for (int i = 0; i < DIM; ++i) {
                    T s = T(0);
#pragma unroll
                    for (int a = 0; a < DIM; ++a) {
                        s = fma(G[a][i], d[0][a], s);
                        div = fma(G[a][i], d[1 + i][a], div);
                    }
                    sW[(i * QC + qq) * KB + e] = s;
                }
                sW[(DIM * QC + qq) * KB + e] = div;
            }
        }
        __syncthreads();
        for (int qq = 0; qq < qn; ++qq) {
            const int q = q0 + qq;
            T w[NW];
#pragma unroll
            for (int m = 0; m < NW; ++m) w[m] = sW[(m * QC + qq) * KB + e];
#pragma unroll
            for (int r = 0; r < RJ; ++r) {
                const int j = g + r * NG;
                if (j < Np) {
                    const T pv = __ldg(P.Pq + (size_t)j * Nq + q);
#pragma unroll
                    for (int i = 0; i < DIM; ++i) acc[1 + i][r] = fma(-pv, w[i], acc[1 + i][r]);
                    if (SW) {
                        T s = acc[0][r];
#pragma unroll
                        for (int a = 0; a < DIM; ++a)
                            s = fma(__ldg(P.DTW + (size_t)(a * Np + j) * Nq + q), w[DIM + a], s);
                        acc[0][r] = s;
                    } else {
                        acc[0][r] = fma(-pv, w[DIM], acc[0][r]);
                    }
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RJ; ++r) {
        const int j = g + r * NG;
        if (j < Np) {
#pragma unroll
            for (int f = 0; f < FLD; ++f) rhs[(size_t)(f * Np + j) * S + k] = acc[f][r];
        }
    }
}

// ---------------------------------------------------------------------------
// Surface term: nodal face traces (own + neighbour, permuted by orientation,
// Dirichlet mirror p+ = -p-, u+ = u-), interpolation to face quadrature,
// penalty flux, lift with Pf.  One face at a time through shared memory.
template <typename T, int DIM, int RJ, bool SW>
__global__ void __launch_bounds__(NT)
k_surface(const Prob<T> P, const T *__restrict__ Q, T *__restrict__ rhs, T tau_p, T tau_u,
          int accumulate, int block0, int QF) {
    constexpr int FLD = DIM + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int Np = P.Np, Nfp = P.Nfp, Nfq = P.Nfq, Nf = P.Nf, NFQ = Nf * Nfq;
    T *sM = reinterpret_cast<T *>(smem_raw);
    T *sP = sM + FLD * Nfp * KB;
    T *sG = sP + FLD * Nfp * KB;
    const int e = threadIdx.x % KB, g = threadIdx.x / KB;
    const size_t S = P.Kpad;
    const size_t k = (size_t)(block0 + blockIdx.x) * KB + e;

    T acc[FLD][RJ];
#pragma unroll
    for (int f = 0; f < FLD; ++f)
#pragma unroll
        for (int r = 0; r < RJ; ++r) acc[f][r] = T(0);

    for (int f = 0; f < Nf; ++f) {
        const int nb = P.nbr[(size_t)f * S + k];
        const int code = P.ncode[(size_t)f * S + k];
        for (int r = g; r < FLD * Nfp; r += NG) {
            const int fld = r / Nfp, i = r - fld * Nfp;
            const T m = Q[(size_t)(fld * Np + P.fmask[f * Nfp + i]) * S + k];
            T pv;
            if (nb >= 0) {
                pv = Q[(size_t)(fld * Np + P.ext_node[code * Nfp + i]) * S + nb];
            } else if (nb == -1) {
                pv = (fld == 0) ? -m : m;
            } else {
                const int h = -nb - 2, o = code % P.nor;
                pv = P.halo[((size_t)h * FLD + fld) * Nfp + P.fperm[o * Nfp + i]];
            }
            sM[r * KB + e] = m;
            sP[r * KB + e] = pv;
        }
        __syncthreads();
        for (int c0 = 0; c0 < Nfq; c0 += QF) {
            const int cn = min(QF, Nfq - c0);
            for (int cc = g; cc < cn; cc += NG) {
                const int fq = c0 + cc;
                T mM[FLD], mP[FLD];
#pragma unroll
                for (int c = 0; c < FLD; ++c) { mM[c] = T(0); mP[c] = T(0); }
                const T *Vrow = P.Vfi + (size_t)fq * Nfp;
                for (int i = 0; i < Nfp; ++i) {
                    const T v = __ldg(Vrow + i);
#pragma unroll
                    for (int c = 0; c < FLD; ++c) {
                        mM[c] = fma(v, sM[(c * Nfp + i) * KB + e], mM[c]);
                        mP[c] = fma(v, sP[(c * Nfp + i) * KB + e], mP[c]);
                    }
                }
                const int idx = f * Nfq + fq;
                T n[DIM];
#pragma unroll
                for (int d = 0; d < DIM; ++d) n[d] = P.fgeo[(size_t)(d * NFQ + idx) * S + k];
                const T sJh = P.fgeo[(size_t)(DIM * NFQ + idx) * S + k];
                const T dp = mP[0] - mM[0];
                T dUn = T(0), avg = T(0);
#pragma unroll
                for (int d = 0; d < DIM; ++d) {
                    dUn += (mP[1 + d] - mM[1 + d]) * n[d];
                    avg += (mP[1 + d] + mM[1 + d]) * n[d];
                }
                const T fp = (SW ? avg : dUn) - tau_p * dp;
                const T fu = dp - tau_u * dUn;
                sG[cc * KB + e] = fp * sJh;
#pragma unroll
                for (int d = 0; d < DIM; ++d) sG[((1 + d) * QF + cc) * KB + e] = fu * (sJh * n[d]);
            }
            __syncthreads();
            for (int cc = 0; cc < cn; ++cc) {
                T w[FLD];
#pragma unroll
                for (int c = 0; c < FLD; ++c) w[c] = sG[(c * QF + cc) * KB + e];
#pragma unroll
                for (int r = 0; r < RJ; ++r) {
                    const int j = g + r * NG;
                    if (j < Np) {
                        const T pf = __ldg(P.Pf + (size_t)j * NFQ + f * Nfq + c0 + cc);
#pragma unroll
                        for (int c = 0; c < FLD; ++c) acc[c][r] = fma(-pf, w[c], acc[c][r]);
                    }
                }
            }
            __syncthreads();
        }
    }
#pragma unroll
    for (int r = 0; r < RJ; ++r) {
        const int j = g + r * NG;
        if (j < Np) {
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                const size_t o = (size_t)(c * Np + j) * S + k;
                rhs[o] = accumulate ? rhs[o] + acc[c][r] : acc[c][r];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// WADG mass inverse Pu diag(w) Vu per field (w = c^2/J for p, 1/J for u);
// MODE 0: out = result;  MODE 1: res = a res + dt result, Q += b res.
template <typename T, int DIM, int RJ, int MODE>
__global__ void __launch_bounds__(NT)
k_update(const Prob<T> P, const T *__restrict__ rhs, T *__restrict__ out, T *__restrict__ Qo,
         T a, T b, T dt, int QC) {
    constexpr int FLD = DIM + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int Np = P.Np, Nqu = P.Nqu;
    T *sR = reinterpret_cast<T *>(smem_raw);
    T *sZ = sR + FLD * Np * KB;
    const int e = threadIdx.x % KB, g = threadIdx.x / KB;
    const size_t S = P.Kpad;
    const size_t k = (size_t)blockIdx.x * KB + e;

    for (int r = g; r < FLD * Np; r += NG) sR[r * KB + e] = rhs[(size_t)r * S + k];
    __syncthreads();

    T acc[FLD][RJ];
#pragma unroll
    for (int f = 0; f < FLD; ++f)
#pragma unroll
        for (int r = 0; r < RJ; ++r) acc[f][r] = T(0);

    for (int q0 = 0; q0 < Nqu; q0 += QC) {
        const int qn = min(QC, Nqu - q0);
        for (int qq = g; qq < qn; qq += NG) {
            const int q = q0 + qq;
            const T wu = P.wu[(size_t)q * S + k];
            const T wp = P.wp ? P.wp[(size_t)q * S + k] : P.c2 * wu;
            T z[FLD];
#pragma unroll
            for (int c = 0; c < FLD; ++c) z[c] = T(0);
            const T *Vrow = P.Vu + (size_t)q * Np;
#pragma unroll 4
            for (int j = 0; j < Np; ++j) {
                const T v = __ldg(Vrow + j);
#pragma unroll
                for (int c = 0; c < FLD; ++c) z[c] = fma(v, sR[(c * Np + j) * KB + e], z[c]);
            }
            sZ[qq * KB + e] = wp * z[0];
#pragma unroll
            for (int c = 1; c < FLD; ++c) sZ[(c * QC + qq) * KB + e] = wu * z[c];
        }
        __syncthreads();
        for (int qq = 0; qq < qn; ++qq) {
            const int q = q0 + qq;
            T w[FLD];
#pragma unroll
            for (int c = 0; c < FLD; ++c) w[c] = sZ[(c * QC + qq) * KB + e];
#pragma unroll
            for (int r = 0; r < RJ; ++r) {
                const int j = g + r * NG;
                if (j < Np) {
                    const T pu = __ldg(P.Pu + (size_t)j * Nqu + q);
#pragma unroll
                    for (int c = 0; c < FLD; ++c) acc[c][r] = fma(pu, w[c], acc[c][r]);
                }
            }
        }
        __syncthreads();
    }
    if constexpr (MODE == 0) {
#pragma unroll
        for (int r = 0; r < RJ; ++r) {
            const int j = g + r * NG;
            if (j < Np) {
#pragma unroll
                for (int c = 0; c < FLD; ++c) out[(size_t)(c * Np + j) * S + k] = acc[c][r];
            }
        }
        return;
    } else {
    // LSRK: the old res / Q values of one node row (all fields) are loaded
    // before its stores (the stores could alias the loads, so the compiler
    // would otherwise serialise one load-store round trip per value)
#pragma unroll
    for (int r = 0; r < RJ; ++r) {
        const int j = g + r * NG;
        if (j < Np) {
            T ro[FLD], qo[FLD];
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                const size_t o = (size_t)(c * Np + j) * S + k;
                ro[c] = (a != T(0)) ? out[o] : T(0);
                qo[c] = Qo[o];
            }
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                const size_t o = (size_t)(c * Np + j) * S + k;
                const T rr = a * ro[c] + dt * acc[c][r];
                out[o] = rr;
                Qo[o] = qo[c] + b * rr;
            }
        }
    }
    }
}

// ---------------------------------------------------------------------------
template <typename T, int DIM>
__global__ void __launch_bounds__(NT)
k_energy(const Prob<T> P, const T *__restrict__ Q, double *__restrict__ partial) {
    constexpr int FLD = DIM + 1;
    __shared__ double red[NT];
    const int e = threadIdx.x % KB, g = threadIdx.x / KB;
    const size_t S = P.Kpad;
    const size_t k = (size_t)blockIdx.x * KB + e;
    const int Np = P.Np;
    double sum = 0.0;
    for (int q = g; q < P.Ne; q += NG) {
        T v[FLD];
#pragma unroll
        for (int c = 0; c < FLD; ++c) v[c] = T(0);
        for (int j = 0; j < Np; ++j) {
            const T x = __ldg(P.Ve + (size_t)q * Np + j);
#pragma unroll
            for (int c = 0; c < FLD; ++c) v[c] = fma(x, Q[(size_t)(c * Np + j) * S + k], v[c]);
        }
        double uu = 0.0;
#pragma unroll
        for (int c = 1; c < FLD; ++c) uu += (double)v[c] * (double)v[c];
        const double wq = (double)P.we[q];
        const double ap = (double)P.ewp[(size_t)q * S + k], au = (double)P.ewu[(size_t)q * S + k];
        const double pp = (double)v[0] * (double)v[0];
        sum += P.e_recip ? wq * (pp / ap + uu / au) : wq * (pp * ap + uu * au);
    }
    red[threadIdx.x] = sum;
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = 0.5 * red[0];
}

__global__ void k_reduce(const double *__restrict__ partial, int n, double *__restrict__ out) {
    __shared__ double red[1024];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = red[0];
}

template <typename T, int DIM>
__global__ void k_pack_halo(const Prob<T> P, const T *__restrict__ Q, const int32_t *__restrict__ send_k,
                            const int32_t *__restrict__ send_f, int n_send, T *__restrict__ buf) {
    constexpr int FLD = DIM + 1;
    const int Nfp = P.Nfp;
    const int64_t total = (int64_t)n_send * FLD * Nfp;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % Nfp);
        const int fld = (int)((t / Nfp) % FLD);
        const int s = (int)(t / ((int64_t)Nfp * FLD));
        const int node = P.fmask[send_f[s] * Nfp + i];
        buf[t] = Q[(size_t)(fld * P.Np + node) * P.Kpad + send_k[s]];
    }
}

template <typename T>
__global__ void k_axpy(int64_t n, const T *__restrict__ d, T *__restrict__ res, T *__restrict__ Q,
                       T a, T b, T dt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const T rr = (a == T(0)) ? dt * d[i] : a * res[i] + dt * d[i];
        res[i] = rr;
        Q[i] = Q[i] + b * rr;
    }
}

}  // namespace wadg

// ===========================================================================
// C ABI
using namespace wadg;

static thread_local char g_err[512] = "";

static int fail(const char *msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return 1;
}

static int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
        return 2;
    }
    return 0;
}

static int rows_per_thread(int Np) {
    const int rj = (Np + NG - 1) / NG;
    if (rj <= 2) return 2;
    if (rj <= 4) return 4;
    if (rj <= 8) return 8;
    if (rj <= 16) return 16;
    return -1;
}

static int validate(const wadg_problem *P) {
    if (!P) return fail("null problem");
    if (P->dim != 2 && P->dim != 3) return fail("dim must be 2 or 3");
    if (P->dtype != WADG_F64 && P->dtype != WADG_F32) return fail("bad dtype");
    if (P->Kpad % KB != 0 || P->Kpad < P->K) return fail("Kpad must be a multiple of 32 and >= K");
    if (rows_per_thread(P->Np) < 0) return fail("Np too large (max 128)");
    return 0;
}

template <typename KernelT>
static int set_smem(KernelT kern, size_t bytes) {
    if (bytes > 227 * 1024) return fail("shared-memory requirement exceeds 227 KB");
    if (bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return fail(cudaGetErrorString(e));
    }
    return 0;
}

// quadrature chunk: multiple of NG, bounded by the shared-memory budget
static int pick_qc(int nq, size_t fixed_bytes, size_t per_q_bytes) {
    int qc = ((nq + NG - 1) / NG) * NG;
    if (qc > 64) qc = 64;
    while (qc > NG && fixed_bytes + per_q_bytes * qc > 96 * 1024) qc -= NG;
    return qc;
}

template <typename T, int DIM, int RJ>
static int launch_volume(const wadg_problem *Pc, const void *Q, void *rhs, cudaStream_t st) {
    Prob<T> P = make_prob<T>(*Pc);
    constexpr int FLD = DIM + 1;
    const bool sw = Pc->formulation == WADG_STRONG_WEAK;
    const int NW = sw ? 2 * DIM : DIM + 1;
    const size_t fixed = (size_t)FLD * P.Np * KB * sizeof(T);
    const int qc = pick_qc(P.Nq, fixed, (size_t)NW * KB * sizeof(T));
    const size_t smem = fixed + (size_t)NW * qc * KB * sizeof(T);
    const dim3 grid(P.Kpad / KB);
    if (sw) {
        if (set_smem(k_volume<T, DIM, RJ, true>, smem)) return 1;
        k_volume<T, DIM, RJ, true><<<grid, NT, smem, st>>>(P, (const T *)Q, (T *)rhs, qc);
    } else {
        if (set_smem(k_volume<T, DIM, RJ, false>, smem)) return 1;
        k_volume<T, DIM, RJ, false><<<grid, NT, smem, st>>>(P, (const T *)Q, (T *)rhs, qc);
    }
    return check_launch("wadg_volume");
}

template <typename T, int DIM, int RJ>
static int launch_surface(const wadg_problem *Pc, const void *Q, void *rhs, double tp, double tu,
                          int accumulate, int b0, int b1, cudaStream_t st) {
    Prob<T> P = make_prob<T>(*Pc);
    constexpr int FLD = DIM + 1;
    const int nblk = P.Kpad / KB;
    if (b1 < 0 || b1 > nblk) b1 = nblk;
    if (b0 < 0) b0 = 0;
    if (b1 <= b0) return 0;
    const size_t fixed = (size_t)FLD * 2 * P.Nfp * KB * sizeof(T);
    const int qf = pick_qc(P.Nfq, fixed, (size_t)FLD * KB * sizeof(T));
    const size_t smem = fixed + (size_t)FLD * qf * KB * sizeof(T);
    const dim3 grid(b1 - b0);
    if (Pc->formulation == WADG_STRONG_WEAK) {
        if (set_smem(k_surface<T, DIM, RJ, true>, smem)) return 1;
        k_surface<T, DIM, RJ, true><<<grid, NT, smem, st>>>(P, (const T *)Q, (T *)rhs, (T)tp, (T)tu,
                                                            accumulate, b0, qf);
    } else {
        if (set_smem(k_surface<T, DIM, RJ, false>, smem)) return 1;
        k_surface<T, DIM, RJ, false><<<grid, NT, smem, st>>>(P, (const T *)Q, (T *)rhs, (T)tp, (T)tu,
                                                             accumulate, b0, qf);
    }
    return check_launch("wadg_surface");
}

template <typename T, int DIM, int RJ, int MODE>
static int launch_update(const wadg_problem *Pc, const void *rhs, void *out, void *Q, double a,
                         double b, double dt, cudaStream_t st) {
    Prob<T> P = make_prob<T>(*Pc);
    constexpr int FLD = DIM + 1;
    const size_t fixed = (size_t)FLD * P.Np * KB * sizeof(T);
    const int qc = pick_qc(P.Nqu, fixed, (size_t)FLD * KB * sizeof(T));
    const size_t smem = fixed + (size_t)FLD * qc * KB * sizeof(T);
    if (set_smem(k_update<T, DIM, RJ, MODE>, smem)) return 1;
    k_update<T, DIM, RJ, MODE><<<P.Kpad / KB, NT, smem, st>>>(P, (const T *)rhs, (T *)out, (T *)Q,
                                                              (T)a, (T)b, (T)dt, qc);
    return check_launch("wadg_update");
}

// dispatch helpers -----------------------------------------------------------
#define WADG_DISPATCH(P, FN, ...)                                                   \
    do {                                                                            \
        const int rj_ = rows_per_thread((P)->Np);                                   \
        if ((P)->dtype == WADG_F64) {                                               \
            if ((P)->dim == 2) {                                                    \
                switch (rj_) {                                                      \
                    case 2: return FN<double, 2, 2>(__VA_ARGS__);                   \
                    case 4: return FN<double, 2, 4>(__VA_ARGS__);                   \
                    case 8: return FN<double, 2, 8>(__VA_ARGS__);                   \
                    default: return FN<double, 2, 16>(__VA_ARGS__);                 \
                }                                                                   \
            } else {                                                                \
                switch (rj_) {                                                      \
                    case 2: return FN<double, 3, 2>(__VA_ARGS__);                   \
                    case 4: return FN<double, 3, 4>(__VA_ARGS__);                   \
                    case 8: return FN<double, 3, 8>(__VA_ARGS__);                   \
                    default: return FN<double, 3, 16>(__VA_ARGS__);                 \
                }                                                                   \
            }                                                                       \
        } else {                                                                    \
            if ((P)->dim == 2) {                                                    \
                switch (rj_) {                                                      \
                    case 2: return FN<float, 2, 2>(__VA_ARGS__);                    \
                    case 4: return FN<float, 2, 4>(__VA_ARGS__);                    \
                    case 8: return FN<float, 2, 8>(__VA_ARGS__);                    \
                    default: return FN<float, 2, 16>(__VA_ARGS__);                  \
                }                                                                   \
            } else {                                                                \
                switch (rj_) {                                                      \
                    case 2: return FN<float, 3, 2>(__VA_ARGS__);                    \
                    case 4: return FN<float, 3, 4>(__VA_ARGS__);                    \
                    case 8: return FN<float, 3, 8>(__VA_ARGS__);                    \
                    default: return FN<float, 3, 16>(__VA_ARGS__);                  \
                }                                                                   \
            }                                                                       \
        }                                                                           \
    } while (0)

template <typename T, int DIM, int RJ>
static int upd_minv(const wadg_problem *P, const void *rhs, void *out, cudaStream_t st) {
    return launch_update<T, DIM, RJ, 0>(P, rhs, out, nullptr, 0.0, 0.0, 0.0, st);
}
template <typename T, int DIM, int RJ>
static int upd_lsrk(const wadg_problem *P, const void *rhs, void *res, void *Q, double a, double b,
                    double dt, cudaStream_t st) {
    return launch_update<T, DIM, RJ, 1>(P, rhs, res, Q, a, b, dt, st);
}

// ---- ExactCurvedMass comparator -----------------------------------------------
// One thread per element applies the stored dense operator A_k = M_k^-1 Mhat
// (R/.../solver.py:302-306 with the Mhat product folded in at setup):
//   mode 0: out = A rhs;   mode 1: res = a res + dt A rhs, Q += b res.
// Coalesced: element index fastest in A ([j][l][Kpad]), rhs, out and Q.  The
// kernel is bound by reading A: 2 Np^2 words per element (p and u operators),
// the storage the paper's weight-adjusted inverse avoids.
namespace wadg {
template <typename T, int MODE>
__global__ void __launch_bounds__(128) k_dense_minv(int Kpad, int Np, int fld, const T *__restrict__ Ap,
                                                    const T *__restrict__ Au, const T *__restrict__ rhs,
                                                    T *__restrict__ out, T *__restrict__ Q, T a, T b, T dt) {
    const int e = blockIdx.x * 128 + threadIdx.x;
    if (e >= Kpad) return;
    const size_t S = Kpad;
    for (int c = 0; c < fld; ++c) {
        const T *A = c == 0 ? Ap : Au;
        const T *x = rhs + (size_t)c * Np * S + e;
        for (int j = 0; j < Np; ++j) {
            const T *Aj = A + (size_t)j * Np * S + e;
            T acc = 0;
            for (int l = 0; l < Np; ++l) acc += Aj[(size_t)l * S] * x[(size_t)l * S];
            const size_t o = ((size_t)c * Np + j) * S + e;
            if (MODE == 0) {
                out[o] = acc;
            } else {
                const T r = (a == (T)0) ? dt * acc : a * out[o] + dt * acc;
                out[o] = r;
                Q[o] += b * r;
            }
        }
    }
}
}  // namespace wadg

static int dense_minv(const wadg_problem *P, const void *rhs, void *out, void *Q, int mode, double a,
                      double b, double dt, cudaStream_t st) {
    if (!P->minv_u) return fail("minv_p set but minv_u is NULL");
    const dim3 grid((P->Kpad + 127) / 128);
    const int fld = P->dim + 1;
    if (P->dtype == WADG_F64) {
        if (mode == 0)
            wadg::k_dense_minv<double, 0><<<grid, 128, 0, st>>>(P->Kpad, P->Np, fld, (const double *)P->minv_p,
                                                                (const double *)P->minv_u, (const double *)rhs,
                                                                (double *)out, nullptr, 0., 0., 0.);
        else
            wadg::k_dense_minv<double, 1><<<grid, 128, 0, st>>>(P->Kpad, P->Np, fld, (const double *)P->minv_p,
                                                                (const double *)P->minv_u, (const double *)rhs,
                                                                (double *)out, (double *)Q, a, b, dt);
    } else {
        if (mode == 0)
            wadg::k_dense_minv<float, 0><<<grid, 128, 0, st>>>(P->Kpad, P->Np, fld, (const float *)P->minv_p,
                                                               (const float *)P->minv_u, (const float *)rhs,
                                                               (float *)out, nullptr, 0.f, 0.f, 0.f);
        else
            wadg::k_dense_minv<float, 1><<<grid, 128, 0, st>>>(P->Kpad, P->Np, fld, (const float *)P->minv_p,
                                                               (const float *)P->minv_u, (const float *)rhs,
                                                               (float *)out, (float *)Q, (float)a, (float)b,
                                                               (float)dt);
    }
    return check_launch("dense mass inverse");
}

// ---- fused tetrahedral stage -------------------------------------------------
static long long *g_prof = nullptr;   // debug: per-CTA phase clocks of the next fused launches

template <typename T>
static fused::FProb<T> make_fprob(const wadg_problem &p) {
    fused::FProb<T> q;
    q.K = p.K; q.Kpad = p.Kpad;
    q.opVA = (const T *)p.opVA; q.opVB = (const T *)p.opVB; q.opU1 = (const T *)p.opU1;
    q.opU2 = (const T *)p.opU2; q.liftT = (const T *)p.liftT; q.Vfi = (const T *)p.Vfi;
    q.fmask = p.fmask; q.ext_node = p.ext_node; q.fperm = p.fperm;
    q.geo = (const T *)p.geo; q.fgeo = (const T *)p.fgeo; q.wu = (const T *)p.wu;
    q.wp = (const T *)p.wp; q.c2 = (T)p.c2; q.nbr = p.nbr; q.ncode = p.ncode;
    q.halo = (const T *)p.halo; q.nor = p.n_orient;
    q.prof = g_prof;
    q.geo_il = (const T *)p.geo_il; q.fgeo_il = (const T *)p.fgeo_il;
    q.wu_il = (const T *)p.wu_il; q.wp_il = (const T *)p.wp_il;
    q.wbar = (const T *)p.wbar;
    return q;
}

static int g_fused_variant = -1;   // debug override of the packing choice: 0 CUDA-core, 2 tcgen05, 3 DMMA,
                                   // 4 split-TF32 mma.sync, -1 default

// cudaFuncSetAttribute (max dynamic shared memory) is per device: one flag per
// (kernel instantiation, device)
static bool attr_once(bool (&done)[64], const void *fn, size_t smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
    if (!done[dev]) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return false;
        done[dev] = true;
    }
    return true;
}

// tcgen05 (TMEM / TMA) fused stage: fp32, orders whose 128-element tile fits
template <typename T, int N>
static constexpr bool umma_available() {
    if constexpr (sizeof(T) == 4 && N >= 2 && N <= 4) return uk::CfgU<N>::SMEM <= 227 * 1024;
    return false;
}

// default for every order it compiles for: fastest in B200 A/B timings
//
template <typename T, int N>
static bool use_umma() {
    if (!umma_available<T, N>()) return false;
    if (g_fused_variant >= 0) return g_fused_variant == 2;
    return true;
}

// DMMA (FP64 tensor core) fused stage: fp64, N = 2..7 (strong-weak), and the
// strong form at N = 2..5 (its sufficiency rules at N_geo = N)
template <typename T, int N, bool SW = true>
static constexpr bool dmma_available() {
    if constexpr (sizeof(T) == 8 && N >= 2 && N <= (SW ? 7 : 5)) return dk::CfgD<N, SW>::SMEM <= 227 * 1024;
    return false;
}

// default for every order it compiles for (N = 2..7): faster than the DFMA
// tiles at every one in B200 A/B timings
template <typename T, int N, bool SW = true>
static bool use_dmma() {
    if (!dmma_available<T, N, SW>()) return false;
    if (g_fused_variant >= 0) return g_fused_variant == 3;
    return true;
}

// split-TF32 mma.sync fused stage: fp32 at the orders the tcgen05 tile does not fit
// (strong-weak at N = 5..7, below which tcgen05 is faster; the strong form at
// N = 2..5, its only fp32 fused stage)
template <typename T, int N, bool SW = true>
static constexpr bool tmma_available() {
    if constexpr (sizeof(T) == 4 && (SW ? (N >= 5 && N <= 7) : (N >= 2 && N <= 5)))
        return tk::CfgT<N, SW>::SMEM <= 227 * 1024;
    return false;
}

// default for every order it compiles for (N = 5..7): faster than the FFMA
// tiles at each (config-5 mesh: 11.1 -> 13.2, 5.8 -> 8.6, 5.6 -> 7.3 GDOF/s)
template <typename T, int N, bool SW = true>
static bool use_tmma() {
    if (!tmma_available<T, N, SW>()) return false;
    if (g_fused_variant >= 0) return g_fused_variant == 4;
    return true;
}

// thread-per-element register stage (strong-weak, N = 1, 2), both precisions:
// the default at N = 1, faster than the tiled CUDA-core kernel there
//
template <typename T, int N, bool SW = true>
static bool use_reg() {
    // (the strong form at N = 2 on this stage ran level with the mma.sync one in
    // fp32, 16.8 vs 16.5 GDOF/s, and at half the DMMA one in fp64: not offered)
    if constexpr (N > 2 || (!SW && N != 1)) return false;
    if (g_fused_variant >= 0) return g_fused_variant == 5;
    return N == 1;
}

// info[8] = {kind, elems_per_block, qchunk, n_chunks, K-extent over nodes (NPP),
//            quad-chunk row stride, node row stride, padded face points}
template <typename T, int N>
static int fused_cfg(int32_t *info, int64_t *smem, int formulation = WADG_STRONG_WEAK) {
    size_t sm = 0;
    int32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool done = false;
    if (formulation != WADG_STRONG_WEAK) {   // strong form: the DMMA (fp64) or mma.sync tf32 (fp32) stage,
                                             // the register stage at N = 1
        if (use_reg<T, N, false>()) {
            using C = rk::CfgR<N, false>;
            const int32_t w[8] = {5, rk::KB, C::NQ, 1, C::NPS, C::NFPS, C::NP, C::OP_TOTAL};
            if (info)
                for (int i = 0; i < 8; ++i) info[i] = w[i];
            if (smem) *smem = 0;
            return 0;
        }
        if constexpr (tmma_available<T, N, false>()) {
            if (use_tmma<T, N, false>()) {
                using C = tk::CfgT<N, false>;
                const int32_t w[8] = {4, C::KB, C::QC, C::NCH, C::NPP, C::NFPK, C::NFQP, (int32_t)C::OP_TOTAL};
                if (info)
                    for (int i = 0; i < 8; ++i) info[i] = w[i];
                if (smem) *smem = (int64_t)C::SMEM;
                return 0;
            }
        }
        if constexpr (dmma_available<T, N, false>()) {
            if (use_dmma<T, N, false>()) {
                using C = dk::CfgD<N, false>;
                const int32_t w[8] = {3, C::KB, C::QC, C::NCH, C::NPP, C::NFPK, C::NFQP, (int32_t)C::OP_TOTAL};
                if (info)
                    for (int i = 0; i < 8; ++i) info[i] = w[i];
                if (smem) *smem = (int64_t)C::SMEM;
                return 0;
            }
        }
        return 1;
    }
    if constexpr (umma_available<T, N>()) {
        if (use_umma<T, N>()) {
            using C = uk::CfgU<N>;
            const int32_t w[8] = {2, C::ME, C::QC, C::NCH, C::NPK, C::NPN, C::NFPK, C::NFH};
            for (int i = 0; i < 8; ++i) v[i] = w[i];
            sm = C::SMEM;
            done = true;
        }
    }
    if constexpr (dmma_available<T, N>()) {
        if (!done && use_dmma<T, N>()) {
            using C = dk::CfgD<N>;
            const int32_t w[8] = {3, C::KB, C::QC, C::NCH, C::NPP, C::NFPK, C::NFQP, (int32_t)C::OP_TOTAL};
            for (int i = 0; i < 8; ++i) v[i] = w[i];
            sm = C::SMEM;
            done = true;
        }
    }
    if constexpr (tmma_available<T, N>()) {
        if (!done && use_tmma<T, N>()) {
            using C = tk::CfgT<N>;
            const int32_t w[8] = {4, C::KB, C::QC, C::NCH, C::NPP, C::NFPK, C::NFQP, (int32_t)C::OP_TOTAL};
            for (int i = 0; i < 8; ++i) v[i] = w[i];
            sm = C::SMEM;
            done = true;
        }
    }
    if (!done && use_reg<T, N>()) {
        using C = rk::CfgR<N>;
        const int32_t w[8] = {5, rk::KB, C::NQ, 1, C::NPS, C::NFPS, C::NP, C::OP_TOTAL};
        for (int i = 0; i < 8; ++i) v[i] = w[i];
        sm = 0;
        done = true;
    }
    if (!done) {
        using C = fused::Cfg<T, N>;
        const int32_t w[8] = {0, C::KB, C::QC, C::NCH, C::NPP, C::QC, C::NPP, C::NFQ};
        for (int i = 0; i < 8; ++i) v[i] = w[i];
        sm = C::SMEM;
    }
    if (info)
        for (int i = 0; i < 8; ++i) info[i] = v[i];
    if (smem) *smem = (int64_t)sm;
    return sm <= 227 * 1024 ? 0 : 1;
}

template <int N, int LAY>
static int launch_umma_lay(const wadg_problem *Pc, const void *Qin, void *Qout, void *res, double tp,
                           double tu, double a, double b, double dt, int b0, int b1, cudaStream_t st) {
    using C = uk::CfgU<N>;
    if (Pc->Kpad % C::ME) return fail("Kpad must be a multiple of the fused block size");
    if (!Pc->geo_il || !Pc->fgeo_il || !Pc->wu_il || (Pc->wp && !Pc->wp_il))
        return fail("tcgen05 stage needs the block-interleaved geo_il / fgeo_il / wu_il / wp_il");
    const int nblk = Pc->Kpad / C::ME;
    if (b1 < 0 || b1 > nblk) b1 = nblk;
    if (b0 < 0) b0 = 0;
    if (b1 <= b0) return 0;
    static bool attr_set[64] = {};
    if (!attr_once(attr_set, (const void *)uk::k_stage_umma<N, LAY>, C::SMEM))
        return fail("cudaFuncSetAttribute failed for the tcgen05 stage");
    // programmatic dependent launch: consecutive stage kernels on a stream overlap
    // the next one's prologue with this one's tail (the kernel waits on
    // griddepcontrol.wait before touching data the previous kernel wrote)
    // persistent CTAs (one per SM, the tcgen05 tile's shared memory and TMEM
    // allow no more): each loops over tiles b0 + blockIdx.x, + gridDim.x, ...
    static int nsm_dev[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail("cudaGetDevice failed");
    if (!nsm_dev[dev] && cudaDeviceGetAttribute(&nsm_dev[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return fail("cudaDeviceGetAttribute failed");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((C::PERSIST && b1 - b0 > nsm_dev[dev]) ? nsm_dev[dev] : b1 - b0);
    cfg.blockDim = dim3(C::NTH);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, uk::k_stage_umma<N, LAY>, make_fprob<float>(*Pc), (const float *)Qin,
                                       (float *)Qout, (float *)res, (float)tp, (float)tu, (float)a, (float)b,
                                       (float)dt, b0, b1);
    if (e != cudaSuccess) return fail(cudaGetErrorString(e));
    return check_launch("wadg_stage_fused(umma)");
}

template <int N>
static int fused_launch_umma(const wadg_problem *Pc, const void *Qin, void *Qout, void *res, double tp,
                             double tu, double a, double b, double dt, int b0, int b1, int lay, cudaStream_t st) {
    switch (lay) {
        case 0: return launch_umma_lay<N, 0>(Pc, Qin, Qout, res, tp, tu, a, b, dt, b0, b1, st);
        case 1: return launch_umma_lay<N, 1>(Pc, Qin, Qout, res, tp, tu, a, b, dt, b0, b1, st);
        case 2: return launch_umma_lay<N, 2>(Pc, Qin, Qout, res, tp, tu, a, b, dt, b0, b1, st);
        default: return fail("row layout on both Q_in and Q_out is not supported");
    }
}

template <int N, bool SW>
static int launch_dmma(const wadg_problem *Pc, const void *Qin, void *Qout, void *res, double tp, double tu,
                       double a, double b, double dt, int b0, int b1, cudaStream_t st) {
    using C = dk::CfgD<N, SW>;
    if (Pc->Kpad % C::KB) return fail("Kpad must be a multiple of the fused block size");
    const int nblk = Pc->Kpad / C::KB;
    if (b1 < 0 || b1 > nblk) b1 = nblk;
    if (b0 < 0) b0 = 0;
    if (b1 <= b0) return 0;
    static bool attr_set[64] = {};
    if (!attr_once(attr_set, (const void *)dk::k_stage_dmma<N, SW>, C::SMEM))
        return fail("cudaFuncSetAttribute failed for the DMMA stage");
    dk::k_stage_dmma<N, SW><<<b1 - b0, C::NTH, C::SMEM, st>>>(make_fprob<double>(*Pc), (const double *)Qin,
                                                            (double *)Qout, (double *)res, tp, tu, a, b, dt, b0);
    return check_launch("wadg_stage_fused(dmma)");
}

template <int N, bool SW>
static int launch_tmma(const wadg_problem *Pc, const void *Qin, void *Qout, void *res, double tp, double tu,
                       double a, double b, double dt, int b0, int b1, cudaStream_t st) {
    using C = tk::CfgT<N, SW>;
    if (Pc->Kpad % C::KB) return fail("Kpad must be a multiple of the fused block size");
    const int nblk = Pc->Kpad / C::KB;
    if (b1 < 0 || b1 > nblk) b1 = nblk;
    if (b0 < 0) b0 = 0;
    if (b1 <= b0) return 0;
    static bool attr_set[64] = {};
    if (!attr_once(attr_set, (const void *)tk::k_stage_tmma<N, SW>, C::SMEM))
        return fail("cudaFuncSetAttribute failed for the split-TF32 mma.sync stage");
    tk::k_stage_tmma<N, SW><<<b1 - b0, C::NTH, C::SMEM, st>>>(make_fprob<float>(*Pc), (const float *)Qin, (float *)Qout,
                                                         (float *)res, (float)tp, (float)tu, (float)a, (float)b,
                                                         (float)dt, b0);
    return check_launch("wadg_stage_fused(tmma)");
}

template <typename T, int N>
static int fused_launch(const wadg_problem *Pc, const void *Qin, void *Qout, void *res, double tp,
                        double tu, double a, double b, double dt, int b0, int b1, int lay, cudaStream_t st) {
    // dispatch on the kernel kind the operators were packed for (P->fused_kind),
    // not on the current packing preference
    if (Pc->fused_kind == 2) {
        if constexpr (umma_available<T, N>())
            return fused_launch_umma<N>(Pc, Qin, Qout, res, tp, tu, a, b, dt, b0, b1, lay, st);
        return fail("operators packed for the tcgen05 stage, which is not compiled for this dtype / order");
    }
    if (Pc->fused_kind == 3) {
        if (lay) return fail("row-layout fields need the tcgen05 stage (fp32, N = 2..4)");
        if (Pc->formulation == WADG_STRONG_WEAK) {
            if constexpr (dmma_available<T, N, true>())
                return launch_dmma<N, true>(Pc, Qin, Qout, res, tp, tu, a, b, dt, b0, b1, st);
        } else {
            if constexpr (dmma_available<T, N, false>())
                return launch_dmma<N, false>(Pc, Qin, Qout, res, tp, tu, a, b, dt, b0, b1, st);
        }
        return fail("operators packed for the DMMA stage, which is not compiled for this dtype / order / form");
    }
    if (Pc->fused_kind == 4) {
        if (lay) return fail("row-layout fields need the tcgen05 stage (fp32, N = 2..4)");
        if (Pc->formulation == WADG_STRONG_WEAK) {
            if constexpr (tmma_available<T, N, true>())
                return launch_tmma<N, true>(Pc, Qin, Qout, res, tp, tu, a, b, dt, b0, b1, st);
        } else {
            if constexpr (tmma_available<T, N, false>())
                return launch_tmma<N, false>(Pc, Qin, Qout, res, tp, tu, a, b, dt, b0, b1, st);
        }
        return fail("operators packed for the split-TF32 mma.sync stage, which is not compiled for this dtype / order / form");
    }
    if (Pc->fused_kind == 5) {
        if constexpr (N <= 2) {
            if (lay) return fail("row-layout fields need the tcgen05 stage (fp32, N = 2..4)");
            if (Pc->Kpad % rk::KB) return fail("Kpad must be a multiple of the fused block size");
            const int nblk = Pc->Kpad / rk::KB;
            if (b1 < 0 || b1 > nblk) b1 = nblk;
            if (b0 < 0) b0 = 0;
            if (b1 <= b0) return 0;
            if (Pc->formulation == WADG_STRONG_WEAK) {
                rk::k_stage_reg<T, N, true><<<b1 - b0, rk::KB, 0, st>>>(
                    make_fprob<T>(*Pc), (const T *)Qin, (T *)Qout, (T *)res, (T)tp, (T)tu, (T)a, (T)b, (T)dt, b0);
            } else {
                if constexpr (N != 1) return fail("the register stage's strong form is compiled for N = 1 only");
                rk::k_stage_reg<T, 1, false><<<b1 - b0, rk::KB, 0, st>>>(
                    make_fprob<T>(*Pc), (const T *)Qin, (T *)Qout, (T *)res, (T)tp, (T)tu, (T)a, (T)b, (T)dt, b0);
            }
            return check_launch("wadg_stage_fused(register stage)");
        }
        return fail("operators packed for the register stage, which is compiled for N = 1, 2 only");
    }
    if (Pc->fused_kind != 0) return fail("unknown fused_kind");
    if (lay) return fail("row-layout fields need the tcgen05 stage (fp32, N = 2..4)");
    using C = fused::Cfg<T, N>;
    if (C::SMEM > 227 * 1024) return fail("fused stage does not fit shared memory for this order");
    if (Pc->Kpad % C::KB) return fail("Kpad must be a multiple of the fused block size");
    const int nblk = Pc->Kpad / C::KB;
    if (b1 < 0 || b1 > nblk) b1 = nblk;
    if (b0 < 0) b0 = 0;
    if (b1 <= b0) return 0;
    static bool attr_set[64] = {};
    if (!attr_once(attr_set, (const void *)fused::k_stage_fused<T, N>, C::SMEM))
        return fail("cudaFuncSetAttribute failed for the fused stage");
    fused::k_stage_fused<T, N><<<b1 - b0, fused::NTF, C::SMEM, st>>>(
        make_fprob<T>(*Pc), (const T *)Qin, (T *)Qout, (T *)res, (T)tp, (T)tu, (T)a, (T)b, (T)dt, b0);
    return check_launch("wadg_stage_fused");
}

#define WADG_FUSED_SWITCH(T, N, FN, ...)          \
    switch (N) {                                  \
        case 1: return FN<T, 1>(__VA_ARGS__);     \
        case 2: return FN<T, 2>(__VA_ARGS__);     \
        case 3: return FN<T, 3>(__VA_ARGS__);     \
        case 4: return FN<T, 4>(__VA_ARGS__);     \
        case 5: return FN<T, 5>(__VA_ARGS__);     \
        case 6: return FN<T, 6>(__VA_ARGS__);     \
        case 7: return FN<T, 7>(__VA_ARGS__);     \
        default: return fail("fused stage compiled for N = 1..7 only"); \
    }

// host row layout (fld, K, Np) <-> device field layout (fld, Np, Kpad) for
// elements [k0, k1): 32 x 32 tiles through shared memory, both sides coalesced
namespace wadg {
// one CTA per 32 elements of one field: the 32 x Np block is one contiguous run
// in the row layout and Np runs of 32 elements in the field layout; both sides
// are read / written linearly (no partly idle node tiles when Np % 32 != 0)
template <typename T, bool TO_FIELDS>
__global__ void __launch_bounds__(256) k_rows_fields(const T *__restrict__ src, T *__restrict__ dst, int K, int Kpad,
                                                      int Np, int k0, int k1) {
    extern __shared__ __align__(16) unsigned char tile_raw[];
    T *tile = reinterpret_cast<T *>(tile_raw);          // [32][Np + 1]
    const int f = blockIdx.y, kb = k0 + 32 * blockIdx.x;
    const int ne = min(32, k1 - kb);
    const size_t rows = (size_t)f * K * Np, flds = (size_t)f * Np * Kpad;
    const int NS = Np + 1;
    if (TO_FIELDS) {
        const T *s0 = src + rows + (size_t)kb * Np;
        for (int t = threadIdx.x; t < ne * Np; t += blockDim.x) {
            const int el = t / Np, j = t - el * Np;
            tile[el * NS + j] = s0[t];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < Np * 32; t += blockDim.x) {
            const int j = t >> 5, el = t & 31;
            if (el < ne) dst[flds + (size_t)j * Kpad + kb + el] = tile[el * NS + j];
        }
    } else {
        for (int t = threadIdx.x; t < Np * 32; t += blockDim.x) {
            const int j = t >> 5, el = t & 31;
            if (el < ne) tile[el * NS + j] = src[flds + (size_t)j * Kpad + kb + el];
        }
        __syncthreads();
        T *d0 = dst + rows + (size_t)kb * Np;
        for (int t = threadIdx.x; t < ne * Np; t += blockDim.x) {
            const int el = t / Np, j = t - el * Np;
            d0[t] = tile[el * NS + j];
        }
    }
}
}  // namespace wadg

template <bool TO_FIELDS>
static int rows_fields(const wadg_problem *P, const void *src, void *dst, int k0, int k1, cudaStream_t st) {
    if (validate(P)) return 1;
    if (k0 < 0 || k1 > P->K || k0 > k1) return fail("element range outside [0, K]");
    if (k0 == k1) return 0;
    const dim3 grid((k1 - k0 + 31) / 32, P->dim + 1);
    const size_t smem = (size_t)32 * (P->Np + 1) * (P->dtype == WADG_F64 ? 8 : 4);
    if (P->dtype == WADG_F64)
        wadg::k_rows_fields<double, TO_FIELDS><<<grid, 256, smem, st>>>((const double *)src, (double *)dst, P->K,
                                                                        P->Kpad, P->Np, k0, k1);
    else
        wadg::k_rows_fields<float, TO_FIELDS><<<grid, 256, smem, st>>>((const float *)src, (float *)dst, P->K,
                                                                       P->Kpad, P->Np, k0, k1);
    return check_launch(TO_FIELDS ? "wadg_rows_to_fields" : "wadg_fields_to_rows");
}

extern "C" {

int wadg_abi_version(void) { return WADG_ABI_VERSION; }

const char *wadg_last_error(void) { return g_err; }

int wadg_volume(const wadg_problem *P, const void *Q, void *rhs, void *stream) {
    if (validate(P)) return 1;
    WADG_DISPATCH(P, launch_volume, P, Q, rhs, (cudaStream_t)stream);
}

int wadg_surface(const wadg_problem *P, const void *Q, void *rhs, double tau_p, double tau_u,
                 int accumulate, int block_begin, int block_end, void *stream) {
    if (validate(P)) return 1;
    if (P->n_halo > 0 && !P->halo) return fail("n_halo > 0 but halo is NULL");
    WADG_DISPATCH(P, launch_surface, P, Q, rhs, tau_p, tau_u, accumulate, block_begin, block_end,
                  (cudaStream_t)stream);
}

int wadg_mass_inverse(const wadg_problem *P, const void *rhs, void *out, void *stream) {
    if (validate(P)) return 1;
    if (P->minv_p) return dense_minv(P, rhs, out, nullptr, 0, 0, 0, 0, (cudaStream_t)stream);
    WADG_DISPATCH(P, upd_minv, P, rhs, out, (cudaStream_t)stream);
}

int wadg_update_lsrk(const wadg_problem *P, const void *rhs, void *res, void *Q, double a, double b,
                     double dt, void *stream) {
    if (validate(P)) return 1;
    if (P->minv_p) return dense_minv(P, rhs, res, Q, 1, a, b, dt, (cudaStream_t)stream);
    WADG_DISPATCH(P, upd_lsrk, P, rhs, res, Q, a, b, dt, (cudaStream_t)stream);
}

int wadg_stage(const wadg_problem *P, void *Q, void *res, void *rhs, double tau_p, double tau_u,
               double a, double b, double dt, void *stream) {
    int rc = wadg_volume(P, Q, rhs, stream);
    if (rc) return rc;
    rc = wadg_surface(P, Q, rhs, tau_p, tau_u, 1, 0, -1, stream);
    if (rc) return rc;
    return wadg_update_lsrk(P, rhs, res, Q, a, b, dt, stream);
}

int wadg_lsrk_axpy(int dtype, int64_t n, const void *d, void *res, void *Q, double a, double b,
                   double dt, void *stream) {
    const int threads = 256;
    int64_t blocks = (n + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    if (dtype == WADG_F64)
        k_axpy<double><<<(int)blocks, threads, 0, (cudaStream_t)stream>>>(
            n, (const double *)d, (double *)res, (double *)Q, a, b, dt);
    else if (dtype == WADG_F32)
        k_axpy<float><<<(int)blocks, threads, 0, (cudaStream_t)stream>>>(
            n, (const float *)d, (float *)res, (float *)Q, (float)a, (float)b, (float)dt);
    else
        return fail("bad dtype");
    return check_launch("wadg_lsrk_axpy");
}

int wadg_energy(const wadg_problem *P, const void *Q, double *partials, double *out_dev, void *stream) {
    if (validate(P)) return 1;
    if (!P->Ve || !P->we || !P->ewp || !P->ewu) return fail("energy quadrature data missing");
    const int nblk = P->Kpad / KB;
    cudaStream_t st = (cudaStream_t)stream;
    if (P->dtype == WADG_F64) {
        if (P->dim == 2) k_energy<double, 2><<<nblk, NT, 0, st>>>(make_prob<double>(*P), (const double *)Q, partials);
        else k_energy<double, 3><<<nblk, NT, 0, st>>>(make_prob<double>(*P), (const double *)Q, partials);
    } else {
        if (P->dim == 2) k_energy<float, 2><<<nblk, NT, 0, st>>>(make_prob<float>(*P), (const float *)Q, partials);
        else k_energy<float, 3><<<nblk, NT, 0, st>>>(make_prob<float>(*P), (const float *)Q, partials);
    }
    if (check_launch("wadg_energy")) return 2;
    k_reduce<<<1, 1024, 0, st>>>(partials, nblk, out_dev);
    return check_launch("wadg_energy_reduce");
}

int wadg_pack_halo(const wadg_problem *P, const void *Q, const int32_t *send_k, const int32_t *send_f,
                   int32_t n_send, void *buf, void *stream) {
    if (validate(P)) return 1;
    if (n_send <= 0) return 0;
    const int64_t total = (int64_t)n_send * (P->dim + 1) * P->Nfp;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    cudaStream_t st = (cudaStream_t)stream;
    if (P->dtype == WADG_F64) {
        if (P->dim == 2) k_pack_halo<double, 2><<<blocks, 256, 0, st>>>(make_prob<double>(*P), (const double *)Q, send_k, send_f, n_send, (double *)buf);
        else k_pack_halo<double, 3><<<blocks, 256, 0, st>>>(make_prob<double>(*P), (const double *)Q, send_k, send_f, n_send, (double *)buf);
    } else {
        if (P->dim == 2) k_pack_halo<float, 2><<<blocks, 256, 0, st>>>(make_prob<float>(*P), (const float *)Q, send_k, send_f, n_send, (float *)buf);
        else k_pack_halo<float, 3><<<blocks, 256, 0, st>>>(make_prob<float>(*P), (const float *)Q, send_k, send_f, n_send, (float *)buf);
    }
    return check_launch("wadg_pack_halo");
}

int wadg_rows_to_fields(const wadg_problem *P, const void *rows, int32_t k0, int32_t k1, void *Q, void *stream) {
    return rows_fields<true>(P, rows, Q, k0, k1, (cudaStream_t)stream);
}

int wadg_fields_to_rows(const wadg_problem *P, const void *Q, int32_t k0, int32_t k1, void *rows, void *stream) {
    return rows_fields<false>(P, Q, rows, k0, k1, (cudaStream_t)stream);
}

int wadg_debug_set_phase_clock_buffer(void *buf) {
    g_prof = (long long *)buf;
    return 0;
}

int wadg_debug_set_fused_variant(int variant) {
    if (variant != -1 && variant != 0 && variant != 2 && variant != 3 && variant != 4 && variant != 5)
        return fail("variant must be -1, 0, 2, 3, 4 or 5");
    g_fused_variant = variant;
    return 0;
}

int wadg_fused_config(int dtype, int order, int32_t *info, int64_t *smem) {
    return wadg_fused_config_form(dtype, order, WADG_STRONG_WEAK, info, smem);
}

int wadg_fused_config_form(int dtype, int order, int formulation, int32_t *info, int64_t *smem) {
    if (dtype == WADG_F64) { WADG_FUSED_SWITCH(double, order, fused_cfg, info, smem, formulation); }
    if (dtype == WADG_F32) { WADG_FUSED_SWITCH(float, order, fused_cfg, info, smem, formulation); }
    return fail("bad dtype");
}

static int stage_fused(const wadg_problem *P, const void *Qin, void *Qout, void *res, double tau_p, double tau_u,
                       double a, double b, double dt, int block_begin, int block_end, int lay, void *stream) {
    if (validate(P)) return 1;
    if (P->dim != 3) return fail("fused stage: tetrahedra only");
    if (P->formulation != WADG_STRONG_WEAK && P->fused_kind != 3 && P->fused_kind != 4 && P->fused_kind != 5)
        return fail("fused stage: the strong form runs on the DMMA (fp64), mma.sync tf32 (fp32) or N = 1 register "
                    "stage only");
    if (P->minv_p) return fail("fused stage: WADG mass inverse only (use wadg_stage for ExactCurvedMass)");
    if (!P->opVA || !P->opVB || !P->opU1 || !P->opU2 || !P->liftT) return fail("fused operators not packed");
    if (Qin == Qout) return fail("fused stage needs distinct Q_in / Q_out buffers");
    if (P->n_halo > 0 && !P->halo) return fail("n_halo > 0 but halo is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    if (P->dtype == WADG_F64) {
        WADG_FUSED_SWITCH(double, P->order, fused_launch, P, Qin, Qout, res, tau_p, tau_u, a, b, dt,
                          block_begin, block_end, lay, st);
    }
    WADG_FUSED_SWITCH(float, P->order, fused_launch, P, Qin, Qout, res, tau_p, tau_u, a, b, dt,
                      block_begin, block_end, lay, st);
}

int wadg_stage_fused(const wadg_problem *P, const void *Qin, void *Qout, void *res, double tau_p,
                     double tau_u, double a, double b, double dt, int block_begin, int block_end,
                     void *stream) {
    return stage_fused(P, Qin, Qout, res, tau_p, tau_u, a, b, dt, block_begin, block_end, 0, stream);
}

int wadg_stage_fused_rows(const wadg_problem *P, const void *Qin, void *Qout, void *res, double tau_p,
                          double tau_u, double a, double b, double dt, int block_begin, int block_end,
                          int layout, void *stream) {
    if (layout < 0 || layout > 2) return fail("layout must be 0, 1 or 2");
    return stage_fused(P, Qin, Qout, res, tau_p, tau_u, a, b, dt, block_begin, block_end, layout, stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// FMA-pipe peak microbenchmark (measurement support for the FP roofline):
// every thread runs 16 independent register-operand FMA chains.
namespace wadg {
template <typename T>
__global__ void __launch_bounds__(256) k_fma_peak(const T *__restrict__ in, T *__restrict__ out, int iters) {
    T a[16];
    const T b = in[threadIdx.x & 7], c = in[8 + (threadIdx.x & 7)];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = in[16 + i] + (T)threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == (T)12345.678) out[threadIdx.x] = s;
}
// packed fp32 (FFMA2): 16 independent float2 chains, 4 flops per chain per iteration
__global__ void __launch_bounds__(256) k_ffma2_peak(const float *__restrict__ in, float *__restrict__ out, int iters) {
    float2 a[16];
    const float2 b = make_float2(in[threadIdx.x & 7], in[(threadIdx.x + 1) & 7]);
    const float2 c = make_float2(in[8 + (threadIdx.x & 7)], in[8 + ((threadIdx.x + 3) & 7)]);
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = make_float2(in[16 + i] + threadIdx.x, in[32 + i] - threadIdx.x);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = __ffma2_rn(a[i], b, c);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
    if (s == 12345.678f) out[threadIdx.x] = s;
}
}  // namespace wadg

// dtype WADG_F64 / WADG_F32 (FFMA / DFMA, 2 * 16 * iters flops per thread) or 2 =
// packed fp32 FFMA2 (4 * 16 * iters flops per thread)
extern "C" int wadg_microbench_fma(int dtype, int blocks, int iters, const void *in, void *out, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == 2) {
        wadg::k_ffma2_peak<<<blocks, 256, 0, st>>>((const float *)in, (float *)out, iters);
        return check_launch("wadg_microbench_fma");
    }
    if (dtype == WADG_F64)
        wadg::k_fma_peak<double><<<blocks, 256, 0, st>>>((const double *)in, (double *)out, iters);
    else
        wadg::k_fma_peak<float><<<blocks, 256, 0, st>>>((const float *)in, (float *)out, iters);
    return check_launch("wadg_microbench_fma");
}

// mma.sync m16n8k8 TF32 throughput probe (design input for the split-TF32 question).
namespace wadg {
__global__ void __launch_bounds__(256) k_mma_tf32_peak(const float *__restrict__ in, float *__restrict__ out, int iters) {
    uint32_t a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(in[i + (threadIdx.x & 3)]);
#pragma unroll
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(in[8 + i + (threadIdx.x & 3)]);
    float c[8][4];
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) c[k][i] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    if (s == 12345.678f) out[threadIdx.x] = s;
}
}  // namespace wadg

extern "C" int wadg_microbench_mma_tf32(int blocks, int iters, const void *in, void *out, void *stream) {
    wadg::k_mma_tf32_peak<<<blocks, 256, 0, (cudaStream_t)stream>>>((const float *)in, (float *)out, iters);
    return check_launch("wadg_microbench_mma_tf32");
}

// mma.sync m8n8k4 FP64 (DMMA) throughput probe: 8 independent accumulators per warp
namespace wadg {
__global__ void __launch_bounds__(256) k_dmma_peak(const double *__restrict__ in, double *__restrict__ out, int iters) {
    const double a = in[threadIdx.x & 7], b = in[8 + (threadIdx.x & 7)];
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[k][0]), "+d"(c[k][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}
}  // namespace wadg

extern "C" int wadg_microbench_dmma(int blocks, int iters, const void *in, void *out, void *stream) {
    wadg::k_dmma_peak<<<blocks, 256, 0, (cudaStream_t)stream>>>((const double *)in, (double *)out, iters);
    return check_launch("wadg_microbench_dmma");
}

// Debug / validation of the tcgen05 primitives (wadg_umma.cuh): one CTA of 128
// threads computes C (128 x N) = A (128 x K) B^T, A row-major (128 x K), B
// row-major (N x K), with split-TF32 tcgen05.mma (A_lo B_hi + A_hi B_lo +
// A_hi B_hi).  mode bit 0: hi operands are the raw fp32 values (the tensor core
// ignores the low mantissa bits) instead of masked copies; bit 1: A_lo comes
// from TMEM (TS form) instead of shared memory; bit 2: plain TF32 (one MMA).
namespace wadg {
__global__ void __launch_bounds__(128) k_umma_test(const float *A, const float *B, float *C, int N, int K, int mode) {
    using namespace umma;
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    uint32_t *slot = reinterpret_cast<uint32_t *>(sm + 8);
    float *sA = reinterpret_cast<float *>(sm + 128);
    float *sAlo = sA + 128 * K;
    float *sB = sAlo + 128 * K;
    float *sBlo = sB + 256 * K;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t SBO = (uint32_t)(K / 4) * 128u;
    auto off = [&](int r, int k) { return (int)(((r >> 3) * SBO + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4) / 4); };
    for (int i = tid; i < 128 * K; i += 128) {
        const int r = i / K, k = i % K;
        const float x = A[i];
        sA[off(r, k)] = (mode & 1) ? x : tf32_hi(x);
        sAlo[off(r, k)] = tf32_lo(x);
    }
    for (int i = tid; i < N * K; i += 128) {
        const int r = i / K, k = i % K;
        const float x = B[i];
        sB[off(r, k)] = (mode & 1) ? x : tf32_hi(x);
        sBlo[off(r, k)] = tf32_lo(x);
    }
    if (tid == 0) {
        fused::mbar_init(bar, 1);
    }
    if (warp == 0) tmem_alloc<512>(slot);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = *slot;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    if (mode & 2) {   // A_lo into TMEM columns 256 + k
        for (int k0 = 0; k0 < K; k0 += 8) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = tf32_lo(A[tid * K + k0 + i]);
            st8(tm + lane_base + 256 + k0, v);
        }
        wait_st();
        fence_before();
        __syncthreads();
        fence_after();
    }
    if (tid == 0) {
        const uint32_t id = idesc_tf32(128, N);
        for (int ks = 0; ks < K / 8; ++ks) {
            const uint64_t ah = desc_k(su32(sA) + ks * 256, 128, SBO), al = desc_k(su32(sAlo) + ks * 256, 128, SBO);
            const uint64_t bh = desc_k(su32(sB) + ks * 256, 128, SBO), bl = desc_k(su32(sBlo) + ks * 256, 128, SBO);
            if (mode & 4) {
                mma_ss(tm, ah, bh, id, ks > 0);
            } else {
                if (mode & 2)
                    mma_ts(tm, tm + 256 + ks * 8, bh, id, ks > 0);
                else
                    mma_ss(tm, al, bh, id, ks > 0);
                mma_ss(tm, ah, bl, id, 1);
                mma_ss(tm, ah, bh, id, 1);
            }
        }
        commit(bar);
    }
    mbar_wait_bounded(bar, 0);
    fence_after();
    for (int c0 = 0; c0 < N; c0 += 8) {
        float v[8];
        ld8(tm + lane_base + c0, v);
        wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) C[tid * N + c0 + i] = v[i];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tm);
}
}  // namespace wadg

extern "C" int wadg_debug_umma_test(const void *A, const void *B, void *C, int N, int K, int mode, void *stream) {
    if (N % 8 || N < 8 || N > 256 || K % 8 || K < 8 || K > 64) return fail("umma test: bad N / K");
    const size_t smem = 128 + (size_t)(2 * 128 * K + 2 * 256 * K) * 4;
    cudaFuncSetAttribute(wadg::k_umma_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    wadg::k_umma_test<<<1, 128, smem, (cudaStream_t)stream>>>((const float *)A, (const float *)B, (float *)C, N, K,
                                                              mode);
    return check_launch("wadg_debug_umma_test");
}

// Debug / measurement: tcgen05.mma issue rate from one warp.  CTA of 128 threads;
// warp 0 issues `count` MMAs (M=128, K=8, N=n) back to back on zeroed operands and
// commits; returns clock64 cycles between the first issue and the commit completion.
// mode 0: A from shared memory (SS) via the per-MMA elected wrapper; 1: A from TMEM
// (TS); 2: SS with 8 MMAs per asm block under one elect (descriptor adds in PTX).
namespace wadg {
__global__ void __launch_bounds__(128) k_umma_rate(long long *out, int n, int count, int mode) {
    using namespace umma;
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    uint32_t *slot = reinterpret_cast<uint32_t *>(sm + 8);
    float *sA = reinterpret_cast<float *>(sm + 1024);
    float *sB = sA + 128 * 8;
    for (int i = threadIdx.x; i < 128 * 8 + 256 * 8; i += 128) sA[i] = 0.f;
    const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    if (threadIdx.x == 0) fused::mbar_init(bar, 1);
    if (warp == 0) tmem_alloc<512>(slot);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = *slot;
    if (warp == 0) {
        const uint32_t id = idesc_tf32(128, n);
        const uint64_t da = desc_k(su32(sA), 128, 256), db = desc_k(su32(sB), 128, 256);
        const long long t0 = clock64();
        if (mode == 0) {
            for (int i = 0; i < count; ++i) mma_ss_w(tm, da, db, id, i > 0);
        } else if (mode == 1) {
            for (int i = 0; i < count; ++i) mma_ts_w(tm, tm + 256, db, id, i > 0);
        } else {
            for (int i = 0; i < count; i += 8) {
                asm volatile(
                    "{\n\t.reg .pred e;\n\t.reg .b32 t;\n\t"
                    "elect.sync t|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t}\n" ::"r"(tm),
                    "l"(da), "l"(db), "r"(id)
                    : "memory");
            }
        }
        const long long t1 = clock64();
        commit_w(bar);
        mbar_wait_bounded(bar, 0);
        const long long t2 = clock64();
        if ((threadIdx.x & 31) == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tm);
}
}  // namespace wadg

extern "C" int wadg_debug_umma_rate(void *out, int n, int count, int mode, void *stream) {
    const size_t smem = 1024 + (128 * 8 + 256 * 8) * 4;
    cudaFuncSetAttribute(wadg::k_umma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    wadg::k_umma_rate<<<1, 128, smem, (cudaStream_t)stream>>>((long long *)out, n, count, mode);
    return check_launch("wadg_debug_umma_rate");
}

// Chip-wide tcgen05 kind::tf32 throughput: `blocks` CTAs each issue `count`
// M=128, K=8 MMAs of width n (timed by the caller with CUDA events)
extern "C" int wadg_microbench_umma(int blocks, int n, int count, int mode, void *out, void *stream) {
    const size_t smem = 1024 + (128 * 8 + 256 * 8) * 4;
    cudaFuncSetAttribute(wadg::k_umma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    wadg::k_umma_rate<<<blocks, 128, smem, (cudaStream_t)stream>>>((long long *)out, n, count, mode);
    return check_launch("wadg_microbench_umma");
}
