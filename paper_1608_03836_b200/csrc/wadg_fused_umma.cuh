// Fused LSRK45 stage for fp32 tetrahedra on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM, operators staged by TMA bulk
// copies).  Same algebra as k_stage_fused / k_stage_fused_tc (strong-weak
// volume, upwind/penalty surface, WADG update and LSRK axpy of
// R/pkg/src/wadg/solver.py:207-301, 348-363) in one kernel per stage with Q
// ping-ponged.
//
// Every dense contraction is a CTA-wide GEMM with the 128 elements of the
// CTA as the M dimension (one element per TMEM lane):
//   D[e, n] (+)= sum_k A[e, k] B[n, k]
// A = per-element data (fields, quadrature values, flux), B = a reference
// operator tile.  fp32 accuracy comes from the split x = hi + lo (hi = x with
// the low 13 mantissa bits cleared, lo = x - hi exactly): three MMAs
// A_lo B_hi + A_hi B_lo + A_hi B_hi per product (the dropped A_lo B_lo is
// O(2^-22) relative).  Operator hi/lo images are packed on the host in the
// canonical K-major no-swizzle layout (wadg_umma.cuh) and arrive by one
// cp.async.bulk per tile; per-element A operands are written by the threads,
// either into shared memory (fields, neighbour face nodes) or straight into
// TMEM with tcgen05.st (quadrature values, flux), which is where the
// epilogue thread of an element already holds them.
//
// Phases per CTA (one CTA of 512 threads per SM, TMEM 512 columns):
//   load    Q -> sQ (raw fp32 = tf32 hi operand) and sQlo
//   volume  per 16-point quadrature chunk:
//           V1: dp_a = D_a p (N = 48), U_i = Vq u_i (N = 16 each)        -> TMEM
//           epilogue: gp_i = sum_a G_ai dp_a, F_a = sum_i G_ai U_i       -> TMEM (hi, lo)
//           V2: R_p += sum_a DTW_a F_a, R_u_i += (-Pq) gp_i              -> TMEM R
//   surface per face, per 16-point half of the face rule:
//           own / exterior traces Vfi (own face nodes, gathered neighbour face nodes)
//           epilogue: upwind/penalty flux * sJ/2 (* n_i)                 -> TMEM (hi, lo)
//           lift: R_c += (-Pf) g_c
//   update  per field pair: R_c -> shared (hi, lo); per 32-point chunk
//           z = Vu R_c, omega z (c^2/J or 1/J), R_c (+)= Pu (omega z)
//   LSRK    res = a res + dt R, Q_out = Q_in + b res
#pragma once

namespace wadg {
namespace uk {

// debug: fine-grained clocks of the tcgen05 stage (slots 8..31 of a 32-slot
// per-CTA record in P.prof; phase marks use WADG_PROF_MARK as elsewhere)
#define UMMA_MARK0(slot) UMMA_MARK(slot, threadIdx.x == 0)
#ifdef WADG_MMA_TRACE   // debug build only: MMA-warp timeline marks in slots 6..29
#define MMA_TRACE(slot) UMMA_MARK(slot, threadIdx.x == 16 * 32)
#else
#define MMA_TRACE(slot) do { } while (0)
#endif
#define UMMA_MARK(slot, cond)                                                                  \
    do {                                                                                       \
        if (P.prof && (cond)) P.prof[(blk - (size_t)block0) * 32 + (slot)] = clock64();        \
    } while (0)

using fused::cdiv;
using fused::rup;

template <int N>
struct CfgU {
    static constexpr int NP = fused::np_tet(N);
    static constexpr int NPK = rup(NP, 8);      // K extent over nodes (MMA K step 8)
    static constexpr int NPN = NPK;             // N extent over nodes (M = 128 accepts N % 8 == 0 on sm_100a)
    static constexpr int NQ = (N + 1) * (N + 1) * (N + 1);
    static constexpr int QC = 16, NCH = cdiv(NQ, QC);       // volume quadrature chunks
    static constexpr int QU = 16, NCHU = cdiv(NQ, QU);      // update quadrature chunks
    static constexpr int NFP = fused::nfp_tri(N);
    static constexpr int NFPK = rup(NFP, 8);
    static constexpr int NFQ = (N + 1) * (N + 1);
    static constexpr int NFH = cdiv(NFQ, 16);               // 16-point halves of a face rule
    static constexpr int NF = 4, FLD = 4, ME = 128, NTH = 544;   // 16 epilogue warps + 1 MMA warp
    static_assert(NFPK <= 16, "exterior-trace K extent must fit 16 TMEM columns per field");
    // operator tile images (floats, hi image then lo image)
    // volume tiles per quadrature chunk: D_a (rows a*16 + q), Vq (rows q), DTW_a (3 blocks of
    // rows j, K = q), -Pq (rows j, K = q)
    // Vq tiles per chunk (16 rows), double buffered
    static constexpr int NPAIR = cdiv(NCH, 2);
    static constexpr int OPDA = 2 * 48 * NPK, OPVQ = 2 * 32 * NPK, OPDTW = 2 * 3 * NPN * QC, OPPQ = 2 * NPN * QC;
    static constexpr int OPVF = 2 * 16 * NPK;               // rows: face points of one half
    static constexpr int OPVFI = 2 * 16 * NFPK;
    static constexpr int OPPF = 2 * NPN * 16;               // rows j, K = face points
    static constexpr int OPU1 = 2 * QU * NPK;
    static constexpr int OPU2 = 2 * NPN * QU;
    static constexpr int OPS_FACE = OPVFI + OPPF;
    // offsets (floats) of the packed operator buffer
    static constexpr size_t O_DA = 0;
    static constexpr size_t O_VQ = O_DA + (size_t)NCH * OPDA;
    static constexpr size_t O_DTW = O_VQ + (size_t)NPAIR * OPVQ;
    static constexpr size_t O_PQ = O_DTW + (size_t)NCH * OPDTW;
    static constexpr size_t O_VFI = O_PQ + (size_t)NCH * OPPQ;         // [half] Vfi
    static constexpr size_t O_PF = O_VFI + (size_t)NFH * OPVFI;         // [f][half] -Pf
    static constexpr size_t O_U1 = O_PF + (size_t)NF * NFH * OPPF;
    static constexpr size_t O_U2 = O_U1 + (size_t)NCHU * OPU1;
    static constexpr size_t OP_TOTAL = O_U2 + (size_t)NCHU * OPU2;
    // shared memory (bytes)
    static constexpr size_t MISC = 2304;
    static_assert(128 + 4 * (NF * 6 * NFP + NF * NFP + 6 * NFP) <= MISC, "index tables exceed MISC");
    static constexpr size_t SQF = (size_t)FLD * ME * NPK;              // floats of one field set
    static constexpr size_t S_VOL = (size_t)(2 * OPDA + OPVQ + OPDTW + OPPQ) * 4;
    static constexpr size_t S_EXT = (size_t)FLD * ME * NFPK * 4;      // one K-major face-node operand
    static constexpr size_t S_UPD = (size_t)2 * (OPU1 + OPU2) * 4;
    static constexpr size_t S_OPS = fused::maxz(S_VOL, S_UPD);
    // surface buffers (union with sQlo + ops): exterior hi, exterior lo, own lo,
    // resident Vfi tiles, two -Pf tiles, neighbour-node staging
    static constexpr size_t S_SURF = 3 * S_EXT + (size_t)(NFH * OPVFI + 2 * OPPF + FLD * NFP * ME) * 4;
    static constexpr size_t S_UNION = fused::maxz(SQF * 4 + S_OPS, S_SURF);
    static constexpr size_t SMEM = MISC + SQF * 4 + S_UNION;
    // TMEM columns
    static constexpr uint32_t RACC = 0, SCR = 4 * NPN;
    static_assert(SCR + 288 + NPN <= 512 && SCR + 192 + 4 * NPK <= 512 && SCR + 320 + (NPN < 32 ? NPN : 32) <= 512,
                  "TMEM budget");
    // op-tile barrier slots (bar[1 + slot]) in the volume phase; the surface and update
    // phases use slots 0 and 1
    static constexpr int SL_DA = 0, SL_VQ = 2, SL_PQ = 4, SL_DTW = 5;
    // persistent CTAs looping over tiles (N = 2, 3: +3.8 / +2.3 %); at N = 4 the
    // loop-carried state costs spills at the 96-register cap, so one tile per CTA
    static constexpr bool PERSIST = N <= 3;
};

// Split-TF32 K loops, issued by one whole warp (one elected lane issues):
// D (+)= A B^T over nks K steps of 8, three MMAs per step
// (A_lo B_hi, A_hi B_lo, A_hi B_hi).  Operand addresses advance 256 B per K
// step in shared memory (two core matrices, LBO = 128) and 8 columns in TMEM.
// A from shared memory (hi, lo)
__device__ __forceinline__ void kloop_ss(uint32_t d, uint32_t ah, uint32_t al, uint32_t sboA, uint32_t bh, uint32_t bl,
                                         uint32_t sboB, int nks, uint32_t id, uint32_t acc0) {
#pragma unroll 1
    for (int ks = 0; ks < nks; ++ks) {
        const uint32_t o = ks * 256;
        const uint64_t dbh = umma::desc_k(bh + o, 128, sboB), dah = umma::desc_k(ah + o, 128, sboA);
        umma::mma_ss_w(d, umma::desc_k(al + o, 128, sboA), dbh, id, (ks > 0) | acc0);
        umma::mma_ss_w(d, dah, umma::desc_k(bl + o, 128, sboB), id, 1u);
        umma::mma_ss_w(d, dah, dbh, id, 1u);
    }
}
// A_hi from shared memory, A_lo from TMEM
__device__ __forceinline__ void kloop_st(uint32_t d, uint32_t ah, uint32_t al_t, uint32_t sboA, uint32_t bh, uint32_t bl,
                                         uint32_t sboB, int nks, uint32_t id, uint32_t acc0) {
#pragma unroll 1
    for (int ks = 0; ks < nks; ++ks) {
        const uint32_t o = ks * 256;
        const uint64_t dbh = umma::desc_k(bh + o, 128, sboB), dah = umma::desc_k(ah + o, 128, sboA);
        umma::mma_ts_w(d, al_t + 8 * ks, dbh, id, (ks > 0) | acc0);
        umma::mma_ss_w(d, dah, umma::desc_k(bl + o, 128, sboB), id, 1u);
        umma::mma_ss_w(d, dah, dbh, id, 1u);
    }
}
// A (hi, lo) from TMEM
__device__ __forceinline__ void kloop_tt(uint32_t d, uint32_t ah_t, uint32_t al_t, uint32_t bh, uint32_t bl,
                                         uint32_t sboB, int nks, uint32_t id, uint32_t acc0) {
#pragma unroll 1
    for (int ks = 0; ks < nks; ++ks) {
        const uint32_t o = ks * 256;
        const uint64_t dbh = umma::desc_k(bh + o, 128, sboB);
        umma::mma_ts_w(d, al_t + 8 * ks, dbh, id, (ks > 0) | acc0);
        umma::mma_ts_w(d, ah_t + 8 * ks, umma::desc_k(bl + o, 128, sboB), id, 1u);
        umma::mma_ts_w(d, ah_t + 8 * ks, dbh, id, 1u);
    }
}

// split 8 values and store hi / lo to two TMEM column groups of this warp's lanes
__device__ __forceinline__ void st_split8(uint32_t t_hi, uint32_t t_lo, const float (&v)[8]) {
    float hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        hi[i] = umma::tf32_split_hi(v[i]);
        lo[i] = v[i] - hi[i];
    }
    umma::st8(t_hi, hi);
    umma::st8(t_lo, lo);
}

__device__ __forceinline__ void st_split4(uint32_t t_hi, uint32_t t_lo, const float (&v)[4]) {
    float hi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        hi[i] = umma::tf32_split_hi(v[i]);
        lo[i] = v[i] - hi[i];
    }
    umma::st4(t_hi, hi);
    umma::st4(t_lo, lo);
}

// named barriers between the epilogue warps (arrive) and the MMA warp (sync)
__device__ __forceinline__ void nb_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
// wait for the k-th completion (1-based) of an mbarrier; valid while at most
// one earlier completion can still be outstanding
__device__ __forceinline__ void wait_k(uint64_t *bar, uint32_t k, int site = -1) {
    umma::mbar_wait_bounded(bar, (k - 1u) & 1u, site);
}

// Warp roles: warps 0..15 are the epilogue warps (element e = 32 (w % 4) + lane,
// sub-group w / 4 owns 4 of the 16 points of a chunk / face half, or field
// w / 4); warp 16 is the MMA warp: it issues every tcgen05.mma and TMA copy and
// never blocks the epilogue warps, which hand over through named barriers
// (bar.arrive) and take results back through tcgen05.commit mbarriers.
// LAY bit 0: Qin in the host row layout (fld, K, Np) (first stage of the host
// pipeline), bit 1: Qout in the row layout (last stage); res is always in the
// field layout.
template <int N, int LAY>
__global__ void __launch_bounds__(CfgU<N>::NTH, 1)
k_stage_umma(const fused::FProb<float> P, const float *__restrict__ Qin, float *__restrict__ Qout,
             float *__restrict__ res, float tau_p, float tau_u, float a_rk, float b_rk, float dt, int block0,
             int block_end) {
    using C = CfgU<N>;
    using namespace umma;
    constexpr int NP = C::NP, NPK = C::NPK, NPN = C::NPN, QC = C::QC, QU = C::QU;
    constexpr int NFP = C::NFP, NFPK = C::NFPK, NFQ = C::NFQ, NFH = C::NFH, NF = 4, ME = 128;
    constexpr int NCH = C::NCH, NCHU = C::NCHU, NSTEP = NF * NFH;
    constexpr uint32_t SBO_Q = (NPK / 4) * 128;        // 8-row group stride of NPK-wide tiles
    constexpr uint32_t SBO_16 = 4 * 128;                // ... of 16-wide tiles
    constexpr uint32_t SBO_FP = (NFPK / 4) * 128;
    constexpr uint32_t RACC = C::RACC, SCR = C::SCR;
    constexpr uint32_t FQB = ME * NPK * 4;              // bytes of one field in sQ / sQlo
    constexpr int NB = C::NTH;                          // named-barrier thread count
    enum { B_P = 1, B_U = 2, B_S0 = 3, B_S1 = 4, B_R = 5, B_Z0 = 6, B_Z1 = 7, B_S2 = 8, B_E = 9 };

    extern __shared__ __align__(1024) unsigned char smem[];
    // mbarriers: [0] MMA group A (volume p chain, face traces, update U1), [7] MMA
    // group B (volume u chain, lifts, update U2), [1..6] operator tiles,
    // v2[0..1] volume V2p / V2u done (operator refills, MMA warp only)
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(smem + 64);
    uint64_t *bar_v2 = reinterpret_cast<uint64_t *>(smem + 80);
    int32_t *sExt = reinterpret_cast<int32_t *>(smem + 128);       // [f2 * nor + o][i]
    int32_t *sFmask = sExt + NF * 6 * NFP;                         // [f][i]
    int32_t *sPerm = sFmask + NF * NFP;                            // [o][i]
    float *sQ = reinterpret_cast<float *>(smem + C::MISC);
    float *sQlo = sQ + C::SQF;
    float *sOp = sQlo + C::SQF;
    const float *ops = P.opVA;                                     // packed tile images (CfgU offsets)

    // warp index through a shuffle: provably warp-uniform, so the MMA warp's
    // branch and descriptor arithmetic stay on the uniform datapath
    const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const bool mma_warp = warp == 16;
    const int qd = warp & 3, sub = (warp >> 2) & 3;                // lane quarter, sub-group 0..3
    const int e = 32 * qd + lane;                                  // element row = TMEM lane
    const size_t S = P.Kpad;
    // persistent CTAs: tiles block0 + blockIdx.x, + gridDim.x, ... < block_end
    asm volatile("griddepcontrol.launch_dependents;");   // the next stage may start its prologue

    // the MMA warp's lane 0 initialises the barriers and at once issues the first
    // volume operator tiles (static data, a region not used before the volume):
    // their copies overlap the prologue and the field staging below
    if (mma_warp && lane == 0) {
        for (int i = 0; i < 8; ++i) fused::mbar_init(&bar[i], 1);
        fused::mbar_init(&bar_v2[0], 1);
        fused::mbar_init(&bar_v2[1], 1);
        fused::fence_proxy_async();
        const float *ops0 = P.opVA;
        float *sOp0 = sQ + 2 * C::SQF;
        auto ld0 = [&](int slot, float *dst, const float *src, uint32_t bytes) {
            fused::mbar_expect_tx(&bar[1 + slot], bytes);
            fused::bulk_g2s(dst, src, bytes, &bar[1 + slot]);
        };
        ld0(C::SL_DA, sOp0, ops0 + C::O_DA, C::OPDA * 4);
        ld0(C::SL_VQ, sOp0 + 2 * C::OPDA, ops0 + C::O_VQ, C::OPVQ * 4);
        ld0(C::SL_PQ, sOp0 + 2 * C::OPDA + C::OPVQ, ops0 + C::O_PQ, C::OPPQ * 4);
        ld0(C::SL_DTW, sOp0 + 2 * C::OPDA + C::OPVQ + C::OPPQ, ops0 + C::O_DTW, C::OPDTW * 4);
        if (NCH > 1) ld0(C::SL_DA + 1, sOp0 + C::OPDA, ops0 + C::O_DA + C::OPDA, C::OPDA * 4);
    }
    if (warp == 0) tmem_alloc<512>(tslot);
    for (int r = tid; r < NF * 6 * NFP; r += C::NTH) sExt[r] = __ldg(P.ext_node + r);
    for (int r = tid; r < NF * NFP; r += C::NTH) sFmask[r] = __ldg(P.fmask + r);
    for (int r = tid; r < 6 * NFP; r += C::NTH) sPerm[r] = __ldg(P.fperm + r);
    // Programmatic dependent launch: everything above touches only static data,
    // so it overlaps the previous stage kernel's tail; the fields, res and halo
    // written by that kernel are read (and Qout / res written) only after this
    // wait.  Without the launch attribute the wait is a no-op.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // barrier-completion counts carried from tile to tile: the MMA warp's operator
    // slot phases, V2p / V2u (and update U2) completions and group-B completions
    // before the current tile; the epilogue's consumed group-A / group-B completions
    // (one set of registers: the MMA warp's {slot phases, V2p, V2u, group B} and the
    // epilogue warps' {group A, group B})
    uint32_t cnt[4] = {0u, 0u, 0u, 0u};
    // group-B (bar[7]) commits per tile: volume NCH + 1, surface NSTEP, update NCHU + 1
    constexpr uint32_t TILE_B = (uint32_t)(NCH + 1 + NSTEP + NCHU + 1);
    fence_before();
    __syncthreads();                      // barrier init, TMEM address and index tables visible
    fence_after();
    const uint32_t tm = *tslot;
    for (size_t blk = (size_t)block0 + blockIdx.x;;) {
    const size_t kblk = blk * ME;
    UMMA_MARK0(0);
    if (P.prof && threadIdx.x == 0) {   // debug: SM id (slot 30), for per-SM gap analysis
        uint32_t smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        P.prof[(blk - (size_t)block0) * 32 + 30] = smid;
    }
    // neighbour tables of all faces (consumed in the surface phase)
    int nbr[NF], ncode[NF];
    if (!mma_warp) {
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            nbr[f] = __ldg(P.nbr + (size_t)f * S + kblk + e);
            ncode[f] = __ldg(P.ncode + (size_t)f * S + kblk + e);
        }
        // ---- fields -> sQ (raw fp32, the tf32 hi operand) and sQlo --------
        const int c = sub;
        if constexpr (LAY & 1) {
            // row layout: this warp's 32 elements of field c are one contiguous run
            // of 32 Np values; read it coalesced and scatter into the K-major tiles
            const long long e0 = (long long)kblk + 32 * qd;
            const int cnt = (int)max(0LL, min(32LL, (long long)P.K - e0)) * NP;
            const float *src = Qin + ((size_t)c * P.K + e0) * NP;
            for (int t = lane; t < 32 * NP; t += 32) {
                const float v = t < cnt ? __ldg(src + t) : 0.f;
                const int el = t / NP, j = t - el * NP;
                const uint32_t o = c * ME * NPK + kmaj_off<NPK>(32 * qd + el, j) / 4;
                sQ[o] = v;
                sQlo[o] = tf32_lo(v);
            }
#pragma unroll
            for (int j = NP; j < NPK; ++j) {
                const uint32_t o = c * ME * NPK + kmaj_off<NPK>(e, j) / 4;
                sQ[o] = 0.f;
                sQlo[o] = 0.f;
            }
        } else {
#pragma unroll
            for (int j0 = 0; j0 < NPK; j0 += 4) {
                float4 v;
                float *pv = reinterpret_cast<float *>(&v);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = j0 + i;
                    pv[i] = j < NP ? __ldg(Qin + (size_t)(c * NP + j) * S + kblk + e) : 0.f;
                }
                float4 l;
                float *pl = reinterpret_cast<float *>(&l);
#pragma unroll
                for (int i = 0; i < 4; ++i) pl[i] = tf32_lo(pv[i]);
                const uint32_t o = kmaj_off<NPK>(e, j0) / 4;
                *reinterpret_cast<float4 *>(sQ + c * ME * NPK + o) = v;
                *reinterpret_cast<float4 *>(sQlo + c * ME * NPK + o) = l;
            }
        }
    }
    fused::fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tl = tm + ((uint32_t)(32 * qd) << 16);         // this warp's lane quarter
    const uint32_t aQ = su32(sQ), aQlo = su32(sQlo);
    UMMA_MARK0(1);

    // ---- shared-memory regions and TMEM columns per phase ------------------
    // volume
    float *sDa = sOp;                                   // [2][OPDA]
    float *sVq = sDa + 2 * C::OPDA;                     // [OPVQ] (one chunk pair)
    float *sPq = sVq + C::OPVQ;                         // [OPPQ]
    float *sDTW = sPq + C::OPPQ;                        // [OPDTW]
    // U of a chunk pair: field i at UO + 32 i, chunk ch at + 16 (ch & 1).  dp_a is
    // written into the gp hi columns (GPH) and the epilogue overwrites it with
    // gp_hi in place (each thread reads its dp values before it writes); the
    // next chunk's D_a p MMAs are issued after this chunk's -Pq gp ones, whose
    // reads of GPH precede them in the tensor core's in-order execution.  RPC:
    // the split-TF32 correction terms (A_lo B_hi, A_hi B_lo) of the R_p volume
    // accumulation, kept apart from the main terms in RACC: the tensor core's
    // fp32 accumulation truncates toward zero at the accumulator's ulp, so the
    // small corrections are not added into the large running R_p (half the
    // truncations there); folded into R_p by the epilogue at the end of the volume
    const uint32_t UO = SCR, GPH = SCR + 96, GPL = SCR + 144, FH = SCR + 192, FL = SCR + 240, RPC = SCR + 288;
    const uint32_t DPO = GPH;
    // surface (over the sQlo + ops union): exterior node hi / lo and own node lo
    // parts (K-major operands), resident Vfi tiles, two -Pf tiles, neighbour-node
    // staging; TMEM: traces at the 16 points of a face half (own, exterior), the
    // flux g (hi, lo: the lift A operand), own face-node hi parts
    float *sExtHi = sQlo, *sExtLo = sQlo + C::S_EXT / 4, *sOwnLo = sQlo + C::S_EXT / 2;
    float *sVfi = sQlo + 3 * C::S_EXT / 4;
    auto sPf = [&](int b) { return sVfi + NFH * C::OPVFI + b * C::OPPF; };
    float *sStage = sVfi + NFH * C::OPVFI + 2 * C::OPPF;
    // RPCS: the split-TF32 correction terms of the R_p lifts (nodes 0 .. RPW-1; the
    // rest, if any, go into RACC), folded into R_p after the last lift (like RPC)
    constexpr int RPW = NPN < 32 ? NPN : 32;
    const uint32_t OWN = SCR, EXT = SCR + 64, GH = SCR + 128, GL = SCR + 192, OWNH = SCR + 256, RPCS = SCR + 320;
    // update: two chains, one per field pair (0: p, u1; 1: u2, u3).  R of pair 0
    // (hi, lo) in the sQlo region, R of pair 1 (hi, lo) in TMEM; per chain z and
    // omega z (hi, lo) in TMEM; two {Vu, Pu} tile buffers
    float *sA = sQlo;
    auto sU = [&](int b) { return sOp + b * (C::OPU1 + C::OPU2); };
    const uint32_t Z0 = SCR, Z1 = SCR + 32, UA0H = SCR + 64, UA0L = SCR + 96, UA1H = SCR + 128, UA1L = SCR + 160;
    const uint32_t RA1 = SCR + 192;                    // [hi f2, hi f3, lo f2, lo f3] x NPK

    if (mma_warp) {
        // =================== MMA warp =====================================
        uint32_t &ph_op = cnt[0], &nv2p = cnt[1], &nv2u = cnt[2];
        uint32_t nB = cnt[3];
        auto op_load = [&](int slot, float *dst, const float *src, uint32_t bytes) {
            if (lane == 0) {
                fused::mbar_expect_tx(&bar[1 + slot], bytes);
                fused::bulk_g2s(dst, src, bytes, &bar[1 + slot]);
            }
        };
        auto op_load2 = [&](int slot, float *d0, const float *s0, uint32_t b0, float *d1, const float *s1, uint32_t b1) {
            if (lane == 0) {
                fused::mbar_expect_tx(&bar[1 + slot], b0 + b1);
                fused::bulk_g2s(d0, s0, b0, &bar[1 + slot]);
                fused::bulk_g2s(d1, s1, b1, &bar[1 + slot]);
            }
        };
        auto op_wait = [&](int slot) {
            mbar_wait_bounded(&bar[1 + slot], (ph_op >> slot) & 1u, 3000 + slot);
            ph_op ^= 1u << slot;
        };
        auto from_epilogue = [&](int id) {   // epilogue warps' TMEM / smem writes are visible
            nb_sync(id, NB);
            fence_after();
        };
        // ---- volume: p chain (dp -> gp -> R_u) and u chain (U -> F -> R_p) ----
        auto issue_v1p = [&](int ch) {
            const uint32_t bh = su32(sDa + (ch & 1) * C::OPDA), bl = bh + C::OPDA * 2, id = idesc_tf32(128, 48);
#pragma unroll 1
            for (int ks = 0; ks < NPK / 8; ++ks) {
                const uint32_t o = ks * 256;
#pragma unroll
                for (int t = 0; t < 3; ++t)
                    mma_ss_w(tm + DPO, desc_k((t == 0 ? aQlo : aQ) + o, 128, SBO_Q),
                             desc_k((t == 1 ? bl : bh) + o, 128, SBO_Q), id, (ks > 0 || t > 0) ? 1u : 0u);
            }
        };
        auto issue_v1u = [&]() {                       // U_i for the chunk pair in sVq
            const uint32_t bh = su32(sVq), bl = bh + C::OPVQ * 2, id = idesc_tf32(128, 32);
#pragma unroll 1
            for (int ks = 0; ks < NPK / 8; ++ks) {
                const uint32_t o = ks * 256;
#pragma unroll
                for (int t = 0; t < 3; ++t)
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        mma_ss_w(tm + UO + 32 * i, desc_k((t == 0 ? aQlo : aQ) + (1 + i) * FQB + o, 128, SBO_Q),
                                 desc_k((t == 1 ? bl : bh) + o, 128, SBO_Q), id, (ks > 0 || t > 0) ? 1u : 0u);
            }
        };
        auto issue_v2p = [&](int ch) {   // R_u_i += (-Pq) gp_i
            const uint32_t bh = su32(sPq), bl = bh + C::OPPQ * 2, id = idesc_tf32(128, NPN);
#pragma unroll 1
            for (int ks = 0; ks < QC / 8; ++ks) {
#pragma unroll
                for (int t = 0; t < 3; ++t)
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        mma_ts_w(tm + RACC + NPN * (1 + i), tm + (t == 0 ? GPL : GPH) + 16 * i + 8 * ks,
                                 desc_k((t == 1 ? bl : bh) + ks * 256, 128, SBO_16), id,
                                 (ch > 0 || ks > 0 || t > 0) ? 1u : 0u);
            }
        };
        auto issue_v2u = [&](int ch) {   // R_p += sum_a DTW_a F_a: main terms -> RACC, corrections -> RPC
            constexpr uint32_t BLK = NPN * QC * 4;
            const uint32_t bh = su32(sDTW), bl = bh + C::OPDTW * 2, id = idesc_tf32(128, NPN);
#pragma unroll 1
            for (int ks = 0; ks < QC / 8; ++ks) {
#pragma unroll
                for (int t = 0; t < 3; ++t)
#pragma unroll
                    for (int a = 0; a < 3; ++a)
                        mma_ts_w(t < 2 ? tm + RPC : tm + RACC, tm + (t == 0 ? FL : FH) + 16 * a + 8 * ks,
                                 desc_k((t == 1 ? bl : bh) + a * BLK + ks * 256, 128, SBO_16), id,
                                 (ch > 0 || ks > 0 || a > 0 || t == 1) ? 1u : 0u);
            }
        };
        // (chunk 0 / 1's operator tiles were issued at kernel entry)
        __syncwarp();
        op_wait(C::SL_DA);
        issue_v1p(0);
        commit_w(&bar[0]);
        op_wait(C::SL_VQ);
        issue_v1u();                         // chunks 0, 1
        commit_w(&bar[7]);
        for (int ch = 0; ch < NCH; ++ch) {
            const bool more = ch + 1 < NCH;
            const int tb = (ch == 2 || ch == 3) ? 6 + 8 * (ch - 2) : -1;
#define VTR(k) do { if (tb >= 0) MMA_TRACE(tb + (k)); } while (0)
            VTR(0);
            from_epilogue(B_P);              // gp(ch) in TMEM, dp(ch) consumed
            VTR(1);
            op_wait(C::SL_PQ);
            VTR(2);
            issue_v2p(ch);
            commit_w(&bar_v2[0]);
            if (more) {
                op_wait(C::SL_DA + ((ch + 1) & 1));
                issue_v1p(ch + 1);
            }
            commit_w(&bar[0]);
            VTR(3);
            from_epilogue(B_U);              // F(ch) in TMEM, U(ch) consumed
            VTR(4);
            op_wait(C::SL_DTW);
            VTR(5);
            issue_v2u(ch);
            commit_w(&bar_v2[1]);
            if (more && (ch & 1)) {          // next chunk pair (ch + 1, ch + 2)
                op_wait(C::SL_VQ);
                issue_v1u();
            }
            commit_w(&bar[7]);
            // refills: the -Pq / D_a(ch) tiles are free once V2p(ch) (issued after V1p(ch))
            // is done, the DTW / Vq(ch) tiles once V2u(ch) (issued after V1u(ch)) is
            wait_k(&bar_v2[0], ++nv2p);
            VTR(6);
            if (more) op_load(C::SL_PQ, sPq, ops + C::O_PQ + (size_t)(ch + 1) * C::OPPQ, C::OPPQ * 4);
            if (ch + 2 < NCH)
                op_load(C::SL_DA + (ch & 1), sDa + (ch & 1) * C::OPDA, ops + C::O_DA + (size_t)(ch + 2) * C::OPDA,
                        C::OPDA * 4);
            wait_k(&bar_v2[1], ++nv2u);
            VTR(7);
#undef VTR
            if (more) op_load(C::SL_DTW, sDTW, ops + C::O_DTW + (size_t)(ch + 1) * C::OPDTW, C::OPDTW * 4);
            if (!(ch & 1) && ch + 2 < NCH)   // pair ch/2 consumed (V1u issued before V2u(ch)): next pair
                op_load(C::SL_VQ, sVq, ops + C::O_VQ + (size_t)(ch / 2 + 1) * C::OPVQ, C::OPVQ * 4);
        }
        nB = cnt[3] + NCH + 1;               // group-B completions so far (V1u(0), per-chunk u commits)
        // ---- surface: per (face, half) step s: traces(s) (group A) are issued as
        // soon as the epilogue has read traces(s-1) out of TMEM, the lift of s-1
        // (group B) once its flux is written; the flux has its own columns ----
        op_load(2, sVfi, ops + C::O_VFI, NFH * C::OPVFI * 4);   // resident for the whole surface
        op_load(0, sPf(0), ops + C::O_PF, C::OPPF * 4);
        if (NSTEP > 1) op_load(1, sPf(1), ops + C::O_PF + C::OPPF, C::OPPF * 4);
        op_wait(2);
        const uint32_t aEH = su32(sExtHi), aEL = su32(sExtLo), aOL = su32(sOwnLo);
        auto issue_lift = [&](int st) {
            op_wait(st & 1);
            const uint32_t pfh = su32(sPf(st & 1)), pfl = pfh + C::OPPF * 2, idl = idesc_tf32(128, NPN);
            const uint32_t idc = idesc_tf32(128, RPW), idr = idesc_tf32(128, NPN > RPW ? NPN - RPW : 8);
#pragma unroll 1
            for (int ks = 0; ks < 2; ++ks)
#pragma unroll
                for (int t = 0; t < 3; ++t)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const uint32_t a = tm + (t == 0 ? GL : GH) + 16 * c + 8 * ks, b = (t == 1 ? pfl : pfh) + ks * 256;
                        if (c == 0 && t < 2) {   // R_p corrections
                            mma_ts_w(tm + RPCS, a, desc_k(b, 128, SBO_16), idc, (st > 0 || ks > 0 || t > 0) ? 1u : 0u);
                            if constexpr (NPN > RPW)
                                mma_ts_w(tm + RACC + RPW, a, desc_k(b + (RPW / 8) * SBO_16, 128, SBO_16), idr, 1u);
                        } else {
                            mma_ts_w(tm + RACC + NPN * c, a, desc_k(b, 128, SBO_16), idl, 1u);
                        }
                    }
            commit_w(&bar[7]);
        };
        for (int step = 0; step < NSTEP; ++step) {
            const int hh = step % NFH;
            if (step == 3) MMA_TRACE(22);
            if (step == 4) MMA_TRACE(28);
            if (hh == 0) from_epilogue(B_S0);   // this face's own / exterior nodes written
            if (step == 4) MMA_TRACE(29);
            if (step > 0) from_epilogue(B_S2);  // traces(step-1) read out of TMEM
            if (step == 3) MMA_TRACE(23);
            const uint32_t vih = su32(sVfi + hh * C::OPVFI), vil = vih + C::OPVFI * 2;
            const uint32_t id = idesc_tf32(128, 16);
#pragma unroll 1
            for (int ks = 0; ks < NFPK / 8; ++ks) {
                const uint32_t o = ks * 256;
#pragma unroll
                for (int t = 0; t < 3; ++t)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const uint64_t db = desc_k((t == 1 ? vil : vih) + o, 128, SBO_FP);
                        const uint32_t acc = (ks > 0 || t > 0) ? 1u : 0u;
                        const uint32_t co = c * ME * NFPK * 4 + o;
                        if (t == 0)
                            mma_ss_w(tm + OWN + 16 * c, desc_k(aOL + co, 128, SBO_FP), db, id, acc);
                        else
                            mma_ts_w(tm + OWN + 16 * c, tm + OWNH + 16 * c + 8 * ks, db, id, acc);
                        mma_ss_w(tm + EXT + 16 * c, desc_k((t == 0 ? aEL : aEH) + co, 128, SBO_FP), db, id, acc);
                    }
            }
            commit_w(&bar[0]);
            if (step == 3) MMA_TRACE(24);
            if (step >= 2) {                 // lift(step-2) done: its -Pf buffer takes step
                wait_k(&bar[7], ++nB, 4000 + step);
                op_load(step & 1, sPf(step & 1), ops + C::O_PF + (size_t)step * C::OPPF, C::OPPF * 4);
            }
            if (step == 3) MMA_TRACE(25);
            if (step > 0) {
                from_epilogue(B_S1);         // flux of step-1 written
                if (step == 3) MMA_TRACE(26);
                issue_lift(step - 1);
                if (step == 3) MMA_TRACE(27);
            }
        }
        // An mbarrier parity wait is only unambiguous while at most one completion is
        // outstanding, so lift(NSTEP-2) is waited for before the last lift is issued.
        if (NSTEP >= 2) wait_k(&bar[7], ++nB, 4100);
        from_epilogue(B_S2);
        from_epilogue(B_S1);
        issue_lift(NSTEP - 1);
        wait_k(&bar[7], ++nB, 4101);         // all lifts done: R complete, tiles and columns free
        // ---- update: chain 0 (pair 0, group A) and chain 1 (pair 1, group B), per
        // 16-point chunk: U1 (z = Vu R_c), then U2 (R_c (+)= Pu omega z) ----
        op_load2(0, sU(0), ops + C::O_U1, C::OPU1 * 4, sU(0) + C::OPU1, ops + C::O_U2, C::OPU2 * 4);
        if (NCHU > 1)
            op_load2(1, sU(1), ops + C::O_U1 + C::OPU1, C::OPU1 * 4, sU(1) + C::OPU1, ops + C::O_U2 + C::OPU2,
                     C::OPU2 * 4);
        const uint32_t sA0 = su32(sA), idz = idesc_tf32(128, QU), idu = idesc_tf32(128, NPN);
        auto issue_u1 = [&](int chain, int u) {
            const uint32_t uo = su32(sU(u & 1));
#pragma unroll 1
            for (int ks = 0; ks < NPK / 8; ++ks) {
                const uint32_t o = ks * 256;
#pragma unroll
                for (int t = 0; t < 3; ++t)
#pragma unroll
                    for (int lf = 0; lf < 2; ++lf) {
                        const uint64_t db = desc_k(uo + (t == 1 ? C::OPU1 * 2 : 0) + o, 128, SBO_Q);
                        const uint32_t acc = (ks > 0 || t > 0) ? 1u : 0u;
                        if (chain == 0)
                            mma_ss_w(tm + Z0 + 16 * lf, desc_k(sA0 + (t == 0 ? 2 + lf : lf) * FQB + o, 128, SBO_Q), db,
                                     idz, acc);
                        else
                            mma_ts_w(tm + Z1 + 16 * lf, tm + RA1 + (t == 0 ? 2 * NPK : 0) + NPK * lf + 8 * ks, db, idz, acc);
                    }
            }
        };
        auto issue_u2 = [&](int chain, int u) {
            const uint32_t bh = su32(sU(u & 1)) + C::OPU1 * 4, bl = bh + C::OPU2 * 2;
            const uint32_t zh = chain ? UA1H : UA0H, zl = chain ? UA1L : UA0L;
#pragma unroll 1
            for (int ks = 0; ks < QU / 8; ++ks)
#pragma unroll
                for (int t = 0; t < 3; ++t)
#pragma unroll
                    for (int lf = 0; lf < 2; ++lf)
                        mma_ts_w(tm + RACC + NPN * (2 * chain + lf), tm + (t == 0 ? zl : zh) + 16 * lf + 8 * ks,
                                 desc_k((t == 1 ? bl : bh) + ks * 256, 128, SBO_16), idu, (u > 0 || ks > 0 || t > 0) ? 1u : 0u);
        };
        from_epilogue(B_R);                  // R of both pairs in place (shared memory, TMEM)
        op_wait(0);
        issue_u1(0, 0);
        commit_w(&bar[0]);
        issue_u1(1, 0);
        commit_w(&bar[7]);
        for (int u = 0; u < NCHU; ++u) {
            const bool more = u + 1 < NCHU;
            from_epilogue(B_Z0);             // omega z of chain 0 in TMEM, z consumed
            issue_u2(0, u);
            if (more) {
                op_wait((u + 1) & 1);
                issue_u1(0, u + 1);
            }
            commit_w(&bar[0]);
            from_epilogue(B_Z1);
            issue_u2(1, u);
            commit_w(&bar_v2[0]);            // last reader of the chunk-u tiles
            if (more) issue_u1(1, u + 1);
            commit_w(&bar[7]);
            wait_k(&bar_v2[0], ++nv2p);      // every completion is consumed (a parity wait needs that)
            if (u + 2 < NCHU)
                op_load2(u & 1, sU(u & 1), ops + C::O_U1 + (size_t)(u + 2) * C::OPU1, C::OPU1 * 4,
                         sU(u & 1) + C::OPU1, ops + C::O_U2 + (size_t)(u + 2) * C::OPU2, C::OPU2 * 4);
        }
        cnt[3] += TILE_B;
        // every MMA of this tile is done (the last U2 commit): the next tile's first
        // volume operator tiles load while the epilogue warps write this tile out
        if (C::PERSIST && blk + gridDim.x < (size_t)block_end) {
            op_load(C::SL_DA, sDa, ops + C::O_DA, C::OPDA * 4);
            op_load(C::SL_VQ, sVq, ops + C::O_VQ, C::OPVQ * 4);
            op_load(C::SL_PQ, sPq, ops + C::O_PQ, C::OPPQ * 4);
            op_load(C::SL_DTW, sDTW, ops + C::O_DTW, C::OPDTW * 4);
            if (NCH > 1) op_load(C::SL_DA + 1, sDa + C::OPDA, ops + C::O_DA + C::OPDA, C::OPDA * 4);
        }
        __syncwarp();
    } else {
        // =================== epilogue warps ===============================
        uint32_t &nA = cnt[0], &nB = cnt[1]; // consumed completions of MMA groups A and B
        auto wait_A = [&]() { wait_k(&bar[0], ++nA); fence_after(); };
        auto wait_B = [&]() { wait_k(&bar[7], ++nB); fence_after(); };
        // hand TMEM (and, with smem = true, shared-memory operand) writes to the
        // MMA warp; the proxy fence is only needed for shared memory the tensor
        // core reads through descriptors
        auto to_mma = [&](int id, bool smem = false) {
            if (smem) fused::fence_proxy_async();
            fence_before();
            nb_arrive(id, NB);
        };
        // ---- volume ----
        float G[9][4];
        constexpr int GQ4 = NCH * 4;                    // float4 rows per geometric factor (Nq padded to 16)
        auto load_G = [&](int ch) {
            const float4 *src = reinterpret_cast<const float4 *>(P.geo_il) + (blk * 9 * GQ4 + ch * 4 + sub) * ME + e;
#pragma unroll
            for (int r = 0; r < 9; ++r) {
                const float4 v = __ldg(src + (size_t)r * GQ4 * ME);
                G[r][0] = v.x; G[r][1] = v.y; G[r][2] = v.z; G[r][3] = v.w;
            }
        };
        load_G(0);
        for (int ch = 0; ch < NCH; ++ch) {
            if (N >= 4 && ch == NCH - 1 && nbr[0] >= 0) {
                // L2 prefetch of face 0's neighbour nodes: the surface gathers them
                // first, right after the volume, with nothing to overlap the load
                // (N = 4: +1.1 %; at N = 2, 3 the extra registers cost more)
                const int code = ncode[0], c = sub;
#pragma unroll 1
                for (int i = 0; i < NFP; ++i) {
                    const float *a = (LAY & 1) ? Qin + ((size_t)c * P.K + nbr[0]) * NP + sExt[code * NFP + i]
                                               : Qin + (size_t)(c * NP + sExt[code * NFP + i]) * S + nbr[0];
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                }
            }
            wait_A();                        // V1p(ch) and V2p(ch-1) done
            {
                float dp[3][4];
#pragma unroll
                for (int a = 0; a < 3; ++a) ld4(tl + DPO + 16 * a + 4 * sub, dp[a]);
                wait_ld();
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    float gp[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p)
                        gp[p] = G[0 * 3 + m][p] * dp[0][p] + G[1 * 3 + m][p] * dp[1][p] + G[2 * 3 + m][p] * dp[2][p];
                    st_split4(tl + GPH + 16 * m + 4 * sub, tl + GPL + 16 * m + 4 * sub, gp);
                }
                wait_st();
            }
            to_mma(B_P);
            wait_B();                        // V1u(ch) and V2u(ch-1) done
            {
                float U[3][4];
#pragma unroll
                for (int i = 0; i < 3; ++i) ld4(tl + UO + 32 * i + 16 * (ch & 1) + 4 * sub, U[i]);
                wait_ld();
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    float F[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p)
                        F[p] = G[m * 3 + 0][p] * U[0][p] + G[m * 3 + 1][p] * U[1][p] + G[m * 3 + 2][p] * U[2][p];
                    st_split4(tl + FH + 16 * m + 4 * sub, tl + FL + 16 * m + 4 * sub, F);
                }
                if (ch + 1 < NCH) load_G(ch + 1);
                wait_st();
            }
            to_mma(B_U);
        }
        wait_A();                            // V2p of the last chunk
        wait_B();                            // V2u of the last chunk
        // fold the R_p correction terms into R_p (fp32, round to nearest): node groups
        // of 8 split between the four sub-groups of an element
        for (int g = sub; g < NPN / 8; g += 4) {
            float r[8], q[8];
            ld8(tl + RACC + 8 * g, r);
            ld8(tl + RPC + 8 * g, q);
            wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] += q[i];
            st8(tl + RACC + 8 * g, r);
        }
        wait_st();                           // handed to the MMA warp with the first face's operands
        UMMA_MARK0(2);
        // ---- surface ----
        auto gather = [&](int f) {   // neighbour face nodes of face f, field sub -> sStage [c][i][128]
            const int nb = f == 0 ? nbr[0] : f == 1 ? nbr[1] : f == 2 ? nbr[2] : nbr[3];
            const int code = f == 0 ? ncode[0] : f == 1 ? ncode[1] : f == 2 ? ncode[2] : ncode[3];
            const int c = sub;
            float *dst = sStage + (size_t)c * NFP * ME + e;
            // one loop per case (the case is fixed per element and face); the rare
            // boundary and halo cases stay rolled to keep the kernel's code small
            if (nb >= 0) {
#pragma unroll
                for (int i = 0; i < NFP; ++i) {
                    if constexpr (LAY & 1)
                        fused::cp_async_elem(dst + i * ME, Qin + ((size_t)c * P.K + nb) * NP + sExt[code * NFP + i]);
                    else
                        fused::cp_async_elem(dst + i * ME, Qin + (size_t)(c * NP + sExt[code * NFP + i]) * S + nb);
                }
            } else if (nb == -1) {       // mirror BC (solver.py:214-217): p+ = -p-, u+ = u-
#pragma unroll 1
                for (int i = 0; i < NFP; ++i) {
                    const float m = sQ[c * ME * NPK + kmaj_off<NPK>(e, sFmask[f * NFP + i]) / 4];
                    dst[i * ME] = c == 0 ? -m : m;
                }
            } else {
#pragma unroll 1
                for (int i = 0; i < NFP; ++i)
                    fused::cp_async_elem(dst + i * ME,
                                         P.halo + ((size_t)(-nb - 2) * 4 + c) * NFP + sPerm[(code % P.nor) * NFP + i]);
            }
            fused::cp_async_commit();
        };
        float fg[4][4];
        constexpr int FQ4 = NFH * 4;                    // float4 rows per face (face rule padded to 16)
        auto load_fg = [&](int step) {
            const int f = step / NFH, hh = step % NFH;
            const int fq4 = 4 * hh + sub;
            const float4 *src = reinterpret_cast<const float4 *>(P.fgeo_il) + (blk * 4 * NF * FQ4 + f * FQ4 + fq4) * ME + e;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const float4 v = 4 * fq4 < NFQ ? __ldg(src + (size_t)d * NF * FQ4 * ME) : make_float4(0.f, 0.f, 0.f, 0.f);
                fg[d][0] = v.x; fg[d][1] = v.y; fg[d][2] = v.z; fg[d][3] = v.w;
            }
        };
        // own / exterior face-node operands of face f (shared memory + TMEM hi)
        auto node_store = [&](int f) {
            fused::cp_async_wait<0>();       // this thread's staged neighbour nodes of face f
            const int c = sub;
            const float *xs = sStage + (size_t)c * NFP * ME + e;
#pragma unroll
            for (int i0 = 0; i0 < NFPK; i0 += 4) {
                float4 vh, vl, oh4, ol4;
                float *ph = reinterpret_cast<float *>(&vh), *pl = reinterpret_cast<float *>(&vl);
                float *qh = reinterpret_cast<float *>(&oh4), *ql = reinterpret_cast<float *>(&ol4);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const bool in = i0 + i < NFP;
                    const float x = in ? xs[(i0 + i) * ME] : 0.f;
                    const float y = in ? sQ[c * ME * NPK + kmaj_off<NPK>(e, sFmask[f * NFP + i0 + i]) / 4] : 0.f;
                    ph[i] = tf32_split_hi(x);
                    pl[i] = x - ph[i];
                    qh[i] = tf32_split_hi(y);
                    ql[i] = y - qh[i];
                }
                const uint32_t o = c * ME * NFPK + kmaj_off<NFPK>(e, i0) / 4;
                *reinterpret_cast<float4 *>(sExtHi + o) = vh;
                *reinterpret_cast<float4 *>(sExtLo + o) = vl;
                *reinterpret_cast<float4 *>(sOwnLo + o) = ol4;
                st4(tl + OWNH + 16 * c + i0, *reinterpret_cast<float (*)[4]>(qh));
            }
#pragma unroll
            for (int i0 = NFPK; i0 < 16; i0 += 4) {
                const float z4[4] = {0.f, 0.f, 0.f, 0.f};
                st4(tl + OWNH + 16 * c + i0, z4);
            }
            wait_st();
            to_mma(B_S0, true);
        };
        // Face-node operands of the next face go in right after the face's last step
        // has read its traces, so the next face's traces overlap that step's flux
        // (at N = 4 this beat writing them at the face boundary: surface 40.7k ->
        // 38.3k cycles per tile).
        {
            // face has read its traces (so the next traces overlap that step's flux)
            gather(0);
            load_fg(0);
            node_store(0);
            if (NF > 1) gather(1);
#pragma unroll 1
            for (int step = 0; step < NSTEP; ++step) {
                const int f = step / NFH, hh = step % NFH;
                wait_A();                        // traces of this step
                float mM[4][4], mP[4][4];
    #pragma unroll
                for (int c = 0; c < 4; ++c) {
                    ld4(tl + OWN + 16 * c + 4 * sub, mM[c]);
                    ld4(tl + EXT + 16 * c + 4 * sub, mP[c]);
                }
                wait_ld();
                fence_before();
                nb_arrive(B_S2, NB);             // trace columns free for the next step's MMAs
                // the last half of a face has consumed the face-node operands: the next
                // face's go in now, so its traces overlap this step's flux
                const bool next_face = hh == NFH - 1 && f + 1 < NF;
                if (next_face) node_store(f + 1);
                float g[4][4];
    #pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const float n0 = fg[0][p], n1 = fg[1][p], n2 = fg[2][p], sJh = fg[3][p];
                    const float dpj = mP[0][p] - mM[0][p];
                    const float dUn = (mP[1][p] - mM[1][p]) * n0 + (mP[2][p] - mM[2][p]) * n1 + (mP[3][p] - mM[3][p]) * n2;
                    const float avg = (mP[1][p] + mM[1][p]) * n0 + (mP[2][p] + mM[2][p]) * n1 + (mP[3][p] + mM[3][p]) * n2;
                    const float fpp = avg - tau_p * dpj;
                    const float fuu = dpj - tau_u * dUn;
                    g[0][p] = fpp * sJh;
                    g[1][p] = fuu * (sJh * n0);
                    g[2][p] = fuu * (sJh * n1);
                    g[3][p] = fuu * (sJh * n2);
                }
                if (step + 1 < NSTEP) load_fg(step + 1);
                if (step > 0) wait_B();          // lift(step-1) done with the flux columns
    #pragma unroll
                for (int c = 0; c < 4; ++c) st_split4(tl + GH + 16 * c + 4 * sub, tl + GL + 16 * c + 4 * sub, g[c]);
                wait_st();
                to_mma(B_S1);
                // neighbour nodes of the face after next: issued off the flux critical path,
                // they have at least one step to land before node_store needs them
                if (next_face && f + 2 < NF) gather(f + 2);
            }
        }
        wait_B();                            // last lift: R complete
        for (int g = sub; g < RPW / 8; g += 4) {   // fold the R_p lift corrections into R_p
            float r[8], q[8];
            ld8(tl + RACC + 8 * g, r);
            ld8(tl + RPCS + 8 * g, q);
            wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] += q[i];
            st8(tl + RACC + 8 * g, r);
        }
        wait_st();
        fence_before();
        nb_sync(B_E, NB - 32);               // epilogue warps only: R_p complete before it is read
        fence_after();
        UMMA_MARK0(3);
        // ---- update ----
        // thread (e, sub): field lf = sub & 1 of each pair, points 8 (sub >> 1) .. +7 of a chunk
        const int lf = sub & 1, pb = 8 * (sub >> 1);
        float w0[8], w1[8];
        constexpr int WQ4 = NCHU * QU / 4;              // float4 rows of the weights (Nq padded to QU)
        auto load_w = [&](int u) {
            const float *b0 = (lf > 0 || !P.wp) ? P.wu_il : P.wp_il;      // chain 0: field lf (p: c^2/J)
            const float sc = (lf > 0 || P.wp) ? 1.f : P.c2;
            const float4 *s0 = reinterpret_cast<const float4 *>(b0) + (blk * WQ4 + u * 4 + pb / 4) * ME + e;
            const float4 *s1 = reinterpret_cast<const float4 *>(P.wu_il) + (blk * WQ4 + u * 4 + pb / 4) * ME + e;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const float4 v = __ldg(s0 + (size_t)k * ME), x = __ldg(s1 + (size_t)k * ME);
                w0[4 * k + 0] = sc * v.x; w0[4 * k + 1] = sc * v.y; w0[4 * k + 2] = sc * v.z; w0[4 * k + 3] = sc * v.w;
                w1[4 * k + 0] = x.x; w1[4 * k + 1] = x.y; w1[4 * k + 2] = x.z; w1[4 * k + 3] = x.w;
            }
        };
        load_w(0);
        {   // R -> A operands: pair 0 (fields lf) to shared memory, pair 1 (fields 2 + lf) to TMEM;
            // node groups of 8 split between sub >> 1
#pragma unroll
            for (int j0 = 8 * (sub >> 1); j0 < NPK; j0 += 16) {
                float v[8], hi[8], lo[8];
                ld8(tl + RACC + NPN * lf + j0, v);
                wait_ld();
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    hi[i] = tf32_split_hi(v[i]);
                    lo[i] = v[i] - hi[i];
                }
#pragma unroll
                for (int jj = 0; jj < 8; jj += 4) {
                    const uint32_t o = kmaj_off<NPK>(e, j0 + jj) / 4;
                    *reinterpret_cast<float4 *>(sA + lf * ME * NPK + o) = make_float4(hi[jj], hi[jj + 1], hi[jj + 2], hi[jj + 3]);
                    *reinterpret_cast<float4 *>(sA + (2 + lf) * ME * NPK + o) = make_float4(lo[jj], lo[jj + 1], lo[jj + 2], lo[jj + 3]);
                }
                ld8(tl + RACC + NPN * (2 + lf) + j0, v);
                wait_ld();
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    hi[i] = tf32_split_hi(v[i]);
                    lo[i] = v[i] - hi[i];
                }
                st8(tl + RA1 + NPK * lf + j0, hi);
                st8(tl + RA1 + 2 * NPK + NPK * lf + j0, lo);
            }
            wait_st();
        }
        to_mma(B_R, true);
        {   // L2 prefetch while the update runs on the tensor core: this tile's res rows
            // (read by the LSRK write) and the fields, neighbour tables and first
            // geometric-factor chunk of the tile that will most likely start on this SM
            // next (launch order: one resident CTA per SM)
            const size_t nxt = blk + gridDim.x;                  // this CTA's next tile
            const bool has_next = nxt < (size_t)block_end;
            const int t512 = warp * 32 + lane;                   // 0..511
            auto pf = [](const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); };
            for (int r = t512; r < 4 * NP * 4; r += 512) {     // 4 x 128 B lines per 512 B row
                const size_t row = r >> 2, off = (r & 3) * 32;
                pf(res + row * S + kblk + off);
                if constexpr (LAY & 1) {     // next tile: 4 contiguous runs of 128 Np floats
                    const size_t c = r / (NP * 4), ln = r % (NP * 4);
                    if (has_next && nxt * ME < (size_t)P.K)
                        pf(Qin + (c * P.K + nxt * ME) * NP + ln * 32);
                } else {
                    if (has_next) pf(Qin + row * S + nxt * ME + off);
                }
            }
            if (has_next) {
                for (int r = t512; r < 2 * NF * 4; r += 512) {
                    const int row = r >> 2, off = (r & 3) * 32;
                    pf((row < NF ? P.nbr + (size_t)row * S : P.ncode + (size_t)(row - NF) * S) + nxt * ME + off);
                }
                constexpr int GQ4n = NCH * 4;
                for (int r = t512; r < 9 * 4 * 16; r += 512) {  // chunk 0: 4 float4 rows of 2 KB per factor
                    const int gr = r / 64, q4 = (r / 16) % 4, ln = r % 16;
                    pf(reinterpret_cast<const float4 *>(P.geo_il) + ((nxt * 9 + gr) * GQ4n + q4) * ME + ln * 8);
                }
            }
        }
        for (int u = 0; u < NCHU; ++u) {
            float wa[8], wb[8];
#pragma unroll
            for (int p = 0; p < 8; ++p) { wa[p] = w0[p]; wb[p] = w1[p]; }
            if (u + 1 < NCHU) load_w(u + 1);
            wait_A();                        // chain 0: U1(u) done (and U2(u-1))
            {
                float z[8];
                ld8(tl + Z0 + 16 * lf + pb, z);
                wait_ld();
#pragma unroll
                for (int i = 0; i < 8; ++i) z[i] *= wa[i];
                st_split8(tl + UA0H + 16 * lf + pb, tl + UA0L + 16 * lf + pb, z);
                wait_st();
            }
            to_mma(B_Z0);
            wait_B();                        // chain 1: U1(u) done (and U2(u-1))
            {
                float z[8];
                ld8(tl + Z1 + 16 * lf + pb, z);
                wait_ld();
#pragma unroll
                for (int i = 0; i < 8; ++i) z[i] *= wb[i];
                st_split8(tl + UA1H + 16 * lf + pb, tl + UA1L + 16 * lf + pb, z);
                wait_st();
            }
            to_mma(B_Z1);
        }
        // the first pass's old res values (and w-bar) load while the last U2 MMAs run
        float rv0[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            rv0[i] = (a_rk != 0.f && i < NP) ? __ldg(res + (size_t)(sub * NP + i) * S + kblk + e) : 0.f;
        const float wb = P.wbar ? __ldg(P.wbar + (size_t)(sub == 0 ? 1 : 0) * S + kblk + e) : 0.f;
        wait_A();                            // U2 of the last chunk, chain 0
        wait_B();                            // U2 of the last chunk
        UMMA_MARK0(4);
        // res = a res + dt Minv(rhs); Q_out = Q_in + b res   (field c = sub)
        {
            const int c = sub;
            // WADG update = wbar R + (tensor-core deviation term in RACC); the
            // pre-update R of pair 0 is in shared memory (hi, lo), of pair 1 in TMEM
            // 16 nodes per pass: the old res values are all loaded before the first
            // store (one load latency per pass instead of one per node)
#pragma unroll
            for (int h0 = 0; h0 < NPK; h0 += 16) {
                float rv[16], v[16] = {}, rh[16] = {}, rl[16] = {};
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int j = h0 + i;
                    if (h0 == 0)
                        rv[i] = rv0[i];
                    else
                        rv[i] = (a_rk != 0.f && j < NP) ? __ldg(res + (size_t)(c * NP + j) * S + kblk + e) : 0.f;
                }
#pragma unroll
                for (int hh = 0; hh < 16; hh += 8) {
                    if (h0 + hh < NPK) {
                        float v8[8];
                        ld8(tl + RACC + NPN * c + h0 + hh, v8);
#pragma unroll
                        for (int i = 0; i < 8; ++i) v[hh + i] = v8[i];
                        if (c >= 2) {
                            ld8(tl + RA1 + NPK * (c - 2) + h0 + hh, v8);
#pragma unroll
                            for (int i = 0; i < 8; ++i) rh[hh + i] = v8[i];
                            ld8(tl + RA1 + 2 * NPK + NPK * (c - 2) + h0 + hh, v8);
#pragma unroll
                            for (int i = 0; i < 8; ++i) rl[hh + i] = v8[i];
                        } else {
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                const uint32_t o = kmaj_off<NPK>(e, h0 + hh + i) / 4;
                                rh[hh + i] = sA[c * ME * NPK + o];
                                rl[hh + i] = sA[(2 + c) * ME * NPK + o];
                            }
                        }
                    }
                }
                wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = fmaf(wb, rh[i] + rl[i], v[i]);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int j = h0 + i;
                    if (j < NP) {
                        const size_t o = (size_t)(c * NP + j) * S + kblk + e;
                        const float r = (a_rk == 0.f) ? dt * v[i] : a_rk * rv[i] + dt * v[i];
                        res[o] = r;
                        const uint32_t so = c * ME * NPK + kmaj_off<NPK>(e, j) / 4;
                        const float q = sQ[so] + b_rk * r;
                        if constexpr (LAY & 2)
                            sQ[so] = q;      // in place (this thread's own entry), stored below
                        else
                            Qout[o] = q;
                    }
                }
            }
            if constexpr (LAY & 2) {   // row layout: the warp's 32 elements of field c, one coalesced run
                __syncwarp();
                const long long e0 = (long long)kblk + 32 * qd;
                const int cnt = (int)max(0LL, min(32LL, (long long)P.K - e0)) * NP;
                float *dst = Qout + ((size_t)c * P.K + e0) * NP;
                for (int t = lane; t < cnt; t += 32) {
                    const int el = t / NP, j = t - el * NP;
                    dst[t] = sQ[c * ME * NPK + kmaj_off<NPK>(32 * qd + el, j) / 4];
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    UMMA_MARK0(5);
    if constexpr (!C::PERSIST) break;
    blk += gridDim.x;
    if (blk >= (size_t)block_end) break;
    }   // tiles
    if (warp == 0) tmem_dealloc<512>(tm);
}

}  // namespace uk
}  // namespace wadg
