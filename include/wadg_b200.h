/*
 * wadg_b200.h — C ABI of the B200-native WADG right-hand-side / LSRK45 path.
 *
 * The reference (arXiv 1608.03836 restated as the Python package `wadg`) has
 * no FFI: its boundary is the Python API of wadg.solver.  Each entry point
 * below replaces one of those functions (or the array kernel inside it) for
 * device-resident data; the Python drop-in (paper_1608_03836_b200.solver)
 * binds them with ctypes (INTEGRATION.md shows the binding):
 *
 *   wadg_volume        <- solver._volume_terms            R/pkg/src/wadg/solver.py:241-265
 *   wadg_surface       <- solver._surface_terms + face_traces  solver.py:195-238
 *   wadg_mass_inverse  <- solver.apply_mass_inverse (WADG)     solver.py:290-301
 *                         -> operators.apply_weight_adjusted_inverse operators.py:45-61
 *   wadg_update_lsrk   <- apply_mass_inverse fused with the LSRK stage axpy
 *                         of solver.lsrk_step                  solver.py:348-363
 *   wadg_stage         <- one LSRK stage of lsrk_step(state, dt, rhs_full)
 *                         = volume + surface + update_lsrk
 *   wadg_lsrk_axpy     <- the stage axpy of lsrk_step for an arbitrary rhs_fn
 *   wadg_energy        <- solver.energy                        solver.py:314-321
 *   wadg_pack_halo     <- (new) face-trace halo for element slabs; no reference counterpart
 *
 * Conventions: plain pointers and sizes only.  All array pointers are device
 * pointers in the dtype named by `dtype` (WADG_F64 / WADG_F32) unless typed
 * int32_t.  Element index is the fastest (stride-1) dimension of every
 * per-element array, padded to Kpad (a multiple of WADG_ELEMS_PER_BLOCK).
 * Kernels never allocate and never synchronise; `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Return 0 on success, nonzero on error
 * with a message in wadg_last_error() (thread-local).
 */
#ifndef WADG_B200_H
#define WADG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WADG_ABI_VERSION 6
#define WADG_ELEMS_PER_BLOCK 32

enum { WADG_F64 = 0, WADG_F32 = 1 };
enum { WADG_STRONG = 0, WADG_STRONG_WEAK = 1 };

typedef struct wadg_problem {
    /* sizes */
    int32_t dim;          /* 2 or 3; fields = dim + 1 (p, u_1..u_dim) */
    int32_t dtype;        /* WADG_F64 | WADG_F32 */
    int32_t K, Kpad;      /* elements, padded element stride */
    int32_t Np, Nq, Nqu;  /* nodes, volume quad points, update quad points */
    int32_t Nf, Nfp, Nfq; /* faces, nodes per face, quad points per face */
    int32_t n_orient;     /* face orientation codes (2 in 2D, 6 in 3D) */
    int32_t formulation;  /* WADG_STRONG | WADG_STRONG_WEAK */
    /* reference operators, row-major */
    const void *Vq;       /* [Nq][Np]      volume interpolation            */
    const void *Dq;       /* [dim][Nq][Np] reference derivatives at quad   */
    const void *Pq;       /* [Np][Nq]      Mhat^-1 Vq^T W                  */
    const void *DTW;      /* [dim][Np][Nq] Mhat^-1 D_a^T W (strong-weak p) */
    const void *Vu;       /* [Nqu][Np]     update-rule interpolation       */
    const void *Pu;       /* [Np][Nqu]     update-rule projection          */
    const void *Vfi;      /* [Nfq][Nfp]    face nodes -> face quad points  */
    const void *Pf;       /* [Np][Nf*Nfq]  Mhat^-1 Vf^T Wf (lift)          */
    const int32_t *fmask;    /* [Nf][Nfp] volume node of each face node            */
    const int32_t *ext_node; /* [Nf*n_orient][Nfp] neighbour volume node, by code  */
    const int32_t *fperm;    /* [n_orient][Nfp] face-node permutation, by orient.  */
    /* per-element data, element index fastest */
    const void *geo;      /* [dim*dim][Nq][Kpad]  (dr_a/dx_i) J, row a*dim+i      */
    const void *fgeo;     /* [dim+1][Nf*Nfq][Kpad] n_1..n_dim, sJ/2               */
    const void *wu;       /* [Nqu][Kpad] 1/J at update points                     */
    const void *wp;       /* [Nqu][Kpad] c^2/J, or NULL: use c2 * wu             */
    double c2;            /* constant c^2 when wp == NULL                         */
    const int32_t *nbr;   /* [Nf][Kpad] neighbour element; -1 = Dirichlet mirror;
                             <= -2 = halo slot (-nbr-2)                          */
    const int32_t *ncode; /* [Nf][Kpad] nbr face * n_orient + orientation        */
    /* halo face traces from other ranks: [n_halo][dim+1][Nfp] (sender order)  */
    const void *halo;
    int32_t n_halo;
    /* energy quadrature (diagnostics) */
    int32_t Ne;
    const void *Ve;       /* [Ne][Np] */
    const void *we;       /* [Ne]     */
    const void *ewp;      /* [Ne][Kpad] */
    const void *ewu;      /* [Ne][Kpad] */
    int32_t e_recip;      /* 1: weights are we/ew*, 0: we*ew*                     */
    /* fused tetrahedral stage (wadg_stage_fused): polynomial order and the
     * operators repacked into quadrature chunks of QC points (see
     * wadg_fused_config), NPP = Np rounded up to 4, zero padded:          */
    int32_t order;
    int32_t fused_kind;   /* kernel the operators below are packed for: 0 CUDA cores, 2 tcgen05,
                           * 3 FP64 DMMA, 4 split-TF32 mma.sync (fp32, N >= 5),
                           * 5 N = 1 thread-per-element registers (opVA: one image)     */
    const void *opVA;     /* D_r, D_s, D_t, Vq at (q, j)   (layout: wadg_fused_config) */
    const void *opVB;     /* DTW_r, DTW_s, DTW_t, Pq at (j, q)                         */
    const void *opU1;     /* Vu                                                        */
    const void *opU2;     /* Pu                                                        */
    const void *liftT;    /* Pf transposed                                             */
    /* tcgen05 stage (kind 2): per-element data interleaved by 128-element
     * blocks with 4 consecutive points per element, so that a thread loads 4
     * points of its element with one 16-byte load and a warp reads 512
     * contiguous bytes:  X_il[blk][row][point/4][128][4], points zero padded
     * (geo: rows = dim*dim, points = Nq padded to 16; fgeo: rows = (dim+1)*Nf,
     * points per face padded to 16; wu/wp: one row, points padded to 32).   */
    const void *geo_il;
    const void *fgeo_il;
    const void *wu_il;
    const void *wp_il;    /* NULL when wp is NULL */
    /* tcgen05 stage: per element mean update weight, [2][Kpad]: row 0 the mean
     * of 1/J, row 1 the mean of c^2/J over the update points.  When not NULL,
     * wu_il / wp_il hold the deviations w - wbar and the stage forms the WADG
     * update as wbar R + Pu((w - wbar) Vu R) (exact, since Pu Vu = I); the
     * tensor core then accumulates only the small deviation term, which keeps
     * its round-toward-zero accumulation error small.  NULL: wu_il / wp_il
     * hold the full weights.                                               */
    const void *wbar;
    /* ExactCurvedMass comparator (R/.../solver.py:156-167, 302-306): when minv_p
     * is not NULL, wadg_mass_inverse / wadg_update_lsrk / wadg_stage apply the
     * stored dense per-element operators A_k = M_k^-1 Mhat (M_k the J/c^2- and
     * J-weighted mass matrices at quadrature degree 2N + 2N_geo) instead of the
     * matrix-free WADG inverse:  [Np][Np][Kpad] each, row j, column l.      */
    const void *minv_p;
    const void *minv_u;
} wadg_problem;

int wadg_abi_version(void);
const char *wadg_last_error(void);

/* rhs = volume term of the Mhat^-1-premultiplied RHS (overwrites rhs) */
int wadg_volume(const wadg_problem *P, const void *Q, void *rhs, void *stream);

/* rhs (+)= surface term over element blocks [block_begin, block_end) (units of
 * WADG_ELEMS_PER_BLOCK); block_end < 0 means all blocks */
int wadg_surface(const wadg_problem *P, const void *Q, void *rhs, double tau_p,
                 double tau_u, int accumulate, int block_begin, int block_end,
                 void *stream);

/* out = WADG mass inverse of a premultiplied rhs */
int wadg_mass_inverse(const wadg_problem *P, const void *rhs, void *out, void *stream);

/* res = a*res + dt*Minv(rhs); Q += b*res  (a == 0 ignores the old res) */
int wadg_update_lsrk(const wadg_problem *P, const void *rhs, void *res, void *Q,
                     double a, double b, double dt, void *stream);

/* one LSRK stage: volume -> surface -> update_lsrk (rhs is scratch) */
int wadg_stage(const wadg_problem *P, void *Q, void *res, void *rhs, double tau_p,
               double tau_u, double a, double b, double dt, void *stream);

/* generic stage axpy over n entries: res = a*res + dt*d; Q += b*res */
int wadg_lsrk_axpy(int dtype, int64_t n, const void *d, void *res, void *Q,
                   double a, double b, double dt, void *stream);

/* energy: partials must hold ceil(Kpad/32) doubles; writes the total to
 * out_dev[0] (device double) */
int wadg_energy(const wadg_problem *P, const void *Q, double *partials,
                double *out_dev, void *stream);

/* Layout of the fused tetrahedral stage for (dtype, order), which decides how
 * the host packs opVA/opVB/opU1/opU2/liftT:
 *   info[0] kind: 0 = CUDA-core kernel ([nch][NPP][QC][4], [nch][QC][NPP][4],
 *                 [nch][NPP][QC], [nch][QC][NPP], [Nf*Nfq][NPP]);
 *                 2 = tcgen05 kernel (one buffer of K-major tile images);
 *                 3 = DMMA kernel (one buffer of fragment-order images);
 *                 4 = split-TF32 mma.sync kernel (one buffer of fragment-order
 *                     hi / lo images);
 *                 5 = N = 1 thread-per-element kernel (one 464-value operator
 *                     image, device.reg_operator_image; no dynamic shared memory)
 *   info[1] elements per CTA, [2] QC, [3] nch, [4] NPP (K extent over nodes),
 *   info[5], [6], [7]: kernel-specific extents (device.py reads them).
 * Returns nonzero if the pair is not compiled / does not fit. */
int wadg_fused_config(int dtype, int order, int32_t *info, int64_t *smem_bytes);

/* The same for a formulation (WADG_STRONG_WEAK or WADG_STRONG).  The strong
 * form (the sufficiency rules at N_geo = N) has fused stages at N = 1 (the
 * register stage, kind 5, both precisions) and N = 2..5: fp64 on the FP64
 * tensor cores (kind 3), fp32 on split-TF32 mma.sync (kind 4); other pairs
 * return nonzero. */
int wadg_fused_config_form(int dtype, int order, int formulation, int32_t *info, int64_t *smem_bytes);

/* Debug: force the fused-stage kernel (0: CUDA-core FMA tiles, 2: split-TF32
 * tcgen05 with TMEM accumulators, 3: FP64 DMMA, 4: split-TF32 mma.sync m16n8k8,
 * 5: N = 1 thread-per-element registers, where available); -1 restores
 * the default.  Affects
 * wadg_fused_config, so set it before building a problem. */
int wadg_debug_set_fused_variant(int variant);

/* One whole LSRK stage for tetrahedra in a single kernel (strong-weak, or the
 * strong form where wadg_fused_config_form reports a kernel):
 * Q_out = Q_in + b*res, res = a*res + dt*Minv(volume + surface)(Q_in).
 * Q_in and Q_out must be different buffers (ping-pong).  Blocks are in units
 * of the fused elems_per_block; block_end < 0 means all. */
int wadg_stage_fused(const wadg_problem *P, const void *Q_in, void *Q_out, void *res,
                     double tau_p, double tau_u, double a, double b, double dt,
                     int block_begin, int block_end, void *stream);

/* wadg_stage_fused with fields in the host row layout (see
 * wadg_rows_to_fields): layout 1 = Q_in is (dim+1, K, Np) (the first stage of
 * a step on a host state), 2 = Q_out is (the last stage).  res stays in the
 * field layout.  Only the tcgen05 stage (fp32, N = 2..4) supports 1 and 2;
 * otherwise it fails and the caller converts with wadg_rows_to_fields. */
int wadg_stage_fused_rows(const wadg_problem *P, const void *Q_in, void *Q_out, void *res,
                          double tau_p, double tau_u, double a, double b, double dt,
                          int block_begin, int block_end, int layout, void *stream);

/* Debug: when buf != NULL, each CTA of subsequent wadg_stage_fused launches
 * writes clock64() at 7 phase boundaries to buf[cta*8 + 0..6] (int64). */
int wadg_debug_set_phase_clock_buffer(void *buf);

/* Measurement support: `blocks` x 256 threads, each running 16 independent
 * register-operand FMA chains for `iters` iterations (2*16*iters flops per
 * thread); `in` holds >= 32 values of the dtype, `out` >= 256. */
int wadg_microbench_fma(int dtype, int blocks, int iters, const void *in, void *out, void *stream);

/* Debug: validate the tcgen05 split-TF32 primitives. One CTA computes
 * C (128 x N) = A (128 x K) B^T (row-major fp32 device arrays); mode bit 0: raw
 * fp32 hi operands, bit 1: A_lo from TMEM, bit 2: plain TF32 (one MMA). */
int wadg_debug_umma_test(const void *A, const void *B, void *C, int N, int K, int mode, void *stream);

/* buf[(s*(dim+1) + fld)*Nfp + i] = Q[fld][fmask[send_f[s]][i]][send_k[s]] */
int wadg_pack_halo(const wadg_problem *P, const void *Q, const int32_t *send_k,
                   const int32_t *send_f, int32_t n_send, void *buf, void *stream);

/* Host-layout conversion for element range [k0, k1) (the pipelined
 * host-state LSRK step): `rows` is the FieldState layout, (dim+1) fields of
 * (K, Np) row-major (R/pkg/src/wadg/solver.py:94 FieldState), dense on the
 * device; Q the (dim+1, Np, Kpad) field layout.  Only [k0, k1) is touched. */
int wadg_rows_to_fields(const wadg_problem *P, const void *rows, int32_t k0, int32_t k1, void *Q,
                        void *stream);
int wadg_fields_to_rows(const wadg_problem *P, const void *Q, int32_t k0, int32_t k1, void *rows,
                        void *stream);

/* Debug / measurement: tcgen05.mma issue rate.  One CTA, one warp issues
 * `count` kind::tf32 MMAs (M = 128, K = 8, N = n) back to back; out[0] =
 * clock64 cycles of the issue loop, out[1] = until the commit completed.
 * mode 0: A from shared memory, 1: A from TMEM, 2: as 0, 8 MMAs per asm block. */
int wadg_debug_umma_rate(void *out, int n, int count, int mode, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* WADG_B200_H */
