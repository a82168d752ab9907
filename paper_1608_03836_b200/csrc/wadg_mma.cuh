// Warp-level split-TF32 ("3xTF32") tensor-core MMA for the fp32 fused stage.
//
// mma.sync.m16n8k8 TF32 fragments (per PTX ISA; g = lane / 4, t = lane % 4):
//   A 16x8 row-major:  a0 (g, t)  a1 (g+8, t)  a2 (g, t+4)  a3 (g+8, t+4)
//   B 8x8 (k x n):     b0 (t, g)  b1 (t+4, g)
//   C 16x8:            c0 (g, 2t) c1 (g, 2t+1) c2 (g+8, 2t) c3 (g+8, 2t+1)
// Each fp32 operand x is split as x = hi + lo with hi = tf32(x), lo = tf32(x - hi);
// C += A_hi B_hi + A_hi B_lo + A_lo B_hi keeps ~fp32 accuracy (the dropped
// A_lo B_lo term is O(2^-22) relative), which the 1e-5 fp32 bar requires
// (plain TF32 operators alone give 3.1e-3).
#pragma once

namespace wadg {
namespace mma {

// Split x = hi + lo with hi = x truncated to a TF32 mantissa (bit mask) and
// lo = x - hi computed exactly in fp32; the MMA truncates lo to TF32 itself,
// so the representation error is O(2^-22 |x|).  Two instructions, no cvt.
struct Split {
    uint32_t hi, lo;
};

__device__ __forceinline__ Split split(float x) {
    Split s;
    s.hi = __float_as_uint(x) & 0xffffe000u;
    s.lo = __float_as_uint(x - __uint_as_float(s.hi));
    return s;
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    // not volatile: independent accumulator chains may be interleaved by the scheduler
    asm(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// A fragment (split) from a column-major-in-smem tile: element (row r, col k)
// at base[k * ld + r]  (our layouts keep the element index contiguous).
struct AFrag {
    uint32_t hi[4], lo[4];
};
struct BFrag {
    uint32_t hi[2], lo[2];
};

__device__ __forceinline__ void load_a_colmajor(AFrag &f, const float *base, int ld, int lane) {
    const float *p = base + (lane & 3) * ld + (lane >> 2);
    const float x0 = p[0], x1 = p[8];
    const float x2 = p[4 * ld], x3 = p[4 * ld + 8];
    Split s;
    s = split(x0); f.hi[0] = s.hi; f.lo[0] = s.lo;
    s = split(x1); f.hi[1] = s.hi; f.lo[1] = s.lo;
    s = split(x2); f.hi[2] = s.hi; f.lo[2] = s.lo;
    s = split(x3); f.hi[3] = s.hi; f.lo[3] = s.lo;
}

// B fragment: element (k, n) at base[k * ld + n]
__device__ __forceinline__ void load_b_rowmajor(BFrag &f, const float *base, int ld, int lane) {
    const float *p = base + (lane & 3) * ld + (lane >> 2);
    Split s;
    s = split(p[0]); f.hi[0] = s.hi; f.lo[0] = s.lo;
    s = split(p[4 * ld]); f.hi[1] = s.hi; f.lo[1] = s.lo;
}

__device__ __forceinline__ void mma3(float (&c)[4], const AFrag &a, const BFrag &b) {
    mma_tf32(c, a.lo, b.hi);
    mma_tf32(c, a.hi, b.lo);
    mma_tf32(c, a.hi, b.hi);
}

// C[n] += A B[n] for NT independent accumulators, issued pass by pass so that
// consecutive MMAs never depend on each other
template <int NT>
__device__ __forceinline__ void mma3_row(float (&c)[NT][4], const AFrag &a, const BFrag (&b)[NT]) {
#pragma unroll
    for (int n = 0; n < NT; ++n) mma_tf32(c[n], a.lo, b[n].hi);
#pragma unroll
    for (int n = 0; n < NT; ++n) mma_tf32(c[n], a.hi, b[n].lo);
#pragma unroll
    for (int n = 0; n < NT; ++n) mma_tf32(c[n], a.hi, b[n].hi);
}

}  // namespace mma
}  // namespace wadg

namespace wadg {
namespace mma {

// c[m][n] += A[m] B[n]: MF x NT independent accumulators, split passes
// interleaved across all of them (no back-to-back dependent MMAs)
template <int MF, int NT>
__device__ __forceinline__ void mma3_AB(float (&c)[MF][NT][4], const AFrag (&a)[MF], const BFrag (&b)[NT]) {
#pragma unroll
    for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[m][n], a[m].lo, b[n].hi);
#pragma unroll
    for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[m][n], a[m].hi, b[n].lo);
#pragma unroll
    for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[m][n], a[m].hi, b[n].hi);
}

// c[m][n] += A B[m][n]
template <int MF, int NT>
__device__ __forceinline__ void mma3_aB(float (&c)[MF][NT][4], const AFrag &a, const BFrag (&b)[MF][NT]) {
#pragma unroll
    for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[m][n], a.lo, b[m][n].hi);
#pragma unroll
    for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[m][n], a.hi, b[m][n].lo);
#pragma unroll
    for (int m = 0; m < MF; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[m][n], a.hi, b[m][n].hi);
}

// c[n] += sum_k A[k] B[k][n]
template <int KA, int NT>
__device__ __forceinline__ void mma3_sum(float (&c)[NT][4], const AFrag (&a)[KA], const BFrag (&b)[KA][NT]) {
#pragma unroll
    for (int k = 0; k < KA; ++k)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[n], a[k].lo, b[k][n].hi);
#pragma unroll
    for (int k = 0; k < KA; ++k)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[n], a[k].hi, b[k][n].lo);
#pragma unroll
    for (int k = 0; k < KA; ++k)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_tf32(c[n], a[k].hi, b[k][n].hi);
}

}  // namespace mma
}  // namespace wadg
