// Rounding of mma.sync.m16n8k8 tf32 accumulation on sm_100a (debug probe):
// C[16x8] = A[16xK] B[Kx8], split-TF32 (3 MMAs per k step), one warp.
// mode 0: chained accumulation in C; mode 1: each k step into a fresh C, added in fp32 (RN).
#include <cstdint>
__device__ __forceinline__ uint32_t tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__global__ void k(const float *A, const float *B, float *C, int K, int mode) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    float acc[4] = {0, 0, 0, 0};
    for (int k0 = 0; k0 < K; k0 += 8) {
        float av[4] = {A[g * K + k0 + t], A[(g + 8) * K + k0 + t], A[g * K + k0 + t + 4], A[(g + 8) * K + k0 + t + 4]};
        float bv[2] = {B[(k0 + t) * 8 + g], B[(k0 + t + 4) * 8 + g]};
        uint32_t ah[4], al[4], bh[2], bl[2];
        for (int i = 0; i < 4; ++i) { ah[i] = tf32_rn(av[i]); al[i] = tf32_rn(av[i] - __uint_as_float(ah[i])); }
        for (int i = 0; i < 2; ++i) { bh[i] = tf32_rn(bv[i]); bl[i] = tf32_rn(bv[i] - __uint_as_float(bh[i])); }
        if (mode == 0) {
            hmma(acc, al, bh); hmma(acc, ah, bl); hmma(acc, ah, bh);
        } else {
            float d[4] = {0, 0, 0, 0};
            hmma(d, al, bh); hmma(d, ah, bl); hmma(d, ah, bh);
            for (int i = 0; i < 4; ++i) acc[i] += d[i];
        }
    }
    C[g * 8 + 2 * t] = acc[0]; C[g * 8 + 2 * t + 1] = acc[1];
    C[(g + 8) * 8 + 2 * t] = acc[2]; C[(g + 8) * 8 + 2 * t + 1] = acc[3];
}
extern "C" int hmma_probe(const float *A, const float *B, float *C, int K, int mode) {
    k<<<1, 32>>>(A, B, C, K, mode);
    return (int)cudaDeviceSynchronize();
}
