// dmsgm_pair.cuh -- paired fp32 arithmetic for sm_100a (device only).
#pragma once
#include <cuda_runtime.h>

namespace dmsgm {

// Paired fp32 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2): each lane is one IEEE
// round-to-nearest operation, bitwise equal to the scalar __f*_rn; a scalar operand
// (make_float2(s, s)) becomes the instruction's broadcast operand.  Used where the
// canonical order applies the same operation to the apparent and candidate model (x = A,
// y = C) or to the two coordinates of the projection.
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
    float2 r;
    asm("{.reg .b64 ta, tb, tc, td;\n\tmov.b64 ta, {%2, %3};\n\tmov.b64 tb, {%4, %5};\n\tmov.b64 tc, {%6, %7};\n\t"
        "fma.rn.f32x2 td, ta, tb, tc;\n\tmov.b64 {%0, %1}, td;}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
    float2 r;
    asm("{.reg .b64 ta, tb, td;\n\tmov.b64 ta, {%2, %3};\n\tmov.b64 tb, {%4, %5};\n\t"
        "mul.rn.f32x2 td, ta, tb;\n\tmov.b64 {%0, %1}, td;}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
    float2 r;
    asm("{.reg .b64 ta, tb, td;\n\tmov.b64 ta, {%2, %3};\n\tmov.b64 tb, {%4, %5};\n\t"
        "add.rn.f32x2 td, ta, tb;\n\tmov.b64 {%0, %1}, td;}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
    float2 r;
    asm("{.reg .b64 ta, tb, td;\n\tmov.b64 ta, {%2, %3};\n\tmov.b64 tb, {%4, %5};\n\t"
        "sub.rn.f32x2 td, ta, tb;\n\tmov.b64 {%0, %1}, td;}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 f2_bc(float s) { return make_float2(s, s); }

// ptxas contracts a paired multiply whose result feeds a paired add (mul.rn.f32x2 or
// fma.rn.f32x2(a, b, -0) followed by add.rn.f32x2 becomes one FFMA2) despite the explicit
// .rn, which the scalar forms honour; it does not contract when the two flush-to-zero
// modes differ.  Where a paired product feeds a paired add, one of the two is therefore
// the .ftz form below -- chosen where flushing a subnormal provably cannot change the
// result (stated at each use).
__device__ __forceinline__ float2 f2_mul_ftz(float2 a, float2 b) {
    float2 r;
    asm("{.reg .b64 ta, tb, td;\n\tmov.b64 ta, {%2, %3};\n\tmov.b64 tb, {%4, %5};\n\t"
        "mul.rn.ftz.f32x2 td, ta, tb;\n\tmov.b64 {%0, %1}, td;}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 f2_add_ftz(float2 a, float2 b) {
    float2 r;
    asm("{.reg .b64 ta, tb, td;\n\tmov.b64 ta, {%2, %3};\n\tmov.b64 tb, {%4, %5};\n\t"
        "add.rn.ftz.f32x2 td, ta, tb;\n\tmov.b64 {%0, %1}, td;}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}

// x + y with round-toward-zero in both lanes (FADD2.RZ); with a magic addend in
// [2^23, 2^24) it yields floor() of a small value as an exact float whose bits hold the
// integer (the frame-warp kernel's floor without F2I / FRND conversions).
__device__ __forceinline__ float2 f2_add_rz(float2 a, float2 b) {
    float2 r;
    asm("{.reg .b64 ta, tb, td;\n\tmov.b64 ta, {%2, %3};\n\tmov.b64 tb, {%4, %5};\n\t"
        "add.rz.f32x2 td, ta, tb;\n\tmov.b64 {%0, %1}, td;}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}

}  // namespace dmsgm
