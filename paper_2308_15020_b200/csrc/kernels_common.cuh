// kernels_common.cuh -- device helpers shared by the eval and solve kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffsat {
namespace dev {

// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic-serialization attribute may
// start while its predecessor drains; pdl_wait() blocks until the predecessor grid has completed and its memory
// is visible (a no-op for a normal launch), pdl_trigger() lets this grid's dependents be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ float fmaT(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmaT(double a, double b, double c) { return ::fma(a, b, c); }
__device__ __forceinline__ float clamp1(float v) { return fminf(fmaxf(v, -1.0f), 1.0f); }
__device__ __forceinline__ double clamp1(double v) { return fmin(fmax(v, -1.0), 1.0); }

template <typename T>
struct cplx {
    T re, im;
};
template <typename T>
__device__ __forceinline__ cplx<T> cmul(const cplx<T>& a, const cplx<T>& b) {
    return {fmaT(a.re, b.re, -a.im * b.im), fmaT(a.re, b.im, a.im * b.re)};
}

__device__ __forceinline__ bool rule_sat(int t, int tmin, int tmax, int parity) {
    bool ok = t >= tmin && t <= tmax;
    if (parity == 1) ok = ok && (t & 1);
    if (parity == 2) ok = ok && !(t & 1);
    return ok;
}

// ---- device images of the host layout (uploaded by ffsat.cu)
struct FastBucketDev {
    int32_t k, kp, nch, pad0;
    int64_t pos_begin, word_off, slot_off;
    double g0;
    double c0[2], c1[2], g[2];   // channel factor a = c0 + c1 * l, FE += g * prod a
    int32_t tmin, tmax, parity;
    int32_t red;                 // satisfaction as a bit reduction of the literals' truth bits (wide kernel):
                                 // 1 any-true (OR), 2 all-true (AND), 3 parity (XOR); +4: satisfied iff the
                                 // reduced bit is 0 (NOR / NAND / XNOR); 0 = count True literals
};

struct UnitDev {                 // a run of constraints of one bucket at positions [pos_begin, pos_begin + count)
    int32_t bucket;              // (tiled path: a var-disjoint class); 16 bytes so a header prefetch is 4 registers
    int32_t count_kp;            // count | kp << 16 (kp = literal words per constraint row of the bucket)
    int32_t pos_begin;
    int32_t word_begin;          // first literal word of the unit (rows of kp words, contiguous)
};
__device__ __forceinline__ int unit_count(const UnitDev& u) { return u.count_kp & 0xffff; }
__device__ __forceinline__ int unit_kp(const UnitDev& u) { return u.count_kp >> 16; }

struct SymSigDev {
    int32_t k, Mp, tmin, tmax, parity, pad;
    int64_t coef_off;
    double g0;
};


}  // namespace dev
}  // namespace ffsat
