// pmg_otpw.cuh — hand-written sm_100a device primitives of the OTPW + hybrid-tiling group kernels.
//
// Included (from memory, by NVRTC) by every generated group kernel.  Everything here is warp-scoped:
// an overlapped tile is owned by ONE warp (§3, §4), so the only
// synchronisation is __syncwarp / per-warp mbarriers — no block barrier (bar.sync) is ever emitted.
//
//  * TMA 1-D bulk copies (cp.async.bulk ... mbarrier::complete_tx) stage input rows (tile + halo) into a
//    warp-private shared-memory ring; completion is tracked by one mbarrier per ring slot.
//  * shuffles implement the paper's producer-load types (3) and (4) (Fig. 4; Fig. 7 lines
//    757-799): a neighbour lane's register in the same parallelogram (chunk) tile, or the last lanes of
//    the previous chunk; one shuffle per exchanged element (the sender pre-selects the chunk).
//  * exact-IEEE f32 helpers (round-to-nearest per op, no contraction) so fused results are bit-identical
//    to the stage-by-stage definition (reading R3).
#pragma once

typedef unsigned int u32;
typedef unsigned long long u64;
typedef long long i64;

#define PMG_FULL 0xffffffffu

struct PmgTensor {           // one planar [c][y][x] device tensor (56 bytes; mirrored in runtime.cpp)
  const char* ptr;
  i64 row_pitch;             // bytes
  i64 plane_pitch;           // bytes
  i64 frame_stride;          // bytes between batch frames (0 for tables / single images)
  int row_base;              // global row index of buffer row 0 (bands)
  int nrows;                 // rows present in the buffer: stores outside [row_base, row_base + nrows) are dropped
  int H, W;                  // full extent of the tensor's image (rows, columns): clamping of scaled reads
  int pad0_, pad1_;
};

// ------------------------------------------------------------------ float semantics (reading R3)
__device__ __forceinline__ float pmg_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float pmg_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float pmg_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float pmg_div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float pmg_sqrt(float a) { return __fsqrt_rn(a); }
// a + (m * b) where m = 2^k (k >= 0): m*b is exact, so one rounding == the written two roundings
__device__ __forceinline__ float pmg_fma_exact(float m, float b, float a) { return __fmaf_rn(m, b, a); }
// packed pairs (sm_100a FADD2 / FMUL2 / FFMA2): two elements per instruction, each rounded exactly as
// its scalar counterpart (a - b == a + (-b) exactly in IEEE 754)
__device__ __forceinline__ float2 pmg_add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 pmg_sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 pmg_mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 pmg_fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 pmg_neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 pmg_bc2(float c) { return make_float2(c, c); }
__device__ __forceinline__ float pmg_fmin(float a, float b) { return (b < a) ? b : a; }
__device__ __forceinline__ float pmg_fmax(float a, float b) { return (b > a) ? b : a; }
__device__ __forceinline__ float pmg_i2f(int a) { return __int2float_rn(a); }
// truncate toward zero; cvt.rzi.s32.f32 saturates out-of-range values and maps NaN to 0 (reading R4)
__device__ __forceinline__ int pmg_f2i(float a) { return __float2int_rz(a); }

// ------------------------------------------------------------------ int32 semantics (reading R4)
__device__ __forceinline__ int pmg_iadd(int a, int b) { return (int)((u32)a + (u32)b); }
__device__ __forceinline__ int pmg_isub(int a, int b) { return (int)((u32)a - (u32)b); }
__device__ __forceinline__ int pmg_imul(int a, int b) { return (int)((u32)a * (u32)b); }
__device__ __forceinline__ int pmg_ineg(int a) { return (int)(0u - (u32)a); }
// floor division / divisor-signed remainder (reading R4): x/0 == 0, x%0 == 0, INT_MIN/-1 wraps to INT_MIN
__device__ __forceinline__ int pmg_idiv(int a, int b) {
  if (b == 0) return 0;
  if (b == -1) return pmg_ineg(a);
  int q = a / b;
  return (((a % b) != 0) && ((a < 0) != (b < 0))) ? q - 1 : q;
}
__device__ __forceinline__ int pmg_imod(int a, int b) {
  if (b == 0 || b == -1) return 0;
  int r = a % b;
  return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r;
}
// shift counts are clamped to [0, 32] (reading R4): a<<c = a*2^c mod 2^32, a>>c = floor(a/2^c)
__device__ __forceinline__ int pmg_ishl(int a, int b) { return b <= 0 ? a : (b >= 32 ? 0 : (int)((u32)a << b)); }
__device__ __forceinline__ int pmg_ishr(int a, int b) { return b <= 0 ? a : a >> (b >= 31 ? 31 : b); }
__device__ __forceinline__ int pmg_iabs(int a) { return a < 0 ? pmg_ineg(a) : a; }
__device__ __forceinline__ int pmg_imin(int a, int b) { return (b < a) ? b : a; }
__device__ __forceinline__ int pmg_imax(int a, int b) { return (b > a) ? b : a; }
__device__ __forceinline__ int pmg_clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
__device__ __forceinline__ int pmg_to_u8(int a) { return (int)(unsigned char)a; }
__device__ __forceinline__ int pmg_to_u16(int a) { return (int)(unsigned short)a; }
__device__ __forceinline__ int pmg_to_i16(int a) { return (int)(short)a; }

// ------------------------------------------------------------------ typed loads / stores
template <typename T> struct PmgElem;
template <> struct PmgElem<float> { typedef float C; __device__ static float cv(float v) { return v; } };
template <> struct PmgElem<int> { typedef int C; __device__ static int cv(int v) { return v; } };
template <> struct PmgElem<short> { typedef int C; __device__ static int cv(short v) { return (int)v; } };
template <> struct PmgElem<unsigned short> { typedef int C; __device__ static int cv(unsigned short v) { return (int)v; } };
template <> struct PmgElem<unsigned char> { typedef int C; __device__ static int cv(unsigned char v) { return (int)v; } };

template <typename T>
__device__ __forceinline__ typename PmgElem<T>::C pmg_ldg(const char* base, i64 off_elems) {
  return PmgElem<T>::cv(__ldg(reinterpret_cast<const T*>(base) + off_elems));
}

template <typename T>
__device__ __forceinline__ typename PmgElem<T>::C pmg_lds(const char* smem, int idx) {
  return PmgElem<T>::cv(reinterpret_cast<const T*>(smem)[idx]);
}

// N consecutive elements viewed as one 1/2/4/8/16-byte word (type punning through a union)
template <typename T, int N>
union PmgVec {
  T e[N];
  uint4 w16;
  uint2 w8;
  unsigned w4;
  unsigned short w2;
};

// store N consecutive elements with one vector store (address aligned to N*sizeof(T))
template <typename T, int N>
__device__ __forceinline__ void pmg_stg_vec(char* dst, const T (&v)[N]) {
  constexpr int B = N * (int)sizeof(T);
  if constexpr (B > 16 && B % 32 == 0) {  // V = 8 f32 lanes: two 16-byte stores
    pmg_stg_vec<T, N / 2>(dst, reinterpret_cast<const T(&)[N / 2]>(v));
    pmg_stg_vec<T, N / 2>(dst + B / 2, reinterpret_cast<const T(&)[N / 2]>(v[N / 2]));
    return;
  }
  PmgVec<T, N> u;
#pragma unroll
  for (int i = 0; i < N; ++i) u.e[i] = v[i];
  if constexpr (B == 16) *reinterpret_cast<uint4*>(dst) = u.w16;
  else if constexpr (B == 8) *reinterpret_cast<uint2*>(dst) = u.w8;
  else if constexpr (B == 4) *reinterpret_cast<unsigned*>(dst) = u.w4;
  else if constexpr (B == 2) *reinterpret_cast<unsigned short*>(dst) = u.w2;
  else {
#pragma unroll
    for (int i = 0; i < N; ++i) reinterpret_cast<T*>(dst)[i] = v[i];
  }
}

// one elected lane: proxy fence, expect_tx(total), and one bulk copy (single stream) -- one asm block so that
// ptxas sees a single elect.sync predicate around the uniform-operand copy
__device__ __forceinline__ void pmg_refill1_elect(u32 bar, u32 total, u32 dst, const void* src, u32 bytes) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "@p fence.proxy.async.shared::cta;\n\t"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %4, [%0];\n}"
      ::"r"(bar), "r"(total), "r"(dst), "l"(src), "r"(bytes) : "memory");
}

// the same without the proxy fence -- experiment only (PMG_FENCE=0): without the fence the lanes' reads of the
// slot are not ordered before the bulk copy that overwrites it, and a full-size run lost elements once
__device__ __forceinline__ void pmg_refill1_elect_nf(u32 bar, u32 total, u32 dst, const void* src, u32 bytes) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %4, [%0];\n}"
      ::"r"(bar), "r"(total), "r"(dst), "l"(src), "r"(bytes) : "memory");
}

// N elements at every other position (stride 2): a quad-resolution phase stored straight into its full-resolution
// interleaved liveout (runtime.cpp interleave fusion)
template <typename T, int N>
__device__ __forceinline__ void pmg_stg_str2(char* dst, const T (&v)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) reinterpret_cast<T*>(dst)[2 * i] = v[i];
}
template <typename T, int N>
__device__ __forceinline__ void pmg_stg_str2_if(char* dst, const T (&v)[N], bool p) {
  if (p) pmg_stg_str2<T, N>(dst, v);
}

// predicated vector store (no branch: the interior body stays one basic block)
template <typename T, int N>
__device__ __forceinline__ void pmg_stg_vec_if(char* dst, const T (&v)[N], bool p) {
  constexpr int B = N * (int)sizeof(T);
  if constexpr (B > 16 && B % 32 == 0) {
    pmg_stg_vec_if<T, N / 2>(dst, reinterpret_cast<const T(&)[N / 2]>(v), p);
    pmg_stg_vec_if<T, N / 2>(dst + B / 2, reinterpret_cast<const T(&)[N / 2]>(v[N / 2]), p);
    return;
  }
  PmgVec<T, N> u;
#pragma unroll
  for (int i = 0; i < N; ++i) u.e[i] = v[i];
  if constexpr (B == 16)
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.v4.b32 [%0], {%1, %2, %3, %4};\n}" ::"l"(dst),
                 "r"(u.w16.x), "r"(u.w16.y), "r"(u.w16.z), "r"(u.w16.w), "r"((int)p) : "memory");
  else if constexpr (B == 8)
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.b32 [%0], {%1, %2};\n}" ::"l"(dst),
                 "r"(u.w8.x), "r"(u.w8.y), "r"((int)p) : "memory");
  else if constexpr (B == 4)
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.b32 [%0], %1;\n}" ::"l"(dst), "r"(u.w4),
                 "r"((int)p) : "memory");
  else if (p) pmg_stg_vec<T, N>(dst, v);
}

// load N consecutive shared-memory elements (aligned) with one vector load
template <typename T, int N>
__device__ __forceinline__ void pmg_lds_vec(const char* src, T (&v)[N]) {
  constexpr int B = N * (int)sizeof(T);
  if constexpr (B > 16 && B % 32 == 0) {
    pmg_lds_vec<T, N / 2>(src, reinterpret_cast<T(&)[N / 2]>(v));
    pmg_lds_vec<T, N / 2>(src + B / 2, reinterpret_cast<T(&)[N / 2]>(v[N / 2]));
    return;
  }
  PmgVec<T, N> u;
  if constexpr (B == 16) u.w16 = *reinterpret_cast<const uint4*>(src);
  else if constexpr (B == 8) u.w8 = *reinterpret_cast<const uint2*>(src);
  else if constexpr (B == 4) u.w4 = *reinterpret_cast<const unsigned*>(src);
  else if constexpr (B == 2) u.w2 = *reinterpret_cast<const unsigned short*>(src);
  else {
#pragma unroll
    for (int i = 0; i < N; ++i) u.e[i] = reinterpret_cast<const T*>(src)[i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = u.e[i];
}

// ------------------------------------------------------------------ mbarrier + TMA bulk copy (sm_90+)
__device__ __forceinline__ u32 pmg_smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void pmg_mbar_init(u32 bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void pmg_mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void pmg_mbar_expect_tx(u32 bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pmg_mbar_wait(u32 bar, u32 phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "PMG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra PMG_WAIT_%=;\n}" ::"r"(bar), "r"(phase) : "memory");
}
// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void pmg_bulk_g2s(u32 dst, const void* src, u32 bytes, u32 bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// predicated variants: every lane executes the instruction stream (no divergence), only `p` lanes act
__device__ __forceinline__ void pmg_mbar_expect_tx_if(u32 bar, u32 bytes, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
               "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}" ::"r"(bar), "r"(bytes), "r"((int)p) : "memory");
}
__device__ __forceinline__ void pmg_bulk_g2s_if(u32 dst, const void* src, u32 bytes, u32 bar, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
               "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "r"((int)p) : "memory");
}
__device__ __forceinline__ void pmg_fence_proxy_async_if(bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q fence.proxy.async.shared::cta;\n}" ::"r"((int)p) : "memory");
}
__device__ __forceinline__ void pmg_fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ int pmg_lane() { int l; asm("mov.u32 %0, %%laneid;" : "=r"(l)); return l; }

// ------------------------------------------------------------------ shuffles (load types 3 / 4)
__device__ __forceinline__ float pmg_shfl(float v, int src) { return __shfl_sync(PMG_FULL, v, src); }
__device__ __forceinline__ int pmg_shfl(int v, int src) { return __shfl_sync(PMG_FULL, v, src); }
