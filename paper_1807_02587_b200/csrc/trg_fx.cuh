// Order-independent (exact) accumulation of FP64 sums, and the bulk-copy
// (TMA engine, cp.async.bulk) + mbarrier helpers the tile pipelines use.
//
// Why fixed point: the reference merges its per-chunk partial sums in chunk
// order so its totals do not depend on the worker count
// (parallel.hpp:30-33).  On the GPU every contribution (a warp's run of
// deposits into one node, a tile's moment record) is converted ONCE to a
// signed fixed-point integer split in three 42-bit limbs and added with
// integer atomics (RED.ADD.64, no return): integer addition is associative,
// so the total is the same for any grid, any SM budget, any CTA schedule,
// and any number of shards whose boundaries keep the 32-entry warp windows
// (the NCCL all-reduce of the limbs is exact too).  Scale: the caller bounds
// |contribution| < 2^bound_exp; the unit is 2^(bound_exp - 96), i.e. each
// contribution keeps >= 96 bits, and 2^21 contributions of that size fit
// each limb without overflow.  Reading back normalises the carries and
// rounds once to double (<= 1 ulp of the exact total).
#pragma once
#include <stdint.h>

namespace trg {

// Accumulator layout is PLANAR: limb l of value m of node j lives at
// acc[(3 m + l) * stride + j].  The limbs of one node are then in different
// cache lines (different L2 slices), so the reductions of one contribution
// proceed in parallel instead of queueing at one slice's atomics unit.
struct FxScale {
  double up;    // 2^S: contribution -> units
  double down;  // 2^-S
};

// Scale for contributions bounded by |v| <= bound (any bound >= 0).
__host__ __device__ __forceinline__ FxScale fx_scale(double bound) {
  int e = -900;
  if (bound > 0.0 && bound < 1e300) {
    e = ilogb(bound) + 1;  // bound < 2^e
    if (e < -900) e = -900;
  }
  FxScale s;
  s.up = ldexp(1.0, 96 - e);
  s.down = ldexp(1.0, e - 96);
  return s;
}

constexpr double kFx42 = 4398046511104.0;                 // 2^42
constexpr double kFxInv42 = 1.0 / 4398046511104.0;        // 2^-42
constexpr double kFx84 = 19342813113834066795298816.0;    // 2^84
constexpr double kFxInv84 = 1.0 / 19342813113834066795298816.0;

// v -> (l0, l1, l2) with v * up = l2 2^84 + l1 2^42 + l0 (l0 rounded to the
// unit; every other step is exact: the nearest-integer splits leave
// remainders that fit a double's significand).
__device__ __forceinline__ void fx_split(double v, double up, long long& l0, long long& l1,
                                         long long& l2) {
  const double V = v * up;
  const double h = rint(V * kFxInv84);
  const double r = fma(-h, kFx84, V);
  const double m = rint(r * kFxInv42);
  const double r2 = fma(-m, kFx42, r);
  l2 = (long long)h;
  l1 = (long long)m;
  l0 = __double2ll_rn(r2);
}

// Value v into the planar limbs a[0], a[stride], a[2 stride] (three integer
// reductions; no return value: the warp never waits on the L2 atomics unit).
__device__ __forceinline__ void fx_red(long long* a, size_t stride, double v, double up) {
  long long l0, l1, l2;
  fx_split(v, up, l0, l1, l2);
  if (l0) asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a), "l"(l0) : "memory");
  if (l1) asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a + stride), "l"(l1) : "memory");
  if (l2) asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a + 2 * stride), "l"(l2) : "memory");
}

// Limb triple -> double (carries normalised in integers, then one rounding
// per limb add).
__host__ __device__ __forceinline__ double fx_value(long long l0, long long l1, long long l2,
                                                    double down) {
  long long c = (l0 + (1ll << 41)) >> 42;
  l0 -= c << 42;
  l1 += c;
  c = (l1 + (1ll << 41)) >> 42;
  l1 -= c << 42;
  l2 += c;
  const double hi = (double)l2 * kFx84 + (double)l1 * kFx42;
  return (hi + (double)l0) * down;
}

// Value m of node j from planar accumulators another CTA (or the L2
// atomics unit) updated.
__device__ __forceinline__ double fx_load(const long long* acc, size_t stride, int j, int m,
                                          double down) {
  const long long* a = acc + (size_t)(3 * m) * stride + j;
  return fx_value(__ldcg(a), __ldcg(a + stride), __ldcg(a + 2 * stride), down);
}

// Deposit of one warp: lane i holds (key_i, v_i[NM]) for the i-th entry of
// a fixed 32-entry window (key < 0: nothing).  Runs of equal keys in lane
// order are summed by a segmented inclusive scan (a fixed tree per window:
// deterministic), and each run's tail adds its sums to node key's limbs with
// the scale of moment order ord[m] (0: mass, 1: first, 2: second moments).
// Must be called by all 32 lanes.
template <int NM>
__device__ __forceinline__ void warp_run_deposit(int key, double v[NM], long long* acc,
                                                 size_t stride, const FxScale* sc, const int* ord) {
  const int lane = threadIdx.x & 31;
  const int prev = __shfl_up_sync(0xffffffffu, key, 1);
  const int next = __shfl_down_sync(0xffffffffu, key, 1);
  const bool head = lane == 0 || prev != key;
  const bool tail = lane == 31 || next != key;
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  if (heads == 0xffffffffu) {
    // every lane is its own run (incoherent order): no scan needed
  } else {
    // distance to this run's head: the scan steps stop at it
    const unsigned below = heads & (0xffffffffu >> (31 - lane));  // heads at lanes <= lane
    const int h = 31 - __clz(below);
    const int span = lane - h;  // lanes [h, lane] belong to the run
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        const double o = __shfl_up_sync(0xffffffffu, v[m], off);
        if (off <= span) v[m] += o;
      }
    }
  }
#ifdef TRG_NO_DEPOSIT
  if (tail && key == -12345) {
#else
  if (tail && key >= 0) {
#endif
#pragma unroll
    for (int m = 0; m < NM; ++m) fx_red(acc + (size_t)(3 * m) * stride + key, stride, v[m], sc[ord[m]].up);
  }
}

// ------------------------------------------------------------ bulk copies
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// makes the barrier's initialisation visible to the async proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Global data other CTAs wrote (ordered by a grid barrier) becomes visible
// to the async proxy (the bulk-copy engine) issued after this fence.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Shared memory the generic proxy wrote/read before becomes safe to
// overwrite by the async proxy.
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// One thread issues: copies `bytes` (any size) from src to dst as 16-byte
// aligned bulk chunks (<= 64 KB each... the engine takes up to 2^20 - 16);
// returns the bytes it armed on `bar` (the caller arrives with that count).
// The unaligned head/tail (if any) is NOT copied: callers keep buffers
// 16-byte aligned and sizes multiples of 16.
__device__ __forceinline__ void bulk_g2s_issue(void* dst, const void* src, unsigned bytes,
                                               uint64_t* bar) {
  mbar_arrive_tx(bar, bytes);
  unsigned off = 0;
  while (off < bytes) {
    const unsigned c = min(bytes - off, 32768u);
    bulk_g2s(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, c, bar);
    off += c;
  }
}

}  // namespace trg
