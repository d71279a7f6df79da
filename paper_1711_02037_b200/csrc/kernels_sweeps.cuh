// kernels_sweeps.cuh — the compressed HALS loop as ONE persistent, cooperatively launched kernel.
//
// Restates, per sweep (UpdateOrder::Grouped):
//   rhals_update_W   p/src/rhals.cpp:107-114 -> rhals_w_component :23-32
//   rhals_h_phase    p/src/rhals.cpp:49-58   -> clamped_row_update p/src/hals.cpp:75-81
//   compressed_pgrad p/src/rhals.cpp:150-158 -> projected_sq_norm  p/src/hals.cpp:55-65
//   stop rule        p/src/rhals.cpp:195-200
//
// Decomposition (one CTA per SM, grid G):
//   * CTA g owns rows [g m/G, (g+1) m/G) of Q and W and columns [g n/G, (g+1) n/G) of B and H.
//     When they fit, the Q / W row slabs live in shared memory for the whole launch; the B / H
//     column slabs always do.  W~ (l x k), T = B H^T, V = H H^T, E = residc H^T, S = W~^T W~ and
//     ||W(:,j)||^2 are replicated (fp64) in every CTA.
//   * W phase: per column j every CTA computes the identical W~ step, lifts and clamps its rows
//     (W(:,j) = [Q W~(:,j) - beta/d]_+), and contributes [Q^T W(:,j); ||W(:,j)||^2] partials; one
//     grid barrier later every CTA reduces the G partials in the same fixed order, so the new
//     W~(:,j) is bitwise identical everywhere.  k dependent grid steps per sweep, no relaunch.
//   * H phase: warp per owned column; the k sequential row updates of the reference run down the
//     column (h in registers, warp-shuffle dot products).  The same pass forms residc(:,c), the
//     compressed objective and the projected grad_H, and the CTA's contribution to next sweep's
//     T, V and to E.  A two-level fixed-order reduction (2 grid barriers) makes them global.
//   * grad_W = -2 Q E is formed row-locally and reduced (1 grid barrier) -> pgrad; CTA 0 writes
//     the trace entry, every CTA evaluates the identical stop test and leaves the loop together.
// Partial buffers alternate between two slots so a CTA that runs ahead never overwrites
// partials another CTA is still reading.
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <algorithm>
#include <cstdlib>

namespace rnmf_gpu {

namespace {

constexpr int kSwThreads = 256;
constexpr int kSwWarps = kSwThreads / 32;
constexpr int kMaxPerLane = 4;  // k, l <= 128
constexpr double kDivisionFloor = 1e-12;  // p/include/rnmf/hals.hpp:67
constexpr int kMaxLSlots = 5;     // (l + 1) / 32 lane slots in the recompress reduction
constexpr int kMaxResSlots = 8;   // l / 16 lane slots for residc
constexpr int kRedStride = 132;   // >= l + 1
constexpr int kRedLen = kSwWarps * kRedStride > kSwThreads ? kSwWarps * kRedStride : kSwThreads;

#ifndef RNMF_SWEEP_PROF
#define RNMF_SWEEP_PROF 0
#endif
constexpr bool kSweepProf = RNMF_SWEEP_PROF != 0;
// profile buckets (cycles of CTA 0, thread 0)
enum {
  kPfWStep, kPfLift, kPfRecomp, kPfBarrier1, kPfReduce1, kPfHCols, kPfHProducts, kPfBarrier2, kPfReduce2a,
  kPfReduce2b, kPfPgw, kPfOther, kPfHS, kPfHInit, kPfHUpd, kPfSweeps, kPfCount
};

struct SmemLayout {
  // fp64 region
  size_t wt, tm, em, vm, sm, wn, pm, colold, colnew, invd, rdw, red, scal, doubles_end;
  // T region (offsets in bytes from the start)
  size_t qs, wst, wcold, bc, hc, rc, total;
  // streamed Q slabs through a 2-stage bulk-copy ring (0: not used): stage = kSwThreads rows
  size_t qring, qring_stage, qbars, qring_n;
  // fp32 streamed path: colnew as fp32 (lp floats, zero past l), E as fp32 (l x k) for grad_W
  size_t cnf, ef;
  // wide: the B / H / residc column slabs stay in global memory (row stride n; H updated in place,
  // residc in SweepArgs::rc), E is read from the reduction buffer and P = W~ V is not kept --
  // shared memory independent of n (BASELINE C5: n = 100,000, l = 96, k = 64)
  bool wide;
};

constexpr int kQRingMax = 6;  // bulk-copy ring stages (fewer when shared memory is short)
template <typename T>
SmemLayout make_layout(int l, int k, int64_t RM, int64_t NCM, bool qs, int ring = 0, int f32s_lp = 0,
                       bool wide = false) {
  SmemLayout L{};
  L.wide = wide;
  size_t d = 0;
  auto take = [&](size_t count) {  // 16-byte aligned (double2 loads)
    const size_t off = d;
    d += (count + 1) / 2 * 2;
    return off;
  };
  L.wt = take(size_t(l) * (k + 1));
  L.tm = take(size_t(l) * (k + 1));
  L.em = wide ? 0 : take(size_t(l) * (k + 1));
  L.vm = take(size_t(k) * k);
  L.sm = take(size_t(k) * k);
  L.wn = take(size_t(k));
  L.pm = wide ? 0 : take(size_t(l) * (k + 1));
  L.colold = take(size_t(l));
  L.colnew = take(size_t(l) > 64 ? size_t(l) : 64);  // zero past l: branch-free padded dot products
  L.invd = take(size_t(k));
  L.rdw = take(size_t(k));
  L.red = take(kRedLen + 2 * kSwWarps);
  L.scal = take(16);
  L.doubles_end = d * sizeof(double);
  size_t b = (L.doubles_end + 15) / 16 * 16;
  auto takeT = [&](size_t count) {
    const size_t off = b;
    b += (count * sizeof(T) + 15) / 16 * 16;
    return off;
  };
  const size_t ncp = size_t(NCM) + 1;
  auto takeD = [&](size_t count) {
    const size_t off = b;
    b += (count * sizeof(double) + 15) / 16 * 16;
    return off;
  };
  L.qs = qs ? takeD(size_t(RM) * (l + 1)) : 0;
  // the ring and fp32 streamed paths keep the lifted column in registers
  L.wcold = (ring || f32s_lp) ? 0 : takeD(size_t(RM));
  L.wst = qs ? takeT(size_t(k) * RM) : 0;
  if (!wide) {
    L.bc = takeT(size_t(l) * ncp);
    L.hc = takeT(size_t(k) * ncp);
    L.rc = takeT(size_t(l) * ncp);
  }
  if (f32s_lp) {
    L.cnf = takeT(size_t(f32s_lp));
    L.ef = takeT(size_t(l) * ((k + 7) & ~7));
  }
  if (ring) {
    b = (b + 127) / 128 * 128;
    L.qring_stage = size_t(kSwThreads) * l * sizeof(T);
    L.qring = b;
    L.qring_n = size_t(ring);
    b += size_t(ring) * L.qring_stage;
    L.qbars = b;
    b += 8 * size_t(ring);
  }
  L.total = b;
  return L;
}

// LREG > 0 with QS: every CTA row slab has <= kSwThreads rows and l + 1 <= LREG <= 64; thread t keeps
// Q row t in fp64 registers for the whole launch (lift = register dot product, recompress = warp
// reduce-scatter), which removes the shared-memory round trips from the column chain.
// LREG > 0 without QS (slab too large for shared memory, e.g. C3/C4): rows are streamed from L2 with
// coalesced 16-byte loads, one row per thread per 256-row chunk; lift, clamp and the recompress
// accumulation happen on the row while it is in registers (one pass over the slab per column).
template <typename T, bool QS, int LREG>
struct Sweeper {
  // fp32 X with the Q slab not resident on chip: coalesced float4-column Q (a.q4), fp32 FMA lift and
  // recompress (no fp64 conversions on the row stream), column-major W scratch (a.wc)
  static constexpr bool F32S = !QS && LREG > 0 && sizeof(T) == 4;
  const SweepArgs<T>& a;
  int G, g, tid, lane, wid, l, k;
  int64_t r0, R, c0, NC, RM;
  int ncp, lq, kp;  // kp = k + 1: odd fp64 row stride of the l x k arrays (bank-conflict free columns)
  double *Wt, *Tm, *Em, *Vm, *Sm, *wn, *Pm, *colold, *colnew, *invd, *rdw, *red, *scal;
  double *Qs, *wcold;
  T *WsT, *Bc, *Hc, *Rc;
  float *cnf = nullptr, *ef = nullptr;
  bool wide = false;
  const double* efin = nullptr;  // wide: E (l x k, row stride k) in the last h_phase reduction buffer
  unsigned epoch = 0;
  int slot = 0;
  unsigned long long* colacc;  // fixed-point column accumulators (3-slot ring)
  // streamed Q slab ring (L.qring): chunks of kSwThreads rows, 2 stages, prefetch runs ahead across
  // columns (Q is constant, so the next pass's first chunks load while the column reduction waits)
  const T* qring = nullptr;
  uint64_t* qbars = nullptr;
  size_t qstage_elems = 0;
  int qst = 0;  // stages
  int64_t qnch = 0, qissued = 0, qused = 0;
  unsigned xepoch = 0;         // cross-GPU barriers passed (row-sharded runs)
  unsigned x2epoch = 0;        // hierarchical cross_allreduce calls (row-sharded runs)
  unsigned cur_t = 0;          // sweep being computed (reseed_dead liveness stamps)
  bool wpos = false;           // this thread lifted a positive W entry in the current column
  int xslot = 0;               // exchange-buffer slot of the next cross_allreduce
  unsigned cstep = 0;          // column steps done in this launch (ring position)
  double qrow[(QS && LREG > 0) ? LREG : 1];
  // optional cycle profile of CTA 0 / thread 0 (built with RNMF_SWEEP_PROF=1 and args.prof != nullptr;
  // compiled out otherwise, the runtime test alone costs a reconvergence point per tick)
  bool prof_on = false;
  long long prof_last = 0;
  long long prof_acc[kPfCount] = {};
  __device__ __forceinline__ void prof_tick(int bucket) {
    if (kSweepProf && prof_on) {
      const long long now = clock64();
      prof_acc[bucket] += now - prof_last;
      prof_last = now;
    }
  }
  int64_t part_slot_len;  // doubles per slot of a.part
  int64_t fin_slot_len;

  __device__ Sweeper(const SweepArgs<T>& args, unsigned char* smem, const SmemLayout& L, int64_t RM_, int64_t NCM)
      : a(args) {
    G = gridDim.x;
    g = blockIdx.x;
    tid = threadIdx.x;
    lane = lane_id();
    wid = warp_id();
    l = a.l;
    k = a.k;
    r0 = a.m * g / G;
    R = a.m * (g + 1) / G - r0;
    c0 = a.n * g / G;
    NC = a.n * (g + 1) / G - c0;
    RM = RM_;
    // (the wide layout never has Q in shared memory: QS variants keep the on-chip slabs statically)
    const bool wl = !QS && L.wide;
    ncp = wl ? int(a.n) : int(NCM) + 1;
    lq = l + 1;
    kp = k + 1;
    double* D = reinterpret_cast<double*>(smem);
    Wt = D + L.wt;
    Tm = D + L.tm;
    Em = wl ? nullptr : D + L.em;
    Vm = D + L.vm;
    Sm = D + L.sm;
    wn = D + L.wn;
    Pm = wl ? nullptr : D + L.pm;
    colold = D + L.colold;
    colnew = D + L.colnew;
    invd = D + L.invd;
    rdw = D + L.rdw;
    red = D + L.red;
    scal = D + L.scal;
    Qs = QS ? reinterpret_cast<double*>(smem + L.qs) : nullptr;
    wcold = reinterpret_cast<double*>(smem + L.wcold);
    WsT = QS ? reinterpret_cast<T*>(smem + L.wst) : nullptr;
    if (wl) {
      Bc = const_cast<T*>(a.b) + c0;
      Hc = a.h + c0;
      Rc = a.rc + c0;
    } else {
      Bc = reinterpret_cast<T*>(smem + L.bc);
      Hc = reinterpret_cast<T*>(smem + L.hc);
      Rc = reinterpret_cast<T*>(smem + L.rc);
    }
    wide = wl;
    if (L.cnf) {
      cnf = reinterpret_cast<float*>(smem + L.cnf);
      ef = reinterpret_cast<float*>(smem + L.ef);
    }
    colacc = reinterpret_cast<unsigned long long*>(reinterpret_cast<unsigned char*>(a.barrier) + 128);
    if (L.qring) {
      qring = reinterpret_cast<const T*>(smem + L.qring);
      qbars = reinterpret_cast<uint64_t*>(smem + L.qbars);
      qstage_elems = size_t(kSwThreads) * l;
      qnch = (R + kSwThreads - 1) / kSwThreads;
      qst = int(L.qring_n);
      if (tid == 0) {
        for (int s2 = 0; s2 < qst; ++s2) tc::mbar_init(&qbars[s2], 1);
        tc::fence_mbar_init();
      }
    }
    part_slot_len = sweep_part_len(l, k) * G;
    fin_slot_len = sweep_part_len(l, k);
    prof_on = kSweepProf && a.prof != nullptr && g == 0 && tid == 0;
    if (prof_on) prof_last = clock64();
  }

  __device__ __forceinline__ double q(int64_t r, int i) const {
    if constexpr (QS)
      return Qs[r * lq + i];
    else
      return double(__ldg(a.q + (r0 + r) * l + i));
  }
  __device__ __forceinline__ T w_get(int64_t r, int j) const {
    if constexpr (QS)
      return WsT[int64_t(j) * RM + r];
    else
      return a.w[(r0 + r) * k + j];
  }
  __device__ __forceinline__ double wcol_get(int64_t r) const { return wcold[r]; }
  // Row r of this CTA's Q slab into registers (streamed path).  fp32 Q: 16-byte vector loads when
  // the row pitch allows.  Out-of-range rows / columns read as 0.
  template <typename F>
  __device__ __forceinline__ void load_row(int64_t r, F (&qf)[LREG > 0 ? LREG : 1]) const {
    if (r >= R) {
#pragma unroll
      for (int i = 0; i < (LREG > 0 ? LREG : 1); ++i) qf[i] = F(0);
      return;
    }
    const T* qr = a.q + (r0 + r) * l;
    if constexpr (sizeof(T) == 4 && LREG > 0) {
      if ((l % 4) == 0) {
#pragma unroll
        for (int i4 = 0; i4 < LREG / 4; ++i4) {
          if (i4 * 4 < l) {
            const float4 v4 = __ldg(reinterpret_cast<const float4*>(qr) + i4);
            qf[4 * i4] = v4.x, qf[4 * i4 + 1] = v4.y, qf[4 * i4 + 2] = v4.z, qf[4 * i4 + 3] = v4.w;
          } else {
            qf[4 * i4] = qf[4 * i4 + 1] = qf[4 * i4 + 2] = qf[4 * i4 + 3] = F(0);
          }
        }
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < (LREG > 0 ? LREG : 1); ++i) qf[i] = i < l ? F(__ldg(qr + i)) : F(0);
  }

  __device__ __forceinline__ double* part_base() { return a.part + int64_t(slot) * part_slot_len; }
  __device__ __forceinline__ double* fin_base() { return a.fin + int64_t(slot) * fin_slot_len; }
  __device__ __forceinline__ void next_slot() { slot ^= 1; }

  // Grid barrier over kBarReps replicated counters: CTA g arrives (release) on counter g % reps,
  // lanes 0..reps-1 of warp 0 poll one counter each (acquire) until their sum reaches the target.
  __device__ void barrier() {
    __syncthreads();
    epoch += 1;
    if (tid < 32) {
      unsigned* ctr = reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(a.barrier) + kSweepBarOffset);
      constexpr int kLine = 128 / int(sizeof(unsigned));
      if (tid == 0) red_release_gpu_add(ctr + (g % kBarReps) * kLine, 1u);
      const unsigned target = epoch * unsigned(G);
      while (true) {
        const unsigned v = tid < kBarReps ? ld_acquire_gpu(ctr + tid * kLine) : 0u;
        if (__reduce_add_sync(0xffffffffu, v) >= target) break;
      }
    }
    __syncthreads();
  }

  // ---- row sharding across GPUs (a.world >= 1; one process per GPU, peers mapped by IPC) ------
  __device__ __forceinline__ bool sharded() const { return a.world > 0; }
  __device__ __forceinline__ unsigned* xcounter(int p) const {
    return reinterpret_cast<unsigned*>(a.peer_sync[p] + 64);
  }
  __device__ __forceinline__ double* xbuf(int p, int slot_, int from) const {
    return reinterpret_cast<double*>(a.peer_sync[p] + kSweepXbufOffset) + (int64_t(slot_) * kMaxWorld + from) * kXMax;
  }
  // Barrier over every CTA of every GPU: each CTA arrives (release, system scope) on the counter of
  // every GPU and waits for its own counter to reach xepoch * (sum of all grids).
  __device__ void xbarrier() {
    __syncthreads();
    xepoch += 1;
    if (tid == 0) {
      for (int p = 0; p < a.world; ++p) red_release_sys_add(xcounter(p), 1u);
      const unsigned target = unsigned(xepoch * a.xtotal);
      while (ld_acquire_sys(xcounter(a.rank)) < target) {
      }
    }
    __syncthreads();
  }
  // thread 0: bulk-copy chunk c (global chunk counter; chunk c % qnch of the slab) into stage c & 1
  __device__ void qring_issue(int64_t c) {
    const int st = int(c % qst);
    const int64_t cc = c % qnch, rows = min(int64_t(kSwThreads), R - cc * kSwThreads);
    const uint32_t bytes = uint32_t(rows * l * int64_t(sizeof(T)));
    tc::mbar_arrive_expect_tx(&qbars[st], bytes);
    tc::bulk_load(const_cast<T*>(qring) + st * qstage_elems, a.q + (r0 + cc * kSwThreads) * l, bytes, &qbars[st]);
  }
  // before the CTA exits: every issued chunk has landed (no bulk copy may target a dead CTA)
  __device__ void qring_drain() {
    if (!qring) return;
    for (int64_t c = qused; c < qissued; ++c) tc::mbar_wait(&qbars[c % qst], uint32_t((c / qst) & 1));
  }

  // All-reduce over GPUs of L values that are already identical in every CTA of a GPU (the result
  // of a GPU-local reduction): CTA 0 stores its GPU's values into slot [xslot][rank] of every
  // GPU's exchange buffer, one cross barrier, then every CTA sums the world contributions in rank
  // order -- the same bits on every GPU.  put(e, v) runs after all reads of get().
  template <typename Get, typename Put>
  __device__ void cross_allreduce(int L, Get&& get, Put&& put) {
    if (!sharded()) return;
    if (!(a.flags & kXFlat)) {
      // hierarchical: a local grid barrier (every CTA here finished reading the slot the peers may
      // rewrite next), CTA 0 writes and meets the other GPUs' CTA 0s, then releases this GPU's CTAs
      barrier();
      x2epoch += 1;
      unsigned* flag2 = reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(a.barrier) + kSweepFlagOffset + 64);
      if (g == 0) {
        for (int e = tid; e < L; e += kSwThreads) {
          const double v = get(e);
          for (int p = 0; p < a.world; ++p) xbuf(p, xslot, a.rank)[e] = v;
        }
        __syncthreads();
        if (tid == 0) {
          for (int p = 0; p < a.world; ++p)
            red_release_sys_add(reinterpret_cast<unsigned*>(a.peer_sync[p] + kSweepXcolOffset + 64), 1u);
          const unsigned target = x2epoch * unsigned(a.world);
          while (ld_acquire_sys(reinterpret_cast<const unsigned*>(a.peer_sync[a.rank] + kSweepXcolOffset + 64)) <
                 target) {
          }
          st_release_gpu(flag2, x2epoch);
        }
        __syncthreads();
      } else {
        if (tid == 0)
          while (ld_acquire_gpu(flag2) < x2epoch) {
          }
        __syncthreads();
      }
      for (int e = tid; e < L; e += kSwThreads) {
        double s2 = 0.0;
        for (int r = 0; r < a.world; ++r) s2 += __ldcg(xbuf(a.rank, xslot, r) + e);
        put(e, s2);
      }
      xslot ^= 1;
      __syncthreads();
      return;
    }
    if (g == 0)
      for (int e = tid; e < L; e += kSwThreads) {
        const double v = get(e);
        for (int p = 0; p < a.world; ++p) xbuf(p, xslot, a.rank)[e] = v;
      }
    xbarrier();
    for (int e = tid; e < L; e += kSwThreads) {
      double s2 = 0.0;
      for (int r = 0; r < a.world; ++r) s2 += __ldcg(xbuf(a.rank, xslot, r) + e);
      put(e, s2);
    }
    xslot ^= 1;
    __syncthreads();
  }

  // Partial layout is CTA-major: p[g * L + e] holds CTA g's contribution to entry e of an
  // L-long vector.  wr(e, sum_g p[g][e]) for e in [e0, e1): consecutive threads take consecutive
  // entries (coalesced), S thread-slices per entry stride over g with all loads independent, and
  // the slices are combined in fixed order through shared memory.  Every thread of the CTA must
  // call this (it contains __syncthreads).
  template <typename Writer>
  __device__ void reduce_entries(const double* p, int L, int e0, int e1, Writer&& wr) {
    const int E = e1 - e0;
    if (E <= 0) return;
    for (int eb = 0; eb < E; eb += kSwThreads) {
      const int EB = min(kSwThreads, E - eb);
      const int S = max(1, min(G, kSwThreads / EB));
      const int el = tid % EB, sidx = tid / EB;
      double acc = 0.0;
      if (sidx < S) {
        const double* src = p + e0 + eb + el;
        for (int gb = sidx; gb < G; gb += 32 * S) {
          double v[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int gg = gb + u * S;
            v[u] = gg < G ? ld_cg(src + int64_t(gg) * L) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 32; ++u) acc += v[u];
        }
      }
      red[tid] = acc;
      __syncthreads();
      if (tid < EB) {
        double v = 0.0;
        for (int q2 = 0; q2 < S; ++q2) v += red[q2 * EB + tid];
        wr(e0 + eb + tid, v);
      }
      __syncthreads();
    }
  }

  // every CTA: wr(e, sum_g part[e][g]) for e < L (fixed order)
  template <typename Writer>
  __device__ void reduce_all(int L, Writer&& wr) {
    reduce_entries(part_base(), L, 0, L, wr);
  }

  // Single-level all-reduce of vectors already written to part_base(): one barrier.
  template <typename Writer>
  __device__ void allreduce1(int L, Writer&& wr) {
    prof_tick(kPfOther);
    barrier();
    prof_tick(kPfBarrier1);
    reduce_all(L, wr);
    next_slot();
    __syncthreads();
    prof_tick(kPfReduce1);
  }

  // Column-step all-reduce of [Q^T W(:,j); ||W(:,j)||^2] (L1 = l + 1 entries; thread e < L1 holds
  // the CTA's partial v of entry e).  Each partial becomes a 64-bit fixed-point integer and is
  // added with one integer atomic into its entry's accumulator (one 128-byte L2 line per entry, so
  // the G atomics of different entries proceed in parallel); after ONE grid barrier every CTA
  // reads the L1 sums.  Integer addition is exact and associative, so the sums have the same bits
  // whatever the arrival order: deterministic, bitwise-identical W~ on every CTA, without reading
  // G partial vectors (the ordered-partials path, kColOrdered, is kept as a testing knob).
  //   Scale: Q has orthonormal columns, so ||W(:,j)|| <= ||Q colnew|| = ||colnew|| =: B, and every
  //   partial -- and every sum of partials over any subset of CTAs -- of entry i < l is bounded by
  //   B, of the norm entry by B^2 (Cauchy-Schwarz over the rows involved).  With the margin 2B
  //   and scale 2^(54 - e), 2B < 2^e, all running sums stay below 2^54 in magnitude; the quantum
  //   2^(e-54) ~ 2^-53 * 2B is at the fp64 rounding level of an ordered sum of the partials.
  //   Ring: 3 slots; CTA 0 zeroes the next step's slot before it arrives here -- every CTA read
  //   that slot two steps ago, before arriving at the previous step's barrier.
  // wr(e, value) runs on thread e; the caller synchronises the block afterwards.
  // col_scales: the fixed-point scales from the per-warp ||colnew||^2 by exponent arithmetic (no
  // sqrt / frexp): with b2 in [2^(E-1023), 2^(E-1022)), 2 sqrt(b2) < 2^e1 and 4 b2 < 2^e2; entries
  // < l are scaled by 2^(54-e1), the norm entry by 2^(54-e2), clamped to the normal range (a norm
  // below 2^-1000 then quantises to 0).  Call after the block barrier that follows col_prepare.
  __device__ __forceinline__ void col_scales(double (&sc)[2], double (&inv)[2]) const {
    double b2 = 0.0;
    for (int w = 0; w * 32 < l; ++w) b2 += scal[4 + w];
    const int E = int((__double_as_longlong(b2) >> 52) & 0x7ff);
    const int e1 = 1 + ((E - 1021) >> 1);  // 1 + ceil((E - 1022) / 2), arithmetic shift
    const int e2 = E - 1020;
    const int s1 = min(1000, max(-1000, 54 - e1)), s2 = min(1000, max(-1000, 54 - e2));
    sc[0] = __longlong_as_double(static_cast<long long>(s1 + 1023) << 52);
    sc[1] = __longlong_as_double(static_cast<long long>(s2 + 1023) << 52);
    inv[0] = __longlong_as_double(static_cast<long long>(1023 - s1) << 52);
    inv[1] = __longlong_as_double(static_cast<long long>(1023 - s2) << 52);
  }

  template <typename Writer>
  __device__ void col_allreduce(int L1, double v, const double (&sc)[2], const double (&inv)[2], Writer&& wr) {
    if (a.flags & kColOrdered) {
      if (tid < L1) part_base()[int64_t(g) * L1 + tid] = v;
      allreduce1(L1, wr);
      return;
    }
    const int64_t slot0 = (cstep % 3) * kColAccStride;
    const int64_t off = slot0 + (int64_t(g % kColAccReps) * kColAccMax + tid) * kColAccSpacing;
    unsigned long long* cur = colacc + off;
    if (sharded() && !(a.flags & kXFlat)) {
      col_allreduce_xgpu(L1, v, sc, inv, slot0, off, wr);
      return;
    }
    if (tid < L1) {
      const long long fx = __double2ll_rn(v * sc[tid < l ? 0 : 1]);  // exact power-of-two scaling
      if (sharded()) {
        // the same integer atomics into every GPU's accumulator (NVLink): all GPUs end with the
        // identical exact sum over all rows of all shards
        for (int p = 0; p < a.world; ++p)
          red_relaxed_sys_add_u64(reinterpret_cast<unsigned long long*>(a.peer_sync[p] + 128) + off,
                                  static_cast<unsigned long long>(fx));
      } else {
        atomicAdd(cur, static_cast<unsigned long long>(fx));
      }
    }
    if (g == 0 && tid < L1)
#pragma unroll
      for (int rp = 0; rp < kColAccReps; ++rp)
        colacc[((cstep + 1) % 3) * kColAccStride + (int64_t(rp) * kColAccMax + tid) * kColAccSpacing] = 0ull;
    prof_tick(kPfOther);
    if (sharded())
      xbarrier();
    else
      barrier();
    prof_tick(kPfBarrier1);
    if (tid < L1) {
      unsigned long long acc = 0ull;
#pragma unroll
      for (int rp = 0; rp < kColAccReps; ++rp)
        acc += ld_cg(colacc + slot0 + (int64_t(rp) * kColAccMax + tid) * kColAccSpacing);
      const long long sum = static_cast<long long>(acc);
      wr(tid, double(sum) * inv[tid < l ? 0 : 1]);
    }
    ++cstep;
    prof_tick(kPfReduce1);
  }

  // Row-sharded column step, hierarchical: (1) every CTA adds its fixed-point partials into this
  // GPU's replicated accumulators, (2) local grid barrier, (3) CTA 0 sums the replicas and adds the
  // GPU's sums into every GPU's global accumulators (world remote adds per entry), arrives on every
  // GPU's CTA-0 counter and waits for all world arrivals on its own, then releases its GPU's CTAs
  // with a flag, (4) every CTA reads the global sums (exact integers: identical bits on every GPU).
  // Ring invariants as in col_allreduce: CTA 0 zeroes slot cstep + 1 (local replicas and global)
  // before arriving at this step's barriers; a peer adds into that slot only after this GPU's CTA 0
  // arrived at this step's cross barrier.
  template <typename Writer>
  __device__ void col_allreduce_xgpu(int L1, double v, const double (&sc)[2], const double (&inv)[2], int64_t slot0,
                                     int64_t off, Writer&& wr) {
    unsigned long long* cur = colacc + off;
    if (tid < L1) atomicAdd(cur, static_cast<unsigned long long>(__double2ll_rn(v * sc[tid < l ? 0 : 1])));
    const int nslot = int((cstep + 1) % 3), cslot = int(cstep % 3);
    auto gacc = [&](int p, int sl, int e) {
      return reinterpret_cast<unsigned long long*>(a.peer_sync[p] + kSweepGaccOffset) +
             (int64_t(sl) * kColAccMax + e) * kColAccSpacing;
    };
    if (g == 0 && tid < L1) {
#pragma unroll
      for (int rp = 0; rp < kColAccReps; ++rp)
        colacc[((cstep + 1) % 3) * kColAccStride + (int64_t(rp) * kColAccMax + tid) * kColAccSpacing] = 0ull;
      *gacc(a.rank, nslot, tid) = 0ull;
    }
    prof_tick(kPfOther);
    barrier();
    unsigned* flag = reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(a.barrier) + kSweepFlagOffset);
    if (g == 0) {
      if (tid < L1) {
        unsigned long long sum = 0ull;
#pragma unroll
        for (int rp = 0; rp < kColAccReps; ++rp)
          sum += ld_cg(colacc + slot0 + (int64_t(rp) * kColAccMax + tid) * kColAccSpacing);
        for (int p = 0; p < a.world; ++p) red_relaxed_sys_add_u64(gacc(p, cslot, tid), sum);
      }
      __syncthreads();
      if (tid == 0) {
        for (int p = 0; p < a.world; ++p)
          red_release_sys_add(reinterpret_cast<unsigned*>(a.peer_sync[p] + kSweepXcolOffset), 1u);
        const unsigned target = (cstep + 1) * unsigned(a.world);
        while (ld_acquire_sys(reinterpret_cast<const unsigned*>(a.peer_sync[a.rank] + kSweepXcolOffset)) < target) {
        }
        st_release_gpu(flag, cstep + 1);
      }
      __syncthreads();
    } else {
      if (tid == 0)
        while (ld_acquire_gpu(flag) < cstep + 1) {
        }
      __syncthreads();
    }
    prof_tick(kPfBarrier1);
    if (tid < L1) {
      const long long sum = static_cast<long long>(ld_cg(gacc(a.rank, cslot, tid)));
      wr(tid, double(sum) * inv[tid < l ? 0 : 1]);
    }
    ++cstep;
    prof_tick(kPfReduce1);
  }

  // Two-level all-reduce (reduce-scatter over CTAs, then all-gather): two barriers.
  template <typename Writer>
  __device__ void allreduce2(int L, Writer&& wr) {
    prof_tick(kPfOther);
    barrier();
    prof_tick(kPfBarrier2);
    const double* p = part_base();
    double* f = fin_base();
    const int e0 = int(int64_t(L) * g / G), e1 = int(int64_t(L) * (g + 1) / G);
    reduce_entries(p, L, e0, e1, [&](int e, double v) { f[e] = v; });
    __syncthreads();
    prof_tick(kPfReduce2a);
    barrier();
    prof_tick(kPfBarrier2);
    constexpr int U = 4;
    for (int e = tid; e < L; e += kSwThreads * U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = (e + kSwThreads * u < L) ? ld_cg(f + e + kSwThreads * u) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (e + kSwThreads * u < L) wr(e + kSwThreads * u, v[u]);
    }
    next_slot();
    __syncthreads();
    prof_tick(kPfReduce2b);
  }

  __device__ double block_sum(double v) {
    v = warp_allreduce_sum(v);
    __syncthreads();
    if (lane == 0) red[kRedLen + wid] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < kSwWarps; ++w) s += red[kRedLen + w];
    __syncthreads();
    return s;
  }

  // ---------------------------------------------------------------------------------------------
  __device__ void load_resident() {
    for (int i = tid; i < 64; i += kSwThreads) colnew[i] = 0.0;  // the padded tail stays zero
    if constexpr (F32S) {
      for (int i = tid; i < LREG; i += kSwThreads) cnf[i] = 0.f;
      // W rows of this CTA into the column-major scratch (the launch works column by column)
      for (int j = 0; j < k; ++j)
        for (int64_t r = tid; r < R; r += kSwThreads) a.wc[int64_t(j) * a.m + r0 + r] = float(a.w[(r0 + r) * k + j]);
    }
    if constexpr (QS) {
      for (int64_t e = tid; e < R * l; e += kSwThreads) {
        const int64_t r = e / l;
        const int i = int(e % l);
        Qs[r * lq + i] = double(a.q[(r0 + r) * l + i]);
      }
      for (int64_t e = tid; e < R * k; e += kSwThreads) {
        const int64_t r = e / k;
        const int j = int(e % k);
        WsT[int64_t(j) * RM + r] = a.w[(r0 + r) * k + j];
      }
    }
    if (!wide) {
      for (int64_t e = tid; e < int64_t(l) * NC; e += kSwThreads) {
        const int i = int(e / NC);
        const int64_t cl = e % NC;
        Bc[i * ncp + cl] = a.b[int64_t(i) * a.n + c0 + cl];
      }
      for (int64_t e = tid; e < int64_t(k) * NC; e += kSwThreads) {
        const int j = int(e / NC);
        const int64_t cl = e % NC;
        Hc[j * ncp + cl] = a.h[int64_t(j) * a.n + c0 + cl];
      }
    }
    if (!(a.flags & kInitWt))
      for (int e = tid; e < l * k; e += kSwThreads) Wt[(e / k) * kp + e % k] = a.wt[e];
    if (!(a.flags & kInitWn))
      for (int e = tid; e < k; e += kSwThreads) wn[e] = a.wn[e];
    if (!(a.flags & (kEval0 | kTvOnly))) {
      for (int e = tid; e < l * k; e += kSwThreads) Tm[(e / k) * kp + e % k] = a.tm[e];
      for (int e = tid; e < k * k; e += kSwThreads) Vm[e] = a.vm[e];
    }
    __syncthreads();
    if constexpr (QS && LREG > 0) {
#pragma unroll
      for (int i = 0; i < LREG; ++i) qrow[i] = (tid < R && i < l) ? Qs[int64_t(tid) * lq + i] : 0.0;
    }
  }

  __device__ void store_back(int64_t last, int stopped) {
    if constexpr (F32S) {
      if ((a.flags & kDoW) || a.order != nullptr)
        for (int j = 0; j < k; ++j)
          for (int64_t r = tid; r < R; r += kSwThreads) a.w[(r0 + r) * k + j] = T(a.wc[int64_t(j) * a.m + r0 + r]);
    }
    if constexpr (QS) {
      for (int64_t e = tid; e < R * k; e += kSwThreads) {
        const int64_t r = e / k;
        const int j = int(e % k);
        a.w[(r0 + r) * k + j] = WsT[int64_t(j) * RM + r];
      }
    }
    if ((a.flags & kDoH) && !wide) {
      for (int64_t e = tid; e < int64_t(k) * NC; e += kSwThreads) {
        const int j = int(e / NC);
        const int64_t cl = e % NC;
        a.h[int64_t(j) * a.n + c0 + cl] = Hc[j * ncp + cl];
      }
    }
    if (g == 0) {
      for (int e = tid; e < l * k; e += kSwThreads) {
        const int pe = (e / k) * kp + e % k;
        a.wt[e] = Wt[pe];
        a.tm[e] = Tm[pe];
        a.em[e] = Em ? Em[pe] : (efin ? efin[e] : 0.0);
      }
      for (int e = tid; e < k * k; e += kSwThreads) a.vm[e] = Vm[e];
      for (int e = tid; e < k; e += kSwThreads) a.wn[e] = wn[e];
      if (tid == 0) {
        a.status[0] = last;
        a.status[1] = stopped;
      }
    }
  }

  // W~ = Q^T W and/or wn = diag(W^T W)   (compress, p/src/rhals.cpp:103; ||W(:,j)||^2 at :53)
  __device__ void init_wt_wn() {
    const int lk = l * k, L = lk + k;
    double* p = part_base();
    if constexpr (QS) {
      for (int e = tid; e < L; e += kSwThreads) {
        double s = 0.0;
        if (e < lk) {
          const int i = e / k, j = e % k;
          for (int64_t r = 0; r < R; ++r) s += q(r, i) * double(w_get(r, j));
        } else {
          const int j = e - lk;
          for (int64_t r = 0; r < R; ++r) {
            const double wv = double(w_get(r, j));
            s += wv * wv;
          }
        }
        p[int64_t(g) * L + e] = s;
      }
    } else {
      // rows staged 4 at a time through shared memory (the red scratch is free here); entry blocks
      // of 8 per thread, one pass over the slab per block
      constexpr int kChunk = 4;
      double* qst = red;                 // [kChunk][l]   (<= 512 doubles)
      double* wst = red + kChunk * 128;  // [kChunk][k]   (<= 256 doubles)
      for (int eb = 0; eb < L; eb += kSwThreads * 8) {
        double accs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) accs[u] = 0.0;
        for (int64_t base = 0; base < R; base += kChunk) {
          const int nr = int(R - base < kChunk ? R - base : kChunk);
          __syncthreads();
          for (int e = tid; e < kChunk * l; e += kSwThreads) {
            const int rr = e / l;
            qst[e] = rr < nr ? double(a.q[(r0 + base + rr) * l + e % l]) : 0.0;
          }
          for (int e = tid; e < kChunk * k; e += kSwThreads) {
            const int rr = e / k;
            wst[e] = rr < nr ? double(a.w[(r0 + base + rr) * k + e % k]) : 0.0;
          }
          __syncthreads();
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = eb + tid + kSwThreads * u;
            if (e < L) {
              double sacc = 0.0;
              if (e < lk) {
                const int i = e / k, jj = e % k;
#pragma unroll
                for (int rr = 0; rr < kChunk; ++rr) sacc += qst[rr * l + i] * wst[rr * k + jj];
              } else {
                const int jj = e - lk;
#pragma unroll
                for (int rr = 0; rr < kChunk; ++rr) sacc += wst[rr * k + jj] * wst[rr * k + jj];
              }
              accs[u] += sacc;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = eb + tid + kSwThreads * u;
          if (e < L) p[int64_t(g) * L + e] = accs[u];
        }
      }
      __syncthreads();
    }
    const bool do_wt = a.flags & kInitWt, do_wn = a.flags & kInitWn;
    allreduce2(L, [&](int e, double v) {
      if (e < lk) {
        if (do_wt) Wt[(e / k) * kp + e % k] = v;
      } else if (do_wn) {
        wn[e - lk] = v;
      }
    });
    // row-sharded: W~ = Q^T W and ||W(:,j)||^2 are sums over the rows of every GPU
    cross_allreduce(
        L, [&](int e) { return e < lk ? Wt[(e / k) * kp + e % k] : wn[e - lk]; },
        [&](int e, double v) {
          if (e < lk) {
            if (do_wt) Wt[(e / k) * kp + e % k] = v;
          } else if (do_wn) {
            wn[e - lk] = v;
          }
        });
  }

  // P = W~ V (l x k), recomputed at the start of every W phase and then kept current with a
  // rank-1 update after each column, so the step of column j costs one FMA per entry instead
  // of a k-long dot product (same value as W~ * V(:,j) in rhals_w_component, up to rounding).
  __device__ void compute_p() {
    for (int e = tid; e < (Pm ? l * k : 0); e += kSwThreads) {
      const int i = e / k, c = e % k;
      const double* wi = Wt + i * kp;
      double s0 = 0.0, s1 = 0.0;
      int t = 0;
      for (; t + 1 < k; t += 2) {
        s0 += wi[t] * Vm[t * k + c];
        s1 += wi[t + 1] * Vm[(t + 1) * k + c];
      }
      if (t < k) s0 += wi[t] * Vm[t * k + c];
      Pm[i * kp + c] = s0 + s1;
    }
    // reciprocal step denominators of the sweep's columns (off the column chain)
    for (int j = tid; j < k; j += kSwThreads) rdw[j] = 1.0 / fmax(Vm[j * k + j] + a.alpha_w, kDivisionFloor);
    __syncthreads();
  }

  // Column-j prologue of rhals_w_component (p/src/rhals.cpp:25-29), row-local to thread i < l:
  // colnew(i) = W~(i,j) + (T(i,j) - P(i,j) - alpha W~(i,j)) / denom_j, plus the per-warp
  // ||colnew||^2 that bounds the fixed-point column reduction (fixed order: identical on every
  // CTA).  Caller synchronises before colnew is read by other threads.
  __device__ void col_prepare(int j, bool fresh = false) {
    const double alpha = a.alpha_w;
    // grouped sweeps: 1 / denom precomputed in compute_p (the fresh orders recompute V(j,j))
    const double rden = fresh ? 1.0 / fmax(Vm[j * k + j] + alpha, kDivisionFloor) : rdw[j];
    if (wid * 32 < l) {
      double nw = 0.0;
      if (tid < l) {
        const double cur = Wt[tid * kp + j];
        double pij;
        if (QS || Pm) {  // (the wide layout, Pm == nullptr, never has Q in shared memory)
          pij = Pm[tid * kp + j];
        } else {  // wide: (W~ V)(i, j) directly
          const double* wi = Wt + tid * kp;
          double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
          int c = 0;
          for (; c + 3 < k; c += 4) {
            p0 = fma(wi[c], Vm[c * k + j], p0);
            p1 = fma(wi[c + 1], Vm[(c + 1) * k + j], p1);
            p2 = fma(wi[c + 2], Vm[(c + 2) * k + j], p2);
            p3 = fma(wi[c + 3], Vm[(c + 3) * k + j], p3);
          }
          for (; c < k; ++c) p0 = fma(wi[c], Vm[c * k + j], p0);
          pij = (p0 + p1) + (p2 + p3);
        }
        nw = cur + (Tm[tid * kp + j] - pij - alpha * cur) * rden;
        colold[tid] = cur;
        colnew[tid] = nw;
        if constexpr (F32S) cnf[tid] = float(nw);
      }
      const double sq = warp_allreduce_sum(nw * nw);
      if (lane == 0) scal[4 + wid] = sq;
    }
  }

  // One column step of rhals_w_component (p/src/rhals.cpp:23-32); col_prepare(j) has run.  With
  // `chain`, the prologue of column j + 1 (grouped order) follows.
  __device__ void w_column(int j, bool chain = true) {
    const double alpha = a.alpha_w, beta = a.beta_w;
    const double denom = fmax(Vm[j * k + j] + alpha, kDivisionFloor);
    prof_tick(kPfWStep);
    double sc[2], inv[2];
    col_scales(sc, inv);
    const double shift = beta != 0.0 ? beta / denom : 0.0;
    const int L1 = l + 1;
    if constexpr (QS && LREG > 0) {
      // lift: thread t owns row t (register-resident Q row)
      double wd = 0.0;
      if (tid < R) {
        double u[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < LREG; ++i)
          if (i < l) u[i & 3] += qrow[i] * colnew[i];
        double uu = (u[0] + u[1]) + (u[2] + u[3]);
        if (beta != 0.0) uu -= shift;
        wd = fmax(uu, 0.0);
        wpos = wd > 0.0;
        wcold[tid] = wd;
        if constexpr (QS)
          WsT[int64_t(j) * RM + tid] = T(wd);
        else
          a.w[(r0 + tid) * k + j] = T(wd);
      }
      prof_tick(kPfLift);
      // recompress partial: v_i = Q(t,i) w_t (i < l), v_l = w_t^2; warp reduce-scatter over the 32
      // rows of the warp (lane L ends with entry L of each 32-entry chunk), then cross-warp in order
#pragma unroll
      for (int chunk = 0; chunk < (LREG + 31) / 32; ++chunk) {
        auto val = [&](int i) -> double {  // entry i of this thread's contribution vector
          return (i < l) ? qrow[i < LREG ? i : 0] * wd : (i == l ? wd * wd : 0.0);
        };
        if (chunk > 0 && chunk * 32 < L1 && L1 - chunk * 32 <= 8) {
          // short tail chunk (<= 8 live entries, e.g. l = 36): 3-stage reduce-scatter of 8 values,
          // then a 2-stage all-reduce within lane quads -- 9 shuffles instead of 31
          double v[4];
          {
            const bool hi = (lane & 16) != 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int ia = chunk * 32 + e, ib = ia + 4;
              const double va = (ia < LREG || ia == l) ? val(ia) : 0.0;
              const double vb = (ib < LREG || ib == l) ? val(ib) : 0.0;
              v[e] = (hi ? vb : va) + __shfl_xor_sync(0xffffffffu, hi ? va : vb, 16);
            }
          }
          {
            const bool hi = (lane & 8) != 0;
#pragma unroll
            for (int e = 0; e < 2; ++e) v[e] = (hi ? v[e + 2] : v[e]) + __shfl_xor_sync(0xffffffffu, hi ? v[e] : v[e + 2], 8);
          }
          {
            const bool hi = (lane & 4) != 0;
            v[0] = (hi ? v[1] : v[0]) + __shfl_xor_sync(0xffffffffu, hi ? v[0] : v[1], 4);
          }
          v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
          v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
          const int i = chunk * 32 + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
          if ((lane & 3) == 0 && i < L1) red[wid * kRedStride + i] = v[0];
        } else if (chunk * 32 < L1) {
          double v[16];
          {
            const bool hi = (lane & 16) != 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int ia = chunk * 32 + e, ib = ia + 16;
              const double va = (ia < LREG || ia == l) ? val(ia) : 0.0;
              const double vb = (ib < LREG || ib == l) ? val(ib) : 0.0;
              const double send = hi ? va : vb;
              const double mine = hi ? vb : va;
              v[e] = mine + __shfl_xor_sync(0xffffffffu, send, 16);
            }
          }
#pragma unroll
          for (int off = 8; off >= 1; off >>= 1) {
            const bool hi = (lane & off) != 0;
#pragma unroll
            for (int e = 0; e < off; ++e) {
              const double send = hi ? v[e] : v[e + off];
              const double mine = hi ? v[e + off] : v[e];
              v[e] = mine + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
          const int i = chunk * 32 + lane;
          if (i < L1) red[wid * kRedStride + i] = v[0];
        }
      }
    } else if constexpr (F32S) {
      // fp32 streamed rows: thread t takes rows t, t + 256, ...; the row's float4 columns are
      // coalesced 512-byte warp loads from a.q4; lift u = Q(r,:) colnew and the recompress partials
      // Q(r,:)^T w, ||w||^2 in fp32 FMA (per-thread partials over a few rows), then the warp
      // reduce-scatter switches to fp64 after two levels (partials over <= 4 threads' rows in fp32)
      constexpr int L4 = LREG / 4;
      constexpr int UNR = LREG <= 32 ? 4 : LREG <= 64 ? 2 : 1;  // rows whose loads are in flight together
      float acc[LREG];
      float accn = 0.f;
#pragma unroll
      for (int i = 0; i < LREG; ++i) acc[i] = 0.f;
      const float shiftf = float(shift);
      const float4* q4 = reinterpret_cast<const float4*>(a.q4);
      const float4* c4 = reinterpret_cast<const float4*>(cnf);
      float* wcol = a.wc + int64_t(j) * a.m + r0;
      for (int64_t rb = tid; rb < R; rb += int64_t(kSwThreads) * UNR) {
        float4 qv[UNR][L4];
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) {
          const int64_t r = rb + int64_t(kSwThreads) * uu;
          const int64_t rr = r < R ? r0 + r : r0;  // clamped: in-range address, result unused
#pragma unroll
          for (int i4 = 0; i4 < L4; ++i4) qv[uu][i4] = __ldg(q4 + int64_t(i4) * a.m + rr);
        }
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) {
          const int64_t r = rb + int64_t(kSwThreads) * uu;
          if (r >= R) continue;
          float u0 = 0.f, u1 = 0.f, u2 = 0.f, u3 = 0.f;
#pragma unroll
          for (int i4 = 0; i4 < L4; ++i4) {
            const float4 c = c4[i4];
            u0 = fmaf(qv[uu][i4].x, c.x, u0);
            u1 = fmaf(qv[uu][i4].y, c.y, u1);
            u2 = fmaf(qv[uu][i4].z, c.z, u2);
            u3 = fmaf(qv[uu][i4].w, c.w, u3);
          }
          float uf = (u0 + u1) + (u2 + u3);
          if (beta != 0.0) uf -= shiftf;
          const float wd = fmaxf(uf, 0.f);
          wpos |= wd > 0.f;
          wcol[r] = wd;
#pragma unroll
          for (int i4 = 0; i4 < L4; ++i4) {
            acc[4 * i4] = fmaf(qv[uu][i4].x, wd, acc[4 * i4]);
            acc[4 * i4 + 1] = fmaf(qv[uu][i4].y, wd, acc[4 * i4 + 1]);
            acc[4 * i4 + 2] = fmaf(qv[uu][i4].z, wd, acc[4 * i4 + 2]);
            acc[4 * i4 + 3] = fmaf(qv[uu][i4].w, wd, acc[4 * i4 + 3]);
          }
          accn = fmaf(wd, wd, accn);
        }
      }
      prof_tick(kPfLift);
#pragma unroll
      for (int chunk = 0; chunk < (LREG + 32) / 32; ++chunk) {
        if (chunk * 32 < L1) {
          // entry i of this thread's vector: acc[i] (i < l; zero for l <= i < LREG), accn at i = l
          auto val = [&](int i) -> float {
            return (i < LREG ? acc[i < LREG ? i : 0] : 0.f) + (i == l ? accn : 0.f);
          };
          float v16[16];
          {
            const bool hi = (lane & 16) != 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float va = val(chunk * 32 + e), vb = val(chunk * 32 + e + 16);
              v16[e] = (hi ? vb : va) + __shfl_xor_sync(0xffffffffu, hi ? va : vb, 16);
            }
          }
          double v[8];
          {
            const bool hi = (lane & 8) != 0;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              v[e] = double((hi ? v16[e + 8] : v16[e]) + __shfl_xor_sync(0xffffffffu, hi ? v16[e] : v16[e + 8], 8));
          }
#pragma unroll
          for (int off = 4; off >= 1; off >>= 1) {
            const bool hi = (lane & off) != 0;
#pragma unroll
            for (int e = 0; e < off; ++e) {
              const double send = hi ? v[e] : v[e + off];
              const double mine = hi ? v[e + off] : v[e];
              v[e] = mine + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
          const int i = chunk * 32 + lane;
          if (i < L1) red[wid * kRedStride + i] = v[0];
        }
      }
    } else if constexpr (LREG > 0) {
      // streamed rows (Q slab not resident): one pass, row in registers, fp64 accumulators
      double acc[LREG], accn = 0.0;
#pragma unroll
      for (int i = 0; i < LREG; ++i) acc[i] = 0.0;
      if (qring) {
        // the slab arrives chunk by chunk through the bulk-copy ring; thread t takes row t of a chunk
        if (qissued == 0) {
          if (tid == 0)
            for (int c2 = 0; c2 < qst; ++c2) qring_issue(c2);
          qissued = qst;
        }
        for (int64_t cc = 0; cc < qnch; ++cc) {
          const int64_t c = qused;
          tc::mbar_wait(&qbars[c % qst], uint32_t((c / qst) & 1));
          const int64_t r = cc * kSwThreads + tid;
          if (r < R) {
            const T* qr = qring + (c % qst) * qstage_elems + int64_t(tid) * l;
            T qf[LREG];
            if constexpr (sizeof(T) == 4) {
#pragma unroll
              for (int i4 = 0; i4 < LREG / 4; ++i4) {
                if (i4 * 4 < l) {
                  const float4 v4 = reinterpret_cast<const float4*>(qr)[i4];
                  qf[4 * i4] = v4.x, qf[4 * i4 + 1] = v4.y, qf[4 * i4 + 2] = v4.z, qf[4 * i4 + 3] = v4.w;
                } else {
                  qf[4 * i4] = qf[4 * i4 + 1] = qf[4 * i4 + 2] = qf[4 * i4 + 3] = T(0);
                }
              }
            } else {
#pragma unroll
              for (int i2 = 0; i2 < LREG / 2; ++i2) {
                if (i2 * 2 < l) {
                  const double2 v2 = reinterpret_cast<const double2*>(qr)[i2];
                  qf[2 * i2] = v2.x, qf[2 * i2 + 1] = v2.y;
                } else {
                  qf[2 * i2] = qf[2 * i2 + 1] = T(0);
                }
              }
            }
            double u[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int i = 0; i < LREG; ++i)
              u[i & 3] += double(qf[i]) * colnew[i];  // qf, colnew zero past l
            double uu2 = (u[0] + u[1]) + (u[2] + u[3]);
            if (beta != 0.0) uu2 -= shift;
            const double wd = fmax(uu2, 0.0);
            wpos |= wd > 0.0;
            a.w[(r0 + r) * k + j] = T(wd);
#pragma unroll
            for (int i = 0; i < LREG; ++i) acc[i] += double(qf[i]) * wd;
            accn += wd * wd;
          }
          __syncthreads();  // stage c % qst consumed by every thread
          qused = c + 1;
          if (tid == 0) qring_issue(c + qst);
          qissued = c + 1 + qst;
        }
      } else {
      // UNR rows per thread per iteration, all their loads issued before any is used
      constexpr int UNR = (sizeof(T) == 4 && LREG <= 32) ? 4 : 1;
      for (int64_t rb = tid; rb < R; rb += int64_t(kSwThreads) * UNR) {
        T qf[UNR][LREG];
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) {
          const int64_t r = rb + int64_t(kSwThreads) * uu;
          load_row(r, qf[uu]);
        }
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) {
          const int64_t r = rb + int64_t(kSwThreads) * uu;
          if (r >= R) continue;
          double u[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int i = 0; i < LREG; ++i)
            u[i & 3] += double(qf[uu][i]) * colnew[i];
          double uu2 = (u[0] + u[1]) + (u[2] + u[3]);
          if (beta != 0.0) uu2 -= shift;
          const double wd = fmax(uu2, 0.0);
          wpos |= wd > 0.0;
          a.w[(r0 + r) * k + j] = T(wd);
#pragma unroll
          for (int i = 0; i < LREG; ++i) acc[i] += double(qf[uu][i]) * wd;
          accn += wd * wd;
        }
      }
      }
      prof_tick(kPfLift);
#pragma unroll
      for (int chunk = 0; chunk < (LREG + 31) / 32; ++chunk) {
        if (chunk * 32 < L1) {
          double v[16];
          {
            const bool hi = (lane & 16) != 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int ia = chunk * 32 + e, ib = ia + 16;
              // entry l (the squared norm) lives in accn; acc[l] is zero (qf is zero past l)
              const double va = (ia < LREG ? acc[ia < LREG ? ia : 0] : 0.0) + (ia == l ? accn : 0.0);
              const double vb = (ib < LREG ? acc[ib < LREG ? ib : 0] : 0.0) + (ib == l ? accn : 0.0);
              const double send = hi ? va : vb;
              const double mine = hi ? vb : va;
              v[e] = mine + __shfl_xor_sync(0xffffffffu, send, 16);
            }
          }
#pragma unroll
          for (int off = 8; off >= 1; off >>= 1) {
            const bool hi = (lane & off) != 0;
#pragma unroll
            for (int e = 0; e < off; ++e) {
              const double send = hi ? v[e] : v[e + off];
              const double mine = hi ? v[e + off] : v[e];
              v[e] = mine + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
          const int i = chunk * 32 + lane;
          if (i < L1) red[wid * kRedStride + i] = v[0];
        }
      }
    } else {
    for (int64_t r = tid; r < R; r += kSwThreads) {
      double u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0;
      int i = 0;
      for (; i + 3 < l; i += 4) {
        u0 += q(r, i) * colnew[i];
        u1 += q(r, i + 1) * colnew[i + 1];
        u2 += q(r, i + 2) * colnew[i + 2];
        u3 += q(r, i + 3) * colnew[i + 3];
      }
      for (; i < l; ++i) u0 += q(r, i) * colnew[i];
      double u = (u0 + u1) + (u2 + u3);
      if (beta != 0.0) u -= shift;
      const double wd = fmax(u, 0.0);
      wpos |= wd > 0.0;
      wcold[r] = wd;
      if constexpr (QS)
        WsT[int64_t(j) * RM + r] = T(wd);
      else
        a.w[(r0 + r) * k + j] = T(wd);
    }
    __syncthreads();
    prof_tick(kPfLift);
    // partials of [Q^T W(:,j); ||W(:,j)||^2] over this CTA's rows: warp w takes rows w, w+8, ..
    // (two interleaved accumulators); lane slot u covers output i = lane + 32 u, where output l
    // is the squared norm ("column l of Q" is W(:,j) itself).  Branch-free: inactive lanes
    // multiply by zero.
    {
      const int nslots = (L1 + 31) / 32;
      double a0[kMaxLSlots], a1[kMaxLSlots];
#pragma unroll
      for (int u = 0; u < kMaxLSlots; ++u) a0[u] = a1[u] = 0.0;
      int64_t r = wid;
      for (; r + kSwWarps < R; r += 2 * kSwWarps) {
        const double w0 = wcol_get(r), w1 = wcol_get(r + kSwWarps);
#pragma unroll
        for (int u = 0; u < kMaxLSlots; ++u) {
          if (u < nslots) {
            const int i = lane + 32 * u;
            const int ic = i < l ? i : l - 1;
            const double sel = i < l ? 1.0 : 0.0;
            const double q0 = sel * q(r, ic) + (i == l ? w0 : 0.0);
            const double q1 = sel * q(r + kSwWarps, ic) + (i == l ? w1 : 0.0);
            a0[u] += q0 * w0;
            a1[u] += q1 * w1;
          }
        }
      }
      if (r < R) {
        const double w0 = wcol_get(r);
#pragma unroll
        for (int u = 0; u < kMaxLSlots; ++u) {
          if (u < nslots) {
            const int i = lane + 32 * u;
            const int ic = i < l ? i : l - 1;
            const double q0 = (i < l ? q(r, ic) : 0.0) + (i == l ? w0 : 0.0);
            a0[u] += q0 * w0;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kMaxLSlots; ++u) {
        const int i = lane + 32 * u;
        if (u < nslots && i < L1) red[wid * kRedStride + i] = a0[u] + a1[u];
      }
    }
    }
    __syncthreads();
    double cpart = 0.0;
    if (tid < L1)
      for (int w = 0; w < kSwWarps; ++w) cpart += red[w * kRedStride + tid];
    if (a.flags & kReseed) {
      // reseed_dead: stamp column j alive in this sweep if any of the CTA's rows lifted positive
      if (__syncthreads_or(wpos) && tid == 0) atomicMax(a.alive + j, cur_t);
      wpos = false;
    }
    prof_tick(kPfRecomp);
    // W~(:,j) <- Q^T W(:,j) and P(i,:) += (W~_new(i,j) - W~_old(i,j)) V(j,:): thread i owns row i
    // of W~ and P, so the next column's prologue follows without a block barrier
    col_allreduce(L1, cpart, sc, inv, [&](int e, double v) {
      if (e < l) {
        const double d = v - colold[e];
        Wt[e * kp + j] = v;
        if constexpr (!QS) {
          if (!Pm) return;
        }
        double* pe = Pm + e * kp;
        const double* vj = Vm + j * k;
        int c = 0;
        for (; c + 8 <= k; c += 8) {
          double pv[8], vv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) pv[u] = pe[c + u], vv[u] = vj[c + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) pe[c + u] = pv[u] + d * vv[u];
        }
        for (; c < k; ++c) pe[c] += d * vj[c];
      } else {
        wn[j] = v;
      }
    });
    if (chain && j + 1 < k) col_prepare(j + 1);
    __syncthreads();
  }

  // Interleaved / Shuffled orders (p/src/rhals.cpp:34-45,73-78): component j alone, with T(:,j) and
  // V(:,j) recomputed from the current H (rhals_w_component_fresh), then row j of H against the
  // new W~(:,j) (rhals_h_component_fresh -> clamped_row_update, p/src/hals.cpp:75-81).
  __device__ void fresh_component(int j) {
    // (a) t_j = B H(j,:)^T (l), v_j = H H(j,:)^T (k): partials over this CTA's columns, one barrier
    const int L = l + k;
    for (int e = tid; e < L; e += kSwThreads) {
      const T* xa = e < l ? Bc + e * ncp : Hc + (e - l) * ncp;
      const T* xb = Hc + j * ncp;
      double s0 = 0.0, s1 = 0.0;
      int64_t c = 0;
      for (; c + 1 < NC; c += 2) {
        s0 += double(xa[c]) * double(xb[c]);
        s1 += double(xa[c + 1]) * double(xb[c + 1]);
      }
      if (c < NC) s0 += double(xa[c]) * double(xb[c]);
      part_base()[int64_t(g) * L + e] = s0 + s1;
    }
    allreduce1(L, [&](int e, double v) {
      if (e < l) {
        Tm[e * kp + j] = v;
      } else {
        Vm[(e - l) * k + j] = v;
        Vm[j * k + (e - l)] = v;
      }
    });
    // P(:, j) = W~ v_j for the prologue
    for (int i = tid; i < l; i += kSwThreads) {
      double s = 0.0;
      for (int c = 0; c < k; ++c) s += Wt[i * kp + c] * Vm[c * k + j];
      if (Pm) Pm[i * kp + j] = s;
    }
    __syncthreads();
    col_prepare(j, true);
    __syncthreads();
    w_column(j, false);
    // (b) row j of H: s = W~^T W~(:,j) (replicated), then every owned column c (no reduction)
    double* sv = colold;  // free after the column step (l >= k)
    for (int i = tid; i < k; i += kSwThreads) {
      double s = 0.0;
      for (int a2 = 0; a2 < l; ++a2) s += Wt[a2 * kp + i] * Wt[a2 * kp + j];
      sv[i] = s;
    }
    __syncthreads();
    const double alpha = a.alpha_h, beta = a.beta_h;
    const double denom = fmax(wn[j] + alpha, kDivisionFloor);
    bool hp = false;
    for (int64_t c = tid; c < NC; c += kSwThreads) {
      double r = 0.0, sh = 0.0;
      for (int i = 0; i < l; ++i) r += double(Bc[i * ncp + c]) * Wt[i * kp + j];
      for (int i = 0; i < k; ++i) sh += sv[i] * double(Hc[i * ncp + c]);
      const double hj = double(Hc[j * ncp + c]);
      double num = r - sh - alpha * hj;
      if (beta != 0.0) num -= beta;
      const T hv = T(fmax(0.0, hj + num / denom));
      Hc[j * ncp + c] = hv;
      hp |= hv > T(0);
    }
    if (a.flags & kReseed) {
      if (__syncthreads_or(hp) && tid == 0) atomicMax(a.alive + k + j, cur_t);
    }
    __syncthreads();
  }

  // H phase, one owned column per thread (clamped_row_update, p/src/hals.cpp:75-81, applied to the
  // column's k entries in order, p/src/rhals.cpp:52-55).  g_j = (S h)_j - r_j with r = B^T W~ is
  // kept in fp64 registers, so row update j is h_j <- [h_j - (g_j + alpha h_j + beta) / d_j]_+
  // followed by g += S(j, :) (h_j_new - h_j): a register chain without shuffles, 32 columns per
  // warp in flight.  Afterwards g is grad_H / 2 at the new h (grad_valid), the residual column
  // B(:,c) - W~ h goes to Rc (objc; W~^T residc for !grad_valid), and H is stored in place.
  template <int KH>
  __device__ void h_cols_lane(bool update, bool grad_valid, double& objc_l, double& pgh_l,
                              unsigned long long& hmask) {
    const double alpha = a.alpha_h, beta = a.beta_h;
    for (int64_t c = tid; c < NC; c += kSwThreads) {
      double g[KH];
#pragma unroll
      for (int j = 0; j < KH; ++j) g[j] = 0.0;
      // -r_j = -sum_i B(i,c) W~(i,j)
      for (int i = 0; i < l; ++i) {
        const double b = double(Bc[i * ncp + c]);
        const double* wi = Wt + i * kp;
#pragma unroll
        for (int j = 0; j < KH; ++j)
          if (j < k) g[j] = fma(-b, wi[j], g[j]);
      }
      // + (S h)_j
      for (int i = 0; i < k; ++i) {
        const double hi = double(Hc[i * ncp + c]);
        const double* si = Sm + i * k;
#pragma unroll
        for (int j = 0; j < KH; ++j)
          if (j < k) g[j] = fma(si[j], hi, g[j]);
      }
      if (update) {
        for (int j = 0; j < k; ++j) {
          double gj = g[0];  // g[j] without a dynamically indexed register array
#pragma unroll
          for (int i = 1; i < KH; ++i) gj = i == j ? g[i] : gj;
          const double hj = double(Hc[j * ncp + c]);
          double num = -(gj + alpha * hj);
          if (beta != 0.0) num -= beta;
          const double hn = fmax(0.0, hj + num * invd[j]);
          const double d = hn - hj;
          const T hv = T(hn);
          Hc[j * ncp + c] = hv;
          if (hv > T(0)) hmask |= 1ull << j;
          const double* sj = Sm + j * k;
#pragma unroll
          for (int i = 0; i < KH; ++i)
            if (i < k) g[i] = fma(sj[i], d, g[i]);
        }
      }
      if (grad_valid) {
        // grad_H = 2 (S h - r) (p/src/rhals.cpp:154), projected (p/src/hals.cpp:55-65)
#pragma unroll
        for (int j = 0; j < KH; ++j)
          if (j < k) {
            const double gv = 2.0 * g[j];
            const double gp = Hc[j * ncp + c] > T(0) ? gv : fmin(0.0, gv);
            pgh_l += gp * gp;
          }
      }
#pragma unroll
      for (int j = 0; j < KH; ++j) g[j] = 0.0;  // reused for W~^T residc
      // residc(:,c) = B(:,c) - W~ h; objc
      for (int i = 0; i < l; ++i) {
        const double* wi = Wt + i * kp;
        double r0 = double(Bc[i * ncp + c]), r1 = 0.0;
        int j = 0;
        for (; j + 1 < k; j += 2) {
          r0 = fma(-wi[j], double(Hc[j * ncp + c]), r0);
          r1 = fma(-wi[j + 1], double(Hc[(j + 1) * ncp + c]), r1);
        }
        if (j < k) r0 = fma(-wi[j], double(Hc[j * ncp + c]), r0);
        const double res = r0 + r1;
        objc_l += res * res;
        Rc[i * ncp + c] = T(res);
        if (!grad_valid) {
#pragma unroll
          for (int jj = 0; jj < KH; ++jj)
            if (jj < k) g[jj] = fma(wi[jj], res, g[jj]);
        }
      }
      if (!grad_valid) {
        // grad_H = -2 W~^T residc (p/src/rhals.cpp:155)
#pragma unroll
        for (int j = 0; j < KH; ++j)
          if (j < k) {
            const double gv = -2.0 * g[j];
            const double gp = Hc[j * ncp + c] > T(0) ? gv : fmin(0.0, gv);
            pgh_l += gp * gp;
          }
      }
    }
  }

  // S = W~^T W~ (k x k), replicated; invd_j = 1 / max(||W(:,j)||^2 + alpha_h, floor)
  __device__ void compute_s() {
    for (int e = tid; e < k; e += kSwThreads) invd[e] = 1.0 / fmax(wn[e] + a.alpha_h, kDivisionFloor);
    for (int e = tid; e < k * k; e += kSwThreads) {
      const int x = e / k, y = e % k;
      double s = 0.0;
      for (int i = 0; i < l; ++i) s += Wt[i * kp + x] * Wt[i * kp + y];
      Sm[e] = s;
    }
    __syncthreads();
  }

  // H phase and/or compressed evaluation over this CTA's columns, then the global reduction of
  // T, V, E, objc, pgrad_H.
  //   update:     apply clamped_row_update for j = 0..k-1 (p/src/rhals.cpp:52-55)
  //   grad_valid: grad_H = 2 (S H - R^T) (scratch valid, :154); else -2 W~^T residc (:155)
  // A column is handled by LPC lanes (16 when k <= 16, two columns per warp; else 32).  Lane j
  // keeps h_j, r_j = (B^T W~)(c, j) and the running dot acc_j = sum_i S(i,j) h_i; the sequential
  // row update j broadcasts only the change of h_j, so each of the k steps costs one shuffle
  // and one FMA per lane instead of a k-long reduction.  After the loop acc_j = (S h)_j, which is
  // exactly the first term of grad_H.
  __device__ void h_phase(bool update, bool grad_valid, double& objc, double& pgh) {
    prof_tick(kPfOther);
    compute_s();
    prof_tick(kPfHS);
    const double alpha = a.alpha_h, beta = a.beta_h;
    int LPC = k <= 16 ? 16 : 32;
    // narrower column groups when the CTA owns more columns than one round of LPC-lane groups
    // covers (e.g. 17 columns at LPC 16 would take two full rounds while the grid waits)
    while (LPC > 4 && NC > int64_t(kSwWarps) * (32 / LPC) && (k + LPC / 2 - 1) / (LPC / 2) <= kMaxPerLane &&
           (l + LPC / 2 - 1) / (LPC / 2) <= kMaxResSlots)
      LPC /= 2;
    const int CPW = 32 / LPC;
    const int sub = lane / LPC, sl = lane % LPC;
    double objc_l = 0.0, pgh_l = 0.0;
    unsigned long long hmask = 0ull;  // rows j of H with a positive entry here (reseed_dead)
    // lane-per-column path (h_cols_lane) where its k-long fp64 register array fits beside the
    // kernel's resident Q rows; the warp-per-column path below otherwise
    constexpr int kHCap = !QS || LREG == 0 ? 64 : LREG <= 32 ? 32 : 0;
    const int kh = k <= 32 ? 32 : k <= 64 ? 64 : 0;
    if (kh != 0 && kh <= kHCap && !(a.flags & kHWarpCols)) {
      if constexpr (kHCap >= 32) {
        if (kh == 32)
          h_cols_lane<32>(update, grad_valid, objc_l, pgh_l, hmask);
        else if constexpr (kHCap >= 64) {
          // k <= 48 (C4: k = 40): a 48-long register array instead of 64 -- the unrolled j loops issue
          // their predicated-off tail too, a quarter of the phase's DFMA / LDS slots at k = 40
          if (k <= 48)
            h_cols_lane<48>(update, grad_valid, objc_l, pgh_l, hmask);
          else
            h_cols_lane<64>(update, grad_valid, objc_l, pgh_l, hmask);
        }
      }
    } else
    for (int64_t cb = int64_t(wid) * CPW; cb < NC; cb += int64_t(kSwWarps) * CPW) {
      const int64_t cl = cb + sub;
      const bool valid = cl < NC;
      const int64_t clx = valid ? cl : 0;
      double h[kMaxPerLane], r[kMaxPerLane], acc[kMaxPerLane];
#pragma unroll
      for (int t = 0; t < kMaxPerLane; ++t) {
        const int j = sl + LPC * t;
        h[t] = (valid && j < k) ? double(Hc[j * ncp + clx]) : 0.0;
        double r0v = 0.0, r1v = 0.0;
        if (j < k) {
          int i = 0;
          for (; i + 1 < l; i += 2) {
            r0v += double(Bc[i * ncp + clx]) * Wt[i * kp + j];
            r1v += double(Bc[(i + 1) * ncp + clx]) * Wt[(i + 1) * kp + j];
          }
          if (i < l) r0v += double(Bc[i * ncp + clx]) * Wt[i * kp + j];
        }
        r[t] = r0v + r1v;
        acc[t] = 0.0;
      }
      prof_tick(kPfHInit);
      // acc_j = sum_i S(i, j) h_i
      // (the source slot ts is a compile-time index: register arrays stay in registers)
#pragma unroll
      for (int ts = 0; ts < kMaxPerLane; ++ts) {
        for (int o = 0; o < LPC && ts * LPC + o < k; ++o) {
          const int i = ts * LPC + o;
          const double hi = __shfl_sync(0xffffffffu, h[ts], o, LPC);
#pragma unroll
          for (int t = 0; t < kMaxPerLane; ++t) {
            const int j = sl + LPC * t;
            if (j < k) acc[t] += Sm[i * k + j] * hi;
          }
        }
      }
      if (update) {
#pragma unroll
        for (int ts = 0; ts < kMaxPerLane; ++ts) {
          for (int owner = 0; owner < LPC && ts * LPC + owner < k; ++owner) {
            const int j = ts * LPC + owner;
            // branch-free: every lane evaluates its own candidate, the owner's is broadcast
            double num = r[ts] - acc[ts] - alpha * h[ts];
            if (beta != 0.0) num -= beta;
            const double hn = fmax(0.0, h[ts] + num * invd[j]);
            const double dj = __shfl_sync(0xffffffffu, hn - h[ts], owner, LPC);
            if (sl == owner) h[ts] = hn;
#pragma unroll
            for (int t = 0; t < kMaxPerLane; ++t) {
              const int jj = sl + LPC * t;
              if (jj < k) acc[t] += Sm[j * k + jj] * dj;
            }
          }
        }
      }
      prof_tick(kPfHUpd);
      // residc(:,c) = B(:,c) - W~ h
      double res[kMaxResSlots];
#pragma unroll
      for (int u = 0; u < kMaxResSlots; ++u) {
        const int i = sl + LPC * u;
        res[u] = (i < l) ? double(Bc[i * ncp + clx]) : 0.0;
      }
#pragma unroll
      for (int ts = 0; ts < kMaxPerLane; ++ts) {
        for (int o = 0; o < LPC && ts * LPC + o < k; ++o) {
          const int j = ts * LPC + o;
          const double hj = __shfl_sync(0xffffffffu, h[ts], o, LPC);
#pragma unroll
          for (int u = 0; u < kMaxResSlots; ++u) {
            const int i = sl + LPC * u;
            if (i < l) res[u] -= Wt[i * kp + j] * hj;
          }
        }
      }
      double gs[kMaxPerLane];
#pragma unroll
      for (int t = 0; t < kMaxPerLane; ++t) gs[t] = 0.0;
      if (!grad_valid) {
        // -2 W~^T residc: broadcast residc entries across the column's lanes
#pragma unroll
        for (int us = 0; us < kMaxResSlots; ++us) {
          for (int o = 0; o < LPC && us * LPC + o < l; ++o) {
            const int i = us * LPC + o;
            const double ri = __shfl_sync(0xffffffffu, res[us], o, LPC);
#pragma unroll
            for (int t = 0; t < kMaxPerLane; ++t) {
              const int jj = sl + LPC * t;
              if (jj < k) gs[t] += Wt[i * kp + jj] * ri;
            }
          }
        }
      }
      if (valid) {
#pragma unroll
        for (int u = 0; u < kMaxResSlots; ++u) {
          const int i = sl + LPC * u;
          if (i < l) {
            objc_l += res[u] * res[u];
            Rc[i * ncp + cl] = T(res[u]);
          }
        }
#pragma unroll
        for (int t = 0; t < kMaxPerLane; ++t) {
          const int j = sl + LPC * t;
          if (j < k) {
            if (update) {
              const T hv = T(h[t]);
              Hc[j * ncp + cl] = hv;
              if (hv > T(0)) hmask |= 1ull << j;
            }
            const double gval = grad_valid ? 2.0 * (acc[t] - r[t]) : -2.0 * gs[t];
            const double gp = h[t] > 0.0 ? gval : fmin(0.0, gval);
            pgh_l += gp * gp;
          }
        }
      }
    }
    __syncthreads();
    if (update && (a.flags & kReseed)) {
      // reseed_dead: stamp the rows of H that keep a positive entry in this CTA's columns
      __shared__ unsigned long long mask_s;
      if (tid == 0) mask_s = 0ull;
      __syncthreads();
      if (hmask) atomicOr(&mask_s, hmask);
      __syncthreads();
      if (tid == 0)
        for (int j = 0; j < k; ++j)
          if ((mask_s >> j) & 1ull) atomicMax(a.alive + k + j, cur_t);
    }
    prof_tick(kPfHCols);
    // CTA partial products: [T (l k) | V (k k) | E (l k) | objc | pgh]
    const int lk = l * k, kk = k * k, L = 2 * lk + kk + 2;
    double* p = part_base();
    if constexpr (sizeof(T) == 4) {
      // [T; V; E] = [B; H; R] H^T over this CTA's columns: rows a of the stacked operand map to
      // partial index a k + j.  4 x 8 output tiles per thread, fp32 products summed in blocks of 32
      // columns (the operands are fp32-rounded already) and the blocks added in fp64 -- no fp64
      // conversion per product.
      // (2 x 8 tiles on the register-resident Q path, whose Q rows occupy 128 registers)
      constexpr int TI = (QS && LREG >= 64) ? 2 : 4;
      const int AR = 2 * l + k;
      const int ntJ = (k + 7) / 8, ntiles = ((AR + TI - 1) / TI) * ntJ;
      for (int tile = tid; tile < ntiles; tile += kSwThreads) {
        const int a0 = (tile / ntJ) * TI, j0 = (tile % ntJ) * 8;
        const T* ap[TI];
        const T* hp[8];
#pragma unroll
        for (int u = 0; u < TI; ++u) {
          const int ar = min(a0 + u, AR - 1);
          ap[u] = ar < l ? Bc + ar * ncp : ar < l + k ? Hc + (ar - l) * ncp : Rc + (ar - l - k) * ncp;
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) hp[v] = Hc + min(j0 + v, k - 1) * ncp;
        double accd[TI][8];
#pragma unroll
        for (int u = 0; u < TI; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v) accd[u][v] = 0.0;
        for (int64_t cb = 0; cb < NC; cb += 32) {
          const int64_t ce = min(NC, cb + 32);
          float accf[TI][8];
#pragma unroll
          for (int u = 0; u < TI; ++u)
#pragma unroll
            for (int v = 0; v < 8; ++v) accf[u][v] = 0.f;
          for (int64_t c = cb; c < ce; ++c) {
            float av[TI], hv[8];
#pragma unroll
            for (int u = 0; u < TI; ++u) av[u] = float(ap[u][c]);
#pragma unroll
            for (int v = 0; v < 8; ++v) hv[v] = float(hp[v][c]);
#pragma unroll
            for (int u = 0; u < TI; ++u)
#pragma unroll
              for (int v = 0; v < 8; ++v) accf[u][v] = fmaf(av[u], hv[v], accf[u][v]);
          }
#pragma unroll
          for (int u = 0; u < TI; ++u)
#pragma unroll
            for (int v = 0; v < 8; ++v) accd[u][v] += double(accf[u][v]);
        }
#pragma unroll
        for (int u = 0; u < TI; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v)
            if (a0 + u < AR && j0 + v < k) p[int64_t(g) * L + (a0 + u) * k + j0 + v] = accd[u][v];
      }
    } else
    for (int e = tid; e < 2 * lk + kk; e += kSwThreads) {
      const T *xa, *xb;
      if (e < lk) {
        xa = Bc + (e / k) * ncp;
        xb = Hc + (e % k) * ncp;
      } else if (e < lk + kk) {
        const int f = e - lk;
        xa = Hc + (f / k) * ncp;
        xb = Hc + (f % k) * ncp;
      } else {
        const int f = e - lk - kk;
        xa = Rc + (f / k) * ncp;
        xb = Hc + (f % k) * ncp;
      }
      double s0 = 0.0, s1 = 0.0;
      int64_t c = 0;
      for (; c + 1 < NC; c += 2) {
        s0 += double(xa[c]) * double(xb[c]);
        s1 += double(xa[c + 1]) * double(xb[c + 1]);
      }
      if (c < NC) s0 += double(xa[c]) * double(xb[c]);
      p[int64_t(g) * L + e] = s0 + s1;
    }
    {
      const double o = warp_allreduce_sum(objc_l), ph = warp_allreduce_sum(pgh_l);
      if (lane == 0) {
        red[kRedLen + wid] = o;
        red[kRedLen + kSwWarps + wid] = ph;
      }
      __syncthreads();
      if (tid == 0) {
        double so = 0.0, sp = 0.0;
        for (int w = 0; w < kSwWarps; ++w) so += red[kRedLen + w], sp += red[kRedLen + kSwWarps + w];
        p[int64_t(g) * L + L - 2] = so;
        p[int64_t(g) * L + L - 1] = sp;
      }
    }
    prof_tick(kPfHProducts);
    efin = fin_base() + lk + kk;  // wide: E stays in this reduction buffer until the next h_phase
    allreduce2(L, [&](int e, double v) {
      if (e < lk) {
        Tm[(e / k) * kp + e % k] = v;
      } else if (e < lk + kk) {
        Vm[e - lk] = v;
      } else if (e < 2 * lk + kk) {
        if (QS || Em) Em[((e - lk - kk) / k) * kp + (e - lk - kk) % k] = v;
      } else {
        scal[e - (2 * lk + kk)] = v;  // scal[0] = objc, scal[1] = pgh
      }
    });
    objc = scal[0];
    pgh = scal[1];
    __syncthreads();
  }

  // projected ||grad_W||^2 with grad_W = -2 Q E (E = residc H^T), reduced over the grid.
  // Thread per row, 16 independent accumulators per pass (throughput- not latency-bound).
  __device__ double pgrad_w() {
    double acc = 0.0;
    // E = residc H^T: shared memory, or (wide) the last h_phase reduction buffer
    const double* Ep = (QS || Em) ? Em : efin;
    const int es = (QS || Em) ? kp : k;
    if constexpr (F32S) {
      // fp32: E (fp64, replicated) -> fp32 copy in shared memory; per row the float4 columns of Q,
      // the row's W from the column-major scratch, grad_W(r, j0..j0+7) by fp32 FMA
      const int k8 = (k + 7) & ~7;  // row stride of the fp32 copy: zero pad, 16-byte rows
      for (int e = tid; e < l * k8; e += kSwThreads) {
        const int i = e / k8, j = e % k8;
        ef[e] = j < k ? float(Ep[i * es + j]) : 0.f;
      }
      __syncthreads();
      // UNR rows per thread: all their Q / W loads are in flight together (the pass streams the Q
      // slab and W from L2) and every broadcast load of E feeds UNR rows' FMAs
      constexpr int L4 = LREG / 4;
      constexpr int UNR = LREG <= 32 ? 4 : 2;
      const float4* q4 = reinterpret_cast<const float4*>(a.q4);
      for (int64_t rb = tid; rb < R; rb += int64_t(kSwThreads) * UNR) {
        float4 qv[UNR][L4];
        int64_t rr[UNR];
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) {
          const int64_t r = rb + int64_t(kSwThreads) * uu;
          rr[uu] = r < R ? r0 + r : r0;  // clamped: in-range address, result unused
#pragma unroll
          for (int i4 = 0; i4 < L4; ++i4) qv[uu][i4] = __ldg(q4 + int64_t(i4) * a.m + rr[uu]);
        }
        float accf[UNR];
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) accf[uu] = 0.f;
        for (int j0 = 0; j0 < k; j0 += 8) {
          float sacc[UNR][8], wv[UNR][8];
#pragma unroll
          for (int uu = 0; uu < UNR; ++uu) {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              sacc[uu][t] = 0.f;
              wv[uu][t] = j0 + t < k ? a.wc[int64_t(j0 + t) * a.m + rr[uu]] : 0.f;
            }
          }
#pragma unroll
          for (int i4 = 0; i4 < L4; ++i4) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int i = 4 * i4 + c;
              if (i < l) {
                const float4* ei = reinterpret_cast<const float4*>(ef + i * k8 + j0);
                const float4 e0 = ei[0], e1 = ei[1];
#pragma unroll
                for (int uu = 0; uu < UNR; ++uu) {
                  const float qv1 = c == 0 ? qv[uu][i4].x : c == 1 ? qv[uu][i4].y : c == 2 ? qv[uu][i4].z : qv[uu][i4].w;
                  sacc[uu][0] = fmaf(qv1, e0.x, sacc[uu][0]);
                  sacc[uu][1] = fmaf(qv1, e0.y, sacc[uu][1]);
                  sacc[uu][2] = fmaf(qv1, e0.z, sacc[uu][2]);
                  sacc[uu][3] = fmaf(qv1, e0.w, sacc[uu][3]);
                  sacc[uu][4] = fmaf(qv1, e1.x, sacc[uu][4]);
                  sacc[uu][5] = fmaf(qv1, e1.y, sacc[uu][5]);
                  sacc[uu][6] = fmaf(qv1, e1.z, sacc[uu][6]);
                  sacc[uu][7] = fmaf(qv1, e1.w, sacc[uu][7]);
                }
              }
            }
          }
#pragma unroll
          for (int uu = 0; uu < UNR; ++uu) {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              if (j0 + t < k) {
                const float gv = -2.f * sacc[uu][t];
                const float gp = wv[uu][t] > 0.f ? gv : fminf(0.f, gv);
                accf[uu] = fmaf(gp, gp, accf[uu]);
              }
            }
          }
        }
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu)
          if (rb + int64_t(kSwThreads) * uu < R) acc += double(accf[uu]);
      }
    } else if constexpr (!QS && LREG > 0) {
      constexpr int UNR = (sizeof(T) == 4 && LREG <= 32) ? 4 : 1;
      for (int64_t rb = tid; rb < R; rb += int64_t(kSwThreads) * UNR) {
        T qf[UNR][LREG];
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) load_row(rb + int64_t(kSwThreads) * uu, qf[uu]);
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) {
          const int64_t r = rb + int64_t(kSwThreads) * uu;
          if (r >= R) continue;
          const T* wr = a.w + (r0 + r) * k;
          for (int j0 = 0; j0 < k; j0 += 8) {
            double sacc[8];
            T wv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              sacc[t] = 0.0;
              wv[t] = j0 + t < k ? wr[j0 + t] : T(0);
            }
#pragma unroll
            for (int i = 0; i < LREG; ++i) {
              if (i < l) {
                const double qv = double(qf[uu][i]);
                const double* ei = Ep + i * es + j0;
#pragma unroll
                for (int t = 0; t < 8; ++t)
                  if (j0 + t < k) sacc[t] += qv * ei[t];
              }
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              if (j0 + t < k) {
                const double gv = -2.0 * sacc[t];
                const double gp = wv[t] > T(0) ? gv : fmin(0.0, gv);
                acc += gp * gp;
              }
            }
          }
        }
      }
    } else {
    bool done = false;
    if constexpr (QS && LREG > 0) {
      // register-resident Q rows: E packed (even row stride, zero pad) into the red scratch so each
      // i step is 16-byte broadcast loads + DFMAs against the row already in registers
      const int kE = (k + 1) & ~1;
      if (l * kE <= kRedLen) {
        __syncthreads();
        for (int e = tid; e < l * kE; e += kSwThreads) {
          const int i = e / kE, j = e % kE;
          red[e] = j < k ? Ep[i * es + j] : 0.0;
        }
        __syncthreads();
        if (tid < R) {
          for (int j0 = 0; j0 < k; j0 += 8) {
            double sacc[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) sacc[t] = 0.0;
#pragma unroll
            for (int i = 0; i < LREG; ++i) {
              if (i < l) {
                const double2* ep = reinterpret_cast<const double2*>(red + i * kE + j0);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  if (j0 + 2 * u < k) {
                    const double2 ev = ep[u];
                    sacc[2 * u] += qrow[i] * ev.x;
                    sacc[2 * u + 1] += qrow[i] * ev.y;
                  }
                }
              }
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              if (j0 + t < k) {
                const double gv = -2.0 * sacc[t];
                const double gp = w_get(tid, j0 + t) > T(0) ? gv : fmin(0.0, gv);
                acc += gp * gp;
              }
            }
          }
        }
        __syncthreads();  // red is block_sum's scratch next
        done = true;
      }
    }
    if (!done)
    for (int64_t r = tid; r < R; r += kSwThreads) {
      for (int j0 = 0; j0 < k; j0 += 16) {
        double sacc[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) sacc[u] = 0.0;
        for (int i = 0; i < l; ++i) {
          const double qv = q(r, i);
          const double* ei = Ep + i * es + j0;
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (j0 + u < k) sacc[u] += qv * ei[u];
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          if (j0 + u < k) {
            const double gv = -2.0 * sacc[u];
            const double gp = w_get(r, j0 + u) > T(0) ? gv : fmin(0.0, gv);
            acc += gp * gp;
          }
        }
      }
    }
    }
    const double tot = block_sum(acc);
    if (tid == 0) part_base()[g] = tot;
    prof_tick(kPfPgw);
    allreduce1(1, [&](int, double v) { scal[2] = v; });
    cross_allreduce(1, [&](int) { return scal[2]; }, [&](int, double v) { scal[2] = v; });
    const double out = scal[2];
    __syncthreads();
    return out;
  }

  __device__ void record(int64_t t, double objc, double pgrad) {
    if (g == 0 && tid == 0) {
      a.trace_objc[t] = objc;
      a.trace_pgrad[t] = pgrad;
      a.trace_time[t] = globaltimer_ns();
    }
  }

  __device__ void run() {
    const long long t_start = clock64();
    load_resident();
    if (a.flags & (kInitWt | kInitWn)) init_wt_wn();
    double pgrad0 = 0.0;
    if (a.flags & (kEval0 | kTvOnly)) {
      double objc = 0.0, pgh = 0.0;
      h_phase(false, false, objc, pgh);
      if (a.flags & kEval0) {
        const double pgw = pgrad_w();
        pgrad0 = pgw + pgh;
        record(0, objc, pgrad0);
        if (g == 0 && tid == 0) a.pgrad0[0] = pgrad0;
      }
    }
    if (!(a.flags & kEval0)) pgrad0 = ld_cg(a.pgrad0);
    int64_t last = a.t_begin - 1;
    int stopped = 0;
    int64_t reseed_at = 0;
    const bool pg_rule = a.stop_rule == 0;
    const bool stationary = (a.flags & kRecord) && pg_rule && !(pgrad0 > 0.0);
    if (a.flags & kEvalPrev) {
      // after a host-side reseed of sweep t_begin - 1: its compressed evaluation with the new W, H
      // (invalid scratch, p/src/rhals.cpp:182-188) and the stop test
      double objc = 0.0, pgh = 0.0;
      h_phase(false, false, objc, pgh);
      const double pgradc = pgrad_w() + pgh;
      record(a.t_begin - 1, objc, pgradc);
      if (pg_rule && pgradc < a.tol * pgrad0) stopped = 1;
    }
    if (!stationary && !stopped) {
      for (int64_t t = a.t_begin; t <= a.t_end; ++t) {
        cur_t = unsigned(t);
        const bool fresh = a.order != nullptr;
        if (fresh) {
          const int* ord = a.order + (t - a.t_begin) * k;
          for (int pos = 0; pos < k; ++pos) fresh_component(ord[pos]);
        } else if (a.flags & kDoW) {
          compute_p();
          col_prepare(0);
          __syncthreads();
          for (int j = 0; j < k; ++j) w_column(j);
        }
        if (a.flags & kDoH) {
          double objc = 0.0, pgh = 0.0;
          // fresh orders: H is already updated; evaluate with grad_H = -2 W~^T residc (the
          // reference's scratch is invalid for them, p/src/rhals.cpp:79,155; also with reseed_dead)
          h_phase(!fresh, !fresh && !(a.flags & kReseed), objc, pgh);
          if (a.flags & kReseed) {
            // a component whose W column or H row has no positive entry left: hand the sweep to the
            // host (reseed draws come from the reference stream), evaluated after the reseed
            bool dead = false;
            for (int j = 0; j < 2 * k; ++j) dead |= ld_cg(a.alive + j) != cur_t;
            if (dead) {
              reseed_at = t;
              break;
            }
          }
          if (a.flags & kRecord) {
            const double pgw = pgrad_w();
            const double pgradc = pgw + pgh;
            record(t, objc, pgradc);
            last = t;
            if (pg_rule && pgradc < a.tol * pgrad0) {
              stopped = 1;
              break;
            }
            continue;
          }
        }
        last = t;
      }
    }
    if (kSweepProf && prof_on) {
      prof_acc[kPfSweeps] = clock64() - t_start;
      for (int b = 0; b < kPfCount; ++b) a.prof[b] = prof_acc[b];
      a.prof[kPfCount] = epoch;
    }
    qring_drain();
    store_back(last, stopped);
    if (g == 0 && tid == 0) a.status[2] = reseed_at;
  }
};

template <typename T, bool QS, int LREG>
__global__ void __launch_bounds__(kSwThreads, 1) rhals_sweeps_kernel(SweepArgs<T> args, SmemLayout L, int64_t RM,
                                                                      int64_t NCM) {
  extern __shared__ __align__(16) unsigned char smem[];
  Sweeper<T, QS, LREG> s(args, smem, L, RM, NCM);
  s.run();
}

}  // namespace

#ifdef RNMF_SWEEPS_COMMON
namespace {
// q4[i4 * m + r] = Q(r, 4 i4 .. 4 i4 + 3), zero past l (the fp32 streamed sweep path's layout)
__global__ void relayout_q_kernel(const float* __restrict__ q, int64_t m, int l, int l4, float4* __restrict__ q4) {
  const int64_t total = m * l4;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i4 = e / m, r = e % m;
    const float* src = q + r * l + 4 * i4;
    float v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = 4 * i4 + c < l ? src[c] : 0.f;
    q4[e] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

}  // namespace

int sweep_relayout_q(const float* q, int64_t m, int l, int l_pad, float* q4, cudaStream_t stream) {
  const int l4 = l_pad / 4;
  const int64_t total = m * l4;
  const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 16));
  if (total > 0) relayout_q_kernel<<<blocks, 256, 0, stream>>>(q, m, l, l4, reinterpret_cast<float4*>(q4));
  RNMF_CUDA(cudaGetLastError());
  return total > 0 ? 1 : 0;
}
#endif

template <typename T>
SweepPlan plan_sweeps(int64_t m, int64_t n, int l, int k, int sm_count, int max_smem) {
  SweepPlan p;
  if (l > 32 * kMaxPerLane || k > 32 * kMaxPerLane) return p;
  const int G = sm_count;
  p.rows_per_cta = ceil_div(m, G);
  p.cols_per_cta = ceil_div(n, G);
  // RNMF_FORCE_NOQS / RNMF_NO_QREG / RNMF_NO_QSTREAM: testing knobs that force the other code paths
  // RNMF_FORCE_WIDE: testing knob, global-memory column slabs even where they fit on chip
  bool wide = std::getenv("RNMF_FORCE_WIDE") != nullptr;
  for (int pass = 0; pass < 2 && p.grid == 0; ++pass, wide = true) {
    for (int qs = (std::getenv("RNMF_FORCE_NOQS") || wide) ? 0 : 1; qs >= 0 && p.grid == 0; --qs) {
      const SmemLayout L = make_layout<T>(l, k, p.rows_per_cta, p.cols_per_cta, qs != 0, 0, 0, wide);
      if (qs && L.total > size_t(max_smem)) continue;
      p.q_in_smem = qs != 0;
      p.wide = wide;
      if (p.q_in_smem) {
        p.smem = L.total;
        p.grid = G;
        if (p.rows_per_cta <= kSwThreads && l + 1 <= 64 && !std::getenv("RNMF_NO_QREG"))
          p.lreg = (l + 1 <= 32) ? 32 : (l + 1 <= 48) ? 48 : 64;
        break;
      }
      if (sizeof(T) == 4 && !std::getenv("RNMF_NO_QSTREAM") && l <= 96) {
        // fp32 streamed path: float4-column Q, fp32 FMA, column-major W scratch
        const int lp = l <= 32 ? 32 : l <= 64 ? 64 : 96;
        const SmemLayout LF = make_layout<T>(l, k, p.rows_per_cta, p.cols_per_cta, false, 0, lp, wide);
        if (LF.total <= size_t(max_smem)) {
          p.f32s = true;
          p.lreg = lp;
          p.smem = LF.total;
          p.grid = G;
          break;
        }
      }
      if (L.total > size_t(max_smem)) break;  // generic path does not fit either: next pass (wide)
      p.smem = L.total;
      p.grid = G;
      if (!std::getenv("RNMF_NO_QSTREAM") && sizeof(T) == 8 && l + 1 <= 32) {
        p.lreg = 32;
        // bulk-copy ring for the streamed slab: 16-byte row pitch, the ring must fit as well
        for (int st = kQRingMax; st >= 2 && !p.qring; --st) {
          const SmemLayout LR = make_layout<T>(l, k, p.rows_per_cta, p.cols_per_cta, false, st, 0, wide);
          if ((int64_t(l) * int64_t(sizeof(T))) % 16 == 0 && LR.total <= size_t(max_smem) &&
              !std::getenv("RNMF_NO_QRING")) {
            p.qring = st;
            p.smem = LR.total;
          }
        }
      }
    }
  }
  if (p.grid == 0) p = SweepPlan{};
  return p;
}

template <typename T>
int launch_sweeps(const SweepArgs<T>& args, const SweepPlan& plan, cudaStream_t stream, bool zero_sync) {
  if (plan.grid <= 0) throw CudaError("sweeps: problem does not fit the persistent kernel");
  const SmemLayout L = make_layout<T>(args.l, args.k, plan.rows_per_cta, plan.cols_per_cta, plan.q_in_smem, plan.qring,
                                     plan.f32s ? plan.lreg : 0, plan.wide);
  if (plan.wide && args.rc == nullptr) throw CudaError("sweeps: wide layout needs the residc buffer");
  if (plan.f32s && (args.q4 == nullptr || args.wc == nullptr))
    throw CudaError("sweeps: fp32 streamed path needs the q4 / wc buffers");
  if (zero_sync) RNMF_CUDA(cudaMemsetAsync(args.barrier, 0, kSweepSyncBytes, stream));
  if (args.l + 1 > kColAccMax) throw CudaError("sweeps: sketch width above the column-reduction capacity");
  SweepArgs<T> a = args;
  // RNMF_COL_ORDERED: testing knob, column-step reduction through the ordered partial buffers
  if (std::getenv("RNMF_COL_ORDERED")) a.flags |= kColOrdered;
  // RNMF_XGPU_FLAT: testing knob, the flat cross-GPU column step (every CTA adds into every GPU)
  if (std::getenv("RNMF_XGPU_FLAT")) a.flags |= kXFlat;
  // RNMF_H_WARP_COLS: testing knob, the warp-per-column H phase
  if (std::getenv("RNMF_H_WARP_COLS")) a.flags |= kHWarpCols;
  int64_t RM = plan.rows_per_cta, NCM = plan.cols_per_cta;
  void* kargs[] = {&a, const_cast<SmemLayout*>(&L), &RM, &NCM};
  const void* stream64 = nullptr;
  const void* stream96 = nullptr;
  if constexpr (sizeof(T) == 4) {
    stream64 = reinterpret_cast<const void*>(rhals_sweeps_kernel<T, false, 64>);
    stream96 = reinterpret_cast<const void*>(rhals_sweeps_kernel<T, false, 96>);
  }
  const void* fn = !plan.q_in_smem ? (plan.lreg == 32   ? reinterpret_cast<const void*>(rhals_sweeps_kernel<T, false, 32>)
                                      : plan.lreg == 64 ? stream64
                                      : plan.lreg == 96 ? stream96
                                                        : reinterpret_cast<const void*>(rhals_sweeps_kernel<T, false, 0>))
                   : plan.lreg == 32 ? reinterpret_cast<const void*>(rhals_sweeps_kernel<T, true, 32>)
                   : plan.lreg == 48 ? reinterpret_cast<const void*>(rhals_sweeps_kernel<T, true, 48>)
                   : plan.lreg == 64 ? reinterpret_cast<const void*>(rhals_sweeps_kernel<T, true, 64>)
                                     : reinterpret_cast<const void*>(rhals_sweeps_kernel<T, true, 0>);
  RNMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(plan.smem)));
  int occ = 0;
  RNMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kSwThreads, plan.smem));
  if (occ < 1) throw CudaError("sweeps: kernel cannot be resident with " + std::to_string(plan.smem) + " B smem");
  RNMF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(plan.grid)), dim3(kSwThreads), kargs, plan.smem, stream));
  return 1;
}

#ifdef RNMF_SWEEPS_T
template SweepPlan plan_sweeps<RNMF_SWEEPS_T>(int64_t, int64_t, int, int, int, int);
template int launch_sweeps<RNMF_SWEEPS_T>(const SweepArgs<RNMF_SWEEPS_T>&, const SweepPlan&, cudaStream_t, bool);
#endif
#ifdef RNMF_SWEEPS_COMMON
bool sweep_prof_compiled() { return kSweepProf; }
#endif

}  // namespace rnmf_gpu
