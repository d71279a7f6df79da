// kernels_sweeps.cu — the compressed HALS loop as ONE persistent, cooperatively launched kernel.
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

#include <algorithm>

namespace rnmf_gpu {

namespace {

constexpr int kSwThreads = 256;
constexpr int kSwWarps = kSwThreads / 32;
constexpr int kMaxPerLane = 4;  // k, l <= 128
constexpr double kDivisionFloor = 1e-12;  // p/include/rnmf/hals.hpp:67

struct SmemLayout {
  // fp64 region
  size_t wt, tm, em, vm, sm, wn, red, scal, doubles_end;
  // T region (offsets in bytes from the start)
  size_t qs, wst, wcol, bc, hc, rc, total;
};

template <typename T>
SmemLayout make_layout(int l, int k, int64_t RM, int64_t NCM, bool qs) {
  SmemLayout L{};
  size_t d = 0;
  auto take = [&](size_t count) {
    const size_t off = d;
    d += count;
    return off;
  };
  L.wt = take(size_t(l) * k);
  L.tm = take(size_t(l) * k);
  L.em = take(size_t(l) * k);
  L.vm = take(size_t(k) * k);
  L.sm = take(size_t(k) * k);
  L.wn = take(size_t(k));
  L.red = take(kSwThreads + 2 * kSwWarps);
  L.scal = take(16);
  L.doubles_end = d * sizeof(double);
  size_t b = (L.doubles_end + 15) / 16 * 16;
  auto takeT = [&](size_t count) {
    const size_t off = b;
    b += (count * sizeof(T) + 15) / 16 * 16;
    return off;
  };
  const size_t ncp = size_t(NCM) + 1;
  L.qs = qs ? takeT(size_t(RM) * (l + 1)) : 0;
  L.wst = qs ? takeT(size_t(k) * RM) : 0;
  L.wcol = qs ? 0 : takeT(size_t(RM));
  L.bc = takeT(size_t(l) * ncp);
  L.hc = takeT(size_t(k) * ncp);
  L.rc = takeT(size_t(l) * ncp);
  L.total = b;
  return L;
}

template <typename T, bool QS>
struct Sweeper {
  const SweepArgs<T>& a;
  int G, g, tid, lane, wid, l, k;
  int64_t r0, R, c0, NC, RM;
  int ncp, lq;
  double *Wt, *Tm, *Em, *Vm, *Sm, *wn, *red, *scal;
  T *Qs, *WsT, *wcol, *Bc, *Hc, *Rc;
  unsigned epoch = 0;
  int slot = 0;
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
    ncp = int(NCM) + 1;
    lq = l + 1;
    double* D = reinterpret_cast<double*>(smem);
    Wt = D + L.wt;
    Tm = D + L.tm;
    Em = D + L.em;
    Vm = D + L.vm;
    Sm = D + L.sm;
    wn = D + L.wn;
    red = D + L.red;
    scal = D + L.scal;
    Qs = QS ? reinterpret_cast<T*>(smem + L.qs) : nullptr;
    WsT = QS ? reinterpret_cast<T*>(smem + L.wst) : nullptr;
    wcol = QS ? nullptr : reinterpret_cast<T*>(smem + L.wcol);
    Bc = reinterpret_cast<T*>(smem + L.bc);
    Hc = reinterpret_cast<T*>(smem + L.hc);
    Rc = reinterpret_cast<T*>(smem + L.rc);
    part_slot_len = sweep_part_len(l, k) * G;
    fin_slot_len = sweep_part_len(l, k);
  }

  __device__ __forceinline__ double q(int64_t r, int i) const {
    if constexpr (QS)
      return double(Qs[r * lq + i]);
    else
      return double(__ldg(a.q + (r0 + r) * l + i));
  }
  __device__ __forceinline__ T w_get(int64_t r, int j) const {
    if constexpr (QS)
      return WsT[int64_t(j) * RM + r];
    else
      return a.w[(r0 + r) * k + j];
  }
  __device__ __forceinline__ T wcol_get(int64_t r, int j) const {
    if constexpr (QS)
      return WsT[int64_t(j) * RM + r];
    else
      return wcol[r];
  }
  __device__ __forceinline__ double* part_base() { return a.part + int64_t(slot) * part_slot_len; }
  __device__ __forceinline__ double* fin_base() { return a.fin + int64_t(slot) * fin_slot_len; }
  __device__ __forceinline__ void next_slot() { slot ^= 1; }

  __device__ void barrier() { grid_barrier(a.barrier, epoch); }

  // every CTA: dst(e) = sum_g part[e][g] for e < L (fixed order), writer(e, value)
  template <typename Writer>
  __device__ void reduce_all(int L, Writer&& wr) {
    const double* p = part_base();
    for (int e = wid; e < L; e += kSwWarps) {
      double s = 0.0;
      for (int gg = lane; gg < G; gg += 32) s += ld_cg(p + int64_t(e) * G + gg);
      s = warp_allreduce_sum(s);
      if (lane == 0) wr(e, s);
    }
  }

  // Single-level all-reduce of vectors already written to part_base(): one barrier.
  template <typename Writer>
  __device__ void allreduce1(int L, Writer&& wr) {
    barrier();
    reduce_all(L, wr);
    next_slot();
    __syncthreads();
  }

  // Two-level all-reduce (reduce-scatter over CTAs, then all-gather): two barriers.
  template <typename Writer>
  __device__ void allreduce2(int L, Writer&& wr) {
    barrier();
    const double* p = part_base();
    double* f = fin_base();
    const int e0 = int(int64_t(L) * g / G), e1 = int(int64_t(L) * (g + 1) / G);
    for (int e = e0 + wid; e < e1; e += kSwWarps) {
      double s = 0.0;
      for (int gg = lane; gg < G; gg += 32) s += ld_cg(p + int64_t(e) * G + gg);
      s = warp_allreduce_sum(s);
      if (lane == 0) f[e] = s;
    }
    barrier();
    for (int e = tid; e < L; e += kSwThreads) wr(e, ld_cg(f + e));
    next_slot();
    __syncthreads();
  }

  __device__ double block_sum(double v) {
    v = warp_allreduce_sum(v);
    __syncthreads();
    if (lane == 0) red[kSwThreads + wid] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < kSwWarps; ++w) s += red[kSwThreads + w];
    __syncthreads();
    return s;
  }

  // ---------------------------------------------------------------------------------------------
  __device__ void load_resident() {
    if constexpr (QS) {
      for (int64_t e = tid; e < R * l; e += kSwThreads) {
        const int64_t r = e / l;
        const int i = int(e % l);
        Qs[r * lq + i] = a.q[(r0 + r) * l + i];
      }
      for (int64_t e = tid; e < R * k; e += kSwThreads) {
        const int64_t r = e / k;
        const int j = int(e % k);
        WsT[int64_t(j) * RM + r] = a.w[(r0 + r) * k + j];
      }
    }
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
    if (!(a.flags & kInitWt))
      for (int e = tid; e < l * k; e += kSwThreads) Wt[e] = a.wt[e];
    if (!(a.flags & kInitWn))
      for (int e = tid; e < k; e += kSwThreads) wn[e] = a.wn[e];
    if (!(a.flags & (kEval0 | kTvOnly))) {
      for (int e = tid; e < l * k; e += kSwThreads) Tm[e] = a.tm[e];
      for (int e = tid; e < k * k; e += kSwThreads) Vm[e] = a.vm[e];
    }
    __syncthreads();
  }

  __device__ void store_back(int64_t last, int stopped) {
    if constexpr (QS) {
      for (int64_t e = tid; e < R * k; e += kSwThreads) {
        const int64_t r = e / k;
        const int j = int(e % k);
        a.w[(r0 + r) * k + j] = WsT[int64_t(j) * RM + r];
      }
    }
    if (a.flags & kDoH) {
      for (int64_t e = tid; e < int64_t(k) * NC; e += kSwThreads) {
        const int j = int(e / NC);
        const int64_t cl = e % NC;
        a.h[int64_t(j) * a.n + c0 + cl] = Hc[j * ncp + cl];
      }
    }
    if (g == 0) {
      for (int e = tid; e < l * k; e += kSwThreads) {
        a.wt[e] = Wt[e];
        a.tm[e] = Tm[e];
        a.em[e] = Em[e];
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
      p[int64_t(e) * G + g] = s;
    }
    const bool do_wt = a.flags & kInitWt, do_wn = a.flags & kInitWn;
    allreduce2(L, [&](int e, double v) {
      if (e < lk) {
        if (do_wt) Wt[e] = v;
      } else if (do_wn) {
        wn[e - lk] = v;
      }
    });
  }

  // One column step of rhals_w_component (p/src/rhals.cpp:23-32).
  __device__ void w_column(int j) {
    const double alpha = a.alpha_w, beta = a.beta_w;
    const double denom = fmax(Vm[j * k + j] + alpha, kDivisionFloor);
    if (tid < l) {
      double wv = 0.0;
      for (int c = 0; c < k; ++c) wv += Wt[tid * k + c] * Vm[c * k + j];
      const double cur = Wt[tid * k + j];
      Wt[tid * k + j] = cur + (Tm[tid * k + j] - wv - alpha * cur) / denom;
    }
    __syncthreads();
    const double shift = beta != 0.0 ? beta / denom : 0.0;
    for (int64_t r = tid; r < R; r += kSwThreads) {
      double u = 0.0;
      for (int i = 0; i < l; ++i) u += q(r, i) * Wt[i * k + j];
      if (beta != 0.0) u -= shift;
      const T wv = T(fmax(u, 0.0));
      if constexpr (QS) {
        WsT[int64_t(j) * RM + r] = wv;
      } else {
        wcol[r] = wv;
        a.w[(r0 + r) * k + j] = wv;
      }
    }
    __syncthreads();
    // partials of [Q^T W(:,j); ||W(:,j)||^2] over this CTA's rows
    const int L1 = l + 1;
    const int S = kSwThreads / L1;
    if (tid < S * L1) {
      const int i = tid % L1, s = tid / L1;
      double acc = 0.0;
      for (int64_t r = s; r < R; r += S) {
        const double wr = double(wcol_get(r, j));
        acc += (i < l ? q(r, i) : wr) * wr;
      }
      red[s * L1 + i] = acc;
    }
    __syncthreads();
    if (tid < L1) {
      double v = 0.0;
      for (int s = 0; s < S; ++s) v += red[s * L1 + tid];
      part_base()[int64_t(tid) * G + g] = v;
    }
    allreduce1(L1, [&](int e, double v) {
      if (e < l)
        Wt[e * k + j] = v;
      else
        wn[j] = v;
    });
  }

  // S = W~^T W~ (k x k), replicated
  __device__ void compute_s() {
    for (int e = tid; e < k * k; e += kSwThreads) {
      const int x = e / k, y = e % k;
      double s = 0.0;
      for (int i = 0; i < l; ++i) s += Wt[i * k + x] * Wt[i * k + y];
      Sm[e] = s;
    }
    __syncthreads();
  }

  // H phase and/or compressed evaluation over this CTA's columns, then the global reduction of
  // T, V, E, objc, pgrad_H.
  //   update:     apply clamped_row_update for j = 0..k-1 (p/src/rhals.cpp:52-55)
  //   grad_valid: grad_H = 2 (S H - R^T) (scratch valid, :154); else -2 W~^T residc (:155)
  __device__ void h_phase(bool update, bool grad_valid, double& objc, double& pgh) {
    compute_s();
    const double alpha = a.alpha_h, beta = a.beta_h;
    double objc_l = 0.0, pgh_l = 0.0;
    for (int64_t cl = wid; cl < NC; cl += kSwWarps) {
      double h[kMaxPerLane], r[kMaxPerLane];
#pragma unroll
      for (int t = 0; t < kMaxPerLane; ++t) {
        const int j = lane + 32 * t;
        h[t] = j < k ? double(Hc[j * ncp + cl]) : 0.0;
        r[t] = 0.0;
      }
      for (int i = 0; i < l; ++i) {
        const double bi = double(Bc[i * ncp + cl]);
#pragma unroll
        for (int t = 0; t < kMaxPerLane; ++t) {
          const int j = lane + 32 * t;
          if (j < k) r[t] += bi * Wt[i * k + j];
        }
      }
      if (update) {
        for (int j = 0; j < k; ++j) {
          double p = 0.0;
#pragma unroll
          for (int t = 0; t < kMaxPerLane; ++t) {
            const int jj = lane + 32 * t;
            if (jj < k) p += Sm[jj * k + j] * h[t];
          }
          const double dot = warp_allreduce_sum(p);
          if (lane == (j & 31)) {
            const double d = fmax(wn[j] + alpha, kDivisionFloor);
#pragma unroll
            for (int t = 0; t < kMaxPerLane; ++t) {
              if (t == (j >> 5)) {
                double num = r[t] - dot - alpha * h[t];
                if (beta != 0.0) num -= beta;
                h[t] = fmax(0.0, h[t] + num / d);
              }
            }
          }
        }
      }
      // residc(:,c) = B(:,c) - W~ h ; grad accumulators
      double res[kMaxPerLane], gs[kMaxPerLane];
#pragma unroll
      for (int u = 0; u < kMaxPerLane; ++u) {
        const int i = lane + 32 * u;
        res[u] = i < l ? double(Bc[i * ncp + cl]) : 0.0;
        gs[u] = 0.0;
      }
      for (int j = 0; j < k; ++j) {
        double hsrc = 0.0;
#pragma unroll
        for (int t = 0; t < kMaxPerLane; ++t)
          if (t == (j >> 5)) hsrc = h[t];
        const double hj = __shfl_sync(0xffffffffu, hsrc, j & 31);
#pragma unroll
        for (int u = 0; u < kMaxPerLane; ++u) {
          const int i = lane + 32 * u;
          if (i < l) res[u] -= Wt[i * k + j] * hj;
        }
        if (grad_valid) {
#pragma unroll
          for (int t = 0; t < kMaxPerLane; ++t) {
            const int jj = lane + 32 * t;
            if (jj < k) gs[t] += Sm[jj * k + j] * hj;
          }
        }
      }
      if (!grad_valid) {
        // -2 W~^T residc: broadcast residc entries across the warp
        for (int i = 0; i < l; ++i) {
          double rsrc = 0.0;
#pragma unroll
          for (int u = 0; u < kMaxPerLane; ++u)
            if (u == (i >> 5)) rsrc = res[u];
          const double ri = __shfl_sync(0xffffffffu, rsrc, i & 31);
#pragma unroll
          for (int t = 0; t < kMaxPerLane; ++t) {
            const int jj = lane + 32 * t;
            if (jj < k) gs[t] += Wt[i * k + jj] * ri;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kMaxPerLane; ++u) {
        const int i = lane + 32 * u;
        if (i < l) {
          objc_l += res[u] * res[u];
          Rc[i * ncp + cl] = T(res[u]);
        }
      }
#pragma unroll
      for (int t = 0; t < kMaxPerLane; ++t) {
        const int j = lane + 32 * t;
        if (j < k) {
          if (update) Hc[j * ncp + cl] = T(h[t]);
          const double gval = grad_valid ? 2.0 * (gs[t] - r[t]) : -2.0 * gs[t];
          const double gp = h[t] > 0.0 ? gval : fmin(0.0, gval);
          pgh_l += gp * gp;
        }
      }
    }
    __syncthreads();
    // CTA partial products: [T (l k) | V (k k) | E (l k) | objc | pgh]
    const int lk = l * k, kk = k * k, L = 2 * lk + kk + 2;
    double* p = part_base();
    for (int e = tid; e < 2 * lk + kk; e += kSwThreads) {
      double s = 0.0;
      if (e < lk) {
        const T* bi = Bc + (e / k) * ncp;
        const T* hj = Hc + (e % k) * ncp;
        for (int64_t c = 0; c < NC; ++c) s += double(bi[c]) * double(hj[c]);
      } else if (e < lk + kk) {
        const int f = e - lk;
        const T* ha = Hc + (f / k) * ncp;
        const T* hb = Hc + (f % k) * ncp;
        for (int64_t c = 0; c < NC; ++c) s += double(ha[c]) * double(hb[c]);
      } else {
        const int f = e - lk - kk;
        const T* ri = Rc + (f / k) * ncp;
        const T* hj = Hc + (f % k) * ncp;
        for (int64_t c = 0; c < NC; ++c) s += double(ri[c]) * double(hj[c]);
      }
      p[int64_t(e) * G + g] = s;
    }
    const double o = block_sum(objc_l);
    const double ph = block_sum(pgh_l);
    if (tid == 0) {
      p[int64_t(L - 2) * G + g] = o;
      p[int64_t(L - 1) * G + g] = ph;
    }
    allreduce2(L, [&](int e, double v) {
      if (e < lk)
        Tm[e] = v;
      else if (e < lk + kk)
        Vm[e - lk] = v;
      else if (e < 2 * lk + kk)
        Em[e - lk - kk] = v;
      else
        scal[e - (2 * lk + kk)] = v;  // scal[0] = objc, scal[1] = pgh
    });
    objc = scal[0];
    pgh = scal[1];
    __syncthreads();
  }

  // projected ||grad_W||^2 with grad_W = -2 Q E (E = residc H^T), reduced over the grid.
  __device__ double pgrad_w() {
    double acc = 0.0;
    for (int64_t r = tid; r < R; r += kSwThreads) {
      for (int j = 0; j < k; ++j) {
        double s = 0.0;
        for (int i = 0; i < l; ++i) s += q(r, i) * Em[i * k + j];
        const double gv = -2.0 * s;
        const double gp = w_get(r, j) > T(0) ? gv : fmin(0.0, gv);
        acc += gp * gp;
      }
    }
    const double tot = block_sum(acc);
    if (tid == 0) part_base()[g] = tot;
    allreduce1(1, [&](int, double v) { scal[2] = v; });
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
    const bool pg_rule = a.stop_rule == 0;
    const bool stationary = (a.flags & kRecord) && pg_rule && !(pgrad0 > 0.0);
    if (!stationary) {
      for (int64_t t = a.t_begin; t <= a.t_end; ++t) {
        if (a.flags & kDoW)
          for (int j = 0; j < k; ++j) w_column(j);
        if (a.flags & kDoH) {
          double objc = 0.0, pgh = 0.0;
          h_phase(true, true, objc, pgh);
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
    store_back(last, stopped);
  }
};

template <typename T, bool QS>
__global__ void __launch_bounds__(kSwThreads, 1) rhals_sweeps_kernel(SweepArgs<T> args, SmemLayout L, int64_t RM,
                                                                      int64_t NCM) {
  extern __shared__ __align__(16) unsigned char smem[];
  Sweeper<T, QS> s(args, smem, L, RM, NCM);
  s.run();
}

}  // namespace

template <typename T>
SweepPlan plan_sweeps(int64_t m, int64_t n, int l, int k, int sm_count, int max_smem) {
  SweepPlan p;
  if (l > 32 * kMaxPerLane || k > 32 * kMaxPerLane) return p;
  const int G = sm_count;
  p.rows_per_cta = ceil_div(m, G);
  p.cols_per_cta = ceil_div(n, G);
  for (int qs = 1; qs >= 0; --qs) {
    const SmemLayout L = make_layout<T>(l, k, p.rows_per_cta, p.cols_per_cta, qs != 0);
    if (L.total <= size_t(max_smem)) {
      p.q_in_smem = qs != 0;
      p.smem = L.total;
      p.grid = G;
      return p;
    }
  }
  return p;
}

template <typename T>
int launch_sweeps(const SweepArgs<T>& args, const SweepPlan& plan, cudaStream_t stream) {
  if (plan.grid <= 0) throw CudaError("sweeps: problem does not fit the persistent kernel");
  const SmemLayout L = make_layout<T>(args.l, args.k, plan.rows_per_cta, plan.cols_per_cta, plan.q_in_smem);
  RNMF_CUDA(cudaMemsetAsync(args.barrier, 0, sizeof(unsigned), stream));
  SweepArgs<T> a = args;
  int64_t RM = plan.rows_per_cta, NCM = plan.cols_per_cta;
  void* kargs[] = {&a, const_cast<SmemLayout*>(&L), &RM, &NCM};
  const void* fn = plan.q_in_smem ? reinterpret_cast<const void*>(rhals_sweeps_kernel<T, true>)
                                  : reinterpret_cast<const void*>(rhals_sweeps_kernel<T, false>);
  RNMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(plan.smem)));
  int occ = 0;
  RNMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kSwThreads, plan.smem));
  if (occ < 1) throw CudaError("sweeps: kernel cannot be resident with " + std::to_string(plan.smem) + " B smem");
  RNMF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(plan.grid)), dim3(kSwThreads), kargs, plan.smem, stream));
  return 1;
}

template SweepPlan plan_sweeps<float>(int64_t, int64_t, int, int, int, int);
template SweepPlan plan_sweeps<double>(int64_t, int64_t, int, int, int, int);
template int launch_sweeps<float>(const SweepArgs<float>&, const SweepPlan&, cudaStream_t);
template int launch_sweeps<double>(const SweepArgs<double>&, const SweepPlan&, cudaStream_t);

}  // namespace rnmf_gpu
