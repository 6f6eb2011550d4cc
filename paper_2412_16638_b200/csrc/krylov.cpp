#include "krylov.hpp"

#include <array>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>

namespace mprkb {

// ---------------------------------------------------------------------------
// EventTimer
// ---------------------------------------------------------------------------
EventTimer::~EventTimer() {
  for (auto& o : open_) {
    cudaEventDestroy(o.a);
    cudaEventDestroy(o.b);
  }
  for (auto e : pool_) cudaEventDestroy(e);
}

cudaEvent_t EventTimer::get() {
  if (!pool_.empty()) {
    cudaEvent_t e = pool_.back();
    pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  CUDA_CHECK(cudaEventCreate(&e));
  return e;
}

int EventTimer::begin(const char* label, cudaStream_t st) {
  if (!enabled_) return -1;
  Open o{label, get(), get()};
  CUDA_CHECK(cudaEventRecord(o.a, st));
  open_.push_back(o);
  return (int)open_.size() - 1;
}

void EventTimer::end(int id, cudaStream_t st) {
  if (id < 0) return;
  CUDA_CHECK(cudaEventRecord(open_[id].b, st));
}

void EventTimer::resolve() {
  for (auto& o : open_) {
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, o.a, o.b));
    Entry* e = nullptr;
    for (auto& x : entries_)
      if (x.label == o.label) e = &x;
    if (!e) {
      entries_.push_back(Entry{o.label, 0, 0.0});
      e = &entries_.back();
    }
    ++e->count;
    e->seconds += ms * 1e-3;
    pool_.push_back(o.a);
    pool_.push_back(o.b);
  }
  open_.clear();
}

namespace {

using Bracket = TimerBracket;

template <class T> struct HostScalar { using type = T; };
template <> struct HostScalar<c32> { using type = std::complex<float>; };
template <> struct HostScalar<c64> { using type = std::complex<double>; };

// detail::scalar_cast<T>(double) (operators.hpp:30-33)
template <class H>
H scast(double x) {
  if constexpr (std::is_floating_point_v<H>)
    return static_cast<H>(x);
  else
    return static_cast<H>(static_cast<typename H::value_type>(x));
}
template <class H>
H conj_val(H x) {
  if constexpr (std::is_floating_point_v<H>)
    return x;
  else
    return std::conj(x);
}
template <class T, class H>
T to_dev(const H& h) {
  T t;
  static_assert(sizeof(T) == sizeof(H));
  std::memcpy(&t, &h, sizeof(T));
  return t;
}

// Finish the slot-0 reduction a FAST kernel just produced: this rank's fp64
// partial(s), summed across a split grid's ranks in rank order.
template <class T>
std::array<double, 2> finish_red(KrylovWork<T>& w, int nv, cudaStream_t st) {
  stream_sync(st);
  std::array<double, 2> v{0.0, 0.0};
  w.red.result(0, nv, v.data());
  if (w.comm && w.comm->size() > 1) w.comm->allreduce_sum(v.data(), nv);
  return v;
}

// Several single-value FAST reductions in one round trip: one stream
// synchronize, one cross-rank all-reduce of the whole batch.
template <class T, size_t K>
std::array<double, K> finish_slots(KrylovWork<T>& w, const std::array<int, K>& slots, cudaStream_t st) {
  stream_sync(st);
  std::array<double, K> v{};
  for (size_t i = 0; i < K; ++i) w.red.result(slots[i], 1, &v[i]);
  if (w.comm && w.comm->size() > 1) w.comm->allreduce_sum(v.data(), (int)K);
  return v;
}

// detail::dot_real / dot (krylov.hpp:43-67) over the whole (possibly split)
// vector.  PARITY on a split grid keeps the reference's single accumulator
// in global index order: rank r continues from rank r-1's partial sum, handed
// on by one broadcast per rank.
template <class T>
std::array<double, 2> global_dot(KrylovWork<T>& w, bool conj, const T* a, const T* b, Numerics num,
                                 cudaStream_t st) {
  const size_t m = w.size();
  const RedSlot s0 = w.red.slot(0);
  const int nv = conj && is_cplx<T> ? 2 : 1;
  Comm* c = w.comm;
  auto launch = [&](const double* init) {
    if (conj)
      dot_conj<T>(m, a, b, s0, num, st, init);
    else
      dot_real<T>(m, a, b, s0, num, st, init);
  };
  if (num == Numerics::Fast || !c || c->size() == 1) {
    launch(nullptr);
    return finish_red(w, nv, st);
  }
  std::array<double, 2> acc{0.0, 0.0};
  for (int r = 0; r < c->size(); ++r) {
    if (r == c->rank()) {
      launch(acc.data());
      stream_sync(st);
      w.red.result(0, nv, acc.data());
    }
    c->bcast_host(acc.data(), nv, r);
  }
  return acc;
}

}  // namespace

template <class T>
KrylovWork<T>::KrylovWork(size_t m) : red(4), m_(m) {
  for (auto& v : vecs_) v.alloc(m * sizeof(T));
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_host), sizeof(double) * 2 * kMaxH, cudaHostAllocMapped));
  CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_dev), h_host, 0));
}

template <class T>
KrylovWork<T>::~KrylovWork() {
  if (h_host) cudaFreeHost(h_host);
  if (ctl_host_) cudaFreeHost(ctl_host_);
}

template <class T>
void* KrylovWork<T>::basis16(int j) {
  while ((int)basis16_.size() <= j) basis16_.emplace_back(m_ * (is_cplx<T> ? 4 : 2));
  return basis16_[j].get();
}

template <class T>
T* KrylovWork<T>::basis(int j) {
  while ((int)basis_.size() <= j) basis_.emplace_back(m_ * sizeof(T));
  return basis_[j].template as<T>();
}

// ---------------------------------------------------------------------------
// cg<T>  (krylov.hpp:100-168)
// ---------------------------------------------------------------------------
template <class T>
void cg_solve(Op& A, Op* P, const T* b, T* x, const Crit& crit, Numerics num, KrylovWork<T>& w,
              SolveReport& rep, cudaStream_t st, EventTimer* timer, T* x_alt, T** result, CgSpec* spec) {
  using R = real_t<T>;
  const size_t m = w.size();
  if (A.size() != m || (P && P->size() != m)) MPRKB_THROW(2, "cg: operator size != vector length");
  rep = SolveReport{};
  Bracket whole(timer, "solver", st);
  const bool fast = num == Numerics::Fast;
  const StencilSpec* S = fast ? A.stencil() : nullptr;
  const RedSlot s0 = w.red.slot(0);
  T *r = w.v(0), *z = w.v(1), *p = w.v(2), *q = w.v(3);

  auto fetch = [&]() -> R { return (R)finish_red(w, 1, st)[0]; };
  auto rdot = [&](const T* a, const T* c) -> R { return (R)global_dot(w, false, a, c, num, st)[0]; };
  auto op = [&](const T* in, T* out) {
    Bracket br(timer, "stencil", st);
    A.apply(in, out, st);
  };
  auto pre = [&](const T* in, T* out) {
    if (P) {
      Bracket br(timer, "precond", st);
      P->set_timer(timer);  // the preconditioner's own tensor-r/m/l, diag labels
      P->apply(in, out, st);
    } else {
      CUDA_CHECK(cudaMemcpyAsync(out, in, m * sizeof(T), cudaMemcpyDeviceToDevice, st));
    }
  };
  // dst = b - A x, returns dot_real(dst, dst)
  auto residual = [&](T* dst) -> R {
    if (S) {
      Bracket br(timer, "stencil", st);
      stencil_residual<T>(*S, x, b, dst, &s0, st);
      return fetch();
    }
    op(x, q);
    vsub<T>(m, b, q, dst, fast ? &s0 : nullptr, st);
    return fast ? fetch() : rdot(dst, dst);
  };

  // FAST with the fused stencil: the scalars the reference needs one at a time
  // are produced speculatively and read in batches — r0, r.z and p.Ap of the
  // first iteration in ONE round trip, and (for an exact-inverse
  // preconditioner such as FastDiag, where the first update normally
  // converges) ||r|| with the true residual in another.  Every decision is
  // still taken in the reference's order on the same values; work the
  // reference would have skipped only touches scratch vectors (never x).
  const bool batch = fast && S != nullptr;
  const bool spec_true = batch && P != nullptr && P->exact_inverse();
  // ... and (fp32 / fp64 real, a second solution buffer) the first update,
  // ||r1|| and the true residual in one pass that leaves q unwritten
  bool fuse_first = false;
  if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double>) {
    const char* env = std::getenv("MPRKB_CG_FUSED");  // (=0: the unfused kernels, for A/B tests)
    fuse_first = spec_true && x_alt != nullptr && cg_fused_supported(*S) && !(env && env[0] == '0');
  }
  // x may alias b (x0 = rhs without a copy) only with a second buffer: the
  // fused first update writes beside it; otherwise x0 is copied there first
  if (x == b) {
    if (!x_alt) MPRKB_THROW(2, "cg: x aliases b without a second solution buffer");
    if (!fuse_first) {
      CUDA_CHECK(cudaMemcpyAsync(x_alt, b, m * sizeof(T), cudaMemcpyDeviceToDevice, st));
      x = x_alt;
      x_alt = nullptr;
    }
  }
  // (split grid: the tuples are this rank's — alpha needs the global sums:
  // each rank's local pair is formed on the device, all-gathered on the
  // stream (Comm::allgather_dev) and completed in rank order by the update
  // itself, so the split solve keeps ONE round trip; MPRKB_SPLIT_DEVALPHA=0
  // waits for the host's allreduced scalars instead)
  const bool split = w.comm && w.comm->size() > 1;
  const bool dev_alpha = fuse_first && !split;
  const char* sda_env = std::getenv("MPRKB_SPLIT_DEVALPHA");
  const bool gath_alpha = fuse_first && split && !(sda_env && sda_env[0] == '0');
  // (split grid: the judge adds the ranks' all-gathered local sums on the
  // device, so a split solve needs no round trip either)
  const bool speculate = (dev_alpha || gath_alpha) && spec != nullptr && !(gath_alpha && spec->defer);
  const RedSlot s2 = (dev_alpha || gath_alpha) ? w.red.slot_dev(2) : w.red.slot(2);
  const RedSlot s3 = speculate ? w.red.slot_dev(3) : w.red.slot(3);
  double r0;
  R rz{}, pq_first{};
  bool have_pq = false;
  double fused_v[2] = {0.0, 0.0};  // (||r1||^2, ||b - A x1||^2) of the fused first update
  // Pipelined iterations (FAST, fused stencil, a general preconditioner, one
  // rank): right after the update the next iteration's z = P r, r.z,
  // p = z + beta p (beta formed on the device, xpby_dev) and q = A p, p.q are
  // launched speculatively, and ONE round trip returns ||r||, r.z and p.q —
  // instead of one per scalar.  Decisions stay the reference's, in its
  // order; if it stops (converged, breakdown, veto) only p, q, z — scratch
  // from then on — were touched.
  const char* pipe_env = std::getenv("MPRKB_CG_PIPE");  // (=0: one round trip per scalar, for A/B tests)
  const bool pipe = batch && !spec_true && (!w.comm || w.comm->size() == 1) && !(pipe_env && pipe_env[0] == '0');
  R spec_rz{}, spec_pq{};
  bool have_spec = false;
  // Device loop (pipelined FAST CG, fp32, a preconditioner folded into the
  // update, the fused direction pass): batches of iterations run with their
  // scalars formed on the device (blas.cu k_cg_ctl, the host's arithmetic on
  // the same tuples) and ONE round trip per batch instead of one per
  // iteration; the host takes over, in the reference's order, where the
  // device stops (stopping test met -> true-residual confirmation / veto;
  // r.z or p.q not positive -> breakdown).  MPRKB_CG_DEVLOOP=0 disables it.
  bool devloop = false;
  if constexpr (std::is_same_v<T, float>) {
    const char* e = std::getenv("MPRKB_CG_DEVLOOP");
    devloop = pipe && P != nullptr && pq_fused_ok(*S) && !(e && e[0] == '0');
  }
  // batch length: 4 at first, then the iterations the observed residual
  // decay predicts are still needed (+1), so few gated no-op launches follow
  // the stop; capped at CgCtl::kMaxBatch
  int next_batch = 4;
  if (batch) {
    {
      Bracket br(timer, "stencil", st);
      if (speculate) {
        const RedSlot s0d = w.red.slot_dev(0);
        stencil_residual<T>(*S, x, b, r, &s0d, st);
      } else {
        stencil_residual<T>(*S, x, b, r, &s0, st);
      }
    }
    pre(r, z);
    {
      Bracket br(timer, "stencil", st);
      stencil_apply_dot2<T>(*S, z, fuse_first ? nullptr : q, r, s2, st);  // q = A z, (z.q, r.z)
    }
    if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double>) {
      if (speculate && spec->defer) {
        // the caller fuses the update into its next pass and judges it
        spec->dir = z;
        rep.iterations = 1;
        rep.converged = true;
        rep.speculative = true;
        if (result) *result = nullptr;
        return;
      }
      if (dev_alpha) {
        // the first update speculatively, alpha formed on the device from the
        // tuples above: it only writes x_alt, so whatever the host decides
        // below (r0 already small, breakdown) x is untouched
        {
          Bracket br(timer, "stencil", st);
          cg_fused_update(*S, 0.0f, &s2, x, z, b, r, x_alt, s3, st, nullptr, 0, speculate ? spec->x1_finite : nullptr);
        }
        if (speculate) {
          // no round trip: the device judges the one-iteration exit; the
          // caller reads the record after its own synchronize
          cg_spec_judge(w.red.slot_dev(0), s2, s3, crit.tol, spec->rec, spec->fail, st);
          rep.iterations = 1;
          rep.converged = true;
          rep.speculative = true;
          if (result) *result = x_alt;
          return;
        }
      } else if (gath_alpha) {
        const int P = w.comm->size();
        double* lsum = w.scal_dev(2 + 2 * (size_t)P + 5 + 5 * (size_t)P);
        tuple_sums(s2, 2, lsum, st);                     // this rank's (p.Ap, r.z)
        w.comm->allgather_dev(lsum, lsum + 2, 2, st);    // every rank's, in rank order
        {
          Bracket br(timer, "stencil", st);
          cg_fused_update(*S, 0.0f, nullptr, x, z, b, r, x_alt, s3, st, lsum + 2, P,
                          speculate ? spec->x1_finite : nullptr);
        }
        if (speculate) {
          double* l5 = lsum + 2 + 2 * (size_t)P;
          cg_spec_local(w.red.slot_dev(0), s2, s3, l5, st);
          w.comm->allgather_dev(l5, l5 + 5, 5, st);
          cg_spec_ranks(l5 + 5, P, crit.tol, spec->rec, spec->fail, st);
          rep.iterations = 1;
          rep.converged = true;
          rep.speculative = true;
          if (result) *result = x_alt;
          return;
        }
      }
    }
    stream_sync(st);
    double v[5];
    w.red.result(0, 1, &v[0]);
    w.red.result(2, 2, &v[1]);
    if (dev_alpha || gath_alpha) w.red.result(3, 2, &v[3]);
    if (split) w.comm->allreduce_sum(v, gath_alpha ? 5 : 3);  // (rank-order sums: per value as before)
    if (dev_alpha || gath_alpha) {
      fused_v[0] = v[3];
      fused_v[1] = v[4];
    }
    if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double>) {
      if (fuse_first && !dev_alpha && !gath_alpha) {  // split grid: the same pass with the global alpha
        const R a = (R)v[2] / (R)v[1];
        {
          Bracket br(timer, "stencil", st);
          cg_fused_update(*S, a, nullptr, x, z, b, r, x_alt, s3, st);
        }
        stream_sync(st);
        w.red.result(3, 2, fused_v);
        w.comm->allreduce_sum(fused_v, 2);
      }
    }
    r0 = (double)std::sqrt((R)v[0]);
    rz = (R)v[2];
    pq_first = (R)v[1];
    have_pq = true;
  } else {
    r0 = (double)std::sqrt(residual(r));
  }
  rep.history.push_back(r0);
  double rnorm = r0;
  bool x_clean = true;  // ||b - A x|| of the current x is known
  double clean_true = r0;
  if (crit.satisfied(rnorm, r0)) {
    rep.converged = true;
  } else {
    if (!batch) {
      pre(r, z);
      std::swap(p, z);  // p = z
      rz = rdot(r, p);
    } else {
      std::swap(p, z);  // p = z (q = A p already formed)
    }
    for (int k = 0; k < crit.max_iter; ++k) {
      if (!(rz > R{})) {
        rep.failure = 2;
        break;
      }
      R pq;
      if (have_pq) {
        pq = pq_first;
        have_pq = false;
      } else if (S) {
        Bracket br(timer, "stencil", st);
        stencil_apply_dot<T>(*S, p, q, s0, st);
        pq = fetch();
      } else {
        op(p, q);
        pq = rdot(p, q);
      }
      if (!(pq > R{})) {
        rep.failure = 2;
        break;
      }
      const R alpha = rz / pq;
      if constexpr (std::is_same_v<T, float>) {
        if (devloop && !(fuse_first && k == 0)) {
          const int batch = std::min(next_batch, crit.max_iter - k);
          CgCtl* ctl = w.ctl_dev();
          CgCtl& hc = *w.ctl_host();
          hc = CgCtl{};
          hc.alpha = alpha;
          hc.rz = rz;
          hc.r0 = r0;
          hc.tol = crit.tol;
          CUDA_CHECK(cudaMemcpyAsync(ctl, &hc, sizeof(CgCtl), cudaMemcpyHostToDevice, st));
          const RedSlot s1d = w.red.slot_dev(1), s2d = w.red.slot_dev(2);
          T* pn = nullptr;  // the work vector that is none of r, z, p, q
          for (T* c : {w.v(0), w.v(1), w.v(2), w.v(3), w.spare()})
            if (c != r && c != z && c != p && c != q) pn = c;
          T* pp[2] = {p, pn};
          bool ok = true;
          for (int j = 0; j < batch && ok; ++j) {
            {
              Bracket br(timer, "precond", st);
              ok = P->cg_update_apply_dev(ctl, x, pp[j & 1], r, q, z, s1d, st);
            }
            if (!ok) break;
            {
              Bracket br(timer, "stencil", st);
              pq_fused(*S, z, pp[j & 1], s1d, 1, 0.0f, pp[(j + 1) & 1], q, s2d, st, ctl);
            }
            cg_ctl_step(ctl, s1d, 0, 1, s2d, st);
          }
          if (!ok) {
            devloop = false;  // (no storage-level update for this preconditioner: host loop)
          } else {
            CUDA_CHECK(cudaMemcpyAsync(&hc, ctl, sizeof(CgCtl), cudaMemcpyDeviceToHost, st));
            stream_sync(st);
            const int done = hc.iters;  // >= 1: the batch's first iteration is never gated
            p = pp[done & 1];
            for (int i = 0; i < done; ++i) rep.history.push_back(hc.hist[i]);
            rep.iterations += done;
            x_clean = false;
            k += done - 1;
            rnorm = hc.hist[done - 1];
            if (hc.stop == 1) {  // the stopping test was met: confirm with the true residual
              const double rt = (double)std::sqrt(residual(q));
              x_clean = true;
              clean_true = rt;
              if (crit.satisfied(rt, r0)) {
                rep.converged = true;
                break;
              }
              std::swap(r, q);  // r = q (verified residual), restart
              rep.history.back() = rt;
              pre(r, z);
              std::swap(p, z);
              rz = rdot(r, p);
              have_spec = false;
              continue;
            }
            if (hc.stop == 2 || hc.stop == 3) {  // breakdown at the next loop top (unless max_iter ends it)
              if (k + 1 < crit.max_iter) {
                rep.failure = 2;
                break;
              }
              continue;
            }
            rz = hc.rz;  // batch exhausted: carry on with the next one
            pq_first = hc.pq;
            have_pq = true;
            {
              // predicted remaining iterations from the mean decay over the batch
              const double first = done > 1 ? hc.hist[0] : rep.history[rep.history.size() - 2];
              const double last = hc.hist[done - 1], target = std::max(crit.tol, crit.tol * r0);
              const int span = done > 1 ? done - 1 : 1;
              int pred = CgCtl::kMaxBatch;
              if (first > 0.0 && last > 0.0 && last < first) {
                const double rate = std::log(last / first) / span;  // < 0
                pred = (int)std::ceil(std::log(target / last) / rate) + 1;
              }
              next_batch = std::max(2, std::min(pred, (int)CgCtl::kMaxBatch));
            }
            continue;
          }
        }
      }
      bool fused = false;
      if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double>) {
        if (fuse_first && k == 0) {  // already ran (above), with this alpha
          std::swap(x, x_alt);
          fused = true;
        }
      }
      // (pipelined: a preconditioner that folds into the update also forms
      // the next z = P r and r.z in the same pass)
      bool pre_fused = false;
      if (!fused && pipe && P) {
        Bracket br(timer, "precond", st);
        pre_fused = P->cg_update_apply((double)alpha, x, p, r, q, z, w.red.slot_dev(1), st);
      }
      if (!fused && !pre_fused) cg_update<T>(m, alpha, x, p, r, q, fast ? &s0 : nullptr, st);
      x_clean = false;
      ++rep.iterations;
      double rt_spec = -1.0;
      if (fused) {
        rnorm = (double)std::sqrt((R)fused_v[0]);
        rt_spec = (double)std::sqrt((R)fused_v[1]);
        // the pass stored neither r1 nor the true residual: materialise the
        // one the reference continues from
        if (crit.satisfied(rnorm, r0)) {
          if (!crit.satisfied(rt_spec, r0)) {
            Bracket br(timer, "stencil", st);
            stencil_residual<T>(*S, x, b, q, nullptr, st);
          }
        } else {
          Bracket br(timer, "stencil", st);
          stencil_apply<T>(*S, p, q, st);
          cg_update<T>(m, alpha, nullptr, p, r, q, nullptr, st);  // r -= alpha q only
        }
      } else if (pipe) {
        const RedSlot s1d = w.red.slot_dev(1);
        if (!pre_fused) {
          pre(r, z);
          dot_real<T>(m, r, z, s1d, num, st);
        }
        bool pq_done = false;
        if constexpr (std::is_same_v<T, float>) {
          if (pq_fused_ok(*S)) {  // p update + A p + p.q in one pass, p ping-ponged
            Bracket br(timer, "stencil", st);
            T* pn = nullptr;  // the work vector that is none of r, z, p, q
            for (T* c : {w.v(0), w.v(1), w.v(2), w.v(3), w.spare()})
              if (c != r && c != z && c != p && c != q) pn = c;
            pq_fused(*S, z, p, s1d, pre_fused ? 1 : 0, rz, pn, q, s2, st);
            p = pn;
            pq_done = true;
          }
        }
        if (!pq_done) {
          xpby_dev<T>(m, z, s1d, pre_fused ? 1 : 0, rz, p, st);
          Bracket br(timer, "stencil", st);
          stencil_apply_dot<T>(*S, p, q, s2, st);
        }
        stream_sync(st);
        double v[3];
        if (pre_fused) {
          w.red.result(1, 2, &v[0]);  // (||r||^2, r.z) of the fused update
        } else {
          w.red.result(0, 1, &v[0]);
          w.red.result(1, 1, &v[1]);
        }
        w.red.result(2, 1, &v[2]);
        rnorm = (double)std::sqrt((R)v[0]);
        spec_rz = (R)v[1];
        spec_pq = (R)v[2];
        have_spec = true;
      } else if (spec_true) {
        {
          Bracket br(timer, "stencil", st);
          stencil_residual<T>(*S, x, b, q, &s3, st);  // q is free after the update
        }
        const auto v = finish_slots<T, 2>(w, {0, 3}, st);
        rnorm = (double)std::sqrt((R)v[0]);
        rt_spec = (double)std::sqrt((R)v[1]);
      } else {
        rnorm = (double)std::sqrt(fast ? fetch() : rdot(r, r));
      }
      rep.history.push_back(rnorm);
      if (crit.satisfied(rnorm, r0)) {
        const double rt = rt_spec >= 0.0 ? rt_spec : (double)std::sqrt(residual(q));
        x_clean = true;
        clean_true = rt;
        if (crit.satisfied(rt, r0)) {
          rep.converged = true;
          break;
        }
        std::swap(r, q);  // r = q (verified residual), restart
        rep.history.back() = rt;
        pre(r, z);
        std::swap(p, z);
        rz = rdot(r, p);
        have_spec = false;
        continue;
      }
      if (have_spec) {  // z, r.z, p and q = A p are already formed
        have_spec = false;
        rz = spec_rz;
        pq_first = spec_pq;
        have_pq = true;
        continue;
      }
      pre(r, z);
      const R rz_next = rdot(r, z);
      const R beta = rz_next / rz;
      rz = rz_next;
      xpby<T>(m, z, beta, p, st);
    }
    if (!rep.converged && rep.failure == 0) rep.failure = 1;
  }
  // exit true residual (krylov.hpp:164-166): recomputing it for an unchanged
  // x would reproduce the same value, so reuse it.
  rep.true_residual = x_clean ? clean_true : (double)std::sqrt(residual(q));
  if (x == b) {  // converged at x0 = b: the solution leaves the rhs buffer
    CUDA_CHECK(cudaMemcpyAsync(x_alt, b, m * sizeof(T), cudaMemcpyDeviceToDevice, st));
    x = x_alt;
  }
  if (result) *result = x;
}

// ---------------------------------------------------------------------------
// gmres<T>  (krylov.hpp:181-311)
// ---------------------------------------------------------------------------
template <class T>
void gmres_solve(Op& A, Op* P, const T* b, T* x, const Crit& crit, Numerics num, KrylovWork<T>& w,
                 SolveReport& rep, cudaStream_t st, EventTimer* timer, int basis_storage) {
  using R = real_t<T>;
  using H = typename HostScalar<T>::type;
  const size_t m = w.size();
  if (A.size() != m || (P && P->size() != m)) MPRKB_THROW(2, "gmres: operator size != vector length");
  rep = SolveReport{};
  Bracket whole(timer, "solver", st);
  const bool fast = num == Numerics::Fast;
  const RedSlot s0 = w.red.slot(0);
  const int kmax = crit.max_iter;
  const bool b16 = basis_storage == 4;
  if (basis_storage != -1 && !b16) MPRKB_THROW(10, "gmres: basis storage must be the working precision or F16");
  T *t = w.v(0), *wv = w.v(1), *xc = w.v(2), *wt = w.v(3);

  auto norm2 = [&](const T* v) -> R { return std::sqrt((R)global_dot(w, false, v, v, num, st)[0]); };
  auto dotc = [&](const T* a, const T* c) -> H {
    const auto v = global_dot(w, true, a, c, num, st);
    if constexpr (is_cplx<T>)
      return H((R)v[0], (R)v[1]);
    else
      return (R)v[0];
  };
  auto op = [&](const T* in, T* out) {
    Bracket br(timer, "stencil", st);
    A.apply(in, out, st);
  };
  auto pre = [&](const T* in, T* out) {
    if (P) {
      Bracket br(timer, "precond", st);
      P->set_timer(timer);  // the preconditioner's own tensor-r/m/l, diag labels
      P->apply(in, out, st);
    } else {
      CUDA_CHECK(cudaMemcpyAsync(out, in, m * sizeof(T), cudaMemcpyDeviceToDevice, st));
    }
  };
  // dst = b - A v  (fused when the operator is a stencil and numerics FAST)
  auto residual_of = [&](const T* v, T* dst) {
    if (fast && A.stencil()) {
      Bracket br(timer, "stencil", st);
      stencil_residual<T>(*A.stencil(), v, b, dst, nullptr, st);
      return;
    }
    op(v, dst);
    vsub<T>(m, b, dst, dst, nullptr, st);
  };

  double exit_true = -1.0;  // ||b - A x|| at exit when already formed (FAST)
  residual_of(x, t);
  pre(t, wv);  // w = P(b - A x0)
  const double beta = (double)norm2(wv);
  rep.history.push_back(beta);

  if (crit.satisfied(beta, beta) || beta == 0.0) {
    rep.converged = true;
  } else {
    std::vector<std::vector<H>> h_cols;
    h_cols.reserve(kmax);
    std::vector<R> cs(kmax, R{});
    std::vector<H> sn(kmax, H{});
    std::vector<H> s(kmax + 1, H{});
    std::vector<T*> basis;
    std::vector<void*> basis16;
    auto push_basis = [&](int j, H scale) {  // basis_j = w * scale
      if (b16) {
        basis16.push_back(w.basis16(j));
        basis16_scale<T>(m, wv, to_dev<T>(scale), basis16[j], st);
      } else {
        basis.push_back(w.basis(j));
        vscale<T>(m, wv, to_dev<T>(scale), basis[j], st);
      }
    };
    s[0] = scast<H>(beta);
    bool x_built = false;
    double cand_true = -1.0;

    // xc = x + sum_j y_j v_j with y from the rotated triangular system
    auto candidate_into = [&](int cols, T* dst) {
      std::vector<H> y(cols, H{});
      for (int i = cols - 1; i >= 0; --i) {
        H acc = s[i];
        for (int j = i + 1; j < cols; ++j) acc -= h_cols[j][i] * y[j];
        y[i] = acc / h_cols[i][i];
      }
      std::vector<T> yd(cols);
      for (int j = 0; j < cols; ++j) yd[j] = to_dev<T>(y[j]);
      if (b16) {
        basis16_candidate<T>(m, x, basis16.data(), yd.data(), cols, dst, st);
      } else {
        candidate<T>(m, x, basis.data(), yd.data(), cols, dst, st);
      }
    };

    push_basis(0, scast<H>(1.0) / scast<H>(beta));

    int k = 0;
    for (; k < kmax;) {
      const T* vk;
      bool applied = false, pre_applied = false;
      if constexpr (std::is_same_v<T, c32>) {
        // a stencil operator reads the fp16 basis vector itself (widened
        // exactly on load: bitwise the widen + apply; MPRKB_GMRES_H16_OP=0),
        // and a b = 8 block-Jacobi preconditioner folds into that pass
        // (bitwise A then P; MPRKB_GMRES_BJ_FOLD=0)
        const char* ho = std::getenv("MPRKB_GMRES_H16_OP");
        const char* bf = std::getenv("MPRKB_GMRES_BJ_FOLD");
        if (b16 && A.stencil() && !A.stencil()->halo && !(ho && ho[0] == '0')) {
          if (P && !(bf && bf[0] == '0')) {
            Bracket br(timer, "stencil", st);
            pre_applied = applied = P->stencil_then_apply_h16(*A.stencil(), basis16[k], wv, st);
          }
          if (!applied) {
            Bracket br(timer, "stencil", st);
            stencil_apply_h16(*A.stencil(), basis16[k], t, st);
            applied = true;
          }
        }
      }
      if (!applied) {
        if (b16) {  // the operator reads the basis vector widened to T (exact)
          basis16_widen<T>(m, basis16[k], wt, st);
          vk = wt;
        } else {
          vk = basis[k];
        }
        op(vk, t);
      }
      if (!pre_applied) pre(t, wv);
      std::vector<H> h(k + 2, H{});
      // fp16 basis, one rank: each h_j is formed on the device from its dot's
      // tuples (the host's sum order and rounding) and consumed there, so the
      // whole sweep runs without a round trip; the host reads the h_j after
      // the norm's synchronize.
      // (working-precision basis: the same in FAST numerics)
      const char* dh_env = std::getenv("MPRKB_GMRES_DEV_H");  // 0: never, 2: also the working-precision basis
      const int dh = dh_env ? dh_env[0] - '0' : 1;
      const bool dev_h = (dh == 2 ? (b16 || num == Numerics::Fast) : (dh == 1 && b16)) &&
                         (!w.comm || w.comm->size() == 1) && k + 1 <= KrylovWork<T>::kMaxH;
      // (fp16 basis: step j's update and step j + 1's dot share one pass,
      // bitwise the separate kernels; MPRKB_GMRES_FUSE_MGS=0 splits them)
      const char* fm_env = std::getenv("MPRKB_GMRES_FUSE_MGS");
      const bool fuse_mgs = !(fm_env && fm_env[0] == '0');
      bool norm_fused = false;
      if (dev_h) {
        const RedSlot sd = w.red.slot_dev(0);
        for (int j = 0; j <= k; ++j) {
          T* hd = w.h_val() + j;
          if (b16 && fuse_mgs) {
            if (j == 0) {
              basis16_dot<T>(m, basis16[0], wv, sd, st);
              finish_h<T>(sd, hd, w.h_dev, st);
            }
            if (j < k) {
              basis16_axmy_dot<T>(m, hd, basis16[j], basis16[j + 1], wv, sd, st);
              finish_h<T>(sd, hd + 1, w.h_dev + 2 * (j + 1), st);
            } else if (fast) {  // (the last update carries ||w||^2: read below)
              basis16_axmy_norm<T>(m, hd, basis16[j], wv, s0, st);
              norm_fused = true;
            } else {
              basis16_axmy_hp<T>(m, hd, basis16[j], wv, st);
            }
          } else if (b16) {
            basis16_dot<T>(m, basis16[j], wv, sd, st);
            finish_h<T>(sd, hd, w.h_dev + 2 * j, st);
            basis16_axmy_hp<T>(m, hd, basis16[j], wv, st);
          } else {
            dot_conj<T>(m, basis[j], wv, sd, num, st, nullptr);
            finish_h<T>(sd, hd, w.h_dev + 2 * j, st);
            vaxmy_hp<T>(m, hd, basis[j], wv, st);
          }
        }
      }
      for (int j = 0; j <= k && !dev_h; ++j) {  // modified Gram-Schmidt
        H hj;
        if (b16) {
          basis16_dot<T>(m, basis16[j], wv, s0, st);
          const auto v = finish_red(w, is_cplx<T> ? 2 : 1, st);
          if constexpr (is_cplx<T>)
            hj = H((R)v[0], (R)v[1]);
          else
            hj = (R)v[0];
          h[j] = hj;
          basis16_axmy<T>(m, to_dev<T>(hj), basis16[j], wv, st);
        } else {
          hj = dotc(basis[j], wv);
          h[j] = hj;
          vaxmy<T>(m, to_dev<T>(hj), basis[j], wv, st);
        }
      }
      const R wnorm = norm_fused ? std::sqrt((R)finish_red(w, 1, st)[0]) : norm2(wv);
      if (dev_h)
        for (int j = 0; j <= k; ++j) {
          const volatile double* hv = w.h_host + 2 * j;
          if constexpr (is_cplx<T>)
            h[j] = H((R)hv[0], (R)hv[1]);
          else
            h[j] = (R)hv[0];
        }
      h[k + 1] = scast<H>(static_cast<double>(wnorm));
      const bool happy = !(static_cast<double>(wnorm) > 0.0);

      for (int j = 0; j < k; ++j) {
        const H tmp = scast<H>(cs[j]) * h[j] + sn[j] * h[j + 1];
        h[j + 1] = scast<H>(cs[j]) * h[j + 1] - conj_val(sn[j]) * h[j];
        h[j] = tmp;
      }
      const R anorm = std::abs(h[k]);
      const R bnorm = std::abs(h[k + 1]);
      const R rho = std::sqrt(anorm * anorm + bnorm * bnorm);
      if (rho == R{}) {
        cs[k] = R{1};
        sn[k] = H{};
      } else if (anorm == R{}) {
        cs[k] = R{};
        sn[k] = scast<H>(1.0);
      } else {
        cs[k] = anorm / rho;
        sn[k] = (h[k] / scast<H>(static_cast<double>(anorm))) * scast<H>(static_cast<double>(bnorm / rho));
      }
      h[k] = scast<H>(cs[k]) * h[k] + sn[k] * h[k + 1];
      h[k + 1] = H{};
      s[k + 1] = -conj_val(sn[k]) * s[k];
      s[k] = scast<H>(cs[k]) * s[k];
      h_cols.push_back(std::move(h));

      ++rep.iterations;
      ++k;
      const double est = static_cast<double>(std::abs(s[k]));
      rep.history.push_back(est);

      if (happy) {
        rep.converged = true;
        break;
      }
      if (crit.satisfied(est, beta)) {
        candidate_into(k, xc);
        residual_of(xc, t);
        pre(t, wt);
        double rt;
        if (fast) {
          // FAST: ||P t|| and — should the candidate be accepted — the exit
          // true residual ||t|| of the same x in one round trip
          dot_real<T>(m, wt, wt, s0, num, st);
          dot_real<T>(m, t, t, w.red.slot(1), num, st);
          stream_sync(st);
          double v[2];
          w.red.result(0, 1, &v[0]);
          w.red.result(1, 1, &v[1]);
          if (w.comm && w.comm->size() > 1) w.comm->allreduce_sum(v, 2);
          rt = (double)std::sqrt((R)v[0]);
          cand_true = (double)std::sqrt((R)v[1]);
        } else {
          rt = static_cast<double>(norm2(wt));
        }
        if (crit.satisfied(rt, beta)) {
          CUDA_CHECK(cudaMemcpyAsync(x, xc, m * sizeof(T), cudaMemcpyDeviceToDevice, st));
          x_built = true;
          exit_true = cand_true;  // x is the candidate: its true residual is known
          rep.converged = true;
          break;
        }
        rep.history.back() = rt;
      }
      if (k == kmax) break;
      push_basis(k, scast<H>(1.0) / scast<H>(static_cast<double>(wnorm)));
    }
    if (!rep.converged) rep.failure = 1;
    if (!x_built) {
      candidate_into(k, xc);
      CUDA_CHECK(cudaMemcpyAsync(x, xc, m * sizeof(T), cudaMemcpyDeviceToDevice, st));
    }
  }

  if (exit_true >= 0.0) {
    rep.true_residual = exit_true;
  } else {
    residual_of(x, t);
    rep.true_residual = static_cast<double>(norm2(t));
  }
}

template class KrylovWork<float>;
template class KrylovWork<double>;
template class KrylovWork<c32>;
template class KrylovWork<c64>;

template void cg_solve<float>(Op&, Op*, const float*, float*, const Crit&, Numerics, KrylovWork<float>&,
                              SolveReport&, cudaStream_t, EventTimer*, float*, float**, CgSpec*);
template void cg_solve<double>(Op&, Op*, const double*, double*, const Crit&, Numerics, KrylovWork<double>&,
                               SolveReport&, cudaStream_t, EventTimer*, double*, double**, CgSpec*);
#define INST_GMRES(T)                                                                                      \
  template void gmres_solve<T>(Op&, Op*, const T*, T*, const Crit&, Numerics, KrylovWork<T>&, SolveReport&, \
                               cudaStream_t, EventTimer*, int);
INST_GMRES(float)
INST_GMRES(double)
INST_GMRES(c32)
INST_GMRES(c64)

}  // namespace mprkb
