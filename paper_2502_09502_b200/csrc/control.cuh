// FISTA control logic (restart, bound-check cadence, cutoffs, termination),
// executed by a single thread on the device.  Mirrors fista.py:159-212.
#pragma once

#include "engine.cuh"

namespace l0 {

__device__ __forceinline__ bool gap_small(const Params* P, double gap, double obj) {
  if (gap <= P->gap_tol) return true;
  return P->gap_tol_rel > 0.0 && gap <= P->gap_tol_rel * fabs(obj);
}

// Close the solve at iteration st->t (fista.py:208-212).  `d` is the bound at
// the current iterate when one was just evaluated (NaN otherwise).
__device__ __forceinline__ void finalize(State* st, const Params* P, double d) {
  if (!isfinite(st->best_dual) && !isnan(d)) st->best_dual = d;
  st->gap = st->obj - st->best_dual;
  if (st->termination == TERM_ITERATION_LIMIT && gap_small(P, st->gap, st->obj))
    st->termination = TERM_CONVERGED;
  st->dual_pending = 0;
  st->dual_only = 0;
  st->done = 1;
}

// Stop with `term`; if no finite bound exists yet, one final bound pass on the
// current iterate is scheduled first (fista.py:208-209).
__device__ __forceinline__ void request_stop(State* st, const Params* P, int term) {
  st->termination = term;
  if (isfinite(st->best_dual)) {
    finalize(st, P, CUDART_NAN);
  } else {
    st->dual_pending = 1;
    st->check_pending = 0;
    st->dual_only = 1;
  }
}

// After F(X beta_next) is known: composite objective, restart, momentum
// counter, bound-check scheduling, primal cutoff, iteration limit
// (fista.py:166-206).
__device__ __forceinline__ void objective_update(State* st, const Params* P, double loss_total) {
  int64_t t = st->t + 1;
  double obj_next = dadd(loss_total, dmul(P->two_l2, st->g_next));
  if (!isfinite(obj_next)) {
    st->err = ST_NUMERICAL;
    st->err_iter = t;
    st->t = t;
    st->done = 1;
    return;
  }
  bool restarted = P->restart && obj_next >= st->obj;
  if (restarted) {
    st->phi = 1;
    st->restarts += 1;
  } else {
    st->phi += 1;
  }
  st->obj = obj_next;
  st->loss_cur = loss_total;
  st->t = t;
  st->last_restarted = restarted ? 1 : 0;
  bool check = is_check(t, P->bci);
  if (check) {
    st->dual_pending = 1;
    st->check_pending = 1;
  }
  int stop = -1;
  if (!isnan(P->early_primal) && obj_next < P->early_primal) stop = TERM_PRIMAL_BELOW;
  else if (t >= P->max_iter) stop = TERM_ITERATION_LIMIT;
  if (stop >= 0) {
    if (check) {
      st->stop_term = stop;   // applies after the bound check of this iteration
      st->dual_only = 1;
    } else {
      request_stop(st, P, stop);
    }
  }
}

// The bound `d` at iteration st->t has been evaluated (fista.py:182-200).
__device__ __forceinline__ void bound_update(State* st, const Params* P, double d) {
  st->last_dual = d;
  if (!st->check_pending) {  // final pass (fista.py:208-209)
    finalize(st, P, d);
    return;
  }
  st->check_pending = 0;
  st->dual_pending = 0;
  if (d > st->best_dual) st->best_dual = d;   // Python max(best_dual, d)
  st->gap = st->obj - st->best_dual;
  TraceRec& r = st->trace[st->trace_count % kTraceCap];
  r.iteration = (double)st->t;
  r.primal = st->obj;
  r.dual = st->best_dual;
  r.gap = st->gap;
  r.restarted = (double)st->last_restarted;
  st->trace_count += 1;
  if (P->stop_on_gap && gap_small(P, st->gap, st->obj)) {
    st->termination = TERM_CONVERGED;
    finalize(st, P, d);
    return;
  }
  if (!isnan(P->early_dual) && st->best_dual >= P->early_dual) {
    st->termination = TERM_DUAL_ABOVE;
    finalize(st, P, d);
    return;
  }
  if (st->stop_term >= 0) {
    st->termination = st->stop_term;
    finalize(st, P, d);
    return;
  }
}

}  // namespace l0
