// lobra_dispatch: LobRA's per-step workload-balanced dispatch, host only.
//
// PAPER.md §4.3: given the deployed heterogeneous FT replicas p*_i, each
// step buckets the batch by length with a DP over the grid and solves
// Eq. 3
//     min_d max_i T({ceil(d_ij / p_i)}_j ; S_i)
//     s.t. sum_i d_ij = B_j,  d_ij <= B_j p_i
// with the App. D cost T_i = sum_j c_ij * ceil(d_ij / p_i) for PP = 1,
// c_ij = the caller's integer cost of one sequence padded to s_j on group i (linear in
// the per-replica count; reading Q15).
//
// The Eq. 3 ILP is solved EXACTLY and canonically (lexicographically smallest optimal d
// in (group, bucket) order, reading Q12):
//  * 1 deployed group: trivial.
//  * 2 groups: a pseudo-polynomial DP over the first group's cost budget:
//        Suf_j(b) = min cost of group 2 over buckets j..R-1 with group-1 cost <= b
//    then t* = min_b max(b, Suf_0(b)) and the lexicographic reconstruction picks, bucket
//    by bucket, the smallest d_1j whose completion still meets t*.
//  * >2 groups: depth-first search over the leading groups' d (lexicographic order,
//    ascending values) with the 2-group DP as the exact leaf solver; node-capped.
// This is an independent implementation of what oracle/dispatch.py computes by brute
// force / MILP; tests check the two agree bit for bit.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <vector>

#include "common.h"
#include "eq3_bb.h"

namespace {

using i64 = int64_t;
const i64 BIG = INT64_MAX / 4;

inline i64 cdiv(i64 a, i64 b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ bucketing
// Returns boundaries (grid values) minimising cross-interval padding with <= R buckets,
// the lexicographically smallest optimal list.  occ_u / occ_c: occupied grid values and
// their counts, ascending.
std::vector<i64> bucketize(const std::vector<i64>& u, const std::vector<i64>& cnt, int R) {
  const int V = (int)u.size();
  // prefix sums for O(1) segment cost: cost(a..b) = u_b * C(a..b) - S(a..b)
  std::vector<i64> C(V + 1, 0), S(V + 1, 0);
  for (int v = 0; v < V; ++v) {
    C[v + 1] = C[v] + cnt[v];
    S[v + 1] = S[v] + cnt[v] * u[v];
  }
  auto seg = [&](int a, int b) {  // intervals a..b (0-based, inclusive) padded to u[b]
    return u[b] * (C[b + 1] - C[a]) - (S[b + 1] - S[a]);
  };
  // F[k][j]: min padding of intervals k..V-1 with <= j buckets (F[V][*] = 0)
  std::vector<std::vector<i64>> F(V + 1, std::vector<i64>(R + 1, BIG));
  for (int j = 0; j <= R; ++j) F[V][j] = 0;
  for (int k = V - 1; k >= 0; --k)
    for (int j = 1; j <= R; ++j) {
      i64 best = BIG;
      for (int e = k; e < V; ++e) {
        if (F[e + 1][j - 1] >= BIG) continue;
        best = std::min(best, seg(k, e) + F[e + 1][j - 1]);
      }
      F[k][j] = best;
    }
  std::vector<i64> out;
  int k = 0, j = R;
  while (k < V) {
    for (int e = k; e < V; ++e) {
      if (F[e + 1][j - 1] < BIG && seg(k, e) + F[e + 1][j - 1] == F[k][j]) {
        out.push_back(u[e]);
        k = e + 1;
        --j;
        break;
      }
    }
  }
  return out;
}

// ------------------------------------------------------------------ Eq. 3 solver
struct Inst {
  int G = 0, R = 0;
  std::vector<i64> Bj;               // demand per bucket
  std::vector<i64> p;                // replicas per group
  std::vector<int> r;                // supported bucket count per group
  std::vector<std::vector<i64>> c;   // cost per (group, bucket)
  bool sup(int i, int j) const { return j < r[i]; }
  i64 cost(int i, int j, i64 d) const { return d ? c[i][j] * cdiv(d, p[i]) : 0; }
};

struct Budget {
  i64 cap, used = 0;
  bool hit = false;
  bool take(i64 n) {
    used += n;
    if (used > cap) hit = true;
    return !hit;
  }
};

// Two-group exact solver on residual demands D_j with fixed extra loads La, Lb.
// Groups a, b of `in`.  Builds Suf tables over budgets 0..UB for group a's cost.
struct Two {
  const Inst& I;
  int a, b;
  std::vector<i64> D;
  i64 La, Lb, UB;
  std::vector<std::vector<i64>> Suf;   // [R+1][UB+1]
  bool ok = false;

  Two(const Inst& in, int ga, int gb, std::vector<i64> dem, i64 la, i64 lb, i64 ub, Budget& bud)
      : I(in), a(ga), b(gb), D(std::move(dem)), La(la), Lb(lb), UB(ub) {
    if (UB < 0) return;
    Suf.assign(I.R + 1, std::vector<i64>(UB + 1, 0));
    ok = layers(I.R, bud);
  }
  // (Re)compute Suf[j] for j = top-1 .. 0 (Suf[top..R] unchanged).
  bool layers(int top, Budget& bud) {
    i64 cells = 0;
    for (int j = 0; j < top; ++j) cells += (UB + 1) * (cdiv(D[j], I.p[a]) + 2);
    if (!bud.take(cells)) return false;
    for (int j = top - 1; j >= 0; --j) {
      std::vector<i64>& cur = Suf[j];
      const std::vector<i64>& nxt = Suf[j + 1];
      std::fill(cur.begin(), cur.end(), BIG);
      const i64 Dj = D[j];
      if (Dj == 0) {
        cur = nxt;
        continue;
      }
      const bool sa = I.sup(a, j), sb = I.sup(b, j);
      const i64 qmax = sa ? cdiv(Dj, I.p[a]) : 0;
      for (i64 q = 0; q <= qmax; ++q) {
        const i64 da = std::min(Dj, q * I.p[a]);
        const i64 rest = Dj - da;
        if (rest > 0 && !sb) continue;
        const i64 ca = I.c[a][j] * q;
        if (ca > UB) break;
        const i64 cb = rest ? I.c[b][j] * cdiv(rest, I.p[b]) : 0;
        for (i64 bb = ca; bb <= UB; ++bb) {
          const i64 v = nxt[bb - ca];
          if (v >= BIG) continue;
          if (v + cb < cur[bb]) cur[bb] = v + cb;
        }
      }
    }
    return true;
  }
  // New residual demands (same groups, UB, loads): recompute only the layers at and below
  // the last bucket whose demand changed.
  bool update(const std::vector<i64>& dem, Budget& bud) {
    int top = 0;
    for (int j = 0; j < I.R; ++j)
      if (dem[j] != D[j]) top = j + 1;
    D = dem;
    ok = layers(top, bud);
    return ok;
  }
  // min over budgets of max(La + b, Lb + Suf_0(b))
  i64 best() const {
    i64 t = BIG;
    for (i64 bb = 0; bb <= UB; ++bb) {
      if (Suf[0][bb] >= BIG) continue;
      t = std::min(t, std::max(La + bb, Lb + Suf[0][bb]));
    }
    return t;
  }
  // Lexicographically smallest d_a (then d_b = D - d_a) with max <= t; false if none.
  bool lexmin(i64 t, std::vector<i64>& da_out) const {
    const int R = I.R;
    i64 budget = std::min(UB, t - La);
    if (budget < 0) return false;
    i64 usedb = Lb;
    da_out.assign(R, 0);
    if (Suf[0][budget] >= BIG || usedb + Suf[0][budget] > t) return false;
    for (int j = 0; j < R; ++j) {
      const i64 Dj = D[j];
      bool found = (Dj == 0);
      for (i64 d = 0; d <= Dj && !found; ++d) {
        if (d > 0 && !I.sup(a, j)) break;
        if (Dj - d > 0 && !I.sup(b, j)) continue;
        const i64 ca = I.cost(a, j, d);
        if (ca > budget) break;
        const i64 cb = I.cost(b, j, Dj - d);
        const i64 rest = Suf[j + 1][budget - ca];
        if (rest < BIG && usedb + cb + rest <= t) {
          da_out[j] = d;
          budget -= ca;
          usedb += cb;
          found = true;
        }
      }
      if (!found) return false;
    }
    return true;
  }
};

i64 objective(const Inst& I, const std::vector<std::vector<i64>>& d) {
  i64 t = 0;
  for (int i = 0; i < I.G; ++i) {
    i64 s = 0;
    for (int j = 0; j < I.R; ++j) s += I.cost(i, j, d[i][j]);
    t = std::max(t, s);
  }
  return t;
}

// By-length dispatch (Fig. 4(c)); always feasible when every bucket is supported.
std::vector<std::vector<i64>> by_length(const Inst& I, const std::vector<i64>& tp) {
  std::vector<std::vector<i64>> d(I.G, std::vector<i64>(I.R, 0));
  for (int j = 0; j < I.R; ++j) {
    int bi = -1;
    i64 bv = BIG;
    for (int i = 0; i < I.G; ++i)
      if (I.sup(i, j) && I.c[i][j] * tp[i] < bv) bv = I.c[i][j] * tp[i], bi = i;
    if (bi >= 0) d[bi][j] = I.Bj[j];
  }
  return d;
}

// Eq. 3 with G >= 3 deployed groups (reading Q12: the lexicographically smallest optimal
// d in (group, bucket) order).
//  1. t* = the smallest t for which the covering program of eq3_bb.cpp (q_ij rounds, loads
//     <= t) is feasible, scanning up from the LP / Lagrangian lower bound;
//  2. groups 0..G-3, bucket by bucket: the smallest d_ij that still admits a completion with
//     max load <= t*.  "d_ij <= u feasible" is monotone in u, so each variable costs one
//     proof that d_ij <= (incumbent value - 1) is infeasible, plus one search per improved
//     incumbent.  d_ij <= u splits into q_ij <= floor(u / p_i) and (when p_i does not
//     divide u) q_ij = ceil(u / p_i) covering exactly u;
//  3. the last two groups: the exact 2-group DP's lexicographic reconstruction.
// Every decision is exact (lobra::eq3::feasible either returns an integer certificate or proves
// infeasibility); only an exhausted node budget leaves a decision open (LOBRA_ERR_BUDGET).
struct MultiLex {
  const Inst& I;
  lobra::eq3::Stats& st;
  bool budget_hit = false;
  MultiLex(const Inst& in, lobra::eq3::Stats& s) : I(in), st(s) {}

  lobra::eq3::Cover cover(const std::vector<i64>& tau, const std::vector<i64>& D,
                   const std::vector<std::vector<char>>& fixed) const {
    lobra::eq3::Cover cv;
    cv.G = I.G;
    cv.R = I.R;
    cv.p = I.p;
    cv.c = I.c;
    cv.tau = tau;
    cv.D = D;
    cv.qhi.assign(I.G, std::vector<i64>(I.R, 0));
    for (int i = 0; i < I.G; ++i)
      for (int j = 0; j < I.R; ++j)
        if (I.sup(i, j) && !fixed[i][j] && D[j] > 0) cv.qhi[i][j] = cdiv(D[j], I.p[i]);
    return cv;
  }
  // d from a covering certificate q of the residual (D, fixed): in every bucket the later
  // groups take as much as their rounds allow, the earlier ones the rest (smallest
  // incumbent values for the lexicographic scan).
  void to_d(const lobra::eq3::Cover& cv, const std::vector<std::vector<i64>>& q,
            std::vector<std::vector<i64>>& d) const {
    for (int j = 0; j < I.R; ++j) {
      i64 rem = cv.D[j];
      for (int i = 0; i < I.G; ++i) {
        if (cv.qhi[i][j] <= 0) {
          if (!fixed_[i][j]) d[i][j] = 0;   // not fixed, no rounds allowed: takes nothing
          continue;
        }
        i64 later = 0;
        for (int k = i + 1; k < I.G; ++k)
          if (cv.qhi[k][j] > 0) later += I.p[k] * q[k][j];
        const i64 v = std::max<i64>(0, rem - later);
        d[i][j] = v;
        rem -= v;
      }
    }
  }
  std::vector<std::vector<char>> fixed_;   // variables of the lexicographic prefix
  int feas(const lobra::eq3::Cover& cv, std::vector<std::vector<i64>>& q) {
#ifdef EQ3_TRACE
    const i64 n0 = st.nodes;
#endif
    const int r = lobra::eq3::feasible(cv, q, st);
#ifdef EQ3_TRACE
    i64 sd = 0;
    for (auto v : cv.D) sd += v;
    fprintf(stderr, "feas r=%d nodes=%lld sumD=%lld tau0=%lld\n", r, (long long)(st.nodes - n0), (long long)sd, (long long)cv.tau[0]);
#endif
    if (r < 0) budget_hit = true;
    return r;
  }

  // t_only: stop after step 1 (dl = a certificate attaining t*, not the canonical d)
  bool run(std::vector<std::vector<i64>>& dl, i64 UB, bool t_only = false) {
    const int G = I.G, R = I.R;
    fixed_.assign(G, std::vector<char>(R, 0));
    std::vector<std::vector<char>>& fixed = fixed_;
    std::vector<i64> tau(G, 0), D = I.Bj;
    // 1. t*
    i64 t;
    {
      lobra::eq3::Cover cv = cover(tau, D, fixed);
      const double lb = lobra::eq3::lower_bound(cv, st);
      t = (i64)std::ceil(lb - 1e-6);
      if (!(lb > -1e300)) t = 0;
    }
    std::vector<std::vector<i64>> q, inc(G, std::vector<i64>(R, 0));
    for (;; ++t) {
      if (t >= UB) {   // the length-based dispatch attains UB
        t = UB;
        inc = dl;
        break;
      }
      std::fill(tau.begin(), tau.end(), t);
      lobra::eq3::Cover cv = cover(tau, D, fixed);
      const int r = feas(cv, q);
      if (r < 0) return false;
      if (r == 1) {
        to_d(cv, q, inc);
        break;
      }
    }
    std::fill(tau.begin(), tau.end(), t);
    if (t_only) {
      dl = inc;
      return true;
    }
    // 2. groups 0..G-3
    std::vector<std::vector<i64>> d(G, std::vector<i64>(R, 0));
    for (int i = 0; i + 2 < G; ++i)
      for (int j = 0; j < R; ++j) {
        if (!I.sup(i, j) || D[j] == 0) {
          fixed[i][j] = 1;
          continue;
        }
        while (inc[i][j] > 0) {
          const i64 u = inc[i][j] - 1;
          bool improved = false;
          // (A) q_ij <= floor(u / p_i)
          {
            lobra::eq3::Cover cv = cover(tau, D, fixed);
            cv.qhi[i][j] = std::min(cv.qhi[i][j], u / I.p[i]);
            const int r = feas(cv, q);
            if (r < 0) return false;
            if (r == 1) {
              std::vector<std::vector<i64>> nd = inc;
              to_d(cv, q, nd);
              for (int jj = j; jj < R; ++jj) inc[i][jj] = nd[i][jj];
              for (int ii = i + 1; ii < G; ++ii) inc[ii] = nd[ii];
              improved = true;
            }
          }
          // (B) q_ij = ceil(u / p_i) covering exactly u
          if (!improved && u % I.p[i] != 0) {
            std::vector<i64> tau2 = tau, D2 = D;
            tau2[i] -= I.c[i][j] * cdiv(u, I.p[i]);
            D2[j] -= u;
            std::vector<std::vector<char>> fx = fixed;
            fx[i][j] = 1;
            lobra::eq3::Cover cv = cover(tau2, D2, fx);
            const int r = feas(cv, q);
            if (r < 0) return false;
            if (r == 1) {
              std::vector<std::vector<i64>> nd = inc;
              to_d(cv, q, nd);
              nd[i][j] = u;
              for (int jj = j; jj < R; ++jj) inc[i][jj] = nd[i][jj];
              for (int ii = i + 1; ii < G; ++ii) inc[ii] = nd[ii];
              improved = true;
            }
          }
          if (!improved) break;
          if (inc[i][j] > u) {   // a certificate of d_ij <= u must lower the incumbent
            lobra::set_error("internal: Eq. 3 incumbent did not improve");
            return false;
          }
        }
        const i64 v = inc[i][j];
        d[i][j] = v;
        tau[i] -= I.cost(i, j, v);
        D[j] -= v;
        fixed[i][j] = 1;
      }
    // 3. the last two groups
    Budget bud{(i64)4000000000LL};
    Two two(I, G - 2, G - 1, D, 0, 0, t, bud);
    std::vector<i64> da;
    if (!two.ok || !two.lexmin(t, da)) {
      // cannot happen: the incumbent restricted to the last two groups is a witness
      lobra::set_error("internal: Eq. 3 lexicographic completion failed");
      return false;
    }
    for (int j = 0; j < R; ++j) {
      d[G - 2][j] = da[j];
      d[G - 1][j] = D[j] - da[j];
    }
    dl = d;
    return true;
  }
};

// Exact Eq. 3 over the deployed groups of L: the lexicographically smallest optimal d
// (reading Q12).  false = solver budget exhausted (dl then holds the length-based d).
bool eq3_exact(const Inst& L, const std::vector<i64>& tp, Budget& bud, i64 node_cap, i64& nodes,
               std::vector<std::vector<i64>>& dl, bool t_only = false) {
  dl = by_length(L, tp);
  if (L.G == 1) {
    dl[0] = L.Bj;
    return true;
  }
  const i64 UB = objective(L, dl);
  if (L.G == 2) {
    Two two(L, 0, 1, L.Bj, 0, 0, UB, bud);
    std::vector<i64> da;
    if (two.ok) {
      const i64 t = two.best();
      if (two.lexmin(t, da))
        for (int j = 0; j < L.R; ++j) dl[0][j] = da[j], dl[1][j] = L.Bj[j] - da[j];
    }
    nodes = bud.used;
    return !bud.hit;
  }
  lobra::eq3::Stats st;
  st.cap = node_cap > 0 ? node_cap : (i64)1000000;
  // the branch-and-bound subtrees run on a pool (exact either way; only the certificates
  // met on the way may differ, never the canonical d)
  lobra::eq3::Pool pool(lobra::eq3::default_threads());
  st.pool = &pool;
  MultiLex ml(L, st);
  std::vector<std::vector<i64>> d = dl;
  const bool ok = ml.run(d, UB, t_only);
  nodes = st.nodes;
  if (ok) dl = d;
  else dl = by_length(L, tp);
  return ok;
}

}  // namespace

extern "C" lobra_status lobra_dispatch(const lobra_deployment* dep, const lobra_batch* batch,
                                       int32_t grid_step, int32_t grid_max, int32_t R,
                                       int32_t mode, int32_t chunking, int64_t node_cap,
                                       lobra_dispatch_out* out) {
  using lobra::fail;
  lobra::clear_error();
  if (!dep || !batch || !out) return fail(LOBRA_ERR_INPUT, "null argument");
  if (grid_step < 1 || grid_max < grid_step || grid_max % grid_step)
    return fail(LOBRA_ERR_INPUT, "grid_max must be a positive multiple of grid_step");
  if (R < 1) return fail(LOBRA_ERR_INPUT, "R must be >= 1");
  if (mode < 0 || mode > 2) return fail(LOBRA_ERR_INPUT, "unknown mode %d", mode);
  if (chunking != 0 && chunking != 1) return fail(LOBRA_ERR_INPUT, "unknown chunking %d", chunking);
  const int G = dep->num_groups;
  const int n = batch->num_seqs;
  if (G < 1 || !dep->tp || !dep->replicas || !dep->max_tokens || !dep->cost)
    return fail(LOBRA_ERR_INPUT, "deployment arrays missing");
  if (n < 1 || !batch->seq_lens || !batch->seq_task) return fail(LOBRA_ERR_INPUT, "empty batch");
  if (!out->boundaries || !out->d || !out->seq_bucket || !out->seq_replica || !out->seq_chunk ||
      !out->pack_order || !out->replica_cost)
    return fail(LOBRA_ERR_INPUT, "output arrays missing");
  const int U = grid_max / grid_step;
  std::vector<i64> tp(G), p(G), M(G);
  i64 total_rep = 0;
  for (int i = 0; i < G; ++i) {
    tp[i] = dep->tp[i];
    p[i] = dep->replicas[i];
    M[i] = dep->max_tokens[i];
    if (tp[i] < 1 || p[i] < 0 || M[i] < grid_step || M[i] % grid_step)
      return fail(LOBRA_ERR_INPUT, "group %d: tp>=1, replicas>=0, max_tokens multiple of grid_step", i);
    if (i && (tp[i - 1] > tp[i] || (tp[i - 1] == tp[i] && M[i - 1] > M[i])))
      return fail(LOBRA_ERR_INPUT, "groups must be ordered by (tp, max_tokens)");
    for (int k = 0; k < U; ++k)
      if (dep->cost[(size_t)i * U + k] < 0) return fail(LOBRA_ERR_INPUT, "negative cost");
    total_rep += p[i];
  }
  if (total_rep < 1) return fail(LOBRA_ERR_INPUT, "no replica deployed");
  // 1. histogram on the grid u_k = k * grid_step
  std::vector<i64> hist(U, 0);
  std::vector<int> seq_k(n);
  for (int s = 0; s < n; ++s) {
    const i64 l = batch->seq_lens[s];
    if (l < 1) return fail(LOBRA_ERR_INPUT, "sequence %d has length %lld < 1", s, (long long)l);
    if (l > grid_max)
      return fail(LOBRA_ERR_INFEASIBLE, "sequence %d (length %lld) exceeds the grid maximum %d", s,
                  (long long)l, grid_max);
    seq_k[s] = (int)cdiv(l, grid_step);   // 1-based interval
    hist[seq_k[s] - 1]++;
  }
  // 2-3. compress empty intervals; DP boundaries
  std::vector<i64> ou, oc;
  for (int k = 0; k < U; ++k)
    if (hist[k]) ou.push_back((i64)(k + 1) * grid_step), oc.push_back(hist[k]);
  const std::vector<i64> bnd = bucketize(ou, oc, R);
  const int Rb = (int)bnd.size();
  std::vector<int> seq_b(n);
  std::vector<i64> Bj(Rb, 0);
  for (int s = 0; s < n; ++s) {
    const i64 u = (i64)seq_k[s] * grid_step;
    const int j = (int)(std::lower_bound(bnd.begin(), bnd.end(), u) - bnd.begin());
    seq_b[s] = j;
    Bj[j]++;
  }
  // 4. r_i and costs
  Inst I;
  I.G = G;
  I.R = Rb;
  I.Bj = Bj;
  I.p = p;
  I.r.assign(G, 0);
  I.c.assign(G, std::vector<i64>(Rb, 0));
  for (int i = 0; i < G; ++i) {
    if (p[i] > 0)
      for (int j = 0; j < Rb; ++j) I.r[i] += bnd[j] <= M[i];
    for (int j = 0; j < Rb; ++j) I.c[i][j] = dep->cost[(size_t)i * U + (bnd[j] / grid_step - 1)];
  }
  for (int j = 0; j < Rb; ++j) {
    bool s = false;
    for (int i = 0; i < G; ++i) s |= I.sup(i, j);
    if (!s)
      return fail(LOBRA_ERR_INFEASIBLE, "bucket %lld fits no deployed replica: re-plan required",
                  (long long)bnd[j]);
  }
  // 5-6. Eq. 3 on the deployed groups only
  std::vector<int> live;
  for (int i = 0; i < G; ++i)
    if (p[i] > 0) live.push_back(i);
  Inst L;
  L.G = (int)live.size();
  L.R = Rb;
  L.Bj = Bj;
  std::vector<i64> ltp;
  for (int i : live) L.p.push_back(p[i]), L.r.push_back(I.r[i]), L.c.push_back(I.c[i]), ltp.push_back(tp[i]);
  Budget bud{(i64)4000000000LL};   // 2-group DP cells
  i64 nodes = 0;
  std::vector<std::vector<i64>> dl = by_length(L, ltp);
  lobra_status st = LOBRA_OK;
  if (mode == 2 && L.G != 1)
    return fail(LOBRA_ERR_INPUT, "uniform dispatch (mode 2) needs exactly one deployed group");
  if (mode == 2) {
    for (int j = 0; j < Rb; ++j) dl[0][j] = Bj[j];
  }
  if (mode == 0 && !eq3_exact(L, ltp, bud, node_cap, nodes, dl)) st = LOBRA_ERR_BUDGET;
  // write d (all groups; undeployed rows are 0)
  std::vector<std::vector<i64>> d(G, std::vector<i64>(Rb, 0));
  for (size_t k = 0; k < live.size(); ++k) d[live[k]] = dl[k];
  i64 t_hat = 0;
  for (int i = 0; i < G; ++i) {
    if (!p[i]) continue;
    i64 s = 0;
    for (int j = 0; j < Rb; ++j) s += I.cost(i, j, d[i][j]);
    t_hat = std::max(t_hat, s);
  }
  // 7. sequences of bucket j in ascending index -> groups in order
  std::vector<int> seq_g(n, -1);
  {
    std::vector<std::vector<int>> idx(Rb);
    for (int s = 0; s < n; ++s) idx[seq_b[s]].push_back(s);
    for (int j = 0; j < Rb; ++j) {
      size_t pos = 0;
      for (int i = 0; i < G; ++i)
        for (i64 q = 0; q < d[i][j]; ++q) seq_g[idx[j][pos++]] = i;
    }
  }
  // 8. per-bucket round robin within a group, starting at the smallest running cost
  std::vector<i64> rbase(G + 1, 0);
  for (int i = 0; i < G; ++i) rbase[i + 1] = rbase[i] + p[i];
  std::vector<i64> running(total_rep, 0);
  std::vector<int> seq_rep(n, -1);
  for (int i = 0; i < G && mode == 2; ++i) {   // uniform: k-th sequence -> replica k mod p
    if (!p[i]) continue;
    int k = 0;
    for (int s = 0; s < n; ++s) {
      const int rep = (int)(rbase[i] + (k++) % p[i]);
      seq_rep[s] = rep;
      running[rep] += I.c[i][seq_b[s]];
    }
  }
  for (int i = 0; i < G && mode != 2; ++i) {
    if (!p[i]) continue;
    for (int j = 0; j < Rb; ++j) {
      int start = 0;
      for (int q = 1; q < p[i]; ++q)
        if (running[rbase[i] + q] < running[rbase[i] + start]) start = q;
      int m = 0;
      for (int s = 0; s < n; ++s) {
        if (seq_b[s] != j || seq_g[s] != i) continue;
        const int rep = (int)(rbase[i] + (start + m) % p[i]);
        seq_rep[s] = rep;
        running[rep] += I.c[i][j];
        ++m;
      }
    }
  }
  // 9-10. chunks b_j = floor(M_i / s_j), descending cost; (task, index) inside a chunk
  std::vector<int> seq_chunk(n, -1), pack(n, -1);
  for (int i = 0; i < G; ++i) {
    for (i64 rep = rbase[i]; rep < rbase[i + 1]; ++rep) {
      struct Ch {
        i64 cost;
        int j, ci;
        std::vector<int> seqs;
      };
      std::vector<Ch> chunks;
      if (chunking == 0) {
        for (int j = 0; j < Rb; ++j) {
          std::vector<int> mine;
          for (int s = 0; s < n; ++s)
            if (seq_rep[s] == rep && seq_b[s] == j) mine.push_back(s);
          if (mine.empty()) continue;
          const i64 b = M[i] / bnd[j];
          int ci = 0;
          for (size_t s0 = 0; s0 < mine.size(); s0 += (size_t)b, ++ci) {
            Ch ch;
            ch.j = j;
            ch.ci = ci;
            const size_t e = std::min(mine.size(), s0 + (size_t)b);
            ch.seqs.assign(mine.begin() + s0, mine.begin() + e);
            ch.cost = (i64)ch.seqs.size() * I.c[i][j];
            chunks.push_back(std::move(ch));
          }
        }
      } else {
        // packed: (bucket desc, index asc), next-fit by real tokens <= M_i
        i64 fill = 0;
        int ci = 0;
        for (int j = Rb - 1; j >= 0; --j)
          for (int s = 0; s < n; ++s) {
            if (seq_rep[s] != rep || seq_b[s] != j) continue;
            const i64 L = batch->seq_lens[s];
            if (chunks.empty() || fill + L > M[i]) {
              Ch ch;
              ch.j = 0;
              ch.ci = ci++;
              ch.cost = 0;
              chunks.push_back(std::move(ch));
              fill = 0;
            }
            chunks.back().seqs.push_back(s);
            fill += L;
          }
        // creation order is the execution order: make the sort below a no-op
        for (auto& ch : chunks) ch.cost = 0;
      }
      std::stable_sort(chunks.begin(), chunks.end(), [](const Ch& x, const Ch& y) {
        if (x.cost != y.cost) return x.cost > y.cost;
        if (x.j != y.j) return x.j < y.j;
        return x.ci < y.ci;
      });
      for (size_t k = 0; k < chunks.size(); ++k) {
        std::vector<int> o = chunks[k].seqs;
        std::stable_sort(o.begin(), o.end(), [&](int x, int y) {
          if (batch->seq_task[x] != batch->seq_task[y]) return batch->seq_task[x] < batch->seq_task[y];
          return x < y;
        });
        for (size_t q = 0; q < o.size(); ++q) seq_chunk[o[q]] = (int)k, pack[o[q]] = (int)q;
      }
    }
  }
  out->num_buckets = Rb;
  for (int j = 0; j < Rb; ++j) out->boundaries[j] = (int32_t)bnd[j];
  for (int i = 0; i < G; ++i)
    for (int j = 0; j < R; ++j) out->d[(size_t)i * R + j] = j < Rb ? d[i][j] : 0;
  for (int s = 0; s < n; ++s) {
    out->seq_bucket[s] = seq_b[s];
    out->seq_replica[s] = seq_rep[s];
    out->seq_chunk[s] = seq_chunk[s];
    out->pack_order[s] = pack[s];
  }
  for (i64 q = 0; q < total_rep; ++q) out->replica_cost[q] = running[q];
  out->t_hat = t_hat;
  out->nodes = nodes;
  if (st == LOBRA_ERR_BUDGET) lobra::set_error("Eq. 3 solver node cap hit; incumbent returned");
  return st;
}

// ------------------------------------------------------------------ stage-1 planner
extern "C" lobra_status lobra_plan_deployment(const lobra_candidates* cand, int32_t n_gpus,
                                              const int32_t* lens, int32_t n_lens,
                                              int32_t batch_size, int32_t grid_step,
                                              int32_t grid_max, int32_t R, double threshold,
                                              int64_t node_cap, lobra_plan_out* out) {
  using lobra::fail;
  lobra::clear_error();
  if (!cand || !lens || !out || !out->replicas || !out->boundaries || !out->demands)
    return fail(LOBRA_ERR_INPUT, "null argument");
  const int S = cand->num_configs;
  if (S < 1 || !cand->tp || !cand->max_tokens || !cand->cost)
    return fail(LOBRA_ERR_INPUT, "candidate arrays missing");
  if (n_gpus < 1 || n_lens < 1 || batch_size < 0 || R < 1)
    return fail(LOBRA_ERR_INPUT, "need n_gpus >= 1, n_lens >= 1, batch_size >= 0, R >= 1");
  if (grid_step < 1 || grid_max < grid_step || grid_max % grid_step)
    return fail(LOBRA_ERR_INPUT, "grid_max must be a positive multiple of grid_step");
  const int U = grid_max / grid_step;
  for (int i = 0; i < S; ++i)
    if (cand->tp[i] < 1 || cand->max_tokens[i] < grid_step || cand->max_tokens[i] % grid_step)
      return fail(LOBRA_ERR_INPUT, "candidate %d: tp >= 1, max_tokens multiple of grid_step", i);
  // 1. histogram + dynamic bucketing of the sample
  std::vector<i64> hist(U, 0);
  for (int k = 0; k < n_lens; ++k) {
    const i64 l = lens[k];
    if (l < 1) return fail(LOBRA_ERR_INPUT, "sample length %lld < 1", (long long)l);
    if (l > grid_max) return fail(LOBRA_ERR_INFEASIBLE, "sample length %lld exceeds the grid", (long long)l);
    hist[cdiv(l, grid_step) - 1]++;
  }
  std::vector<i64> ou, oc;
  for (int k = 0; k < U; ++k)
    if (hist[k]) ou.push_back((i64)(k + 1) * grid_step), oc.push_back(hist[k]);
  const std::vector<i64> bnd = bucketize(ou, oc, R);
  const int Rb = (int)bnd.size();
  std::vector<i64> cnt(Rb, 0);
  {
    size_t v = 0;
    for (int j = 0; j < Rb; ++j)
      while (v < ou.size() && ou[v] <= bnd[j]) cnt[j] += oc[v++];
  }
  // 2. demands
  std::vector<i64> Bj(Rb);
  for (int j = 0; j < Rb; ++j)
    Bj[j] = batch_size > 0 ? ((i64)batch_size * cnt[j] + n_lens - 1) / n_lens : cnt[j];
  // per-config support and costs
  std::vector<int> r(S, 0);
  std::vector<std::vector<i64>> c(S, std::vector<i64>(Rb));
  for (int i = 0; i < S; ++i)
    for (int j = 0; j < Rb; ++j) {
      r[i] += bnd[j] <= cand->max_tokens[i];
      c[i][j] = cand->cost[(size_t)i * U + (bnd[j] / grid_step - 1)];
    }
  // 3. configuration proposal: drop dominated candidates with the same GPU count
  std::vector<char> keep(S, 1);
  for (int a = 0; a < S; ++a)
    for (int b = 0; b < S && keep[a]; ++b) {
      if (a == b || !keep[b] || cand->tp[a] != cand->tp[b] || r[b] < r[a]) continue;
      bool dom = true;
      for (int j = 0; j < r[a]; ++j) dom &= c[b][j] <= c[a][j];
      if (!dom) continue;
      bool strict = r[b] > r[a];
      for (int j = 0; j < r[a]; ++j) strict |= c[b][j] < c[a][j];
      if (strict || b < a) keep[a] = 0;
    }
  int last = -1;
  for (int j = 0; j < Rb; ++j)
    if (Bj[j] > 0) last = j;
  int min_n = INT32_MAX;
  for (int i = 0; i < S; ++i)
    if (keep[i]) min_n = std::min(min_n, (int)cand->tp[i]);
  // 4. maximal covering plans
  std::vector<std::vector<int>> plans;
  std::vector<int> p(S, 0);
  std::function<void(int, int)> rec = [&](int i, int left) {
    if (i == S) {
      if (left >= min_n) return;                       // not maximal
      int cover = 0;
      for (int k = 0; k < S; ++k)
        if (p[k]) cover = std::max(cover, r[k]);
      if (cover - 1 < last) return;                    // longest demanded bucket uncovered
      plans.push_back(p);
      return;
    }
    if (!keep[i]) {
      p[i] = 0;
      rec(i + 1, left);
      return;
    }
    for (int q = left / cand->tp[i]; q >= 0; --q) {
      p[i] = q;
      rec(i + 1, left - q * cand->tp[i]);
    }
    p[i] = 0;
  };
  rec(0, n_gpus);
  if (plans.empty()) return fail(LOBRA_ERR_INFEASIBLE, "no deployment plan covers the longest bucket");
  // 5. Theorem-1 lower bounds via length-based dispatch
  struct Cand {
    double lb;
    int idx;
  };
  std::vector<Cand> lbs;
  auto make_inst = [&](const std::vector<int>& pl, std::vector<i64>& tp_l) {
    Inst L;
    L.R = Rb;
    L.Bj = Bj;
    for (int i = 0; i < S; ++i)
      if (pl[i] > 0) {
        L.p.push_back(pl[i]);
        L.r.push_back(r[i]);
        L.c.push_back(c[i]);
        tp_l.push_back(cand->tp[i]);
      }
    L.G = (int)L.p.size();
    return L;
  };
  for (size_t k = 0; k < plans.size(); ++k) {
    std::vector<i64> tpl;
    Inst L = make_inst(plans[k], tpl);
    const auto d = by_length(L, tpl);
    double num = 0, den = 0;
    for (int g = 0; g < L.G; ++g) {
      i64 t = 0;
      for (int j = 0; j < Rb; ++j) t += L.cost(g, j, d[g][j]);
      num += (double)(L.p[g] * tpl[g]) * (double)t;
      den += (double)(L.p[g] * tpl[g]);
    }
    lbs.push_back({num / den, (int)k});
  }
  double min_lb = lbs[0].lb;
  for (auto& e : lbs) min_lb = std::min(min_lb, e.lb);
  // 6. exact Eq. 3 per kept plan
  bool hit = false;
  int solved = 0;
  i64 best_t = BIG;
  int best = -1;
  auto better = [&](i64 t, int k) {
    if (best < 0 || t != best_t) return best < 0 || t < best_t;
    auto key = [&](const std::vector<int>& pl) {
      i64 g = 0, rp = 0;
      for (int i = 0; i < S; ++i) g += (i64)pl[i] * cand->tp[i], rp += pl[i];
      return std::make_pair(g, rp);
    };
    const auto a = key(plans[k]), b = key(plans[best]);
    if (a != b) return a < b;
    return plans[k] < plans[best];
  };
  // kept plans in ascending Theorem-1 bound (good incumbents first); a plan whose exact Eq. 3
  // lower bound (LP / Lagrangian, eq3_bb.cpp) already exceeds the best t found is skipped:
  // it can be neither the best nor tied with it, so the selection stays exact
  // (plans with <= 2 groups first: their exact solve is a cheap DP)
  auto ngroups = [&](int k) {
    int g = 0;
    for (int i = 0; i < S; ++i) g += plans[k][i] > 0;
    return g;
  };
  std::stable_sort(lbs.begin(), lbs.end(), [&](const Cand& a, const Cand& b) {
    const bool ha = ngroups(a.idx) >= 3, hb = ngroups(b.idx) >= 3;
    return ha != hb ? hb : a.lb < b.lb;
  });
  for (auto& e : lbs) {
    if (threshold >= 0 && e.lb > (1.0 + threshold) * min_lb + 1e-9) continue;
    std::vector<i64> tpl;
    Inst L = make_inst(plans[e.idx], tpl);
    if (best >= 0 && L.G >= 3) {
      lobra::eq3::Cover cv;
      cv.G = L.G;
      cv.R = L.R;
      cv.p = L.p;
      cv.c = L.c;
      cv.tau.assign(L.G, 0);
      cv.D = L.Bj;
      cv.qhi.assign(L.G, std::vector<i64>(L.R, 0));
      for (int g = 0; g < L.G; ++g)
        for (int j = 0; j < L.R; ++j)
          if (L.sup(g, j) && L.Bj[j] > 0) cv.qhi[g][j] = cdiv(L.Bj[j], L.p[g]);
      lobra::eq3::Stats s0;
      s0.cap = INT64_MAX;
      const double lbz = lobra::eq3::lower_bound(cv, s0);
      if (lbz > -1e300 && (i64)std::ceil(lbz - 1e-6) > best_t) {
        ++solved;   // decided exactly: proven worse than the incumbent plan
        continue;
      }
    }
    std::vector<std::vector<i64>> d;
    Budget b1{(i64)4000000000LL};
    i64 nodes = 0;
    if (!eq3_exact(L, tpl, b1, node_cap, nodes, d, /*t_only=*/true)) hit = true;
    ++solved;
    const i64 t = objective(L, d);
    if (better(t, e.idx)) best_t = t, best = e.idx;
  }
  for (int i = 0; i < S; ++i) out->replicas[i] = plans[best][i];
  out->num_buckets = Rb;
  for (int j = 0; j < Rb; ++j) out->boundaries[j] = (int32_t)bnd[j], out->demands[j] = Bj[j];
  out->plans_total = (int)plans.size();
  out->plans_solved = solved;
  int g = 0;
  for (int i = 0; i < S; ++i) g += plans[best][i] * cand->tp[i];
  out->gpus_used = g;
  out->t_hat = best_t;
  if (hit) {
    lobra::set_error("a per-plan Eq. 3 solve hit the node cap; incumbents used");
    return LOBRA_ERR_BUDGET;
  }
  return LOBRA_OK;
}

// Configuration proposal (App. A) -- see include/lobra.h and reading Q26.
extern "C" lobra_status lobra_propose_configs(const lobra_thruput_table* tb, int32_t* winner,
                                              int32_t* keep) {
  using lobra::fail;
  lobra::clear_error();
  if (!tb || !winner || !keep) return fail(LOBRA_ERR_INPUT, "null argument");
  const int C = tb->num_configs, L = tb->num_lens, K = tb->num_gpu_counts;
  if (C < 1 || L < 1 || K < 1 || !tb->tp || !tb->pp || !tb->seq_len || !tb->thruput || !tb->gpu_counts)
    return fail(LOBRA_ERR_INPUT, "empty throughput table");
  for (int c = 0; c < C; ++c)
    if (tb->tp[c] < 1 || tb->pp[c] < 1) return fail(LOBRA_ERR_INPUT, "config %d: tp, pp >= 1", c);
  for (int k = 0; k < K; ++k)
    if (tb->gpu_counts[k] < 1) return fail(LOBRA_ERR_INPUT, "gpu_counts[%d] < 1", k);
  for (int c = 0; c < C; ++c) keep[c] = 0;
  for (int k = 0; k < K; ++k) {
    const int g = tb->gpu_counts[k];
    for (int l = 0; l < L; ++l) {
      int best = -1;
      for (int c = 0; c < C; ++c) {
        const int n = tb->tp[c] * tb->pp[c];
        const double v = tb->thruput[(size_t)c * L + l];
        if (n > g || g % n != 0 || !(v > 0.0)) continue;
        if (best < 0) { best = c; continue; }
        const double vb = tb->thruput[(size_t)best * L + l];
        const int nb = tb->tp[best] * tb->pp[best];
        bool better;
        if (v != vb) better = v > vb;
        else if (n != nb) better = n < nb;
        else if (tb->tp[c] != tb->tp[best]) better = tb->tp[c] < tb->tp[best];
        else better = tb->pp[c] < tb->pp[best];   // equal keys: the lower index stays
        if (better) best = c;
      }
      winner[(size_t)k * L + l] = best;
      if (best >= 0) keep[best] = 1;
    }
  }
  return LOBRA_OK;
}

// ------------------------------------------------------------------ App. D replica time
// T = sum_j (m_j t(b_j, s_j) + t(r_j, s_j)) + (p - 1) max over existing chunks
extern "C" lobra_status lobra_replica_time(int32_t R, const int32_t* d, const int32_t* s, int64_t M,
                                          int32_t pp, double c0, double c1, double c2, double* out) {
  using namespace lobra;
  clear_error();
  if (R < 1 || pp < 1 || M < 1 || !d || !s || !out)
    return fail(LOBRA_ERR_INPUT, "replica_time: need num_buckets >= 1, pp_stages >= 1, max_tokens >= 1");
  auto t = [&](int64_t b, int64_t len) {
    return b <= 0 ? 0.0 : c0 + c1 * (double)b * (double)len + c2 * (double)b * (double)len * (double)len;
  };
  double compute = 0.0, longest = 0.0;
  for (int j = 0; j < R; ++j) {
    if (d[j] < 0 || s[j] < 1 || s[j] > M)
      return fail(LOBRA_ERR_INPUT, "replica_time: bucket %d: d = %d, s = %d (need d >= 0, 1 <= s <= M)", j,
                  d[j], s[j]);
    const int64_t b = M / s[j], m = d[j] / b, r = d[j] % b;
    const double full = m > 0 ? t(b, s[j]) : 0.0, rem = r > 0 ? t(r, s[j]) : 0.0;
    compute += (double)m * full + rem;
    longest = std::max(longest, std::max(full, rem));
  }
  *out = compute + (double)(pp - 1) * longest;
  return LOBRA_OK;
}
