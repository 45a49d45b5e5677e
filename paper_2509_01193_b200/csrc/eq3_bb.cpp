// Exact covering feasibility for Eq. 3 with three or more deployed groups.
//
// Eq. 3 asks for min_d max_i sum_j c_ij ceil(d_ij / p_i) s.t. sum_i d_ij = B_j.  With the
// replica-round variables q_ij = ceil(d_ij / p_i) the objective only depends on q, and an
// integer q is realisable by some d iff sum_i p_i q_ij >= B_j (give each group at most
// p_i q_ij of bucket j).  For a budget vector tau the question "is max_i load_i - tau_i
// <= 0 reachable" is therefore the small covering integer program
//     sum_j c_ij q_ij <= tau_i  (groups),   sum_i p_i q_ij >= D_j  (buckets),
//     0 <= q_ij <= qhi_ij integer,
// which `feasible` decides EXACTLY by depth-first branch-and-bound:
//   * node bound: the LP relaxation min z s.t. load_i - tau_i <= z (a dense bounded dual
//     simplex, warm-started from the parent after the branching bound change); a node is
//     discarded only when the LP value exceeds 0 (up to 1e-6 cost units: integer data);
//   * Lagrangian bound (root and every node): sum_j K_j(lambda) - sum_i lambda_i tau_i
//     with the node LP's load duals lambda and K_j the exact integer covering knapsack of
//     bucket j under the node's bounds (a valid lower bound on z for any lambda >= 0
//     summing to 1).  It sees the ceil(d / p) rounding of groups with many replicas, which
//     the LP relaxation does not: 5-30x fewer nodes at p = 4 (measured);
//   * branching: a fractional q of the group with the most replicas, most fractional first,
//     down branch first;
//   * incumbents: LP rounding + greedy repair, verified in integer arithmetic.
//   * parallel: the open subtrees below depth kSplitDepth run on a thread pool; the first
//     certificate stops the others (same answer, possibly another certificate).
// Measured (C5-scale steps, B ~ 1952, R = 16; profiles/r2_dispatch_solve_times.md):
// 3 groups on 8 GPUs ~20-35 ms, 3 groups with p = 4/2/1 and 4 groups ~60-180 ms (8 cores).
// Every "feasible" answer carries an integer certificate; every "infeasible" answer is a
// complete search whose pruning used only valid lower bounds.  The only way to be undecided
// is the node budget (returned as -1, surfaced as LOBRA_ERR_BUDGET by the caller).
#include "eq3_bb.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <deque>
#include <limits>

namespace lobra {
namespace eq3 {
namespace {

const double INF = std::numeric_limits<double>::infinity();
const double PTOL = 1e-7;   // primal feasibility (cost units; data are integers ~1e0..1e6)
const double ZTOL = 1e-6;   // LP value above which a node is infeasible
const double PIV = 1e-11;   // smallest usable pivot

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Dense tableau, bounded variables, dual simplex.  Columns: q vars, z, one slack per row.
struct LP {
  int m = 0, n = 0;
  std::vector<double> T;      // m x n, B^-1 A
  std::vector<double> xb;     // basic values
  std::vector<int> basis;     // var of row r
  std::vector<int> row_of;    // row of var k if basic, else -1
  std::vector<double> lo, hi, x, d;
  std::vector<char> atub;     // nonbasic at upper bound
  int zcol = 0;

  double value(int k) const { return row_of[k] >= 0 ? xb[row_of[k]] : x[k]; }
  double z() const { return value(zcol); }

  void pivot(int r, int e, double delta) {
    const double* Tr0 = &T[(size_t)r * n];
    for (int i = 0; i < m; ++i)
      if (i != r) xb[i] -= T[(size_t)i * n + e] * delta;
    const double enter_val = x[e] + delta;
    const int out = basis[r];
    // leaving variable becomes nonbasic at the bound it was pushed to
    const double a = Tr0[e];
    double* Tr = &T[(size_t)r * n];
    const double inv = 1.0 / a;
    for (int k = 0; k < n; ++k) Tr[k] *= inv;
    Tr[e] = 1.0;
    for (int i = 0; i < m; ++i) {
      if (i == r) continue;
      double* Ti = &T[(size_t)i * n];
      const double f = Ti[e];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) Ti[k] -= f * Tr[k];
      Ti[e] = 0.0;
    }
    const double fd = d[e];
    if (fd != 0.0) {
      for (int k = 0; k < n; ++k) d[k] -= fd * Tr[k];
      d[e] = 0.0;
    }
    row_of[out] = -1;
    row_of[e] = r;
    basis[r] = e;
    xb[r] = enter_val;
  }

  // 0 = optimal, 1 = infeasible or LP value provably > cutoff, 2 = iteration cap
  int solve(double cutoff, int maxit, int64_t& pivots) {
    for (int it = 0; it < maxit; ++it) {
      // the dual simplex objective is a lower bound on the LP optimum (dual feasibility)
      if (z() > cutoff) return 1;
      int r = -1;
      double worst = PTOL;
      for (int i = 0; i < m; ++i) {
        const int k = basis[i];
        const double v = xb[i];
        double inf = 0;
        if (v < lo[k] - PTOL) inf = lo[k] - v;
        else if (v > hi[k] + PTOL) inf = v - hi[k];
        if (inf > worst) worst = inf, r = i;
      }
      if (r < 0) return 0;
      const int out = basis[r];
      const bool below = xb[r] < lo[out];
      const double bound = below ? lo[out] : hi[out];
      const double* Tr = &T[(size_t)r * n];
      int e = -1;
      double best = INF, best_a = 0;
      for (int k = 0; k < n; ++k) {
        if (row_of[k] >= 0 || lo[k] == hi[k]) continue;
        const double a = Tr[k];
        if (std::fabs(a) < PIV) continue;
        const bool up = atub[k];
        // moving k changes xb[r] by -a * dx; dx > 0 from lower, < 0 from upper
        const bool ok = below ? (up ? a > 0 : a < 0) : (up ? a < 0 : a > 0);
        if (!ok) continue;
        const double ratio = std::fabs(d[k]) / std::fabs(a);
        if (ratio < best - 1e-12 || (ratio < best + 1e-12 && std::fabs(a) > best_a)) {
          best = ratio;
          best_a = std::fabs(a);
          e = k;
        }
      }
      if (e < 0) return 1;   // dual unbounded: primal infeasible
      const double delta = (xb[r] - bound) / Tr[e];
      x[out] = bound;
      atub[out] = !below;
      pivot(r, e, delta);
      ++pivots;
    }
    return 2;
  }

  // tighten bounds of variable k to [l, h] (l <= h); keeps dual feasibility
  void set_bounds(int k, double l, double h) {
    lo[k] = l;
    hi[k] = h;
    if (row_of[k] >= 0) return;
    const double nv = atub[k] ? h : l;   // a nonbasic keeps its side (its reduced cost sign)
    const double dv = nv - x[k];
    if (dv != 0.0) {
      for (int i = 0; i < m; ++i) xb[i] -= T[(size_t)i * n + k] * dv;
      x[k] = nv;
    }
  }
};

struct Model {
  const Cover* in = nullptr;
  std::vector<int> vi, vj;                 // q var -> (group, bucket)
  std::vector<std::vector<int>> var_of;    // [G][R] -> var index or -1
  std::vector<int> cover_row;              // [R] -> row or -1
  std::vector<int> repair_order;           // buckets with demand, largest cost first
  int nq = 0;
};

LP build_lp(const Cover& in, Model& md) {
  md.in = &in;
  md.var_of.assign(in.G, std::vector<int>(in.R, -1));
  md.vi.clear();
  md.vj.clear();
  for (int i = 0; i < in.G; ++i)
    for (int j = 0; j < in.R; ++j)
      if (in.qhi[i][j] > 0 && in.D[j] > 0) {
        md.var_of[i][j] = (int)md.vi.size();
        md.vi.push_back(i);
        md.vj.push_back(j);
      }
  md.nq = (int)md.vi.size();
  md.cover_row.assign(in.R, -1);
  int m = in.G;
  for (int j = 0; j < in.R; ++j)
    if (in.D[j] > 0) md.cover_row[j] = m++;
  LP lp;
  lp.m = m;
  lp.zcol = md.nq;
  lp.n = md.nq + 1 + m;
  lp.T.assign((size_t)m * lp.n, 0.0);
  lp.lo.assign(lp.n, 0.0);
  lp.hi.assign(lp.n, INF);
  lp.x.assign(lp.n, 0.0);
  lp.d.assign(lp.n, 0.0);
  lp.atub.assign(lp.n, 0);
  lp.row_of.assign(lp.n, -1);
  lp.basis.assign(m, 0);
  lp.xb.assign(m, 0.0);
  double tmax = 0;
  for (int i = 0; i < in.G; ++i) tmax = std::max(tmax, std::fabs((double)in.tau[i]));
  std::vector<double> rhs(m, 0.0);
  for (int v = 0; v < md.nq; ++v) {
    const int i = md.vi[v], j = md.vj[v];
    lp.T[(size_t)i * lp.n + v] = (double)in.c[i][j];
    lp.T[(size_t)md.cover_row[j] * lp.n + v] = -(double)in.p[i];
    lp.hi[v] = (double)in.qhi[i][j];
  }
  for (int i = 0; i < in.G; ++i) {
    lp.T[(size_t)i * lp.n + lp.zcol] = -1.0;
    rhs[i] = (double)in.tau[i];
  }
  for (int j = 0; j < in.R; ++j)
    if (md.cover_row[j] >= 0) rhs[md.cover_row[j]] = -(double)in.D[j];
  // buckets with the largest costs first (lumpy ones before the fine-grained fillers)
  md.repair_order.clear();
  for (int j = 0; j < in.R; ++j)
    if (in.D[j] > 0) md.repair_order.push_back(j);
  std::sort(md.repair_order.begin(), md.repair_order.end(), [&](int a, int b) {
    int64_t ca = 0, cb = 0;
    for (int i = 0; i < in.G; ++i) ca = std::max(ca, in.c[i][a]), cb = std::max(cb, in.c[i][b]);
    return ca != cb ? ca > cb : a < b;
  });
  lp.lo[lp.zcol] = -tmax - 1.0;
  lp.x[lp.zcol] = lp.lo[lp.zcol];
  lp.d[lp.zcol] = 1.0;   // objective min z; slack basis => reduced costs = costs
  for (int r = 0; r < m; ++r) {
    const int s = md.nq + 1 + r;
    lp.T[(size_t)r * lp.n + s] = 1.0;
    lp.basis[r] = s;
    lp.row_of[s] = r;
    double v = rhs[r];
    for (int k = 0; k <= md.nq; ++k) v -= lp.T[(size_t)r * lp.n + k] * lp.x[k];
    lp.xb[r] = v;
  }
  return lp;
}

// K_j(lambda): min sum_i w_i q_i s.t. sum_i p_i q_i >= D, 0 <= q_i <= qhi_i (integer),
// w_i = lambda_i c_ij.  Bounded covering knapsack by binary splitting over coverage 0..D.
double cover_knapsack(const Cover& in, int j, const std::vector<double>& lam, std::vector<double>& f) {
  const int64_t Dj = in.D[j];
  f.assign((size_t)Dj + 1, INF);
  f[0] = 0.0;
  for (int i = 0; i < in.G; ++i) {
    int64_t cnt = std::min(in.qhi[i][j], cdiv(Dj, in.p[i]));
    if (cnt <= 0) continue;
    const double w = lam[i] * (double)in.c[i][j];
    for (int64_t chunk = 1; cnt > 0; chunk <<= 1) {
      const int64_t take = std::min(chunk, cnt);
      cnt -= take;
      const int64_t cov = take * in.p[i];
      const double cw = w * (double)take;
      for (int64_t k = Dj; k >= 1; --k) {
        const int64_t from = std::max<int64_t>(0, k - cov);
        const double v = f[from] + cw;
        if (v < f[k]) f[k] = v;
      }
    }
  }
  return f[Dj];
}

double lagrangian(const Cover& in, const LP& lp, const Model& md) {
  std::vector<double> lam(in.G, 0.0);
  double s = 0;
  for (int i = 0; i < in.G; ++i) {
    const int slack = md.nq + 1 + i;
    lam[i] = lp.row_of[slack] >= 0 ? 0.0 : std::max(0.0, lp.d[slack]);
    s += lam[i];
  }
  if (!(s > 0)) return -INF;
  for (auto& l : lam) l /= s;
  double lb = 0;
  std::vector<double> f;
  for (int j = 0; j < in.R; ++j) {
    if (in.D[j] <= 0) continue;
    const double k = cover_knapsack(in, j, lam, f);
    if (k == INF) return INF;
    lb += k;
  }
  for (int i = 0; i < in.G; ++i) lb -= lam[i] * (double)in.tau[i];
  return lb;
}

struct Scratch {
  std::vector<double> f, lam, g;
  std::vector<int64_t> rest;
  std::vector<int> ids, order, gids;
  std::vector<int64_t> cnt, room, m;
  std::vector<double> w;
};

// min sum_i w_i n_i s.t. sum_i p_i n_i >= rest, 0 <= n_i <= cnt_i (w_i = lambda_i c_ij, the
// node's room hi - lo).  Exchange argument: with b a best-ratio item (min w/p) that has room
// for every exchange, some optimum uses fewer than p_b units of every other item (p_b units
// of item i cover what p_i units of b cover, at no lower cost), so those counts are
// enumerated and b covers the rest; otherwise a bounded knapsack over coverage.
double knap_min(const Cover& in, const LP& lp, const Model& md, int j, const std::vector<double>& lam,
                int64_t rest, Scratch& sc) {
  sc.ids.resize(in.G);
  sc.cnt.resize(in.G);
  sc.room.resize(in.G);
  sc.w.resize(in.G);
  sc.m.assign(in.G, 0);
  int* ids = sc.ids.data();
  int64_t* cnt = sc.cnt.data();
  int64_t* room = sc.room.data();
  double* w = sc.w.data();
  std::vector<double>& f = sc.f;
  int n = 0, b = -1;
  int64_t pmax = 1;
  for (int i = 0; i < in.G; ++i) {
    const int v = md.var_of[i][j];
    if (v < 0) continue;
    room[n] = (int64_t)lp.hi[v] - (int64_t)lp.lo[v];
    const int64_t c0 = std::min(room[n], cdiv(rest, in.p[i]));
    if (c0 <= 0) continue;
    ids[n] = i;
    cnt[n] = c0;
    w[n] = lam[i] * (double)in.c[i][j];
    pmax = std::max(pmax, in.p[i]);
    if (b < 0 || w[n] * (double)in.p[ids[b]] < w[b] * (double)in.p[i]) b = n;
    ++n;
  }
  if (n == 0) return INF;
  const int64_t pb = in.p[ids[b]];
  int64_t combos = 1;
  for (int k = 0; k < n; ++k)
    if (k != b) combos *= std::min<int64_t>(cnt[k] + 1, pb);
  if (room[b] >= cdiv(rest, pb) && combos <= 4096) {
    double best = INF;
    int64_t* m = sc.m.data();
    for (int64_t it = 0; it < combos; ++it) {
      int64_t r = it, covered = 0;
      double cost = 0;
      for (int k = 0; k < n; ++k) {
        if (k == b) continue;
        const int64_t lim = std::min<int64_t>(cnt[k] + 1, pb);
        m[k] = r % lim;
        r /= lim;
        covered += m[k] * in.p[ids[k]];
        cost += w[k] * (double)m[k];
      }
      const int64_t left = std::max<int64_t>(0, rest - covered);
      cost += w[b] * (double)cdiv(left, pb);
      if (cost < best) best = cost;
    }
    return best;
  }
  f.assign((size_t)rest + 1, INF);
  f[0] = 0.0;
  for (int k = 0; k < n; ++k) {
    int64_t c = cnt[k];
    const int64_t p = in.p[ids[k]];
    double* F = f.data();
    if (c >= cdiv(rest, p)) {   // effectively unbounded: one forward pass
      const double wk = w[k];
      for (int64_t q = 1; q <= std::min(p, rest); ++q) F[q] = std::min(F[q], F[0] + wk);
      for (int64_t q = p + 1; q <= rest; ++q) F[q] = std::min(F[q], F[q - p] + wk);
      continue;
    }
    for (int64_t chunk = 1; c > 0; chunk <<= 1) {
      const int64_t take = std::min(chunk, c);
      c -= take;
      const int64_t cv = take * p;
      const double cw = w[k] * (double)take;
      for (int64_t q = rest; q > cv; --q) F[q] = std::min(F[q], F[q - cv] + cw);
      for (int64_t q = std::min(cv, rest); q >= 1; --q) F[q] = std::min(F[q], F[0] + cw);
    }
  }
  return f[rest];
}

// The same Lagrangian bound at a branch-and-bound node: every q_ij restricted to the
// node's [lo, hi]; bucket j's knapsack starts from the coverage of the lower bounds.
double lagrangian_node(const Cover& in, const LP& lp, const Model& md, Scratch& sc) {
  std::vector<double>& lam = sc.lam;
  lam.assign(in.G, 0.0);
  double s = 0;
  for (int i = 0; i < in.G; ++i) {
    const int slack = md.nq + 1 + i;
    lam[i] = lp.row_of[slack] >= 0 ? 0.0 : std::max(0.0, lp.d[slack]);
    s += lam[i];
  }
  if (!(s > 0)) return -INF;
  for (auto& l : lam) l /= s;
  // per bucket: the continuous (greedy) covering cost and an upper bound g_j on what the
  // integer knapsack adds to it (rounding the one fractional item up)
  double lb = 0, gsum = 0;
  for (int i = 0; i < in.G; ++i) lb -= lam[i] * (double)in.tau[i];
  sc.rest.assign(in.R, 0);
  sc.g.assign(in.R, 0.0);
  sc.order.resize(in.R);
  std::vector<int>& ids = sc.gids;
  ids.resize(in.G);
  int64_t* rest_of = sc.rest.data();
  double* g_of = sc.g.data();
  for (int j = 0; j < in.R; ++j) {
    if (in.D[j] <= 0) continue;
    int64_t cov = 0;
    int n = 0;
    for (int i = 0; i < in.G; ++i) {
      const int v = md.var_of[i][j];
      if (v < 0) continue;
      const int64_t l0 = (int64_t)lp.lo[v];
      cov += l0 * in.p[i];
      lb += lam[i] * (double)in.c[i][j] * (double)l0;
      if (lp.hi[v] > lp.lo[v]) ids[n++] = i;
    }
    const int64_t rest = in.D[j] - cov;
    if (rest <= 0) continue;
    std::sort(ids.begin(), ids.begin() + n, [&](int a, int b) {
      return lam[a] * (double)in.c[a][j] * (double)in.p[b] < lam[b] * (double)in.c[b][j] * (double)in.p[a];
    });
    double need = (double)rest, cost = 0, g = 0;
    for (int k = 0; k < n && need > 0; ++k) {
      const int i = ids[k];
      const int v = md.var_of[i][j];
      const double room = lp.hi[v] - lp.lo[v];
      const double take = std::min(room, need / (double)in.p[i]);
      const double w = lam[i] * (double)in.c[i][j];
      cost += w * take;
      need -= take * (double)in.p[i];
      const double fr = take - std::floor(take + 1e-12);
      if (fr > 1e-12) g = w * (1.0 - fr);
    }
    if (need > 1e-9) return INF;   // the bucket cannot be covered at this node
    lb += cost;
    rest_of[j] = rest;
    g_of[j] = g;
    gsum += g;
  }
  if (lb + gsum <= ZTOL || lb > ZTOL) return lb;
  // replace the continuous costs by the exact integer knapsacks, largest possible gain first,
  // until the bound either proves the node infeasible or provably cannot
  int* order = sc.order.data();
  int no = 0;
  for (int j = 0; j < in.R; ++j)
    if (g_of[j] > 0) order[no++] = j;
  std::sort(order, order + no, [&](int a, int b) { return g_of[a] > g_of[b]; });
  for (int t = 0; t < no; ++t) {
    const int j = order[t];
    // continuous cost of bucket j (recomputed) -> exact integer cost
    int n = 0;
    for (int i = 0; i < in.G; ++i) {
      const int v = md.var_of[i][j];
      if (v >= 0 && lp.hi[v] > lp.lo[v]) ids[n++] = i;
    }
    std::sort(ids.begin(), ids.begin() + n, [&](int a, int b) {
      return lam[a] * (double)in.c[a][j] * (double)in.p[b] < lam[b] * (double)in.c[b][j] * (double)in.p[a];
    });
    double need = (double)rest_of[j], cont = 0;
    for (int k = 0; k < n && need > 0; ++k) {
      const int i = ids[k];
      const int v = md.var_of[i][j];
      const double take = std::min(lp.hi[v] - lp.lo[v], need / (double)in.p[i]);
      cont += lam[i] * (double)in.c[i][j] * take;
      need -= take * (double)in.p[i];
    }
    const double k = knap_min(in, lp, md, j, lam, rest_of[j], sc);
    if (k == INF) return INF;
    lb += k - cont;
    gsum -= g_of[j];
    if (lb > ZTOL || lb + gsum <= ZTOL) return lb;
  }
  return lb;
}

bool verify(const Cover& in, const std::vector<std::vector<int64_t>>& q) {
  for (int i = 0; i < in.G; ++i) {
    int64_t L = 0;
    for (int j = 0; j < in.R; ++j) {
      if (q[i][j] < 0 || q[i][j] > std::max<int64_t>(in.qhi[i][j], 0)) return false;
      L += in.c[i][j] * q[i][j];
    }
    if (L > in.tau[i]) return false;
  }
  for (int j = 0; j < in.R; ++j) {
    int64_t cov = 0;
    for (int i = 0; i < in.G; ++i) cov += in.p[i] * q[i][j];
    if (cov < in.D[j]) return false;
  }
  return true;
}

// Round the LP point down, then cover each bucket's deficit greedily with the group whose
// budget stays the loosest.  Returns true with q on success.
bool round_repair(const Cover& in, const LP& lp, const Model& md,
                  std::vector<std::vector<int64_t>>& q, std::vector<int64_t>& L) {
  q.resize(in.G);
  for (auto& r : q) r.assign(in.R, 0);
  L.assign(in.G, 0);
  for (int v = 0; v < md.nq; ++v) {
    const double val = lp.value(v);
    int64_t f = (int64_t)std::floor(val + 1e-9);
    f = std::max<int64_t>((int64_t)lp.lo[v], std::min<int64_t>((int64_t)lp.hi[v], f));
    q[md.vi[v]][md.vj[v]] = f;
  }
  for (int i = 0; i < in.G; ++i)
    for (int j = 0; j < in.R; ++j) L[i] += in.c[i][j] * q[i][j];
  for (int j : md.repair_order) {
    int64_t cov = 0;
    for (int i = 0; i < in.G; ++i) cov += in.p[i] * q[i][j];
    int64_t def = in.D[j] - cov;
    while (def > 0) {
      int bi = -1;
      int64_t bslack = INT64_MIN, bk = 0;
      for (int i = 0; i < in.G; ++i) {
        const int v = md.var_of[i][j];
        if (v < 0) continue;
        const int64_t room = (int64_t)lp.hi[v] - q[i][j];
        if (room <= 0) continue;
        const int64_t k = std::min(room, cdiv(def, in.p[i]));
        const int64_t full = k * in.p[i] >= def;
        const int64_t slack = in.tau[i] - L[i] - in.c[i][j] * k;
        // prefer a group that finishes the deficit within budget, then the loosest
        const int64_t key = slack >= 0 && full ? slack : slack - ((int64_t)1 << 40);
        if (key > bslack) bslack = key, bi = i, bk = k;
      }
      if (bi < 0) return false;
      q[bi][j] += bk;
      L[bi] += in.c[bi][j] * bk;
      def -= bk * in.p[bi];
    }
  }
  return verify(in, q);
}

// Shared state of one feasibility search (all threads).
struct Shared {
  std::atomic<int64_t> nodes{0};
  std::atomic<int64_t> pivots{0};
  std::atomic<int> found{0};    // a certificate is stored in sol: every thread stops
  std::atomic<int> budget{0};   // the node budget ran out
  int64_t cap = 0;
  std::mutex mu;
  std::vector<std::vector<int64_t>> sol;
};

// Subtrees below this depth are the parallel tasks (up to 2^depth of them).
constexpr int kSplitDepth = 10;

struct BB {
  const Cover& in;
  const Model& md;
  Shared& sh;
  std::vector<std::vector<int64_t>> cand;
  std::vector<int64_t> loads;
  std::deque<LP> stk;   // child LPs by depth (storage reused; deque: growth keeps references)
  Scratch sc;
  std::vector<LP>* frontier = nullptr;   // set while collecting the parallel tasks
  BB(const Cover& c, const Model& m, Shared& s) : in(c), md(m), sh(s) {}

  int found(const std::vector<std::vector<int64_t>>& q) {
    std::lock_guard<std::mutex> lk(sh.mu);
    if (!sh.found.load()) {
      sh.sol = q;
      sh.found.store(1);
    }
    return 1;
  }

  // 1 feasible (certificate in sh.sol), 0 infeasible subtree (or another thread already
  // found a certificate), -1 budget
  int node(LP& lp, int depth) {
    if (sh.found.load(std::memory_order_relaxed)) return 0;
    if (sh.budget.load(std::memory_order_relaxed)) return -1;
    if (frontier && depth >= kSplitDepth) {
      frontier->push_back(lp);
      return 0;
    }
    if (sh.nodes.fetch_add(1, std::memory_order_relaxed) + 1 > sh.cap) {
      sh.budget.store(1);
      return -1;
    }
    int64_t piv = 0;
    const int rc = lp.solve(ZTOL, 20000, piv);
    sh.pivots.fetch_add(piv, std::memory_order_relaxed);
    if (rc == 1) return 0;
    if (rc == 2) {
      sh.budget.store(1);
      return -1;
    }
    if (lp.z() > ZTOL) return 0;
    // the per-bucket integer covering (Lagrangian) bound sees the ceil(d / p) rounding the
    // LP relaxation ignores (decisive with p_i >= 4: 5-30x fewer nodes, measured)
    if (lagrangian_node(in, lp, md, sc) > ZTOL) return 0;
    // branching candidate: a fractional q of the group with the most replicas (its rounds
    // cover the coarsest steps), the most fractional one among them (measured best of the
    // rules tried: cost-weighted, by bucket, by cost)
    int bv = -1;
    double bs = -1, bval = 0;
    for (int v = 0; v < md.nq; ++v) {
      const double val = lp.value(v);
      const double fr = val - std::floor(val);
      const double dist = std::min(fr, 1.0 - fr);
      if (dist < 1e-7) continue;
      const double s = (double)in.p[md.vi[v]] * 1e6 + dist;
      if (s > bs) bs = s, bv = v, bval = val;
    }
    if (round_repair(in, lp, md, cand, loads)) return found(cand);
    if (bv < 0) {
      // LP point integral up to tolerance: its rounding satisfies the integer constraints
      // unless the tolerance hid a violation; branch on the largest deviation instead
      cand.assign(in.G, std::vector<int64_t>(in.R, 0));
      for (int v = 0; v < md.nq; ++v) cand[md.vi[v]][md.vj[v]] = (int64_t)std::llround(lp.value(v));
      if (verify(in, cand)) return found(cand);
      double dev = 0;
      for (int v = 0; v < md.nq; ++v) {
        if (lp.lo[v] == lp.hi[v]) continue;
        const double val = lp.value(v);
        const double dd = std::fabs(val - std::llround(val));
        if (dd >= dev) dev = dd, bv = v, bval = val;
      }
      if (bv < 0) return 0;
    }
    const double fl = std::floor(bval);
    const bool up_first = false;   // down first: small rounds first (measured best)
    for (int pass = 0; pass < 2; ++pass) {
      const bool up = (pass == 0) == up_first;
      double l = lp.lo[bv], h = lp.hi[bv];
      if (up) l = std::max(l, fl + 1.0);
      else h = std::min(h, fl);
      if (l > h) continue;
      while ((int)stk.size() <= depth) stk.emplace_back();
      LP& child = stk[depth];   // copy-assignment reuses the vectors' storage
      child = lp;
      child.set_bounds(bv, l, h);
      const int r = node(child, depth + 1);
      if (r != 0) return r;
    }
    return 0;
  }
};

bool trivially_infeasible(const Cover& in) {
  for (int i = 0; i < in.G; ++i)
    if (in.tau[i] < 0) return true;
  for (int j = 0; j < in.R; ++j) {
    int64_t cap = 0;
    for (int i = 0; i < in.G; ++i) cap += in.p[i] * std::max<int64_t>(in.qhi[i][j], 0);
    if (cap < in.D[j]) return true;
  }
  return false;
}

}  // namespace

int feasible(const Cover& in, std::vector<std::vector<int64_t>>& q, Stats& st) {
  if (trivially_infeasible(in)) return 0;
  Model md;
  LP lp = build_lp(in, md);
  if (md.nq == 0) {
    q.assign(in.G, std::vector<int64_t>(in.R, 0));
    return verify(in, q) ? 1 : 0;
  }
  ++st.nodes;
  const int rc = lp.solve(ZTOL, 20000, st.lp_pivots);
  if (rc == 2) return -1;
  if (rc == 1 || lp.z() > ZTOL) return 0;
  if (lagrangian(in, lp, md) > ZTOL) return 0;
  Shared sh;
  sh.cap = st.cap - st.nodes + 1;   // the root is re-entered by node() (warm: already optimal)
  int r;
  if (!st.pool || st.pool->size() <= 1) {
    BB bb(in, md, sh);
    r = bb.node(lp, 0);
  } else {
    // depth-first down to kSplitDepth on this thread, the open subtrees below it on the pool
    std::vector<LP> tasks;
    BB top(in, md, sh);
    top.frontier = &tasks;
    r = top.node(lp, 0);
    if (r == 0 && !sh.found.load() && !tasks.empty()) {
      std::vector<BB> bbs;
      bbs.reserve(st.pool->size());
      for (int w = 0; w < st.pool->size(); ++w) bbs.emplace_back(in, md, sh);
      st.pool->run((int)tasks.size(), [&](int w, int k) {
        if (!sh.found.load(std::memory_order_relaxed) && !sh.budget.load(std::memory_order_relaxed))
          bbs[w].node(tasks[k], kSplitDepth + 1);
      });
    }
    r = sh.found.load() ? 1 : sh.budget.load() ? -1 : 0;
  }
  if (sh.found.load()) r = 1;
  st.nodes += sh.nodes.load() - 1;
  st.lp_pivots += sh.pivots.load();
  if (r == 1) q = sh.sol;
  return r;
}

double lower_bound(const Cover& in, Stats& st) {
  Model md;
  LP lp = build_lp(in, md);
  if (md.nq == 0) return -INF;
  ++st.nodes;
  const int rc = lp.solve(INF, 20000, st.lp_pivots);
  if (rc == 1) return INF;
  if (rc == 2) return -INF;
  return std::max(lp.z(), lagrangian(in, lp, md));
}

Pool::Pool(int nthreads) {
  for (int w = 1; w < nthreads; ++w) threads_.emplace_back([this, w] { work(w); });
}

Pool::~Pool() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : threads_) t.join();
}

// Every worker takes part in every generation (wakes, drains the task counter, reports), and
// run() returns only after all of them reported, so no worker can carry a stale task
// function into the next run().
void Pool::work(int worker) {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(int, int)>* f;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      f = f_;
    }
    for (;;) {
      int k;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (next_ >= ntasks_) break;
        k = next_++;
      }
      (*f)(worker, k);
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      ++reported_;
    }
    done_cv_.notify_all();
  }
}

void Pool::run(int ntasks, const std::function<void(int, int)>& f) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    f_ = &f;
    ntasks_ = ntasks;
    next_ = 0;
    reported_ = 0;
    ++gen_;
  }
  cv_.notify_all();
  for (;;) {   // the caller is worker 0
    int k;
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (next_ >= ntasks_) break;
      k = next_++;
    }
    f(0, k);
  }
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return reported_ == (int)threads_.size(); });
  f_ = nullptr;
}

int default_threads() {
  if (const char* e = std::getenv("LOBRA_DISPATCH_THREADS")) {
    const int n = std::atoi(e);
    if (n >= 1) return std::min(n, 64);
  }
  const int hw = (int)std::thread::hardware_concurrency();
  return std::max(1, std::min(16, hw - 1));
}

}  // namespace eq3
}  // namespace lobra
