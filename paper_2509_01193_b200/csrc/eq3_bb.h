// Exact covering-feasibility oracle for LobRA's Eq. 3 with three or more deployed groups
// (internal; not part of the ABI).  See eq3_bb.cpp.
#pragma once
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace lobra {
namespace eq3 {

// The Eq. 3 instance in "replica-round" variables q_ij = ceil(d_ij / p_i):
//   group i (p_i replicas) serving bucket j (D_j sequences) in q_ij rounds costs c_ij q_ij
//   and covers up to p_i q_ij sequences.  qhi[i][j] = 0 marks an unsupported / fixed-out
//   pair.  All integers.
struct Cover {
  int G = 0, R = 0;
  std::vector<int64_t> p;                  // [G]
  std::vector<std::vector<int64_t>> c;     // [G][R]
  std::vector<int64_t> tau;                // [G] per-group budgets (cost units)
  std::vector<int64_t> D;                  // [R] demands
  std::vector<std::vector<int64_t>> qhi;   // [G][R] upper bounds on q_ij (0 = not allowed)
};

// A small fork-join pool for the branch-and-bound subtrees of one dispatch call: `run(n, f)`
// calls f(worker, task) for task = 0..n-1 on `size()` threads (the caller is worker 0) and
// returns when every task has finished.  Not reentrant; one owner thread.
class Pool {
 public:
  explicit Pool(int nthreads);
  ~Pool();
  int size() const { return (int)threads_.size() + 1; }
  void run(int ntasks, const std::function<void(int, int)>& f);

 private:
  void work(int worker);
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int, int)>* f_ = nullptr;
  int ntasks_ = 0, next_ = 0, reported_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Worker threads for the >= 3-group solver: LOBRA_DISPATCH_THREADS if set (>= 1), else the
// host's hardware threads minus one (the caller's launch thread), at most 16.
int default_threads();

struct Stats {
  int64_t nodes = 0;      // branch-and-bound nodes (LP solves) so far
  int64_t cap = 0;        // node budget
  int64_t lp_pivots = 0;
  Pool* pool = nullptr;   // optional: explore the subtrees below the root in parallel
  bool hit() const { return nodes > cap; }
};

// Does an integer q (0 <= q_ij <= qhi_ij) exist with sum_j c_ij q_ij <= tau_i for every i
// and sum_i p_i q_ij >= D_j for every j?  1 = yes (q filled, verified in integers), 0 = no
// (proved by the LP / Lagrangian bounds of a complete branch-and-bound), -1 = node budget
// exhausted (undecided).  With st.pool the subtrees below depth kSplitDepth are explored by
// the pool's threads (the first certificate found stops the others); the answer is the
// same, only which certificate q is returned may depend on timing.
int feasible(const Cover& in, std::vector<std::vector<int64_t>>& q, Stats& st);

// Lower bound on min_q max_i (sum_j c_ij q_ij - tau_i) over the covering constraints:
// max of the LP relaxation value and the Lagrangian bound with per-bucket integer covering
// (LP duals as multipliers).  Exact in the sense that the true integer optimum is >= it.
double lower_bound(const Cover& in, Stats& st);

}  // namespace eq3
}  // namespace lobra
