// Eq.1 iteration latency of one candidate plan, on the host: the planner's hot loop
// (hetplan costs.py:204-535 — _compute_per_microbatch :220-249, the pipelined phase
// recurrence :323-360, total_iteration_latency :384-535), restated operation by
// operation from plan/estimate.py so every double is bit-identical to the Python
// restatement (and through it to the reference).  The caller (plan/estimate.py)
// flattens the plan: per ministage its group, round, layer classes, the distinct
// (kind, share) members of its group, the summed AllGather / ReduceScatter times and
// the boundary transfer times; per group its size and parameter counts.
#include "zb_internal.h"

#include <cstdint>
#include <map>
#include <vector>

using namespace zb;

namespace {

struct Phase {
  double t_chain;
  std::vector<std::pair<int, double>> lane_end;  // insertion-ordered {group: end}
  double* find(int g) {
    for (auto& e : lane_end)
      if (e.first == g) return &e.second;
    return nullptr;
  }
};

inline double pmax(double a, double b) { return b > a ? b : a; }  // Python max(a, b)

Phase phase_makespan(const std::vector<int>& grp, const std::vector<double>& chain_mb,
                     const std::vector<double>& lane_round, const std::vector<double>& head_round,
                     const std::vector<double>& rs_tail, const std::vector<double>& d_in,
                     const std::vector<double>& floors, double start) {
  Phase ph;
  double t_chain = start, t_first = start;
  for (size_t i = 0; i < grp.size(); ++i) {
    const int g = grp[i];
    double* le = ph.find(g);
    const double prev = le ? *le : 0.0;
    const double begin = pmax(pmax(t_first + d_in[i], floors[i]), prev);
    double end = pmax(t_chain + chain_mb[i] + d_in[i], begin + head_round[i]);
    if (le) end = pmax(end, *le + lane_round[i]);
    if (le)
      *le = end + rs_tail[i];
    else
      ph.lane_end.push_back({g, end + rs_tail[i]});
    t_chain = end;
    t_first = begin + chain_mb[i];
  }
  ph.t_chain = t_chain;
  return ph;
}

}  // namespace

// part: 0 fwd, 1 bwd (fwd + bwd), 2 bwd only.  fits[(kind * n_cls + cls) * 4 + j],
// j = fwd_alpha, fwd_beta, bwd_alpha, bwd_beta.
static double per_microbatch(int s, int part, const int* lay_off, const int* lay_cls,
                             const int* mem_off, const int* mem_kind, const int* mem_share,
                             int n_cls, const double* fits) {
  double worst = 0.0;
  for (int d = mem_off[s]; d < mem_off[s + 1]; ++d) {
    const double share = (double)mem_share[d];
    double t = 0.0;
    for (int l = lay_off[s]; l < lay_off[s + 1]; ++l) {
      const double* f = fits + ((size_t)mem_kind[d] * n_cls + lay_cls[l]) * 4;
      const double fwd = f[0] + f[1] * share;
      const double bwd = f[2] + f[3] * share;
      t += part == 0 ? fwd : (part == 1 ? fwd + bwd : bwd);
    }
    worst = pmax(worst, t);
  }
  return worst;
}

extern "C" int zb_eq1_latency(int n, int m, int z3, int offloads, int rounds, const int* grp,
                              const int* q, const int* lay_off, const int* lay_cls,
                              const int* mem_off, const int* mem_kind, const int* mem_share,
                              int n_cls, const double* fits, const double* ag, const double* rs,
                              const double* p2p, const double* stage_params, int n_groups,
                              const int* group_size, double optim_per_param, double* out) {
  if (n <= 0 || m <= 0 || !grp || !q || !lay_off || !lay_cls || !mem_off || !mem_kind ||
      !mem_share || !fits || !ag || !rs || !p2p || !stage_params || !group_size || !out)
    return set_error(ZB_ERR_INVALID, "eq1_latency: bad arguments");
  std::vector<double> f_mb(n), b_mb(n), b_only(n);
  for (int s = 0; s < n; ++s) {
    f_mb[s] = per_microbatch(s, 0, lay_off, lay_cls, mem_off, mem_kind, mem_share, n_cls, fits);
    b_mb[s] = per_microbatch(s, 1, lay_off, lay_cls, mem_off, mem_kind, mem_share, n_cls, fits);
    b_only[s] = per_microbatch(s, 2, lay_off, lay_cls, mem_off, mem_kind, mem_share, n_cls, fits);
  }
  auto round_cost = [&](int s, double per_mb, double out_xfer) {
    if (z3) return pmax(m * (per_mb + ag[s]), m * out_xfer);
    return pmax(pmax(m * per_mb, ag[s]), m * out_xfer);
  };
  std::vector<int> gseq(grp, grp + n);
  // forward
  std::vector<double> floors_f(n, 0.0), chain_f(f_mb), rounds_f(n), zeros(n, 0.0);
  std::vector<double> d_in_f(p2p, p2p + n);
  if (z3) {
    for (int s = 0; s < n; ++s)
      if (q[s] > 0) chain_f[s] += ag[s];
  } else {
    std::map<int, double> acc;
    for (int s = 0; s < n; ++s)
      if (q[s] <= 1) {
        auto it = acc.find(grp[s]);
        const double v = (it == acc.end() ? 0.0 : it->second) + ag[s];
        acc[grp[s]] = v;
        floors_f[s] = v;
      }
  }
  for (int s = 0; s < n; ++s) rounds_f[s] = round_cost(s, f_mb[s], s + 1 < n ? p2p[s + 1] : 0.0);
  const double t_fwd = phase_makespan(gseq, chain_f, rounds_f, rounds_f, zeros, d_in_f, floors_f,
                                      0.0).t_chain;
  // backward (stages in reverse)
  std::vector<int> rev_g(n);
  std::vector<double> d_in_b(n), floors_b(n, 0.0), chain_b, heads_b, lanes_b, rs_b(n);
  std::vector<int> visited;
  for (int k = 0; k < n; ++k) {
    const int s = n - 1 - k;
    rev_g[k] = grp[s];
    d_in_b[k] = k == 0 ? 0.0 : p2p[s + 1];
    rs_b[k] = rs[s];
  }
  if (!z3) floors_b[0] = t_fwd + ag[n - 1];
  for (int k = 0; k < n; ++k) {
    const int s = n - 1 - k, g = grp[s];
    bool first_here = true;
    for (int v : visited)
      if (v == g) first_here = false;
    if (first_here) visited.push_back(g);
    const double lane = round_cost(s, b_mb[s], p2p[s]);
    lanes_b.push_back(lane);
    const double recompute = b_mb[s] - b_only[s];
    if (k == 0) {
      chain_b.push_back(b_mb[s] + (z3 ? ag[s] : 0.0));
      heads_b.push_back(lane);
    } else if (first_here) {
      chain_b.push_back(b_only[s]);
      heads_b.push_back(pmax(lane - recompute, m * b_only[s]));
    } else {
      chain_b.push_back(b_only[s] + (z3 ? ag[s] : 0.0));
      heads_b.push_back(lane);
    }
  }
  Phase pb = phase_makespan(rev_g, chain_b, lanes_b, heads_b, rs_b, d_in_b, floors_b, t_fwd);
  // optimizer after each group's final round
  std::vector<double> first_chunk(n_groups, 0.0), all_chunks(n_groups, 0.0);
  std::vector<uint8_t> seen_all(n_groups, 0);
  for (int s = 0; s < n; ++s) {
    const int g = grp[s];
    if (q[s] == 0) first_chunk[g] = stage_params[s];
    all_chunks[g] = (seen_all[g] ? all_chunks[g] : 0.0) + stage_params[s];
    seen_all[g] = 1;
  }
  double t_total = 0.0;
  for (auto& e : pb.lane_end) {
    const int g = e.first;
    const double local = offloads ? first_chunk[g] : all_chunks[g];
    t_total = pmax(t_total, e.second + local / group_size[g] * optim_per_param);
  }
  const int g0 = grp[0];
  const double startup = ag[0] + rs[0] + first_chunk[g0] / group_size[g0] * optim_per_param;
  out[0] = (t_fwd - ag[0]) / rounds;
  out[1] = (t_total - t_fwd + ag[0] - startup) / rounds;
  out[2] = startup;
  return 0;
}
