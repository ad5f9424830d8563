// C++ host over the C-ABI: config 2's dynamics x_{t+1} = tanh(2 Q x_t) + 0.1 x_{t-1}
// on a Haar operator, once probe by probe through the ProbeOperator adapter and
// once as one device-resident hd_run; checks the reference's properties
// (isometry, repeat-free consistency of the two routes) and prints timings.
//   g++ -O2 -std=c++17 -I include examples/cabi_demo.cpp -L paper_2101_07464_b200/lib -lhd_b200 -Wl,-rpath,...
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "b200_probe_operator.hpp"

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 100000;
  const int64_t T = argc > 2 ? std::atoll(argv[2]) : 20;
  std::vector<double> x1(n), x0(n, 0.0);
  for (int64_t i = 0; i < n; ++i) x1[i] = std::sin(0.37 * (double)i + 1.0);
  double nrm = 0.0;
  for (double v : x1) nrm += v * v;
  for (double& v : x1) v /= std::sqrt(nrm);

  // route 1: probe by probe (ProbeOperator adapter, host vectors)
  b200::ProbeOperator op(HD_HAAR, n, n, 1.0, 42);
  std::vector<double> prev = x0, cur = x1;
  double worst_iso = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int64_t t = 0; t < T; ++t) {
    const std::vector<double> y = op.probe(cur, b200::Side::right);
    double ny = 0.0, nx = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      ny += y[i] * y[i];
      nx += cur[i] * cur[i];
    }
    worst_iso = std::fmax(worst_iso, std::fabs(std::sqrt(ny) - std::sqrt(nx)) / std::sqrt(nx));
    std::vector<double> nxt(n);
    for (int64_t i = 0; i < n; ++i) nxt[i] = std::tanh(2.0 * y[i]) + 0.1 * prev[i];
    prev = cur;
    cur = nxt;
  }
  const double ms_probe = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();

  // route 2: the same run device-resident (hd_run, fused tanh-mix update)
  b200::ProbeOperator op2(HD_HAAR, n, n, 1.0, 42);
  std::vector<double> fin(n);
  hd_run_args a{};
  a.update = HD_UPDATE_TANH_MIX;
  a.side_rule = HD_SIDES_RIGHT;
  a.iterations = T;
  a.x1 = x1.data();
  a.x0 = x0.data();
  a.on_device = 0;
  a.final_out = fin.data();
  const auto t1 = std::chrono::steady_clock::now();
  b200::check(hd_run(op2.handle(), &a));
  const double ms_run = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();

  double diff = 0.0, ref = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    diff += (fin[i] - cur[i]) * (fin[i] - cur[i]);
    ref += cur[i] * cur[i];
  }
  const double rel = std::sqrt(diff / ref);
  bool budget_ok = false;
  try {
    b200::ProbeOperator small(HD_HAAR, 2, 2, 1.0, 1);
    small.probe({1.0, 0.0}, b200::Side::right);
    small.probe({0.0, 1.0}, b200::Side::left);
    small.probe({1.0, 1.0}, b200::Side::right);
  } catch (const b200::BudgetExhausted&) {
    budget_ok = true;
  }
  std::printf("{\"n\": %lld, \"T\": %lld, \"probe_route_ms\": %.3f, \"hd_run_ms\": %.3f, \"isometry_err\": %.3g, "
              "\"routes_rel_diff\": %.3g, \"budget_exception\": %s, \"version\": \"%s\"}\n",
              (long long)n, (long long)T, ms_probe, ms_run, worst_iso, rel, budget_ok ? "true" : "false",
              hd_version());
  return (worst_iso < 1e-12 && rel < 1e-12 && budget_ok) ? 0 : 1;
}
