// Dev/test aid: run the host GP fit (space.cpp gp_fit) on a seeded valid observed set of a space and
// write L^-1 (row-major), alpha and ||L^-1||_F as raw FP64 to stdout.  tests/test_host_pool.py
// compares the output of 1 and several host threads bit for bit (AS_HOST_THREADS).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <vector>

#include "../paper_2603_11603_b200/csrc/space.hpp"

using namespace as;

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  std::ifstream f(argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();
  HostSpace H;
  if (!build_space(ss.str().c_str(), H).ok()) return 3;
  const int M = std::atoi(argv[2]);
  std::vector<DV> dv;
  std::vector<uint32_t> act;
  std::vector<double> cost, sim;
  uint64_t x = 12345;
  for (int guard = 0; static_cast<int>(dv.size()) < M && guard < 1000000; ++guard) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    const uint64_t cvi = (x >> 11) % H.n_cvi;
    DV d;
    uint32_t a;
    uint64_t raw;
    cvi_decode(H, cvi, d, a, raw);
    double c, mem;
    bool ok;
    simulate_host(H, d, a, c, ok, mem);
    if (!ok) continue;
    dv.push_back(d);
    act.push_back(a);
    sim.push_back(c);
    cost.push_back(c * (1.0 + 0.001 * static_cast<double>((x >> 20) % 100)));
  }
  GPFit fit;
  if (!gp_fit(H, dv, act, cost, sim, fit, nullptr).ok()) return 4;
  std::fwrite(fit.Wl.data(), 8, fit.Wl.size(), stdout);
  std::fwrite(fit.alpha.data(), 8, fit.alpha.size(), stdout);
  std::fwrite(&fit.w_fro, 8, 1, stdout);
  return 0;
}
