#include <chrono>
#include <cstdio>
#include <vector>
#include <fstream>
#include <sstream>
#include "autoscout.h"
int main() {
  std::ifstream f("/root/repo/spaces/C4.json"); std::stringstream ss; ss << f.rdbuf();
  as_space* s; as_status r = autoscout_space_create(ss.str().c_str(), -1, &s);
  printf("create %d\n", r);
  std::vector<uint64_t> raws; std::vector<double> costs;
  // observed set: first 256 valid CVI positions spread
  uint64_t n_cvi = 357000000;
  for (uint64_t i = 0; raws.size() < 256 && i < 100000; ++i) {
    uint64_t cvi = (i * 1000003ull) % 350000000ull, raw; autoscout_cvi_to_raw(s, cvi, &raw);
    double c, m; int ok; autoscout_simulate(s, raw, &c, &m, &ok); if (!ok) continue;
    raws.push_back(raw); costs.push_back(c * 1.1);
  }
  for (int it = 0; it < 5; ++it) {
    autoscout_observe_clear(s);
    auto t0 = std::chrono::steady_clock::now();
    r = autoscout_observe(s, raws.data(), costs.data(), raws.size(), nullptr);
    auto t1 = std::chrono::steady_clock::now();
    printf("observe %d: %.3f ms\n", r, std::chrono::duration<double, std::milli>(t1 - t0).count());
  }
}
