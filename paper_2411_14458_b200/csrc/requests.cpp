// requests.cpp — deterministic request sources on the host
// (synthetic_requests, bubbletea.cpp:269-284). The draws use libstdc++'s
// mt19937 and distributions, whose algorithms are implementation-defined,
// so the trace is generated with the same standard library as the reference
// and then streamed to the device (SURVEY.md §7 hard part 7).
#include <algorithm>
#include <random>
#include <vector>

#include "../../include/geopipe_batch.h"

extern "C" int gpb_synthetic_requests(int32_t count, uint32_t seed, double horizon_ms,
                                      const gpb_prefill_model* pm, gpb_request* out) {
  if (count < 0 || !pm || (count > 0 && !out)) return GPB_CONFIG_ERROR;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> arr(0.0, std::max(0.0, horizon_ms));
  std::uniform_int_distribution<int> tok(1, pm->max_tokens);
  std::vector<double> arrivals(count);
  for (int i = 0; i < count; ++i) arrivals[i] = arr(rng);
  std::sort(arrivals.begin(), arrivals.end());
  for (int i = 0; i < count; ++i) {
    out[i].id = i;
    out[i].tokens = tok(rng);
    out[i].arrival_ms = arrivals[i];
  }
  return GPB_OK;
}
