// Launch accounting for the bench's "gpu_launches" field: every C-ABI entry
// point adds the number of kernels it launched.
#include <atomic>
#include "bddc_b200.h"

static std::atomic<long long> g_launches{0};

extern "C" {
void bddc_note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long bddc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
int bddc_launch_count_reset(void) {
  g_launches.store(0);
  return 0;
}
}
