// Host side of the symbolic plan (integer index maps, no device work): the
// glob tables of plan.py (_glob_part) in one pass of plain loops.  numpy needs
// ~30 array operations on 10^5-entry arrays for the same tables (~3 ms per
// step at cfg5, on the step's host-bound critical path); this is ~0.2 ms.
//
// Reference call sites replaced: the per-subdomain index work of
// build_subdomain_operator (substructuring.py:85-96: which globs a subdomain
// touches, where each sits in its interface numbering).
#include <vector>

#include "bddc_b200.h"

extern "C" {

int bddc_plan_glob_tables(int G, int N, const int* gsize, const long long* nsh,
                          const long long* sharers, int* sh_start, int* slot_glob,
                          long long* sh_doff, int* sub_globs, int* sub_glob_sh,
                          int* sub_glob_start, int* sub_glob_boff, int* sh_boff, long long* nB,
                          long long* b_starts) {
  if (G < 0 || N < 0) return -1;
  // slots in glob-major order: sh_start, slot_glob, sh_doff (n_g^2 per slot)
  long long ns = 0, doff = 0;
  for (int g = 0; g < G; ++g) {
    sh_start[g] = (int)ns;
    const long long n2 = (long long)gsize[g] * gsize[g];
    for (long long k = 0; k < nsh[g]; ++k) {
      slot_glob[ns] = g;
      sh_doff[ns] = doff;
      doff += n2;
      ++ns;
    }
  }
  sh_start[G] = (int)ns;
  sh_doff[ns] = doff;
  // slots by (sharer, glob): counting sort by sharer, stable in the glob order
  std::vector<int> cnt((size_t)N + 1, 0);
  for (long long s = 0; s < ns; ++s) {
    const long long sub = sharers[s];
    if (sub < 0 || sub >= N) return -2;
    ++cnt[(size_t)sub + 1];
  }
  for (int i = 0; i < N; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
  for (int i = 0; i <= N; ++i) sub_glob_start[i] = cnt[(size_t)i];
  std::vector<int> cur(cnt.begin(), cnt.end() - 1);
  std::vector<long long> gstart((size_t)G + 1, 0);
  for (int g = 0; g < G; ++g) gstart[(size_t)g + 1] = gstart[(size_t)g] + gsize[g];
  for (long long s = 0; s < ns; ++s) {
    const int sub = (int)sharers[s];
    const int pos = cur[(size_t)sub]++;
    sub_globs[pos] = slot_glob[s];
    sub_glob_sh[pos] = (int)s;
  }
  // block offset of every glob inside its sharer's glob-major interface order
  for (int i = 0; i < N; ++i) {
    long long boff = 0;
    for (int k = sub_glob_start[i]; k < sub_glob_start[i + 1]; ++k) {
      sub_glob_boff[k] = (int)boff;
      sh_boff[sub_glob_sh[k]] = (int)boff;
      b_starts[k] = gstart[(size_t)sub_globs[k]];
      boff += gsize[sub_globs[k]];
    }
    nB[i] = boff;
  }
  return 0;
}

}  // extern "C"
