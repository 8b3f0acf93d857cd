// Tuning knobs (not part of the product): read from the environment only in a -DSGM_TUNING build;
// the product library always uses the defaults (tests/test_abi.py checks that it ignores them).
#pragma once
#include <cstdlib>

namespace sgm {
inline int tune_int(const char* name, int dflt) {
#ifdef SGM_TUNING
  const char* s = std::getenv(name);
  return s ? std::atoi(s) : dflt;
#else
  (void)name;
  return dflt;
#endif
}
}  // namespace sgm
