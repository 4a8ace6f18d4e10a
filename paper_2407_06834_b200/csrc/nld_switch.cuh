// A/B switches of the kernel experiments.  They exist only in the test build
// (`make ab`: -DNLD_AB_BUILD -> libnld_b200_ab.so, its own ABI tag, never
// loaded by the package); the product library compiles every switch to its
// default, so no environment variable can change what the product runs.
#pragma once

#ifdef NLD_AB_BUILD
#include <cstdlib>
namespace nld {
inline int ab_switch(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && e[0]) ? (e[0] != '0') : dflt;
}
inline int ab_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && e[0]) ? std::atoi(e) : dflt;
}
}  // namespace nld
#else
namespace nld {
constexpr int ab_switch(const char*, int dflt) { return dflt; }
constexpr int ab_int(const char*, int dflt) { return dflt; }
}  // namespace nld
#endif
