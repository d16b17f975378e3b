// The drop-in B200 roofline profile beside the reference's own table
// (roofline_b200.hpp over src/traffic.cpp, compiled unchanged): no GPU needed.
#include <cstdio>
#include <stdexcept>

#include "gcoo/roofline_b200.hpp"

int main() {
  const gcoo::RooflineModel& b = gcoo::roofline_profile_ext("B200");
  const gcoo::RooflineModel& p = gcoo::roofline_profile_ext("p100");  // the reference's entry
  bool threw = false;
  try {
    gcoo::roofline_profile_ext("h100");
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  const double ridge = b.peak_flops / b.bandwidth;
  const double at_s099 = gcoo::roofline_throughput(19.7, b);  // BASELINE configs[1] OI
  std::printf("{\"name\": \"%.*s\", \"peak_flops\": %.6g, \"bandwidth\": %.6g, \"ridge\": %.4g, "
              "\"attainable_oi19.7\": %.6g, \"p100_peak\": %.6g, \"unknown_throws\": %s}\n",
              (int)b.name.size(), b.name.data(), b.peak_flops, b.bandwidth, ridge, at_s099, p.peak_flops,
              threw ? "true" : "false");
  return (b.name == "b200" && b.peak_flops > 7e13 && b.bandwidth > 6e12 && p.peak_flops == 9.5e12 && threw) ? 0 : 1;
}
