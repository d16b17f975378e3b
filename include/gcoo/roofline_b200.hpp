// roofline_b200.hpp — the B200 entry for the reference's roofline profiles.
//
// The reference's RooflineModel table (src/traffic.cpp:223-227) holds the
// paper's cards (gtx980, titanx, p100) and roofline_profile() (:230-237)
// throws for any other name.  This header adds this pool's measured B200
// (FP32 FFMA peak and HBM copy bandwidth, from libgcoo_cuda.so's
// gcoo_roofline_b200) without touching the reference's traffic.cpp:
//
//   const gcoo::RooflineModel& hw = gcoo::roofline_profile_ext("b200");
//   double attainable = gcoo::roofline_throughput(oi, hw);
//
// Include after (or instead of) <gcoo/traffic.hpp>; link libgcoo_cuda.so.
#pragma once

#include <string>
#include <string_view>

#include <gcoo/traffic.hpp>

#include "../gcoo_capi.h"

namespace gcoo {

/// The measured B200 profile (name "b200").
inline const RooflineModel& roofline_profile_b200() {
  static const RooflineModel hw = [] {
    double peak = 0.0, bw = 0.0;
    gcoo_roofline_b200(&peak, &bw);
    return RooflineModel{"b200", peak, bw};
  }();
  return hw;
}

/// roofline_profile (traffic.cpp:230-237) with "b200" (any case) added; every
/// other name resolves through the reference's table, with its exception.
inline const RooflineModel& roofline_profile_ext(std::string_view name) {
  std::string lower(name);
  for (char& ch : lower) ch = (char)((ch >= 'A' && ch <= 'Z') ? ch - 'A' + 'a' : ch);
  if (lower == "b200") return roofline_profile_b200();
  return roofline_profile(name);
}

}  // namespace gcoo
