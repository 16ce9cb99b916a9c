// buffill.h -- Alg. "Hit buffer filling" (§4 l.184-213), host side.
//
// storeHit(hit): while the buffer holds fewer than b - b_t hits every hit
// joins it and raises toa_max; after that only hits with toa < toa_max +
// t_closing join, later ones go to the next buffer; a hit with toa - toa_max >
// t + t_closing sends the buffer and the next buffer takes its place.  Since
// the stream is t-ordered (l.99-100: toa(h_i) < toa(h_j) + t for i < j), every
// hit after a send has toa >= C = toa_max + t_closing, the sent buffer's cut:
// only clusters with a hit within dt_max of C can still grow (tpx_stream_*
// carries exactly those).  End of stream and cut readings: DESIGN.md R20.
#pragma once
#include <cstdint>
#include <vector>

#include "tpx_cluster.h"

namespace tpx {

template <typename HV, typename GV>  // hit and arrival-index containers
struct buffill_t {
  uint64_t b = 0, b_t = 0, t = 0, t_closing = 0;
  uint64_t toa_max = 0;
  HV buf, next;
  GV buf_g, next_g;  // arrival index of each hit

  // Store one hit; returns true if `buf` must be sent now with cut *cut (the
  // caller consumes buf/buf_g and then calls rotate()).
  bool store(const tpx_hit& h, uint64_t g, uint64_t* cut) {
    if (buf.size() < b - b_t) {
      buf.push_back(h);
      buf_g.push_back(g);
      if (h.toa > toa_max) toa_max = h.toa;
    } else if (h.toa < toa_max + t_closing) {
      buf.push_back(h);
      buf_g.push_back(g);
    } else {
      next.push_back(h);
      next_g.push_back(g);
    }
    if (h.toa > toa_max + t + t_closing) {  // toa(hit) - toa_max > t + t_closing
      *cut = toa_max + t_closing;
      return true;
    }
    return false;
  }

  void rotate() {
    buf.swap(next);
    buf_g.swap(next_g);
    next.clear();
    next_g.clear();
  }
};

using buffill = buffill_t<std::vector<tpx_hit>, std::vector<uint64_t>>;

}  // namespace tpx
