// tsdiscord drop-in API (B200 build): serial-DRAG entry points and the exact
// nearest-neighbour profile.  Mirrors
// /root/reference/proj/include/tsdiscord/drag.hpp:11-41; here every entry point
// runs on the GPU (drag() returns the same range set as pardrag()).
#ifndef TSDISCORD_DRAG_HPP
#define TSDISCORD_DRAG_HPP

#include <vector>

#include "tsdiscord/types.hpp"

namespace tsdiscord {

std::vector<DiscordRecord> drag(const TimeSeries& series, index_t m, double r_sq,
                                bool early_abandon = true);
std::vector<double> brute_force_nn(const TimeSeries& series, index_t m);
std::vector<DiscordRecord> brute_force_topk(const TimeSeries& series, index_t m, index_t k);

}  // namespace tsdiscord

#endif
