// tsdiscord drop-in API (B200 build): serial-DRAG entry points and the exact
// nearest-neighbour profile.  Mirrors
// /root/reference/proj/include/tsdiscord/drag.hpp:11-41; here every entry point
// runs on the GPU (drag() returns the same range set as pardrag()).
//
// drag_select / drag_refine keep their contract (the selection keeps every
// range discord; the refinement returns exactly {c in candidates :
// nn(c)^2 >= r^2} with exact nn), not the serial scan's intermediate set: the
// device decides every row in one try, so the selection returns the discords
// themselves and best_so_far_sq is each one's exact nn^2 (the reference's is
// the minimum over the pairs its left-to-right scan happened to evaluate).
#ifndef TSDISCORD_DRAG_HPP
#define TSDISCORD_DRAG_HPP

#include <vector>

#include "tsdiscord/types.hpp"

namespace tsdiscord {

struct Candidate {
    index_t index = 0;
    double best_so_far_sq = 0;
};

struct CandidateSet {
    std::vector<Candidate> entries;
};

// Throws std::invalid_argument when m < 3, 2m > n or r_sq < 0 (src/drag.cpp:63-64).
CandidateSet drag_select(const TimeSeries& series, index_t m, double r_sq);

std::vector<DiscordRecord> drag_refine(const TimeSeries& series, index_t m, double r_sq,
                                       const CandidateSet& candidates,
                                       bool early_abandon = true);

std::vector<DiscordRecord> drag(const TimeSeries& series, index_t m, double r_sq,
                                bool early_abandon = true);
std::vector<double> brute_force_nn(const TimeSeries& series, index_t m);
std::vector<DiscordRecord> brute_force_topk(const TimeSeries& series, index_t m, index_t k);

}  // namespace tsdiscord

#endif
