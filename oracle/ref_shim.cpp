// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" wrappers around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libtsdref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg / --impl reference) may load it.
//
// Each wrapper calls exactly one public reference entry point:
//   tsdref_gen_randomwalk   -> tsdiscord::gen_randomwalk     (proj/src/io.cpp:110-119)
//   tsdref_init_stats       -> tsdiscord::init_stats         (proj/src/stats.cpp:7-36)
//   tsdref_advance_stats    -> tsdiscord::advance_stats      (proj/src/stats.cpp:38-58)
//   tsdref_brute_force_nn   -> tsdiscord::brute_force_nn     (proj/src/drag.cpp:137-149)
//   tsdref_pardrag          -> tsdiscord::pardrag (overload) (proj/src/pardrag.cpp:429-434)
//   tsdref_merlin           -> tsdiscord::merlin_full        (proj/src/merlin.cpp:57-132)
//   tsdref_discords_csv     -> tsdiscord::write_discords_csv (proj/src/io.cpp:121-130)
//   tsdref_heatmap          -> read_discords_csv + build_heatmap + rank_discords and the three
//                              writers (proj/src/io.cpp:132-160, proj/src/heatmap.cpp:18-83)
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsdiscord/drag.hpp"
#include "tsdiscord/heatmap.hpp"
#include "tsdiscord/io.hpp"
#include "tsdiscord/merlin.hpp"
#include "tsdiscord/pardrag.hpp"
#include "tsdiscord/stats.hpp"

using namespace tsdiscord;

namespace {
thread_local std::string g_err;

struct Rec {
    int64_t index;
    double nn_dist_sq;
    double nn_dist;
};

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}
}  // namespace

#define REF_GUARD(...)                                              \
    try {                                                           \
        __VA_ARGS__;                                                     \
        return 0;                                                   \
    } catch (const std::invalid_argument& e) { return fail(e, 1); } \
    catch (const std::logic_error& e) { return fail(e, 2); }        \
    catch (const std::exception& e) { return fail(e, 3); }

extern "C" {

const char* tsdref_last_error() { return g_err.c_str(); }

int tsdref_gen_randomwalk(int64_t n, uint64_t seed, double* out) {
    REF_GUARD({
        const TimeSeries s = gen_randomwalk(n, seed);
        std::memcpy(out, s.values().data(), sizeof(double) * static_cast<size_t>(n));
    })
}

int tsdref_init_stats(const double* x, int64_t n, int64_t m, double* mu, double* sigma) {
    REF_GUARD({
        const TimeSeries s(std::vector<double>(x, x + n));
        const RollingStats st = init_stats(s, m);
        std::memcpy(mu, st.mu.data(), sizeof(double) * static_cast<size_t>(st.valid_count));
        std::memcpy(sigma, st.sigma.data(), sizeof(double) * static_cast<size_t>(st.valid_count));
    })
}

// Advances from m0 to m1 (m1 >= m0) with advance_stats, starting from init_stats(m0).
int tsdref_advance_stats(const double* x, int64_t n, int64_t m0, int64_t m1, double* mu,
                         double* sigma) {
    REF_GUARD({
        const TimeSeries s(std::vector<double>(x, x + n));
        RollingStats st = init_stats(s, m0);
        for (int64_t m = m0; m < m1; ++m) st = advance_stats(st, s);
        std::memcpy(mu, st.mu.data(), sizeof(double) * static_cast<size_t>(st.valid_count));
        std::memcpy(sigma, st.sigma.data(), sizeof(double) * static_cast<size_t>(st.valid_count));
    })
}

int tsdref_brute_force_nn(const double* x, int64_t n, int64_t m, double* out) {
    REF_GUARD({
        const TimeSeries s(std::vector<double>(x, x + n));
        const auto nn = brute_force_nn(s, m);
        std::memcpy(out, nn.data(), sizeof(double) * nn.size());
    })
}

int tsdref_pardrag(const double* x, int64_t n, int64_t m, double r_sq, int64_t seglen,
                   int64_t workers, void* recs, int64_t cap, int64_t* count) {
    REF_GUARD({
        const TimeSeries s(std::vector<double>(x, x + n));
        const auto out = pardrag(s, m, r_sq, seglen, workers, true);
        *count = static_cast<int64_t>(out.size());
        Rec* r = static_cast<Rec*>(recs);
        for (size_t k = 0; k < out.size() && static_cast<int64_t>(k) < cap; ++k)
            r[k] = {out[k].index, out[k].nn_dist_sq, out[k].nn_dist};
    })
}

// Outputs per length L = maxL-minL+1: counts[L], recs[L*top_k], final_r[L],
// retries[L], failed[L] (1 if the length is in failed_lengths).
int tsdref_merlin(const double* x, int64_t n, int64_t min_len, int64_t max_len, int64_t top_k,
                  int64_t seglen, int64_t workers, int64_t max_retries, int reuse_stats,
                  int64_t* counts, void* recs, double* final_r, int64_t* retries,
                  uint8_t* failed) {
    REF_GUARD({
        const TimeSeries s(std::vector<double>(x, x + n));
        MerlinOptions o;
        o.top_k = top_k;
        o.seglen = seglen;
        o.workers = workers;
        o.max_retries = max_retries;
        o.reuse_stats = reuse_stats != 0;
        const MerlinReport rep = merlin_full(s, min_len, max_len, o);
        const int64_t L = max_len - min_len + 1;
        Rec* r = static_cast<Rec*>(recs);
        for (int64_t k = 0; k < L; ++k) {
            counts[k] = 0;
            failed[k] = 0;
            final_r[k] = rep.final_r[static_cast<size_t>(k)];
            retries[k] = rep.retries[static_cast<size_t>(k)];
        }
        for (index_t m : rep.discords.failed_lengths) failed[m - min_len] = 1;
        for (const auto& [m, lst] : rep.discords.per_length) {
            const int64_t k = m - min_len;
            counts[k] = static_cast<int64_t>(lst.size());
            for (size_t j = 0; j < lst.size(); ++j)
                r[k * top_k + static_cast<int64_t>(j)] = {lst[j].index, lst[j].nn_dist_sq,
                                                          lst[j].nn_dist};
        }
    })
}

// CSV text of merlin(...) as written by write_discords_csv; returns the byte
// length (buffer must hold it; call with cap=0 to size).
int64_t tsdref_merlin_csv(const double* x, int64_t n, int64_t min_len, int64_t max_len,
                          int64_t top_k, int64_t seglen, int64_t workers, char* buf,
                          int64_t cap) {
    try {
        const TimeSeries s(std::vector<double>(x, x + n));
        MerlinOptions o;
        o.top_k = top_k;
        o.seglen = seglen;
        o.workers = workers;
        std::ostringstream os;
        write_discords_csv(merlin(s, min_len, max_len, o), os);
        const std::string str = os.str();
        if (cap >= static_cast<int64_t>(str.size())) std::memcpy(buf, str.data(), str.size());
        return static_cast<int64_t>(str.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Heatmap outputs of a discord CSV, as the reference CLI writes them
// (tools/main.cpp:111-136): which = 0 heatmap CSV, 1 PGM, 2 ranking CSV (k).
// Returns the byte length (call with cap=0 to size), -1 on error.
int64_t tsdref_heatmap(const char* csv, int64_t n, int64_t k, int which, char* buf, int64_t cap) {
    try {
        std::istringstream in(csv);
        const MultiLengthDiscordSet d = read_discords_csv(in);
        const Heatmap h = build_heatmap(d, n);
        std::ostringstream os;
        if (which == 0) write_heatmap_csv(h, os);
        else if (which == 1) write_heatmap_pgm(h, os);
        else write_ranking_csv(rank_discords(h, k), os);
        const std::string str = os.str();
        if (cap >= static_cast<int64_t>(str.size())) std::memcpy(buf, str.data(), str.size());
        return static_cast<int64_t>(str.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
