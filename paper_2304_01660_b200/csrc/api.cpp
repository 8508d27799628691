// C++ drop-in API (namespace tsdiscord) over the C-ABI of libtsdiscord_b200.so.
//
// Callers of the reference library (/root/reference/proj/include/tsdiscord)
// relink against this library unchanged: the same declarations, the same
// exception types for the same preconditions, results equal to the
// reference's.  Every compute entry point goes to the GPU through one
// thread-local context (device from $TSD_DEVICE, default 0); a missing or
// failing GPU raises std::runtime_error — there is no CPU fallback.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <istream>
#include <memory>
#include <ostream>
#include <sstream>
#include <string>
#include <string_view>
#include <thread>

#include "tsdiscord/distance.hpp"
#include "tsdiscord/drag.hpp"
#include "tsdiscord/heatmap.hpp"
#include "tsdiscord/io.hpp"
#include "tsdiscord/merlin.hpp"
#include "tsdiscord/pardrag.hpp"
#include "tsdiscord/stats.hpp"
#include "tsdiscord/types.hpp"
#include "tsdiscord_b200.h"

namespace tsdiscord {

namespace {

[[noreturn]] void rethrow(int code, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (code) {
        case TSD_EINVAL: throw std::invalid_argument(m);
        case TSD_ELOGIC: throw std::logic_error(m);
        default: throw std::runtime_error(m);
    }
}

struct Ctx {
    tsd_ctx* c = nullptr;
    std::vector<double> uploaded;
    Ctx() : Ctx(std::getenv("TSD_DEVICE") ? std::atoi(std::getenv("TSD_DEVICE")) : 0) {}
    explicit Ctx(int device) {
        const int rc = tsd_ctx_create(device, &c);
        if (rc != TSD_OK) rethrow(TSD_ERUNTIME, tsd_create_error());
    }
    ~Ctx() { tsd_ctx_destroy(c); }
    void check(int rc) {
        if (rc != TSD_OK) rethrow(rc, tsd_last_error(c));
    }
    void series(const TimeSeries& s) {
        const auto& v = s.values();
        if (v.size() == uploaded.size() && std::memcmp(v.data(), uploaded.data(), v.size() * 8) == 0)
            return;
        check(tsd_series_set(c, v.data(), (int64_t)v.size()));
        uploaded = v;
    }
};

Ctx& ctx() {
    thread_local std::unique_ptr<Ctx> c;
    if (!c) c = std::make_unique<Ctx>();
    return *c;
}

// A device list of two or more GPUs (MerlinOptions / ParOptions::devices):
// one in-process rank group per calling thread, rebuilt when the list changes.
struct Group {
    tsd_group* g = nullptr;
    std::vector<int> devices;
    std::vector<double> uploaded;
    ~Group() { tsd_group_destroy(g); }
    void check(int rc) {
        if (rc != TSD_OK) rethrow(rc, tsd_group_last_error(g));
    }
    void series(const TimeSeries& s) {
        const auto& v = s.values();
        if (v.size() == uploaded.size() && std::memcmp(v.data(), uploaded.data(), v.size() * 8) == 0)
            return;
        check(tsd_group_series_set(g, v.data(), (int64_t)v.size()));
        uploaded = v;
    }
};

Group* group_for(const std::vector<int>& devices) {
    if (devices.size() < 2) return nullptr;
    thread_local std::unique_ptr<Group> gr;
    if (!gr || gr->devices != devices) {
        gr.reset();
        auto fresh = std::make_unique<Group>();
        const int rc = tsd_group_create(devices.data(), (int)devices.size(), &fresh->g);
        if (rc != TSD_OK) rethrow(rc, tsd_create_error());
        fresh->devices = devices;
        gr = std::move(fresh);
    }
    return gr.get();
}

// one device of the list when it has exactly one entry
Ctx& ctx_for(const std::vector<int>& devices) {
    if (devices.size() == 1) {
        thread_local std::unique_ptr<Ctx> one;
        thread_local int one_dev = -1;
        if (!one || one_dev != devices[0]) {
            one.reset();
            auto c = std::make_unique<Ctx>(devices[0]);
            one = std::move(c);
            one_dev = devices[0];
        }
        return *one;
    }
    return ctx();
}

std::vector<DiscordRecord> to_records(const std::vector<tsd_record>& r, size_t n) {
    std::vector<DiscordRecord> out(n);
    for (size_t i = 0; i < n; ++i) out[i] = {(index_t)r[i].index, r[i].nn_dist_sq, r[i].nn_dist};
    return out;
}

std::vector<DiscordRecord> run_pardrag(const TimeSeries& series, index_t m, double r_sq,
                                       index_t seglen, const RollingStats* stats,
                                       const std::vector<int>& devices = {}) {
    const index_t N = series.n() - m + 1;
    std::vector<tsd_record> buf(std::max<index_t>(N, 1));
    int64_t cnt = 0;
    if (Group* g = group_for(devices)) {  // the group computes its own stats (same values)
        g->series(series);
        g->check(tsd_group_pardrag(g->g, m, r_sq, seglen, buf.data(), (int64_t)buf.size(), &cnt));
        return to_records(buf, (size_t)cnt);
    }
    Ctx& c = ctx_for(devices);
    c.series(series);
    const bool use_stats = stats && (index_t)stats->mu.size() >= N && stats->m == m;
    c.check(tsd_pardrag(c.c, m, r_sq, seglen, use_stats ? stats->mu.data() : nullptr,
                        use_stats ? stats->sigma.data() : nullptr, buf.data(), (int64_t)buf.size(), &cnt));
    return to_records(buf, (size_t)cnt);
}

}  // namespace

// ---- types (reference: src/types.cpp) ---------------------------------------
TimeSeries::TimeSeries(std::vector<double> values) : v_(std::move(values)) {
    if (n() < 3) throw std::invalid_argument("time series needs at least 3 points");
    for (double x : v_)
        if (!std::isfinite(x)) throw std::invalid_argument("time series contains a non-finite value");
}

void sort_discords(std::vector<DiscordRecord>& r) {
    std::sort(r.begin(), r.end(), [](const DiscordRecord& a, const DiscordRecord& b) {
        return a.nn_dist_sq != b.nn_dist_sq ? a.nn_dist_sq > b.nn_dist_sq : a.index < b.index;
    });
}

bool non_self_match(index_t i, index_t j, index_t m) { return (i > j ? i - j : j - i) >= m; }

SegmentLayout compute_layout(index_t n, index_t m, index_t seglen) {
    int64_t o[4];
    const int rc = tsd_compute_layout(n, m, seglen, o);
    if (rc != TSD_OK) rethrow(rc, tsd_last_error(nullptr));
    return SegmentLayout{(index_t)o[0], (index_t)o[1], (index_t)o[2], (index_t)o[3]};
}

// ---- stats -------------------------------------------------------------------
RollingStats init_stats(const TimeSeries& series, index_t m) {
    if (m < 2 || m > series.n() - 1) throw std::invalid_argument("init_stats: length out of range");
    Ctx& c = ctx();
    c.series(series);
    RollingStats s;
    s.m = m;
    s.valid_count = series.n() - m + 1;
    s.mu.resize((size_t)s.valid_count);
    s.sigma.resize((size_t)s.valid_count);
    c.check(tsd_init_stats(c.c, m, s.mu.data(), s.sigma.data()));
    return s;
}

RollingStats advance_stats(const RollingStats& stats, const TimeSeries& series) {
    if (stats.m + 1 > series.n() - 1) throw std::invalid_argument("advance_stats: next length out of range");
    Ctx& c = ctx();
    c.series(series);
    RollingStats next = stats;  // stale tail entries carry over, as in the reference
    next.m = stats.m + 1;
    next.valid_count = stats.valid_count - 1;
    std::vector<double> mu((size_t)next.valid_count), sg((size_t)next.valid_count);
    c.check(tsd_advance_stats(c.c, stats.m, stats.mu.data(), stats.sigma.data(), mu.data(), sg.data()));
    std::copy(mu.begin(), mu.end(), next.mu.begin());
    std::copy(sg.begin(), sg.end(), next.sigma.begin());
    return next;
}

// ---- pardrag / drag ------------------------------------------------------------
std::vector<DiscordRecord> pardrag(const TimeSeries& series, index_t m, double r_sq, index_t seglen,
                                   index_t /*workers*/, bool /*early_exit*/) {
    return run_pardrag(series, m, r_sq, seglen, nullptr);
}

std::vector<DiscordRecord> pardrag(const TimeSeries& series, index_t m, double r_sq,
                                   const RollingStats& stats, const SegmentLayout& layout,
                                   const ParOptions& opts) {
    return run_pardrag(series, m, r_sq, layout.seglen, &stats, opts.devices);
}

// SelectionState: host view of the two-phase state (pardrag.hpp)
SelectionState::SelectionState(const SegmentLayout& layout, index_t real_count)
    : size_(layout.num_seg * layout.seg_n),
      flags_(new Flags[static_cast<std::size_t>(std::max<index_t>(size_, 0))]),
      nn_(new std::atomic<double>[static_cast<std::size_t>(std::max<index_t>(size_, 0))]),
      side_(static_cast<std::size_t>(std::max<index_t>(size_, 0)),
            Side{std::numeric_limits<double>::infinity(), {}, false}) {
    for (index_t i = 0; i < size_; ++i) {
        const unsigned char live = i < real_count;  // pad slots start cleared
        flags_[(size_t)i].cand.store(live, std::memory_order_relaxed);
        flags_[(size_t)i].neighbor.store(live, std::memory_order_relaxed);
        nn_[(size_t)i].store(std::numeric_limits<double>::infinity(), std::memory_order_relaxed);
    }
}

void SelectionState::lower_nn_dist_sq(index_t i, double value) {
    std::atomic<double>& slot = nn_[at(i)];
    double cur = slot.load(std::memory_order_relaxed);
    while (value < cur && !slot.compare_exchange_weak(cur, value, std::memory_order_relaxed)) {
    }
}

void SelectionState::conjoin() {
    for (index_t i = 0; i < size_; ++i)
        if (!flags_[(size_t)i].neighbor.load(std::memory_order_relaxed))
            flags_[(size_t)i].cand.store(0, std::memory_order_relaxed);
}

namespace {
bool stats_fit(const RollingStats& stats, index_t m, index_t N) {
    return stats.m == m && (index_t)stats.mu.size() >= N && (index_t)stats.sigma.size() >= N;
}
}  // namespace

SelectionState par_select(const TimeSeries& series, index_t m, double r_sq, const RollingStats& stats,
                          const SegmentLayout& layout, const ParOptions& opts) {
    const index_t N = series.subseq_count(m);
    SelectionState state(layout, N);
    std::vector<uint8_t> cand((size_t)std::max<index_t>(N, 1));
    std::vector<double> nn((size_t)std::max<index_t>(N, 1));
    if (group_for(opts.devices)) {
        // the rank group runs the same try; survivors carry their exact nn
        const auto recs = run_pardrag(series, m, r_sq, layout.seglen, &stats, opts.devices);
        std::fill(cand.begin(), cand.end(), 0);
        for (const auto& r : recs) {
            cand[(size_t)(r.index - 1)] = 1;
            nn[(size_t)(r.index - 1)] = r.nn_dist_sq;
        }
    } else {
        Ctx& c = ctx_for(opts.devices);
        c.series(series);
        const bool own = stats_fit(stats, m, N);
        c.check(tsd_par_select(c.c, m, r_sq, layout.seglen, own ? stats.mu.data() : nullptr,
                               own ? stats.sigma.data() : nullptr, cand.data(), nn.data()));
    }
    for (index_t i = 1; i <= N; ++i) {
        if (!cand[(size_t)(i - 1)]) {
            state.clear_cand(i);
            state.clear_neighbor(i);
        } else {
            state.lower_nn_dist_sq(i, nn[(size_t)(i - 1)]);
        }
    }
    return state;
}

std::vector<DiscordRecord> par_refine(const TimeSeries& series, index_t m, double r_sq,
                                      const RollingStats& stats, const SegmentLayout& layout,
                                      SelectionState& state, const ParOptions& opts) {
    const index_t N = series.subseq_count(m);
    std::vector<uint8_t> cand((size_t)std::max<index_t>(N, 1), 0);
    bool any = false;
    for (index_t i = 1; i <= N && i <= state.size(); ++i) {
        cand[(size_t)(i - 1)] = state.cand(i) ? 1 : 0;
        any = any || cand[(size_t)(i - 1)];
    }
    if (!any) return {};
    std::vector<DiscordRecord> out;
    if (group_for(opts.devices)) {
        for (const auto& r : run_pardrag(series, m, r_sq, layout.seglen, &stats, opts.devices))
            if (cand[(size_t)(r.index - 1)]) out.push_back(r);
    } else {
        Ctx& c = ctx_for(opts.devices);
        c.series(series);
        const bool own = stats_fit(stats, m, N);
        std::vector<tsd_record> buf((size_t)std::max<index_t>(N, 1));
        int64_t cnt = 0;
        c.check(tsd_par_refine(c.c, m, r_sq, layout.seglen, own ? stats.mu.data() : nullptr,
                               own ? stats.sigma.data() : nullptr, cand.data(), buf.data(),
                               (int64_t)buf.size(), &cnt));
        out = to_records(buf, (size_t)cnt);
    }
    for (const auto& r : out) state.lower_nn_dist_sq(r.index, r.nn_dist_sq);
    return out;
}

namespace {
void drag_checks(const TimeSeries& series, index_t m, double r_sq) {
    // src/drag.cpp:63-64
    if (m < 3 || 2 * m > series.n()) throw std::invalid_argument("drag_select: invalid length");
    if (r_sq < 0) throw std::invalid_argument("drag_select: negative threshold");
}
index_t drag_seglen(const TimeSeries& series, index_t m) {
    return std::min<index_t>(std::max<index_t>(2 * m, 512), series.n());
}
}  // namespace

CandidateSet drag_select(const TimeSeries& series, index_t m, double r_sq) {
    drag_checks(series, m, r_sq);
    const auto recs = run_pardrag(series, m, r_sq, drag_seglen(series, m), nullptr);
    CandidateSet set;
    set.entries.reserve(recs.size());
    for (const auto& r : recs) set.entries.push_back({r.index, r.nn_dist_sq});
    std::sort(set.entries.begin(), set.entries.end(),
              [](const Candidate& a, const Candidate& b) { return a.index < b.index; });
    return set;
}

std::vector<DiscordRecord> drag_refine(const TimeSeries& series, index_t m, double r_sq,
                                       const CandidateSet& candidates, bool) {
    if (candidates.entries.empty()) return {};
    const index_t N = series.subseq_count(m);
    std::vector<uint8_t> keep((size_t)std::max<index_t>(N, 1), 0);
    for (const auto& c : candidates.entries)
        if (c.index >= 1 && c.index <= N) keep[(size_t)(c.index - 1)] = 1;
    std::vector<DiscordRecord> out;
    for (const auto& r : run_pardrag(series, m, r_sq, drag_seglen(series, m), nullptr))
        if (keep[(size_t)(r.index - 1)]) out.push_back(r);
    return out;
}

std::vector<DiscordRecord> drag(const TimeSeries& series, index_t m, double r_sq, bool) {
    drag_checks(series, m, r_sq);
    // same range-discord set; the segment length only shapes the reference's schedule
    return run_pardrag(series, m, r_sq, drag_seglen(series, m), nullptr);
}

// ---- distance building blocks (distance.hpp; host utilities of the API) ---------
std::vector<double> znormalize(std::span<const double> x) {
    const std::size_t m = x.size();
    if (m < 3) throw std::invalid_argument("znormalize: need at least 3 points");
    // one pass of running sums in index order: the rounding the device's exact
    // distance (ref_dist_warp) reproduces
    double s1 = 0.0, s2 = 0.0;
    for (const double v : x) {
        s1 += v;
        s2 += v * v;
    }
    const double mean = s1 / (double)m;
    const double var = s2 / (double)m - mean * mean;
    const double sd = std::sqrt(var > 0.0 ? var : 0.0);
    std::vector<double> z(m, 0.0);
    if (!(sd < kSigmaEps))
        for (std::size_t k = 0; k < m; ++k) z[k] = (x[k] - mean) / sd;
    return z;
}

double sq_ed(std::span<const double> x, std::span<const double> y) {
    if (x.size() != y.size()) throw std::invalid_argument("sq_ed: length mismatch");
    double acc = 0.0;
    for (std::size_t k = 0; k < x.size(); ++k) acc += (x[k] - y[k]) * (x[k] - y[k]);
    return acc;
}

double sq_ednorm_from_dot(double dot, index_t m, double mu_x, double mu_y, double sigma_x, double sigma_y) {
    const double md = (double)m;
    const int flat = (sigma_x < kSigmaEps) + (sigma_y < kSigmaEps);
    if (flat == 2) return 0.0;
    if (flat == 1) return 2.0 * md;
    const double corr = (dot - md * mu_x * mu_y) / (md * sigma_x * sigma_y);
    return std::min(std::max(2.0 * md * (1.0 - corr), 0.0), 4.0 * md);
}

std::optional<double> early_abandon_sq_ed(std::span<const double> xh, std::span<const double> yh,
                                          double bound) {
    if (xh.size() != yh.size()) throw std::invalid_argument("early_abandon_sq_ed: length mismatch");
    double acc = 0.0;
    for (std::size_t k = 0; k < xh.size(); ++k) {
        acc += (xh[k] - yh[k]) * (xh[k] - yh[k]);
        if (acc >= bound) return std::nullopt;
    }
    return acc;
}

DotRow dot_products_block(std::span<const double> query, std::span<const double> window, index_t m,
                          index_t count) {
    if ((index_t)query.size() < m) throw std::invalid_argument("dot_products_block: query shorter than m");
    if ((index_t)window.size() < count + m - 1) throw std::invalid_argument("dot_products_block: window too short");
    DotRow row((size_t)std::max<index_t>(count, 0));
    for (index_t k = 0; k < count; ++k) {
        const double* w = window.data() + k;
        double acc = 0.0;
        for (index_t p = 0; p < m; ++p) acc += query[(size_t)p] * w[p];
        row[(size_t)k] = acc;
    }
    return row;
}

DotRow update_dot_col(const DotRow& prev_col, const DotRow& row, index_t k, std::span<const double> segment,
                      std::span<const double> chunk, index_t m) {
    if (k <= 1 || k > (index_t)row.size()) throw std::invalid_argument("update_dot_col: chunk ordinal out of range");
    DotRow col(prev_col.size());
    if (col.empty()) return col;
    col[0] = row[(size_t)(k - 1)];
    const double in = chunk[(size_t)(k + m - 2)], out = chunk[(size_t)(k - 2)];
    for (std::size_t t = 1; t < col.size(); ++t)
        col[t] = prev_col[t - 1] + segment[t + (size_t)m - 1] * in - segment[t - 1] * out;
    return col;
}

std::vector<double> brute_force_nn(const TimeSeries& series, index_t m) {
    Ctx& c = ctx();
    c.series(series);
    std::vector<double> nn((size_t)(series.n() - m + 1));
    c.check(tsd_brute_force_nn(c.c, m, nn.data()));
    return nn;
}

std::vector<DiscordRecord> brute_force_topk(const TimeSeries& series, index_t m, index_t k) {
    const index_t count = series.subseq_count(m);
    if (k < 1 || k > count) throw std::invalid_argument("brute_force_topk: k out of range");
    const auto nn = brute_force_nn(series, m);
    std::vector<DiscordRecord> all((size_t)count);
    for (index_t i = 0; i < count; ++i) all[(size_t)i] = {i + 1, nn[(size_t)i], std::sqrt(nn[(size_t)i])};
    sort_discords(all);
    all.resize((size_t)k);
    return all;
}

// ---- merlin ---------------------------------------------------------------------
double ThresholdHistory::window_mean() const {
    if (nn_dist.size() < 5) throw std::logic_error("threshold history window too short");
    double s = 0.0;
    for (size_t k = nn_dist.size() - 5; k < nn_dist.size(); ++k) s += nn_dist[k];
    return s / 5.0;
}

double ThresholdHistory::window_std() const {
    const double mu = window_mean();
    double s = 0.0;
    for (size_t k = nn_dist.size() - 5; k < nn_dist.size(); ++k) s += (nn_dist[k] - mu) * (nn_dist[k] - mu);
    return std::sqrt(s / 5.0);
}

double next_threshold(const ThresholdHistory& h, ThresholdPhase phase, index_t min_len, double last_r,
                      bool failed) {
    double out = 0.0;
    const int rc = tsd_next_threshold(h.nn_dist.data(), (int64_t)h.nn_dist.size(),
                                      phase == ThresholdPhase::first ? 0 : phase == ThresholdPhase::warmup ? 1 : 2,
                                      min_len, last_r, failed ? 1 : 0, &out);
    if (rc != TSD_OK) rethrow(rc, tsd_last_error(nullptr));
    return out;
}

MerlinReport merlin_full(const TimeSeries& series, index_t min_len, index_t max_len,
                         const MerlinOptions& opts) {
    const index_t L = std::max<index_t>(max_len - min_len + 1, 1);
    const index_t k = std::max<index_t>(opts.top_k, 1);
    std::vector<int64_t> counts((size_t)L), retries((size_t)L);
    std::vector<tsd_record> recs((size_t)(L * k));
    std::vector<double> final_r((size_t)L);
    std::vector<uint8_t> failed((size_t)L);
    tsd_merlin_opts o{opts.top_k, opts.seglen, opts.workers, opts.max_retries, opts.reuse_stats ? 1 : 0};
    if (Group* g = group_for(opts.devices)) {
        g->series(series);
        g->check(tsd_group_merlin(g->g, min_len, max_len, &o, counts.data(), recs.data(), final_r.data(),
                                  retries.data(), failed.data()));
    } else {
        Ctx& c = ctx_for(opts.devices);
        c.series(series);
        c.check(tsd_merlin(c.c, min_len, max_len, &o, counts.data(), recs.data(), final_r.data(),
                           retries.data(), failed.data()));
    }
    MerlinReport rep;
    rep.discords.min_len = min_len;
    rep.discords.max_len = max_len;
    for (index_t i = 0; i < L; ++i) {
        const index_t m = min_len + i;
        rep.final_r.push_back(final_r[(size_t)i]);
        rep.retries.push_back((index_t)retries[(size_t)i]);
        if (failed[(size_t)i]) {
            rep.discords.failed_lengths.push_back(m);
            continue;
        }
        std::vector<DiscordRecord> lst;
        for (int64_t j = 0; j < counts[(size_t)i]; ++j) {
            const tsd_record& r = recs[(size_t)(i * k + j)];
            lst.push_back({(index_t)r.index, r.nn_dist_sq, r.nn_dist});
        }
        rep.discords.per_length[m] = std::move(lst);
    }
    return rep;
}

MultiLengthDiscordSet merlin(const TimeSeries& series, index_t min_len, index_t max_len,
                             const MerlinOptions& opts) {
    return merlin_full(series, min_len, max_len, opts).discords;
}

// ---- io -------------------------------------------------------------------------
std::string format_double(double value) {
    char buf[40];
    auto res = std::to_chars(buf, buf + sizeof(buf), value);
    return std::string(buf, res.ptr);
}

TimeSeries gen_randomwalk(index_t n, std::uint64_t seed) {
    if (n < 3) throw std::invalid_argument("gen_randomwalk: n must be at least 3");
    std::vector<double> v((size_t)n);
    const int rc = tsd_gen_randomwalk(n, seed, v.data());
    if (rc != TSD_OK) rethrow(rc, tsd_last_error(nullptr));
    return TimeSeries(std::move(v));
}

void write_series(const TimeSeries& series, std::ostream& out) {
    for (double v : series.values()) out << format_double(v) << '\n';
}

void write_discords_csv(const MultiLengthDiscordSet& d, std::ostream& out) {
    out << "length,index,nn_dist,nn_dist_sq,score\n";
    for (const auto& [m, lst] : d.per_length)
        for (const auto& r : lst)
            out << m << ',' << r.index << ',' << format_double(r.nn_dist) << ','
                << format_double(r.nn_dist_sq) << ','
                << format_double(r.nn_dist_sq / (2.0 * static_cast<double>(m))) << '\n';
}

namespace {
std::string strip(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && std::isspace((unsigned char)s[a])) ++a;
    while (b > a && std::isspace((unsigned char)s[b - 1])) --b;
    return s.substr(a, b - a);
}
bool to_double(const std::string& tok, double& out) {
    const std::string t = strip(tok);
    if (t.empty()) return false;
    auto res = std::from_chars(t.data(), t.data() + t.size(), out);
    return res.ec == std::errc() && res.ptr == t.data() + t.size();
}
std::vector<std::string> split_csv(const std::string& line) {
    std::vector<std::string> f;
    std::string cur;
    std::istringstream is(line);
    while (std::getline(is, cur, ',')) f.push_back(cur);
    if (!line.empty() && line.back() == ',') f.emplace_back();
    return f;
}
}  // namespace

MultiLengthDiscordSet read_discords_csv(std::istream& in) {
    // src/io.cpp:132-160: header "length,...", then length,index,nn_dist,nn_dist_sq[,score]
    MultiLengthDiscordSet set;
    std::string line;
    long lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (strip(line).empty()) continue;
        if (lineno == 1) {
            if (line.rfind("length,", 0) != 0) throw std::runtime_error("discord CSV: unexpected header '" + line + "'");
            continue;
        }
        const auto f = split_csv(line);
        if (f.size() < 4)
            throw std::runtime_error("discord CSV line " + std::to_string(lineno) + ": expected at least 4 fields");
        double m, idx, d, d2;
        if (!to_double(f[0], m) || !to_double(f[1], idx) || !to_double(f[2], d) || !to_double(f[3], d2))
            throw std::runtime_error("discord CSV line " + std::to_string(lineno) + ": non-numeric field");
        set.per_length[(index_t)m].push_back(DiscordRecord{(index_t)idx, d2, d});
    }
    if (!set.per_length.empty()) {
        set.min_len = set.per_length.begin()->first;
        set.max_len = set.per_length.rbegin()->first;
    }
    return set;
}

// ---- heatmap (reference: src/heatmap.cpp; built and ranked on the GPU) ---------
namespace {
// Generations are unique process-wide; each thread's context remembers which
// one its device matrix holds.  A Heatmap built on another thread (another
// context) therefore never matches and is uploaded before ranking.
std::atomic<std::uint64_t> g_heatmap_next{0};
std::uint64_t& resident_heatmap() {
    thread_local std::uint64_t g = 0;
    return g;
}
std::uint64_t new_heatmap_gen() {
    const std::uint64_t g = ++g_heatmap_next;
    resident_heatmap() = g;
    return g;
}
}  // namespace

Heatmap::Heatmap(index_t min_len, index_t max_len, index_t n) : min_len_(min_len), max_len_(max_len), n_(n) {
    if (min_len < 3 || min_len > max_len || max_len >= n) throw std::invalid_argument("heatmap: invalid length range");
    scores_.assign(static_cast<std::size_t>(rows() * cols()), 0.0);
}

Heatmap build_heatmap(const MultiLengthDiscordSet& discords, index_t n) {
    Heatmap h(discords.min_len, discords.max_len, n);
    std::vector<int64_t> lens;
    std::vector<tsd_record> recs;
    for (const auto& [m, lst] : discords.per_length)
        for (const auto& r : lst) {
            lens.push_back(m);
            recs.push_back(tsd_record{(int64_t)r.index, r.nn_dist_sq, r.nn_dist});
        }
    Ctx& c = ctx();
    c.check(tsd_heatmap_build(c.c, h.min_len(), h.max_len(), n, lens.data(), recs.data(), (int64_t)recs.size(),
                              h.mutable_scores().data()));
    h.set_device_gen(new_heatmap_gen());
    return h;
}

std::vector<RankedDiscord> rank_discords(const Heatmap& heatmap, index_t k) {
    if (k < 1) throw std::invalid_argument("rank_discords: k must be positive");
    Ctx& c = ctx();
    if (heatmap.device_gen() == 0 || heatmap.device_gen() != resident_heatmap()) {
        c.check(tsd_heatmap_set(c.c, heatmap.min_len(), heatmap.max_len(), heatmap.n(), heatmap.scores().data()));
        heatmap.set_device_gen(new_heatmap_gen());
    }
    std::vector<tsd_ranked> buf((size_t)std::min<index_t>(k, std::max<index_t>(heatmap.cols(), 1)));
    int64_t cnt = 0;
    c.check(tsd_heatmap_rank(c.c, k, buf.data(), &cnt));
    std::vector<RankedDiscord> out((size_t)cnt);
    for (int64_t e = 0; e < cnt; ++e) out[(size_t)e] = RankedDiscord{(index_t)buf[e].index, (index_t)buf[e].length, buf[e].score};
    return out;
}

void write_heatmap_csv(const Heatmap& h, std::ostream& out) {
    for (index_t m = h.min_len(); m <= h.max_len(); ++m) {
        for (index_t i = 1; i <= h.cols(); ++i) {
            if (i > 1) out << ',';
            out << format_double(h.score(m, i));
        }
        out << '\n';
    }
}

void write_heatmap_pgm(const Heatmap& h, std::ostream& out) {
    out << "P5\n" << h.cols() << ' ' << h.rows() << "\n255\n";
    for (index_t m = h.min_len(); m <= h.max_len(); ++m)
        for (index_t i = 1; i <= h.cols(); ++i) {
            const double v = std::clamp(h.score(m, i) / 2.0, 0.0, 1.0);
            out.put(static_cast<char>(static_cast<unsigned char>(std::lround(v * 255.0))));
        }
}

void write_ranking_csv(const std::vector<RankedDiscord>& ranking, std::ostream& out) {
    out << "rank,index,length,score\n";
    for (std::size_t r = 0; r < ranking.size(); ++r)
        out << (r + 1) << ',' << ranking[r].index << ',' << ranking[r].length << ',' << format_double(ranking[r].score)
            << '\n';
}

// load_series (src/io.cpp:48-104) with the reference's semantics and messages,
// parallel: the file is read once, split into lines, and the data lines are
// parsed by all host threads in contiguous chunks; the first error by line
// number is the one reported (the reference stops at it).
namespace {
std::string_view trim_ref(std::string_view s) {  // " \t\r" only, as src/io.cpp:24-29
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string_view::npos) return {};
    const auto e = s.find_last_not_of(" \t\r");
    return s.substr(b, e - b + 1);
}
bool parse_ref(std::string_view tok, double& out) {  // src/io.cpp:31-38
    const std::string_view t = trim_ref(tok);
    if (t.empty()) return false;
    auto res = std::from_chars(t.data(), t.data() + t.size(), out);
    return res.ec == std::errc() && res.ptr == t.data() + t.size();
}
// field f of a CSV line (split on ',', a trailing ',' adds an empty field);
// false when the line has fewer fields
bool csv_field(std::string_view line, long f, std::string_view& out) {
    size_t a = 0;
    for (long k = 0; k < f; ++k) {
        const size_t c = line.find(',', a);
        if (c == std::string_view::npos) return false;
        a = c + 1;
    }
    const size_t c = line.find(',', a);
    out = line.substr(a, c == std::string_view::npos ? std::string_view::npos : c - a);
    return true;
}
}  // namespace

TimeSeries load_series(const std::string& path, const std::string& column) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open input file: " + path);
    const std::string buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    // lines as std::getline splits them (no empty line after a final '\n')
    std::vector<std::string_view> lines;
    {
        size_t a = 0;
        while (a < buf.size()) {
            size_t e = buf.find('\n', a);
            if (e == std::string::npos) e = buf.size();
            lines.emplace_back(buf.data() + a, e - a);
            a = e + 1;
        }
    }
    // header / column resolution on the first non-blank line
    long col = column.empty() ? 0 : -1;
    size_t first = lines.size();
    for (size_t i = 0; i < lines.size(); ++i)
        if (!trim_ref(lines[i]).empty()) {
            first = i;
            break;
        }
    if (first < lines.size()) {
        std::string_view f0;
        csv_field(lines[first], 0, f0);
        double probe;
        if (!parse_ref(f0, probe)) {  // header row
            if (!column.empty()) {
                for (long f = 0;; ++f) {
                    std::string_view fv;
                    if (!csv_field(lines[first], f, fv)) break;
                    if (trim_ref(fv) == column) col = f;
                }
                if (col < 0) {
                    double idx;
                    if (parse_ref(column, idx)) col = static_cast<long>(idx);
                    else throw std::runtime_error("column '" + column + "' not found in header");
                }
            }
            ++first;
        } else if (!column.empty()) {
            double idx;
            if (!parse_ref(column, idx))
                throw std::runtime_error("column '" + column + "' requested but file has no header");
            col = static_cast<long>(idx);
        }
    }
    // parallel parse of lines [first, end)
    const size_t total = lines.size() > first ? lines.size() - first : 0;
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    const size_t nchunk = std::max<size_t>(1, std::min<size_t>(hc, total / 65536 + 1));
    struct Chunk {
        std::vector<double> v;
        size_t err_line = SIZE_MAX;
        std::string err;
    };
    std::vector<Chunk> ch(nchunk);
    auto work = [&](size_t c) {
        const size_t lo = first + total * c / nchunk, hi = first + total * (c + 1) / nchunk;
        Chunk& k = ch[c];
        k.v.reserve(hi - lo);
        for (size_t i = lo; i < hi; ++i) {
            const std::string_view line = lines[i];
            if (trim_ref(line).empty()) continue;
            std::string_view fv;
            if (!csv_field(line, col, fv)) {
                k.err_line = i;
                k.err = "line " + std::to_string(i + 1) + ": missing column " + std::to_string(col);
                return;
            }
            double v;
            if (!parse_ref(fv, v)) {
                k.err_line = i;
                k.err = "line " + std::to_string(i + 1) + ": non-numeric value '" + std::string(trim_ref(fv)) + "'";
                return;
            }
            k.v.push_back(v);
        }
    };
    if (nchunk == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (size_t c = 0; c < nchunk; ++c) th.emplace_back(work, c);
        for (auto& t : th) t.join();
    }
    std::vector<double> values;
    values.reserve(total);
    for (const Chunk& k : ch) {
        if (k.err_line != SIZE_MAX) throw std::runtime_error(k.err);
        values.insert(values.end(), k.v.begin(), k.v.end());
    }
    if (values.size() < 3)
        throw std::runtime_error("series too short: need at least 3 values, got " + std::to_string(values.size()));
    return TimeSeries(std::move(values));
}

}  // namespace tsdiscord
