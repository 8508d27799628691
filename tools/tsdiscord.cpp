// tsdiscord — command-line front end of the B200 library.
//
// Same subcommands, options, outputs and exit codes as the reference CLI
// (/root/reference/proj/tools/main.cpp:184-236), with its own option parser
// (the reference's CLI11 is not vendored):
//   gen-rw        --n N [--seed S] --output PATH
//   discover      --input PATH [--column C] --minl A --maxl B [--topk K] [--seglen L]
//                 [--workers W] --output PATH                     (exit 1 if a length failed)
//   oracle-check  --input PATH [--column C] --minl A --maxl B [--topk K] [--discords CSV]
//   heatmap       --input DISCORDS_CSV --n N --output PREFIX
//   bench         --minl A --maxl B [--topk K] [--seed S] [--sweep-n a,b] [--sweep-seglen ..]
//                 [--sweep-workers ..] [--sweep-width ..] --output PATH
// Discovery runs on the GPU (device $TSD_DEVICE, default 0); --workers is
// accepted and ignored, as in the C-ABI.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsdiscord/drag.hpp"
#include "tsdiscord/heatmap.hpp"
#include "tsdiscord/io.hpp"
#include "tsdiscord/merlin.hpp"

using namespace tsdiscord;

namespace {

using Clock = std::chrono::steady_clock;

struct Args {
    std::string sub;
    std::map<std::string, std::string> opt;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string str(const std::string& k, const std::string& d = "") const {
        auto it = opt.find(k);
        return it == opt.end() ? d : it->second;
    }
    long long num(const std::string& k, long long d) const {
        auto it = opt.find(k);
        if (it == opt.end()) return d;
        size_t pos = 0;
        const long long v = std::stoll(it->second, &pos);
        if (pos != it->second.size()) throw std::invalid_argument("--" + k + ": not an integer");
        return v;
    }
    std::vector<long long> list(const std::string& k) const {
        std::vector<long long> out;
        const std::string s = str(k);
        size_t a = 0;
        while (a < s.size()) {
            size_t b = s.find(',', a);
            if (b == std::string::npos) b = s.size();
            out.push_back(std::stoll(s.substr(a, b - a)));
            a = b + 1;
        }
        return out;
    }
};

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

Args parse(int argc, char** argv, const std::map<std::string, std::vector<std::string>>& known,
           const std::map<std::string, std::vector<std::string>>& required) {
    if (argc < 2) throw Usage("a subcommand is required: gen-rw, discover, oracle-check, heatmap, bench");
    Args a;
    a.sub = argv[1];
    auto it = known.find(a.sub);
    if (it == known.end()) throw Usage("unknown subcommand: " + a.sub);
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) throw Usage("unexpected argument: " + k);
        k = k.substr(2);
        std::string v;
        const size_t eq = k.find('=');
        if (eq != std::string::npos) {
            v = k.substr(eq + 1);
            k = k.substr(0, eq);
        } else {
            if (i + 1 >= argc) throw Usage("--" + k + " needs a value");
            v = argv[++i];
        }
        bool ok = false;
        for (const auto& o : it->second) ok = ok || o == k;
        if (!ok) throw Usage("unknown option for " + a.sub + ": --" + k);
        a.opt[k] = v;
    }
    for (const auto& r : required.at(a.sub))
        if (!a.has(r)) throw Usage("--" + r + " is required");
    return a;
}

std::ofstream open_output(const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open output file: " + path);
    return out;
}

MerlinOptions options(const Args& a) {
    MerlinOptions o;
    o.top_k = a.num("topk", 1);
    o.seglen = a.num("seglen", 512);
    o.workers = a.num("workers", 1);
    return o;
}

double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }

int discover(const Args& a) {
    const TimeSeries s = load_series(a.str("input"), a.str("column"));
    const auto t0 = Clock::now();
    const MultiLengthDiscordSet d = merlin(s, a.num("minl", 0), a.num("maxl", 0), options(a));
    const double el = since(t0);
    auto out = open_output(a.str("output"));
    write_discords_csv(d, out);
    for (const auto& [m, recs] : d.per_length) std::cout << "length " << m << ": " << recs.size() << " discord(s)\n";
    for (index_t m : d.failed_lengths) std::cout << "length " << m << ": FAILED (threshold retries exhausted)\n";
    std::cout << "wall time: " << el << " s\n";
    return d.failed_lengths.empty() ? 0 : 1;
}

int oracle_check(const Args& a) {
    const TimeSeries s = load_series(a.str("input"), a.str("column"));
    if (s.n() > 5000) throw std::runtime_error("oracle-check: series too long (guard is n <= 5000)");
    const index_t lo = a.num("minl", 0), hi = a.num("maxl", 0), k = a.num("topk", 1);
    MultiLengthDiscordSet got;
    if (a.has("discords")) {
        std::ifstream in(a.str("discords"));
        if (!in) throw std::runtime_error("cannot open discord file: " + a.str("discords"));
        got = read_discords_csv(in);
    } else {
        got = merlin(s, lo, hi, options(a));
    }
    bool all = true;
    for (index_t m = lo; m <= hi; ++m) {
        const auto exp = brute_force_topk(s, m, k);
        const auto it = got.per_length.find(m);
        double worst = 0.0;
        bool pass = it != got.per_length.end() && it->second.size() == exp.size();
        for (size_t j = 0; pass && j < exp.size(); ++j) {
            if (it->second[j].index != exp[j].index) pass = false;
            worst = std::max(worst, std::abs(it->second[j].nn_dist - exp[j].nn_dist) / std::max(exp[j].nn_dist, 1e-300));
        }
        if (worst > 1e-7) pass = false;
        std::cout << "length " << m << ": " << (pass ? "PASS" : "FAIL") << " (max nn_dist discrepancy " << worst
                  << ")\n";
        all = all && pass;
    }
    return all ? 0 : 1;
}

int heatmap(const Args& a) {
    std::ifstream in(a.str("input"));
    if (!in) throw std::runtime_error("cannot open discord file: " + a.str("input"));
    const MultiLengthDiscordSet d = read_discords_csv(in);
    if (d.per_length.empty()) throw std::runtime_error("discord file contains no records; nothing to plot");
    const Heatmap h = build_heatmap(d, a.num("n", 0));
    const std::string p = a.str("output");
    {
        auto o = open_output(p + "_heatmap.csv");
        write_heatmap_csv(h, o);
    }
    {
        auto o = open_output(p + "_heatmap.pgm");
        write_heatmap_pgm(h, o);
    }
    {
        auto o = open_output(p + "_ranking.csv");
        write_ranking_csv(rank_discords(h, 10), o);
    }
    std::cout << "heatmap: " << h.rows() << " x " << h.cols() << "\n";
    return 0;
}

int bench(const Args& a) {
    auto out = open_output(a.str("output"));
    out << "axis,n,min_len,max_len,seglen,workers,wall_s,discords,s_per_discord\n";
    const std::uint64_t seed = (std::uint64_t)a.num("seed", 0);
    const index_t lo = a.num("minl", 0), hi = a.num("maxl", 0), seglen = a.num("seglen", 512);
    const index_t workers = a.num("workers", 1), topk = a.num("topk", 1);
    const auto ns = a.list("sweep-n");
    const index_t n0 = ns.empty() ? 100000 : ns.front();
    auto row = [&](const char* axis, index_t n, index_t l, index_t h, index_t sl, index_t w) {
        const TimeSeries s = gen_randomwalk(n, seed);
        MerlinOptions o;
        o.top_k = topk;
        o.seglen = sl;
        o.workers = w;
        const auto t0 = Clock::now();
        const auto d = merlin(s, l, h, o);
        const double el = since(t0);
        size_t found = 0;
        for (const auto& [m, r] : d.per_length) found += r.size();
        out << axis << ',' << n << ',' << l << ',' << h << ',' << sl << ',' << w << ',' << el << ',' << found << ','
            << (found ? el / (double)found : 0.0) << '\n';
        std::cout << axis << " n=" << n << " range=[" << l << ',' << h << "] seglen=" << sl << " workers=" << w
                  << ": " << el << " s\n";
    };
    for (long long n : ns) row("n", n, lo, hi, seglen, workers);
    for (long long w : a.list("sweep-width")) row("range", n0, lo, lo + w - 1, seglen, workers);
    for (long long s : a.list("sweep-seglen")) row("seglen", n0, lo, hi, s, workers);
    for (long long w : a.list("sweep-workers")) row("workers", n0, lo, hi, seglen, w);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const std::map<std::string, std::vector<std::string>> known = {
        {"gen-rw", {"n", "seed", "output"}},
        {"discover", {"input", "column", "minl", "maxl", "topk", "seglen", "workers", "output"}},
        {"oracle-check", {"input", "column", "minl", "maxl", "topk", "seglen", "workers", "discords"}},
        {"heatmap", {"input", "n", "output"}},
        {"bench", {"minl", "maxl", "topk", "seglen", "workers", "seed", "sweep-n", "sweep-seglen", "sweep-workers",
                   "sweep-width", "output"}}};
    const std::map<std::string, std::vector<std::string>> required = {
        {"gen-rw", {"n", "output"}},
        {"discover", {"input", "minl", "maxl", "output"}},
        {"oracle-check", {"input", "minl", "maxl"}},
        {"heatmap", {"input", "n", "output"}},
        {"bench", {"minl", "maxl", "output"}}};
    Args a;
    try {
        a = parse(argc, argv, known, required);
    } catch (const std::exception& e) {
        std::cerr << e.what() << "\nRun with a subcommand: gen-rw | discover | oracle-check | heatmap | bench\n";
        return 106;  // CLI11's parse-error exit code
    }
    try {
        if (a.sub == "gen-rw") {
            const TimeSeries s = gen_randomwalk(a.num("n", 0), (std::uint64_t)a.num("seed", 0));
            auto out = open_output(a.str("output"));
            write_series(s, out);
            return 0;
        }
        if (a.sub == "discover") return discover(a);
        if (a.sub == "oracle-check") return oracle_check(a);
        if (a.sub == "heatmap") return heatmap(a);
        if (a.sub == "bench") return bench(a);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
    return 0;
}
