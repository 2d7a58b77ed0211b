// search.cpp — the host side of the hot path: knob-space encoding, the
// Ansor-style sampler, sharded batch measurement with an all-gather, best-of-N
// and Droplet Search.  Host-only C++; the GPU measurer lives in harness.cu.
//
// Paper: Def. 2.1, Example 2.3, neighbourhood
// (P:290-294), Droplet Search, combined approach,
// Droplet cap of 100 trials.  Readings R-xx: DESIGN.md §3.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <unordered_set>

#include "internal.hpp"
#include "nvtx.hpp"

namespace db200 {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
tuner_status fail(tuner_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

// ---------------------------------------------------------------- encoding (R-T1)
uint64_t Tuner::linear(const Pt& p) const {
    const SketchSpace& s = spaces[p.pos];
    uint64_t lin = 0;
    for (int d = 0; d < s.nknobs(); ++d) lin = lin * s.values[d].size() + (uint64_t)p.idx[d];
    return s.offset + lin;
}

Pt Tuner::from_public(const tuner_point& tp, tuner_status& st) const {
    Pt p;
    st = TUNER_OK;
    int pos = -1;
    for (size_t i = 0; i < spaces.size(); ++i)
        if (spaces[i].sketch == tp.sketch) { pos = (int)i; break; }
    if (pos < 0) { st = fail(TUNER_ERANGE, "point's sketch is not in this tuner's spaces"); return p; }
    const SketchSpace& s = spaces[pos];
    if (tp.n != s.nknobs()) { st = fail(TUNER_EDIM, "index vector length != number of knobs"); return p; }
    p.pos = pos;
    p.n = tp.n;
    for (int d = 0; d < tp.n; ++d) {
        if (tp.idx[d] < 0 || tp.idx[d] >= (int32_t)s.values[d].size()) {
            st = fail(TUNER_ERANGE, "index out of range");
            return p;
        }
        p.idx[d] = tp.idx[d];
    }
    return p;
}

tuner_point Tuner::to_public(const Pt& p) const {
    tuner_point tp;
    std::memset(&tp, 0, sizeof(tp));
    tp.sketch = spaces[p.pos].sketch;
    tp.n = p.n;
    for (int d = 0; d < p.n; ++d) tp.idx[d] = p.idx[d];
    return tp;
}

void Tuner::values_of(const Pt& p, int32_t* v) const {
    const SketchSpace& s = spaces[p.pos];
    for (int d = 0; d < p.n; ++d) v[d] = s.values[d][p.idx[d]];
}

// Neighbourhood: one index step along one coordinate; no diagonals
// (R-D7); out-of-range skipped, no wrap (R-D6); dimension-major, minus before
// plus (R-D3).
// the +-r axis-aligned ring (r = 1: the neighbourhood of P:292-294; r > 1: R-D16), dimension-
// major, minus before plus, out-of-range indices skipped
void Tuner::ring(const Pt& x, std::vector<Pt>& out, int r) const {
    out.clear();
    const SketchSpace& s = spaces[x.pos];
    for (int d = 0; d < x.n; ++d) {
        for (int delta = -r; delta <= r; delta += 2 * r) {
            int i = x.idx[d] + delta;
            if (i < 0 || i >= (int)s.values[d].size()) continue;
            Pt q = x;
            q.idx[d] = i;
            out.push_back(q);
        }
    }
}

// ---------------------------------------------------------------- sharded measurement (R-M1)
namespace {
struct Slot {  // 96 bytes, keyed by batch index so results are rank-independent
    int32_t idx;
    int32_t status;
    double cost_ns;
    double max_err;
    int32_t rank;
    int32_t nsamp;
    float samp[kMaxSamples];
};
static_assert(sizeof(Slot) == 96, "slot layout");
}  // namespace

static void slot_from(Slot& d, int32_t idx, int32_t rank, const Result& r) {
    std::memset(&d, 0, sizeof(Slot));
    d.idx = idx;
    d.rank = rank;
    d.status = r.status;
    d.cost_ns = r.cost_ns;
    d.max_err = r.max_err;
    d.nsamp = r.nsamp;
    std::memcpy(d.samp, r.samp, sizeof(d.samp));
}
static void result_from(Result& x, const Slot& s) {
    x.cost_ns = s.cost_ns;
    x.max_err = s.max_err;
    x.status = s.status;
    x.rank = s.rank;
    x.nsamp = s.nsamp < 0 ? 0 : (s.nsamp > kMaxSamples ? kMaxSamples : s.nsamp);
    std::memcpy(x.samp, s.samp, sizeof(x.samp));
}
static constexpr int32_t kSlotError = -2;  // a slot carrying a rank's failure (status = the error)

tuner_status Tuner::measure_batch(const std::vector<Pt>& batch) {
    if (batch.empty()) return TUNER_OK;
    NvtxRange nv("measure_batch");
    auto t0 = std::chrono::steady_clock::now();
    const int G = opts.world > 1 ? opts.world : 1;
    const int r = opts.world > 1 ? opts.rank : 0;
    std::vector<Pt> local;
    std::vector<int32_t> local_idx;
    for (size_t j = r; j < batch.size(); j += G) {
        local.push_back(batch[j]);
        local_idx.push_back((int32_t)j);
    }
    std::vector<Result> lres;
    const int64_t launches0 = g_launch_counter_ptr()->load();
    tuner_status st = measurer->measure(local, lres, best_cost, true);
    stats.kernel_launches += g_launch_counter_ptr()->load() - launches0;
    for (auto& x : lres) x.rank = r;
    std::vector<Result> res(batch.size());
    if (!comm) {
        if (st != TUNER_OK) return st;
        res = lres;
    } else {
        // every rank takes part in the all-gather even after a local failure (its slot 0
        // then carries the error), so a failing rank never leaves the others blocked
        const size_t per = (batch.size() + G - 1) / G;
        std::vector<Slot> send(per), recv(per * G);
        for (size_t i = 0; i < per; ++i) {
            std::memset(&send[i], 0, sizeof(Slot));
            send[i].idx = -1;
            send[i].rank = r;
            if (st == TUNER_OK && i < lres.size()) slot_from(send[i], local_idx[i], r, lres[i]);
        }
        if (st != TUNER_OK) {
            send[0].idx = kSlotError;
            send[0].status = st;
        }
        tuner_status cs = comm->allgather(send.data(), recv.data(), (int64_t)(per * sizeof(Slot)));
        if (st != TUNER_OK) return st;
        if (cs != TUNER_OK) return cs;
        stats.collectives++;
        size_t filled = 0;
        for (const Slot& s : recv) {
            if (s.idx == kSlotError) return fail((tuner_status)s.status, "another rank failed while measuring");
            if (s.idx < 0) continue;
            if ((size_t)s.idx >= batch.size()) return fail(TUNER_ENCCL, "corrupt all-gather slot");
            result_from(res[s.idx], s);
            ++filled;
        }
        if (filled != batch.size()) return fail(TUNER_ENCCL, "all-gather returned an incomplete batch");
        if (G > 1 && !table_mode && (st = calibrate(batch, res)) != TUNER_OK) return st;
    }
    for (size_t j = 0; j < batch.size(); ++j) {
        tuner_result smp;
        std::memset(&smp, 0, sizeof(smp));
        smp.pt = to_public(batch[j]);
        smp.status = res[j].status;
        smp.cost_ns = res[j].status == TUNER_S_OK ? res[j].cost_ns : INFINITY;
        smp.max_err = res[j].max_err;
        smp.rank = res[j].rank;
        record(batch[j], smp, std::vector<float>(res[j].samp, res[j].samp + res[j].nsamp), true);
    }
    stats.candidates += (int64_t)batch.size();
    stats.batches++;
    stats.measure_wall_ns +=
        std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
    return TUNER_OK;
}

// Per-GPU calibration ("a winner found on rank r is re-timed on rank 0 before
// acceptance"): the batch's first argmin, when it beats the incumbent and was timed on another
// rank, is re-timed on rank 0 (with the precise tier) and rank 0's cost replaces it; repeated,
// at most kCalibrations times per batch, while the new argmin is another such winner.  So every
// incumbent's cost -- every point Droplet or best-of-N accepts -- is a rank-0 cost, and no GPU's
// bias decides an acceptance.  The re-timing result travels in one all-gather (rank 0's slot).
tuner_status Tuner::calibrate(const std::vector<Pt>& batch, std::vector<Result>& res) {
    static constexpr int kCalibrations = 4;
    const int G = opts.world;
    std::vector<char> done(batch.size(), 0);
    for (int it = 0; it < kCalibrations; ++it) {
        size_t js = batch.size();
        for (size_t j = 0; j < batch.size(); ++j)
            if (res[j].status == TUNER_S_OK && (js == batch.size() || res[j].cost_ns < res[js].cost_ns)) js = j;
        if (js == batch.size() || !(res[js].cost_ns < best_cost) || res[js].rank == 0 || done[js]) break;
        done[js] = 1;
        Slot send;
        std::memset(&send, 0, sizeof(send));
        send.idx = -1;
        if (opts.rank == 0) {
            std::vector<Result> rr;
            tuner_status ms = measurer->measure(std::vector<Pt>{batch[js]}, rr, best_cost, false);
            if (ms == TUNER_OK) {
                slot_from(send, (int32_t)js, 0, rr[0]);
            } else {
                send.idx = kSlotError;
                send.status = ms;
            }
        }
        std::vector<Slot> recv(G);
        tuner_status cs = comm->allgather(&send, recv.data(), (int64_t)sizeof(Slot));
        if (cs != TUNER_OK) return cs;
        stats.collectives++;
        if (recv[0].idx == kSlotError) return fail((tuner_status)recv[0].status, "rank 0 failed re-timing a winner");
        if (recv[0].idx != (int32_t)js) return fail(TUNER_ENCCL, "corrupt calibration slot");
        result_from(res[js], recv[0]);
        stats.calibrations++;
    }
    return TUNER_OK;
}

// Append one measured (or replayed) point to the history and the memo; log it (rank 0).
void Tuner::record(const Pt& p, const tuner_result& smp, std::vector<float>&& samples, bool log) {
    memo[linear(p)] = history.size();
    history.push_back(smp);
    hsamples.push_back(std::move(samples));
    if (smp.cost_ns < best_cost) best_cost = smp.cost_ns;
    if (log && trial_log && opts.rank == 0) log_trial(p, smp, hsamples.back());
}

// ---------------------------------------------------------------- trial log
// One JSON object per line:
//   {"key":"<op/shape/dtype>","sketch":S,"vals":[v0,...],"cost_ns":C|null,"max_err":E,"status":s,
//    "rank":r,"samp":[t0,...]}
// Knob VALUES (not indices) are logged, so a log replays into a tuner whose value lists differ;
// lines of another problem or sketch, or with a value outside this tuner's lists, are skipped.
static std::string problem_key(int32_t op, const tuner_shape& s) {
    char buf[320];
    std::snprintf(buf, sizeof buf,
                  "op%d/dt%d/b%lld/m%lld/n%lld/k%lld/N%lld/C%lld/H%lld/W%lld/K%lld/R%lld/S%lld/st%d.%d/pd%d.%d/dl%d.%d",
                  op, s.dtype, (long long)s.b, (long long)s.m, (long long)s.n, (long long)s.k, (long long)s.N,
                  (long long)s.C, (long long)s.H, (long long)s.W, (long long)s.K, (long long)s.R, (long long)s.S,
                  s.stride_h, s.stride_w, s.pad_h, s.pad_w, s.dil_h, s.dil_w);
    return buf;
}

void Tuner::log_trial(const Pt& p, const tuner_result& smp, const std::vector<float>& samples) {
    int32_t v[TUNER_MAX_KNOBS];
    values_of(p, v);
    std::string line = "{\"key\":\"" + key + "\",\"sketch\":" + std::to_string(spaces[p.pos].sketch) + ",\"vals\":[";
    for (int d = 0; d < p.n; ++d) line += (d ? "," : "") + std::to_string(v[d]);
    char num[64];
    line += "],\"cost_ns\":";
    if (std::isfinite(smp.cost_ns)) {
        std::snprintf(num, sizeof num, "%.17g", smp.cost_ns);
        line += num;
    } else {
        line += "null";
    }
    std::snprintf(num, sizeof num, "%.9g", smp.max_err);
    line += ",\"max_err\":" + std::string(num) + ",\"status\":" + std::to_string(smp.status) +
            ",\"rank\":" + std::to_string(smp.rank) + ",\"samp\":[";
    for (size_t i = 0; i < samples.size(); ++i) {
        std::snprintf(num, sizeof num, "%.9g", (double)samples[i]);
        line += (i ? "," : "") + std::string(num);
    }
    line += "]}\n";
    std::fwrite(line.data(), 1, line.size(), trial_log);
    std::fflush(trial_log);
}

// the numbers of a JSON array "[a,b,...]" starting at p (after the '['); returns past ']'
static const char* parse_array(const char* p, std::vector<double>& out) {
    out.clear();
    while (*p == ' ') ++p;
    if (*p == ']') return p + 1;
    for (;;) {
        char* e = nullptr;
        const double x = std::strtod(p, &e);
        if (e == p) return nullptr;
        out.push_back(x);
        p = e;
        while (*p == ' ') ++p;
        if (*p == ']') return p + 1;
        if (*p != ',') return nullptr;
        ++p;
    }
}
static const char* field(const char* line, const char* name) {
    const char* f = std::strstr(line, name);
    return f ? f + std::strlen(name) : nullptr;
}

tuner_status Tuner::replay_log(const char* path) {
    std::FILE* f = std::fopen(path, "r");
    if (!f) return TUNER_OK;  // no log yet: a fresh job
    std::string line;
    char buf[4096];
    int64_t lineno = 0;
    tuner_status st = TUNER_OK;
    std::vector<double> vals, samp;
    while (st == TUNER_OK && std::fgets(buf, sizeof buf, f)) {
        line.assign(buf);
        while (!line.empty() && line.back() != '\n' && std::fgets(buf, sizeof buf, f)) line += buf;
        ++lineno;
        if (line.find_first_not_of(" \t\r\n") == std::string::npos) continue;
        const char* L = line.c_str();
        const char* k = field(L, "\"key\":\"");
        const char* sk = field(L, "\"sketch\":");
        const char* va = field(L, "\"vals\":[");
        const char* co = field(L, "\"cost_ns\":");
        const char* me = field(L, "\"max_err\":");
        const char* ss = field(L, "\"status\":");
        const char* rk = field(L, "\"rank\":");
        const char* sa = field(L, "\"samp\":[");
        if (!k || !sk || !va || !co || !me || !ss || !rk || !sa || !parse_array(va, vals) || !parse_array(sa, samp)) {
            st = fail(TUNER_EINVAL, std::string("malformed trial-log line ") + std::to_string(lineno) + " in " + path);
            break;
        }
        if (std::strncmp(k, key.c_str(), key.size()) != 0 || k[key.size()] != '"') continue;  // another problem
        const int32_t sketch = (int32_t)std::strtol(sk, nullptr, 10);
        int pos = -1;
        for (size_t i = 0; i < spaces.size(); ++i)
            if (spaces[i].sketch == sketch) pos = (int)i;
        if (pos < 0 || (int)vals.size() != spaces[pos].nknobs()) continue;  // a sketch this tuner does not search
        Pt p;
        p.pos = pos;
        p.n = spaces[pos].nknobs();
        bool ok = true;
        for (int d = 0; d < p.n && ok; ++d) {
            const auto& vl = spaces[pos].values[d];
            auto it = std::find(vl.begin(), vl.end(), (int32_t)vals[d]);
            ok = it != vl.end();
            if (ok) p.idx[d] = (int32_t)(it - vl.begin());
        }
        if (!ok || measured(p)) continue;
        tuner_result smp;
        std::memset(&smp, 0, sizeof(smp));
        smp.pt = to_public(p);
        smp.cost_ns = std::strncmp(co, "null", 4) == 0 ? INFINITY : std::strtod(co, nullptr);
        smp.max_err = std::strtod(me, nullptr);
        smp.status = (int32_t)std::strtol(ss, nullptr, 10);
        smp.rank = (int32_t)std::strtol(rk, nullptr, 10);
        if (smp.status != TUNER_S_OK) smp.cost_ns = INFINITY;
        std::vector<float> fs(samp.begin(), samp.end());
        if (fs.size() > (size_t)kMaxSamples) fs.resize(kMaxSamples);
        record(p, smp, std::move(fs), false);
        stats.replayed++;
    }
    std::fclose(f);
    return st;
}

// ---------------------------------------------------------------- sampler (R-S1)
tuner_status Tuner::draw(int32_t n, std::vector<Pt>& out) {
    out.clear();
    std::unordered_set<uint64_t> taken;
    int64_t attempts = 0;
    const int64_t cap = 64ll * n;
    while ((int32_t)out.size() < n && attempts < cap) {
        ++attempts;
        Pt p;
        p.pos = (int32_t)rng.uniform((uint32_t)spaces.size());
        const SketchSpace& s = spaces[p.pos];
        p.n = s.nknobs();
        for (int d = 0; d < p.n; ++d) p.idx[d] = (int32_t)rng.uniform((uint32_t)s.values[d].size());
        if (!valid(p)) continue;
        uint64_t id = linear(p);
        if (memo.count(id) || taken.count(id)) continue;
        taken.insert(id);
        out.push_back(p);
    }
    return TUNER_OK;
}

tuner_status Tuner::measure_chunked(const std::vector<Pt>& pts) {
    for (size_t i = 0; i < pts.size(); i += (size_t)opts.max_batch) {
        size_t e = std::min(pts.size(), i + (size_t)opts.max_batch);
        tuner_status st = measure_batch(std::vector<Pt>(pts.begin() + i, pts.begin() + e));
        if (st != TUNER_OK) return st;
    }
    return TUNER_OK;
}

// ---------------------------------------------------------------- grid search
// AutoTVM's grid search as an exploitation alternative (RQ4): the next n
// statically valid, unmeasured points in enumeration order (union linear id: sketch
// order, then row-major, last knob fastest), from a cursor kept across calls.
void Tuner::grid(int32_t n, std::vector<Pt>& out) {
    out.clear();
    const uint64_t end = spaces.back().offset + spaces.back().size;
    while ((int32_t)out.size() < n && grid_cursor < end) {
        const uint64_t id = grid_cursor++;
        Pt p;
        while (p.pos + 1 < (int32_t)spaces.size() && id >= spaces[p.pos + 1].offset) ++p.pos;
        const SketchSpace& s = spaces[p.pos];
        p.n = s.nknobs();
        uint64_t rem = id - s.offset;
        for (int d = p.n - 1; d >= 0; --d) {
            const uint64_t card = s.values[d].size();
            p.idx[d] = (int32_t)(rem % card);
            rem /= card;
        }
        if (memo.count(id) || !valid(p)) continue;
        out.push_back(p);
    }
}

// ---------------------------------------------------------------- evolutionary exploration
// Ansor's evolution of annotated sketches without the learned cost
// model (every child is measured), R-E1: generation 0 = the sampler; then each
// generation draws children from the `elite` best measured points (cost, then
// measurement order): a = parent[u(E)]; if u(2) == 1, b = parent[u(E)] and, when b
// has a's sketch, each knob takes b's index if u(2) == 1; then one knob d = u(nknobs)
// is resampled, child[d] = u(card_d).  Children must be valid, unmeasured and new in
// their generation (<= 64*pop attempts); an empty generation ends the run.
tuner_status Tuner::evolve(int32_t n, int32_t pop, int32_t elite, std::vector<Pt>& out) {
    out.clear();
    std::vector<Pt> gen;
    bool any_finite = false;
    for (const auto& h : history) any_finite |= std::isfinite(h.cost_ns);
    tuner_status st = TUNER_OK;
    if (!any_finite) {  // a fresh tuner: generation 0 (else continue from the elite)
        draw(std::min(pop, n), gen);
        if ((st = measure_chunked(gen)) != TUNER_OK) return st;
    }
    out = gen;
    int32_t used = (int32_t)gen.size();
    while (used < n) {
        std::vector<std::pair<double, size_t>> ranked;
        for (size_t i = 0; i < history.size(); ++i)
            if (std::isfinite(history[i].cost_ns)) ranked.emplace_back(history[i].cost_ns, i);
        std::sort(ranked.begin(), ranked.end());
        std::vector<Pt> parents;
        for (size_t i = 0; i < ranked.size() && (int32_t)parents.size() < elite; ++i) {
            tuner_status s2;
            parents.push_back(from_public(history[ranked[i].second].pt, s2));
        }
        if (parents.empty()) break;
        const int32_t want = std::min(pop, n - used);
        const uint32_t E = (uint32_t)parents.size();
        gen.clear();
        std::unordered_set<uint64_t> taken;
        for (int64_t attempts = 0; (int32_t)gen.size() < want && attempts < 64ll * pop; ++attempts) {
            const Pt& a = parents[rng.uniform(E)];
            Pt child = a;
            if (rng.uniform(2) == 1) {
                const Pt& b = parents[rng.uniform(E)];
                if (b.pos == a.pos)
                    for (int d = 0; d < child.n; ++d)
                        if (rng.uniform(2) == 1) child.idx[d] = b.idx[d];
            }
            const SketchSpace& sp = spaces[a.pos];
            if (sp.nknobs() > 0) {
                const int d = (int)rng.uniform((uint32_t)sp.nknobs());
                child.idx[d] = (int32_t)rng.uniform((uint32_t)sp.values[d].size());
            }
            if (!valid(child)) continue;
            const uint64_t id = linear(child);
            if (memo.count(id) || taken.count(id)) continue;
            taken.insert(id);
            gen.push_back(child);
        }
        if (gen.empty()) break;
        if ((st = measure_chunked(gen)) != TUNER_OK) return st;
        out.insert(out.end(), gen.begin(), gen.end());
        used += (int32_t)gen.size();
    }
    return TUNER_OK;
}

// ---------------------------------------------------------------- Droplet Search
// P:297-304.  Step 2(a) "If there exists c_i' ... yields a faster kernel ...
// update the current best": the whole ring is measured as one batch and the
// first strictly better argmin in ring order is taken (R-D2, R-D3, R-D4).
// Step 2(b) "If there is no such c_i', then the search terminates."
// GROW (R-D9): after a ring move along u, probe x_prev + 2^j u (j >= 1, clamped
// until the clamp repeats) as one batch; accept ray points in order while each
// is strictly better.  Budget counts new measurements incl. an unmeasured
// start (R-D14); a truncated batch ends the search unconverged (R-D13).
tuner_status Tuner::droplet(const Pt& start, int32_t budget, std::vector<Pt>& traj,
                            tuner_droplet_report& rep) {
    int32_t used = 0, rounds = 0;
    tuner_status st;
    if (!measured(start)) {
        st = measure_batch(std::vector<Pt>{start});
        if (st != TUNER_OK) return st;
        used = 1;
    }
    Pt x = start;
    double c = cost(x);
    traj.assign(1, x);
    auto finish = [&](bool converged) {
        std::memset(&rep, 0, sizeof(rep));
        rep.best = to_public(x);
        rep.best_cost = c;
        rep.trials_used = used;
        rep.rounds = rounds;
        rep.converged = converged ? 1 : 0;
        rep.traj_len = (int32_t)traj.size();
        return TUNER_OK;
    };
    // "yields a faster kernel": strictly lower cost (R-D4) and, with alpha > 0, a
    // significant difference of the repeat timings (Wilcoxon rank-sum p < alpha, R-W1)
    auto better = [&](const Pt& p, const Pt& q) {
        const size_t ip = memo.at(linear(p)), iq = memo.at(linear(q));
        if (!(history[ip].cost_ns < history[iq].cost_ns)) return false;
        if (opts.alpha <= 0.0) return true;
        const auto& a = hsamples[ip];
        const auto& b = hsamples[iq];
        return wilcoxon_p(a.data(), (int)a.size(), b.data(), (int)b.size()) < opts.alpha;
    };
    // the not-yet-measured valid points of `cands`, truncated to the budget left
    auto fresh = [&](const std::vector<Pt>& cands, std::vector<Pt>& q) {
        q.clear();
        size_t n = 0;
        for (const Pt& p : cands) {
            if (measured(p) || !valid(p)) continue;
            ++n;
            if ((int32_t)q.size() < budget - used) q.push_back(p);
        }
        return n > q.size();
    };
    std::vector<Pt> nb, q, ray;
    int r = 1;  // ring radius (RADIUS policy, R-D16)
    for (;;) {
        NvtxRange nv("droplet_round");
        ring(x, nb, r);
        if (r > 1 && nb.empty()) return finish(true);  // every axis line of x examined
        bool trunc = fresh(nb, q);
        if (!q.empty() && (st = measure_batch(q)) != TUNER_OK) return st;
        used += (int32_t)q.size();
        ++rounds;
        int bi = -1;
        double bc = 0.0;
        for (size_t i = 0; i < nb.size(); ++i) {
            if (!measured(nb[i]) || !valid(nb[i])) continue;
            double cp = cost(nb[i]);
            if (bi < 0 || cp < bc) { bi = (int)i; bc = cp; }
        }
        if (bi < 0 || !better(nb[bi], x)) {
            if (opts.policy == TUNER_DS_RADIUS && !trunc) {
                ++r;
                continue;
            }
            return finish(!trunc);
        }
        r = 1;
        const Pt prev = x;
        x = nb[bi];
        c = bc;
        traj.push_back(x);
        if (used == budget) return finish(false);
        if (opts.policy != TUNER_DS_GROW) continue;
        int d = 0;
        while (x.idx[d] == prev.idx[d]) ++d;
        const int step = x.idx[d] - prev.idx[d];
        const int card = (int)spaces[x.pos].values[d].size();
        ray.clear();
        Pt last = x;
        for (int64_t j = 1, span = 2;; ++j, span *= 2) {
            int64_t i = (int64_t)prev.idx[d] + step * span;
            if (i < 0) i = 0;
            if (i > card - 1) i = card - 1;
            Pt qj = x;
            qj.idx[d] = (int32_t)i;
            if (qj == last) break;
            ray.push_back(qj);
            last = qj;
        }
        trunc = fresh(ray, q);
        if (!q.empty() && (st = measure_batch(q)) != TUNER_OK) return st;
        used += (int32_t)q.size();
        ++rounds;
        for (const Pt& p : ray) {
            if (measured(p) && valid(p) && better(p, x)) {
                x = p;
                c = cost(p);
                traj.push_back(x);
            } else {
                break;
            }
        }
        if (trunc) return finish(false);
    }
}

// ---------------------------------------------------------------- cost-table measurer
namespace {
struct TableMeasurer : Measurer {
    Tuner* t;
    std::vector<double> table;
    std::vector<float> samples;  // optional [point][nsamp] repeat timings
    int nsamp = 0;
    TableMeasurer(Tuner* tt, std::vector<double>&& tab) : t(tt), table(std::move(tab)) {}
    tuner_status measure(const std::vector<Pt>& pts, std::vector<Result>& out, double, bool) override {
        out.assign(pts.size(), Result{});
        for (size_t i = 0; i < pts.size(); ++i) {
            const uint64_t id = t->linear(pts[i]);
            out[i].cost_ns = table[id];
            out[i].status = TUNER_S_OK;
            out[i].nsamp = nsamp;
            for (int k = 0; k < nsamp; ++k) out[i].samp[k] = samples[id * nsamp + k];
        }
        return TUNER_OK;
    }
    bool valid(const Pt& p) override { return std::isfinite(table[t->linear(p)]); }
};

struct CallbackComm : Comm {
    tuner_allgather_fn fn;
    void* ctx;
    CallbackComm(tuner_allgather_fn f, void* c) : fn(f), ctx(c) {}
    tuner_status allgather(const void* send, void* recv, int64_t bytes) override {
        int rc = fn(ctx, send, recv, bytes);
        return rc == 0 ? TUNER_OK : fail(TUNER_ENCCL, "host all-gather callback failed");
    }
};
}  // namespace

std::unique_ptr<Measurer> make_table_measurer(Tuner* t, std::vector<double>&& table, const double* samples,
                                              int nsamp) {
    std::unique_ptr<TableMeasurer> m(new TableMeasurer(t, std::move(table)));
    if (samples && nsamp > 0) {
        m->nsamp = nsamp;
        m->samples.assign(samples, samples + m->table.size() * (size_t)nsamp);
    }
    return std::unique_ptr<Measurer>(m.release());
}

std::unique_ptr<Comm> make_callback_comm(tuner_allgather_fn fn, void* ctx) {
    return std::unique_ptr<Comm>(new CallbackComm(fn, ctx));
}

}  // namespace db200

// ================================================================= C ABI
using namespace db200;

#define CHECK_HANDLE(t)                                                        \
    do {                                                                       \
        if (!(t)) return fail(TUNER_EINVAL, "NULL tuner handle");              \
        if ((t)->dead) return fail(TUNER_ESTATE, "tuner handle is dead after a CUDA error"); \
    } while (0)

static tuner_status after(Tuner* t, tuner_status st) {
    if (st == TUNER_ECUDA) t->dead = true;
    return st;
}

extern "C" void tuner_opts_default(tuner_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->warmup = 2;
    o->repeats = 10;
    o->number = 0;
    o->timeout_ms = 1000.0;
    o->seed = 0;
    o->policy = TUNER_DS_GROW;
    o->alpha = 0.0;
    o->max_batch = 512;
    o->verify = 1;
    o->rank = 0;
    o->world = 1;
}

extern "C" const char* tuner_last_error(void) { return g_err.c_str(); }

extern "C" tuner_status tuner_create(int32_t op, const tuner_shape* shape, const tuner_knob_space* spaces,
                                     int32_t nspaces, const tuner_opts* opts, tuner_t** out) {
    if (!out) return fail(TUNER_EINVAL, "out is NULL");
    *out = nullptr;
    if (!shape || !spaces || nspaces < 1 || !opts) return fail(TUNER_EINVAL, "shape/spaces/opts missing");
    std::unique_ptr<tuner> t(new tuner());
    t->op = op;
    t->shape = *shape;
    t->opts = *opts;
    if (!(t->opts.early_cut >= 0.0)) return fail(TUNER_EINVAL, "early_cut must be >= 0");
    if (t->opts.repeats < 1 || t->opts.warmup < 0 || t->opts.number < 0 || t->opts.max_batch < 1)
        return fail(TUNER_EINVAL, "repeats >= 1, warmup >= 0, number >= 0, max_batch >= 1 required");
    if (!(t->opts.alpha >= 0.0 && t->opts.alpha < 1.0)) return fail(TUNER_EINVAL, "alpha must be in [0, 1)");
    if (t->opts.cost_samples && (t->opts.cost_nsamp < 1 || t->opts.cost_nsamp > kMaxSamples))
        return fail(TUNER_EINVAL, "cost_nsamp must be in [1, 16]");
    if (t->opts.policy != TUNER_DS_PLAIN && t->opts.policy != TUNER_DS_GROW && t->opts.policy != TUNER_DS_RADIUS)
        return fail(TUNER_EINVAL, "unknown Droplet policy");
    if (t->opts.world < 1) t->opts.world = 1;
    if (t->opts.rank < 0 || t->opts.rank >= t->opts.world) return fail(TUNER_EINVAL, "rank out of range");
    t->table_mode = opts->cost_table != nullptr;
    std::string why;
    if (!make_shape_info(op, *shape, t->info, why)) {
        if (!t->table_mode) return fail(TUNER_EINVAL, why);
    }
    uint64_t off = 0;
    for (int32_t i = 0; i < nspaces; ++i) {
        const tuner_knob_space& ks = spaces[i];
        if (ks.nknobs < 0 || ks.nknobs > TUNER_MAX_KNOBS || (ks.nknobs > 0 && (!ks.card || !ks.values)))
            return fail(TUNER_EINVAL, "bad knob space");
        for (int32_t j = 0; j < i; ++j)
            if (spaces[j].sketch == ks.sketch) return fail(TUNER_EINVAL, "duplicate sketch id in spaces");
        SketchSpace s;
        s.sketch = ks.sketch;
        const SketchDesc* desc = t->table_mode ? nullptr : sketch_desc(ks.sketch);
        if (!t->table_mode) {
            if (!desc) return fail(TUNER_ERANGE, "unknown sketch id");
            if (!(desc->op_mask & (1 << op)) || desc->dtype != shape->dtype)
                return fail(TUNER_EINVAL, std::string("sketch ") + desc->name + " does not implement this op/dtype");
            if ((size_t)ks.nknobs != desc->values.size()) return fail(TUNER_EDIM, "knob count != sketch's knobs");
        }
        int32_t voff = 0;
        unsigned __int128 size = 1;
        for (int32_t d = 0; d < ks.nknobs; ++d) {
            if (ks.card[d] < 1 || ks.card[d] > TUNER_MAX_VALUES) return fail(TUNER_EINVAL, "knob cardinality");
            std::vector<int32_t> vals(ks.values + voff, ks.values + voff + ks.card[d]);
            voff += ks.card[d];
            for (size_t k = 1; k < vals.size(); ++k)
                if (!(vals[k - 1] < vals[k])) return fail(TUNER_EINVAL, "knob values must be strictly increasing");
            if (desc) {
                for (int32_t v : vals) {
                    bool ok = false;
                    for (int32_t sv : desc->values[d]) ok |= (sv == v);
                    if (!ok)
                        return fail(TUNER_EINVAL, std::string("value ") + std::to_string(v) + " of knob " +
                                                      desc->knob_names[d] + " is not compiled for " + desc->name);
                }
            }
            s.values.push_back(std::move(vals));
            size *= (unsigned __int128)ks.card[d];
            if (size > ((unsigned __int128)1 << 62)) return fail(TUNER_EOVERFLOW, "space larger than 2^62");
        }
        s.size = (uint64_t)size;
        s.offset = off;
        off += s.size;
        if (off > (1ull << 62)) return fail(TUNER_EOVERFLOW, "space larger than 2^62");
        t->spaces.push_back(std::move(s));
    }
    t->total = off;
    t->rng = SplitMix64(opts->seed);
    t->key = problem_key(op, *shape);
    // the exchange step (R-M1): a caller-supplied host all-gather, or NCCL from a unique
    // id; an exchange given at world 1 is used too (one rank gathers its own slots)
    if (opts->allgather) {
        t->comm = make_callback_comm(opts->allgather, opts->allgather_ctx);
    } else if (opts->nccl_unique_id) {
        tuner_status st = make_nccl_comm(opts->nccl_unique_id, t->opts.rank, t->opts.world, opts->stream, t->comm);
        if (st != TUNER_OK) return st;
    } else if (t->opts.world > 1) {
        return fail(TUNER_EINVAL, "world > 1 needs an allgather callback or an NCCL unique id");
    }
    if (t->table_mode) {
        if ((uint64_t)opts->cost_table_len != t->total)
            return fail(TUNER_EINVAL, "cost_table_len != total number of points");
        std::vector<double> tab(opts->cost_table, opts->cost_table + opts->cost_table_len);
        for (double v : tab)
            if (std::isnan(v)) return fail(TUNER_EINVAL, "NaN in cost table");
        t->measurer = make_table_measurer(t.get(), std::move(tab), opts->cost_samples, opts->cost_nsamp);
    } else {
        if (!opts->x || !opts->w || !opts->y) return fail(TUNER_EINVAL, "measured mode needs x, w, y device buffers");
        tuner_status st = make_gpu_measurer(t.get(), t->measurer);
        if (st != TUNER_OK) return st;
    }
    if (opts->trial_log && opts->trial_log[0]) {  // resume from, then append to, the trial log
        tuner_status st = t->replay_log(opts->trial_log);
        if (st != TUNER_OK) return st;
        if (t->opts.rank == 0 && !(t->trial_log = std::fopen(opts->trial_log, "a")))
            return fail(TUNER_EINVAL, std::string("cannot open trial log ") + opts->trial_log);
    }
    t->opts.trial_log = nullptr;  // borrowed for the call only
    *out = t.release();
    return TUNER_OK;
}

extern "C" tuner_status tuner_point_valid(const tuner_t* tc, const tuner_point* pt, int32_t* valid) {
    Tuner* t = const_cast<tuner_t*>(tc);
    CHECK_HANDLE(t);
    if (!pt || !valid) return fail(TUNER_EINVAL, "NULL argument");
    tuner_status st;
    Pt p = t->from_public(*pt, st);
    if (st != TUNER_OK) return st;
    *valid = t->valid(p) ? 1 : 0;
    return TUNER_OK;
}

static void fill_sample(Tuner* t, const Pt& p, tuner_result* out) { *out = t->history[t->memo.at(t->linear(p))]; }

extern "C" tuner_status tuner_sample(tuner_t* t, int32_t n, tuner_result* out, int32_t* n_out) {
    CHECK_HANDLE(t);
    if (n < 0 || (n > 0 && !out) || !n_out) return fail(TUNER_EINVAL, "bad arguments");
    *n_out = 0;
    std::vector<Pt> pts;
    t->draw(n, pts);
    for (size_t i = 0; i < pts.size(); i += (size_t)t->opts.max_batch) {
        size_t e = std::min(pts.size(), i + (size_t)t->opts.max_batch);
        std::vector<Pt> b(pts.begin() + i, pts.begin() + e);
        tuner_status st = t->measure_batch(b);
        if (st != TUNER_OK) return after(t, st);
    }
    for (size_t i = 0; i < pts.size(); ++i) fill_sample(t, pts[i], &out[i]);
    *n_out = (int32_t)pts.size();
    return TUNER_OK;
}

extern "C" tuner_status tuner_grid(tuner_t* t, int32_t n, tuner_result* out, int32_t* n_out) {
    CHECK_HANDLE(t);
    if (n < 0 || (n > 0 && !out) || !n_out) return fail(TUNER_EINVAL, "bad arguments");
    *n_out = 0;
    std::vector<Pt> pts;
    t->grid(n, pts);
    tuner_status st = t->measure_chunked(pts);
    if (st != TUNER_OK) return after(t, st);
    for (size_t i = 0; i < pts.size(); ++i) fill_sample(t, pts[i], &out[i]);
    *n_out = (int32_t)pts.size();
    return TUNER_OK;
}

extern "C" tuner_status tuner_evolve(tuner_t* t, int32_t n, int32_t pop, int32_t elite, tuner_result* out,
                                     int32_t* n_out) {
    CHECK_HANDLE(t);
    if (n < 0 || pop < 1 || elite < 1 || (n > 0 && !out) || !n_out) return fail(TUNER_EINVAL, "bad arguments");
    *n_out = 0;
    std::vector<Pt> pts;
    tuner_status st = t->evolve(n, pop, elite, pts);
    if (st != TUNER_OK) return after(t, st);
    for (size_t i = 0; i < pts.size(); ++i) fill_sample(t, pts[i], &out[i]);
    *n_out = (int32_t)pts.size();
    return TUNER_OK;
}

// ---------------------------------------------------------------- multi-layer budget (R-F3)
// P:244-248 / P:393-396: initial quota min(K/L, 64) per layer, then the remaining
// trials in increments to the layer with the largest weight x best cost, after
// dropping layers below drop_frac of the model total.  Exploration = evolve.
static double weighted_best(tuner_t* t, double w) {
    double b = INFINITY;
    for (const auto& h : t->history)
        if (h.cost_ns < b) b = h.cost_ns;
    return w * b;
}

extern "C" tuner_status tuner_schedule(tuner_t* const* layers, int32_t nlayers, const double* weights, int64_t budget,
                                       int32_t increment, double drop_frac, int32_t pop, int32_t elite,
                                       int64_t* trials) {
    if (!layers || nlayers < 1 || !weights || !trials || budget < 0 || increment < 1 || pop < 1 || elite < 1 ||
        !(drop_frac >= 0.0))
        return fail(TUNER_EINVAL, "bad arguments");
    for (int32_t i = 0; i < nlayers; ++i) {
        CHECK_HANDLE(layers[i]);
        if (!(weights[i] > 0.0)) return fail(TUNER_EINVAL, "weights must be > 0");
        trials[i] = 0;
    }
    const int64_t q = std::max<int64_t>(1, std::min<int64_t>(budget / nlayers, 64));
    int64_t total = 0;
    std::vector<Pt> got;
    for (int32_t i = 0; i < nlayers; ++i) {
        const int64_t n = std::min(q, budget - total);
        if (n <= 0) break;
        tuner_status st = layers[i]->evolve((int32_t)n, pop, elite, got);
        if (st != TUNER_OK) return after(layers[i], st);
        trials[i] += (int64_t)got.size();
        total += (int64_t)got.size();
    }
    std::vector<int32_t> work;
    for (int32_t i = 0; i < nlayers; ++i) work.push_back(i);
    while (total < budget && !work.empty()) {
        double model = 0.0;
        for (int32_t i = 0; i < nlayers; ++i) {
            const double wb = weighted_best(layers[i], weights[i]);
            if (std::isfinite(wb)) model += wb;
        }
        std::vector<int32_t> keep;
        for (int32_t i : work) {
            const double wb = weighted_best(layers[i], weights[i]);
            if (!(std::isfinite(wb) && wb < drop_frac * model)) keep.push_back(i);
        }
        work.swap(keep);
        if (work.empty()) break;
        int32_t pick = work[0];
        for (size_t k = 1; k < work.size(); ++k)
            if (weighted_best(layers[work[k]], weights[work[k]]) > weighted_best(layers[pick], weights[pick]))
                pick = work[k];
        const int64_t n = std::min<int64_t>(increment, budget - total);
        tuner_status st = layers[pick]->evolve((int32_t)n, pop, elite, got);
        if (st != TUNER_OK) return after(layers[pick], st);
        if (got.empty()) {
            work.erase(std::find(work.begin(), work.end(), pick));
            continue;
        }
        trials[pick] += (int64_t)got.size();
        total += (int64_t)got.size();
    }
    return TUNER_OK;
}

extern "C" tuner_status tuner_measure(tuner_t* t, const tuner_point* pts, int32_t n, tuner_result* out) {
    CHECK_HANDLE(t);
    if (n < 0 || (n > 0 && (!pts || !out))) return fail(TUNER_EINVAL, "bad arguments");
    std::vector<Pt> all(n), todo;
    std::vector<char> ok(n, 0);
    std::unordered_set<uint64_t> seen;
    for (int32_t i = 0; i < n; ++i) {
        tuner_status st;
        all[i] = t->from_public(pts[i], st);
        if (st != TUNER_OK) return st;
        ok[i] = t->valid(all[i]);
        uint64_t id = t->linear(all[i]);
        if (ok[i] && !t->memo.count(id) && !seen.count(id)) {
            seen.insert(id);
            todo.push_back(all[i]);
        }
    }
    for (size_t i = 0; i < todo.size(); i += (size_t)t->opts.max_batch) {
        size_t e = std::min(todo.size(), i + (size_t)t->opts.max_batch);
        tuner_status st = t->measure_batch(std::vector<Pt>(todo.begin() + i, todo.begin() + e));
        if (st != TUNER_OK) return after(t, st);
    }
    for (int32_t i = 0; i < n; ++i) {
        if (ok[i]) {
            fill_sample(t, all[i], &out[i]);
        } else {
            std::memset(&out[i], 0, sizeof(out[i]));
            out[i].pt = pts[i];
            out[i].cost_ns = INFINITY;
            out[i].status = TUNER_S_INVALID;
            out[i].rank = -1;
        }
    }
    return TUNER_OK;
}

extern "C" tuner_status tuner_droplet(tuner_t* t, const tuner_point* start, int32_t budget, tuner_point* traj,
                                      int32_t traj_cap, tuner_droplet_report* report) {
    CHECK_HANDLE(t);
    if (!start || !report) return fail(TUNER_EINVAL, "NULL argument");
    if (budget < 1) return fail(TUNER_EINVAL, "budget must be >= 1");
    tuner_status st;
    Pt s = t->from_public(*start, st);
    if (st != TUNER_OK) return st;
    if (!t->valid(s)) return fail(TUNER_ERANGE, "start point is statically invalid");
    std::vector<Pt> tr;
    st = t->droplet(s, budget, tr, *report);
    if (st != TUNER_OK) return after(t, st);
    if (traj)
        for (int32_t i = 0; i < (int32_t)tr.size() && i < traj_cap; ++i) traj[i] = t->to_public(tr[i]);
    return TUNER_OK;
}

extern "C" tuner_status tuner_timings(const tuner_t* tc, const tuner_point* pt, float* out, int32_t cap,
                                      int32_t* n_out) {
    Tuner* t = const_cast<tuner_t*>(tc);
    CHECK_HANDLE(t);
    if (!pt || !n_out || (cap > 0 && !out)) return fail(TUNER_EINVAL, "NULL argument");
    tuner_status st;
    Pt p = t->from_public(*pt, st);
    if (st != TUNER_OK) return st;
    auto it = t->memo.find(t->linear(p));
    if (it == t->memo.end()) return fail(TUNER_ERANGE, "point was never measured");
    const auto& v = t->hsamples[it->second];
    *n_out = (int32_t)v.size();
    for (int32_t i = 0; i < cap && i < (int32_t)v.size(); ++i) out[i] = v[i];
    return TUNER_OK;
}

extern "C" tuner_status tuner_best(const tuner_t* tc, tuner_result* out) {
    Tuner* t = const_cast<tuner_t*>(tc);
    CHECK_HANDLE(t);
    if (!out) return fail(TUNER_EINVAL, "NULL out");
    if (t->history.empty()) return fail(TUNER_ESTATE, "tuner_best before any measurement");
    size_t bi = 0;
    for (size_t i = 1; i < t->history.size(); ++i)
        if (t->history[i].cost_ns < t->history[bi].cost_ns) bi = i;  // first argmin (R-B1)
    *out = t->history[bi];
    return TUNER_OK;
}

extern "C" tuner_status tuner_best_of_sketch(const tuner_t* tc, int32_t sketch, tuner_result* out) {
    Tuner* t = const_cast<tuner_t*>(tc);
    CHECK_HANDLE(t);
    if (!out) return fail(TUNER_EINVAL, "NULL out");
    bool known = false;
    for (const auto& sp : t->spaces) known |= sp.sketch == sketch;
    if (!known) return fail(TUNER_ERANGE, "sketch not in this tuner's spaces");
    size_t bi = t->history.size();
    for (size_t i = 0; i < t->history.size(); ++i) {
        const tuner_result& h = t->history[i];
        if (h.pt.sketch != sketch || !std::isfinite(h.cost_ns)) continue;
        if (bi == t->history.size() || h.cost_ns < t->history[bi].cost_ns) bi = i;  // first argmin (R-B1)
    }
    if (bi == t->history.size()) return fail(TUNER_ESTATE, "no finite measurement of this sketch");
    *out = t->history[bi];
    return TUNER_OK;
}

extern "C" tuner_status tuner_history(const tuner_t* tc, tuner_result* out, int64_t cap, int64_t* n_out) {
    Tuner* t = const_cast<tuner_t*>(tc);
    if (!t) return fail(TUNER_EINVAL, "NULL tuner handle");
    if (!n_out) return fail(TUNER_EINVAL, "NULL n_out");
    *n_out = (int64_t)t->history.size();
    if (out)
        for (int64_t i = 0; i < cap && i < (int64_t)t->history.size(); ++i) out[i] = t->history[i];
    return TUNER_OK;
}

extern "C" tuner_status tuner_get_stats(const tuner_t* tc, tuner_stats* out) {
    if (!tc || !out) return fail(TUNER_EINVAL, "NULL argument");
    *out = tc->stats;
    return TUNER_OK;
}

extern "C" tuner_status kernel_run(const tuner_t* tc, const tuner_point* cfg, const tuner_buffers* buf, void* stream) {
    Tuner* t = const_cast<tuner_t*>(tc);
    CHECK_HANDLE(t);
    if (!cfg || !buf) return fail(TUNER_EINVAL, "NULL argument");
    if (t->table_mode) return fail(TUNER_ESTATE, "kernel_run in cost-table mode");
    tuner_status st;
    Pt p = t->from_public(*cfg, st);
    if (st != TUNER_OK) return st;
    if (!t->valid(p)) return fail(TUNER_ERANGE, "statically invalid schedule");
    return after(t, gpu_kernel_run(t, p, buf, stream ? stream : t->opts.stream));
}

extern "C" tuner_status tuner_reference(const tuner_t* tc, const tuner_buffers* buf, float* y_ref, float* y_absref,
                                        void* stream) {
    Tuner* t = const_cast<tuner_t*>(tc);
    CHECK_HANDLE(t);
    if (!buf || !y_ref || !y_absref) return fail(TUNER_EINVAL, "NULL argument");
    if (t->table_mode) return fail(TUNER_ESTATE, "tuner_reference in cost-table mode");
    return after(t, gpu_reference(t, buf, y_ref, y_absref, stream ? stream : t->opts.stream));
}

extern "C" tuner_status tuner_nccl_unique_id(void* out128) {
    if (!out128) return fail(TUNER_EINVAL, "NULL out");
    return nccl_unique_id(out128);
}

extern "C" void tuner_destroy(tuner_t* t) { delete t; }

extern "C" int64_t tuner_global_launch_count(void) { return g_launch_counter_ptr()->load(); }
