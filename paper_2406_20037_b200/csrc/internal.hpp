// internal.hpp — shared declarations of libdroplet_b200 (not part of the ABI).
#pragma once
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tuner.h"
#include "shape.hpp"

namespace db200 {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
tuner_status fail(tuner_status st, const std::string& msg);

// ---------------------------------------------------------------- PRNG (R-S1)
// SplitMix64; uniform(m) = high 64 bits of z*m (no rejection).
struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t seed) : state(seed) {}
    uint64_t next() {
        state += 0x9E3779B97F4A7C15ull;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint32_t uniform(uint32_t m) {
        return (uint32_t)(((unsigned __int128)next() * (unsigned __int128)m) >> 64);
    }
};

// ---------------------------------------------------------------- knob spaces
struct SketchSpace {
    int32_t sketch = 0;               // template id
    std::vector<std::vector<int32_t>> values;  // per knob, strictly increasing
    uint64_t size = 1;                // product of cardinalities
    uint64_t offset = 0;              // linear-id offset in the union
    int nknobs() const { return (int)values.size(); }
};

// A point in the union of sketch spaces: position of the sketch in the
// tuner's space list + index vector.
struct Pt {
    int32_t pos = 0;
    int32_t n = 0;
    std::array<int32_t, TUNER_MAX_KNOBS> idx{};
    bool operator==(const Pt& o) const {
        if (pos != o.pos || n != o.n) return false;
        for (int i = 0; i < n; ++i)
            if (idx[i] != o.idx[i]) return false;
        return true;
    }
};

// Per-candidate measurement result.
static constexpr int kMaxSamples = 16;  // repeat timings kept per candidate (statistical mode)
struct Result {
    double cost_ns = INFINITY;
    double max_err = 0.0;
    int32_t status = TUNER_S_OK;
    int32_t rank = 0;
    int32_t nsamp = 0;
    float samp[kMaxSamples] = {};  // per-launch times of the repeats (ns)
};
double wilcoxon_p(const float* a, int n1, const float* b, int n2);

// ---------------------------------------------------------------- sketch catalogue
bool make_shape_info(int32_t op, const tuner_shape& s, ShapeInfo& out, std::string& why);

struct SketchDesc {
    int32_t id;
    const char* name;
    int32_t op_mask;  // bit per tuner_op
    int32_t dtype;
    std::vector<const char*> knob_names;
    std::vector<std::vector<int32_t>> values;  // full supported space
};
const SketchDesc* sketch_desc(int32_t id);
// Static validity of concrete knob values for a shape (hardware rules).
bool sketch_valid(int32_t id, const ShapeInfo& sh, const int32_t* v);

// ---------------------------------------------------------------- comm
struct Comm {
    virtual ~Comm() = default;
    virtual tuner_status allgather(const void* send, void* recv, int64_t bytes) = 0;
};
std::unique_ptr<Comm> make_callback_comm(tuner_allgather_fn fn, void* ctx);
tuner_status make_nccl_comm(const void* uid, int rank, int world, void* stream,
                            std::unique_ptr<Comm>& out);
tuner_status nccl_unique_id(void* out128);

// ---------------------------------------------------------------- measurement backends
struct Measurer {
    virtual ~Measurer() = default;
    // measure `pts` (this rank's share of a batch) -> results in the same order.
    // `incumbent` = best cost measured so far; `collective` = every rank is in this call
    // (the batch's shard), false = one rank re-times alone (calibration)
    virtual tuner_status measure(const std::vector<Pt>& pts, std::vector<Result>& out, double incumbent,
                                 bool collective) = 0;
    virtual bool valid(const Pt& p) = 0;
};

struct Tuner;
std::unique_ptr<Measurer> make_table_measurer(Tuner* t, std::vector<double>&& table, const double* samples,
                                              int nsamp);
tuner_status make_gpu_measurer(Tuner* t, std::unique_ptr<Measurer>& out);
tuner_status gpu_kernel_run(Tuner* t, const Pt& p, const tuner_buffers* buf, void* stream);
tuner_status gpu_reference(const Tuner* t, const tuner_buffers* buf, float* y_ref, float* y_absref,
                           void* stream);
extern std::atomic<int64_t>* g_launch_counter_ptr();

// ---------------------------------------------------------------- the tuner
struct Tuner {
    int32_t op = 0;
    tuner_shape shape{};
    ShapeInfo info{};
    tuner_opts opts{};
    std::vector<SketchSpace> spaces;
    uint64_t total = 0;
    bool table_mode = false;
    bool dead = false;
    SplitMix64 rng{0};
    std::vector<tuner_result> history;
    std::vector<std::vector<float>> hsamples;  // repeat timings per history entry
    std::unordered_map<uint64_t, size_t> memo;  // linear id -> history index
    std::unique_ptr<Measurer> measurer;
    std::unique_ptr<Comm> comm;
    tuner_stats stats{};
    double best_cost = INFINITY;
    uint64_t grid_cursor = 0;  // next union linear id tuner_grid examines
    StreamKScratch sk;         // stream-K workspace (tcgen05 SCHED >= 1), allocated on first need

    Tuner() = default;
    Tuner(const Tuner&) = delete;
    Tuner& operator=(const Tuner&) = delete;
    ~Tuner();  // harness.cu: drops the measurer (device synchronised), then frees `sk`

    uint64_t linear(const Pt& p) const;
    Pt from_public(const tuner_point& tp, tuner_status& st) const;  // validates dims/ranges
    tuner_point to_public(const Pt& p) const;
    void values_of(const Pt& p, int32_t* v) const;
    bool valid(const Pt& p) { return measurer->valid(p); }
    void ring(const Pt& x, std::vector<Pt>& out, int r = 1) const;
    bool measured(const Pt& p) const { return memo.count(linear(p)) != 0; }
    double cost(const Pt& p) const { return history[memo.at(linear(p))].cost_ns; }

    std::FILE* trial_log = nullptr;  // append-only JSONL log (opts.trial_log), rank 0 writes
    std::string key;                 // the problem key of the log lines (op, shape, dtype)

    tuner_status measure_batch(const std::vector<Pt>& batch);
    tuner_status calibrate(const std::vector<Pt>& batch, std::vector<Result>& res);
    void record(const Pt& p, const tuner_result& smp, std::vector<float>&& samples, bool log);
    void log_trial(const Pt& p, const tuner_result& smp, const std::vector<float>& samples);
    tuner_status replay_log(const char* path);
    tuner_status draw(int32_t n, std::vector<Pt>& out);
    tuner_status measure_chunked(const std::vector<Pt>& pts);
    tuner_status evolve(int32_t n, int32_t pop, int32_t elite, std::vector<Pt>& out);
    void grid(int32_t n, std::vector<Pt>& out);
    tuner_status droplet(const Pt& start, int32_t budget, std::vector<Pt>& traj,
                         tuner_droplet_report& rep);
};

}  // namespace db200

// the opaque ABI handle is the tuner itself
struct tuner : public db200::Tuner {};
