// planner.cpp — see planner.hpp.  Host integer code, run once in lamb_create.
#include "planner.hpp"

#include <numeric>

namespace lamb {

static inline int64_t round_up(int64_t x, int64_t q) { return (x + q - 1) / q * q; }

std::string build_plan(const int64_t* numel, const int32_t* group, int64_t n_tensors,
                       int32_t world, int32_t rank, int64_t cap, Plan* out) {
    if (n_tensors < 1) return "n_tensors must be >= 1";
    if (world < 1 || world > 8) return "world_size must be in [1, 8]";
    if (rank < 0 || rank >= world) return "rank out of range";
    if (cap < 0) return "bucket cap must be >= 0";
    if (cap == 0) cap = kDefaultCap;
    Plan& p = *out;
    p = Plan();
    p.world = world;
    p.rank = rank;
    p.cap = cap;
    p.numel.assign(numel, numel + n_tensors);
    p.group.resize(n_tensors);
    for (int64_t i = 0; i < n_tensors; ++i) {
        if (numel[i] < 1) return "tensor " + std::to_string(i) + " has numel < 1";
        p.group[i] = group ? group[i] : 0;
    }

    // P1 (table order) + P2 (8-aligned starts) + P3 (greedy close-before-overflow, strict >).
    // Bucket b collects tensors [t_begin, t_end); `fill` is its aligned size so far.
    const int64_t Q = kSliceAlign * (int64_t)std::lcm((int64_t)world, kTensorAlign);  // P4
    p.tensor_off.resize(n_tensors);
    p.tensor_bucket.resize(n_tensors);
    std::vector<int64_t> start_in_bucket(n_tensors);
    int64_t fill = 0, t_begin = 0, base = 0;
    auto close_bucket = [&](int64_t t_end) {
        const int64_t S = round_up(fill, Q);                       // P4
        p.buckets.insert(p.buckets.end(), {base, S, t_begin, t_end});
        for (int64_t j = t_begin; j < t_end; ++j) {
            p.tensor_off[j] = base + start_in_bucket[j];
            p.tensor_bucket[j] = (int64_t)p.buckets.size() / 4 - 1;
        }
        base += S;                                                  // P5
    };
    for (int64_t i = 0; i < n_tensors; ++i) {
        const int64_t a = round_up(numel[i], kTensorAlign);
        if (i > t_begin && fill + a > cap) {
            close_bucket(i);
            t_begin = i;
            fill = 0;
        }
        start_in_bucket[i] = fill;
        fill += a;
    }
    close_bucket(n_tensors);
    p.flat_size = base;
    p.shard_size = base / world;

    // P6: rank r owns slice r of every bucket; shard-local order = bucket order.
    // P7: segments of this rank; straddlers = tensors whose first and last element lie in
    //     different slices (computed for all tensors, identical on every rank).
    const int64_t B = p.n_buckets();
    p.shard_base.resize(B);
    p.is_straddler.assign(n_tensors, 0);
    int64_t sb = 0;
    for (int64_t b = 0; b < B; ++b) {
        const int64_t bbase = p.buckets[4 * b], S = p.buckets[4 * b + 1];
        const int64_t tb = p.buckets[4 * b + 2], te = p.buckets[4 * b + 3];
        const int64_t slice = S / world;
        p.shard_base[b] = sb;
        const int64_t lo = bbase + (int64_t)rank * slice, hi = lo + slice;
        for (int64_t i = tb; i < te; ++i) {
            const int64_t first = p.tensor_off[i], last = first + p.numel[i] - 1;
            if ((first - bbase) / slice != (last - bbase) / slice) p.is_straddler[i] = 1;
            const int64_t s = first > lo ? first : lo;
            const int64_t e = (last + 1) < hi ? (last + 1) : hi;
            if (s < e) p.segments.insert(p.segments.end(), {i, sb + (s - lo), s - first, e - s});
        }
        sb += slice;
    }
    for (int64_t i = 0; i < n_tensors; ++i)
        if (p.is_straddler[i]) p.straddlers.push_back(i);
    return std::string();
}

}  // namespace lamb
