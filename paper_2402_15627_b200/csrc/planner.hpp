// planner.hpp — shard/bucket planner (rules P1-P7).
//
// PAPER.md never describes buckets or shard layouts: ZeRO-2 shards optimizer state and
// gradients over the DP ranks (§2) and overlaps communication per model chunk
// (§3.2).  The layout below is DESIGN.md reading Z17; it is the bit-exact contract
// with the oracle's planner (oracle/plan.py), with which this file shares no code.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace lamb {

constexpr int64_t kTensorAlign = 8;    // P2: tensor starts 8-aligned (16 B bf16, 32 B fp32)
constexpr int64_t kSliceAlign = 128;   // P4/P6: slices are multiples of 128 elements
constexpr int64_t kDefaultCap = 40000000;

struct Plan {
    int32_t world = 1, rank = 0;
    int64_t cap = kDefaultCap;
    std::vector<int64_t> numel;          // [T]
    std::vector<int32_t> group;          // [T]
    std::vector<int64_t> tensor_off;     // [T] flat offset
    std::vector<int64_t> tensor_bucket;  // [T]
    std::vector<int64_t> buckets;        // [B][4] base, S_b, t_begin, t_end
    std::vector<int64_t> shard_base;     // [B] offset of bucket b's slice in the shard
    std::vector<int64_t> segments;       // [n_seg][4] tensor, shard_off, tensor_off, len
    std::vector<int64_t> straddlers;     // ascending tensor ids with >= 2 segments (global)
    std::vector<uint8_t> is_straddler;   // [T]
    int64_t flat_size = 0, shard_size = 0;

    int64_t n_tensors() const { return (int64_t)numel.size(); }
    int64_t n_buckets() const { return (int64_t)buckets.size() / 4; }
    int64_t n_segments() const { return (int64_t)segments.size() / 4; }
};

// Returns an empty string on success, else the reason (-> LAMB_EINVAL).
std::string build_plan(const int64_t* numel, const int32_t* group, int64_t n_tensors,
                       int32_t world, int32_t rank, int64_t cap, Plan* out);

}  // namespace lamb
