// KV-cache bookkeeping, two layers:
//
//  KvBlockPool  - the reference's block-count ledger (splitsim/gpu_model.hpp:79-135):
//                 blocks_for(t) = ceil(t/B); alloc() resizes a request to hold
//                 t tokens atomically or reports AdmissionDenied; free() drops it;
//                 usage_pct() = 100*total/capacity.  Kept with identical
//                 semantics so policies observe the same numbers.
//  PagePool     - NEW: physical page ids for the one HBM arena that backs every
//                 instance.  Lowest-free-id-first, so any replay of the same
//                 alloc/free sequence reproduces the page tables bit for bit
//                 (that replay is how the oracle checks GPU page tables).
#pragma once

#include <functional>
#include <map>
#include <queue>
#include <string>
#include <vector>

#include "base.hpp"

namespace sw {

class KvBlockPool {
public:
    enum class AllocResult { Ok, AdmissionDenied };

    KvBlockPool() = default;
    KvBlockPool(int block_tokens, long long capacity_blocks) : block_tokens_(block_tokens), cap_(capacity_blocks) {
        if (block_tokens_ < 1) throw ConfigError("gpu.block_tokens: must be >= 1");
    }

    int block_tokens() const { return block_tokens_; }
    long long capacity() const { return cap_; }
    long long total_allocated() const { return used_; }
    long long blocks_for(long long tokens) const { return (tokens + block_tokens_ - 1) / block_tokens_; }
    bool has(int rid) const { return held_.find(rid) != held_.end(); }

    long long allocated(int rid) const {
        const auto it = held_.find(rid);
        if (it == held_.end())
            throw ContractViolation("kv pool: request " + std::to_string(rid) + " has no allocation");
        return it->second;
    }

    AllocResult alloc(int rid, long long tokens_resident) {
        const long long want = blocks_for(tokens_resident);
        const auto it = held_.find(rid);
        const long long have = it == held_.end() ? 0 : it->second;
        if (used_ + (want - have) > cap_) return AllocResult::AdmissionDenied;
        used_ += want - have;
        held_[rid] = want;
        return AllocResult::Ok;
    }

    void free(int rid) {
        const auto it = held_.find(rid);
        if (it == held_.end())
            throw ContractViolation("kv pool: free of unallocated request " + std::to_string(rid));
        used_ -= it->second;
        held_.erase(it);
    }

    double usage_pct() const { return 100.0 * static_cast<double>(used_) / static_cast<double>(cap_); }

private:
    int block_tokens_ = 16;
    long long cap_ = 1;
    long long used_ = 0;
    std::map<int, long long> held_;  // ordered map: deterministic iteration
};

// Physical page allocator over [0, n_pages).  Every request owns an ordered
// list of page ids (its page-table row); growing appends the lowest free ids.
class PagePool {
public:
    struct Event {  // one entry of the alloc/free journal (replayed by the oracle)
        int request;
        int pages_after;  // row length after the op; 0 = freed
    };

    explicit PagePool(long long n_pages = 0) : n_pages_(n_pages) {
        for (long long p = 0; p < n_pages; ++p) free_.push(static_cast<int>(p));
    }

    long long n_pages() const { return n_pages_; }
    long long in_use() const { return n_pages_ - static_cast<long long>(free_.size()); }

    const std::vector<int>& row(int rid) const {
        static const std::vector<int> kEmpty;
        const auto it = rows_.find(rid);
        return it == rows_.end() ? kEmpty : it->second;
    }

    // Grow request `rid` to hold `pages` pages; returns the index of the first
    // newly appended page in its row.  Shrinking is not a thing: KV only grows.
    int grow_to(int rid, int pages) {
        auto& r = rows_[rid];
        const int first_new = static_cast<int>(r.size());
        if (pages <= first_new) return first_new;
        if (static_cast<long long>(pages - first_new) > static_cast<long long>(free_.size()))
            throw ContractViolation("page pool: arena exhausted growing request " + std::to_string(rid));
        while (static_cast<int>(r.size()) < pages) {
            r.push_back(free_.top());
            free_.pop();
        }
        journal_.push_back({rid, pages});
        return first_new;
    }

    void release(int rid) {
        const auto it = rows_.find(rid);
        if (it == rows_.end()) throw ContractViolation("page pool: release of unknown request " + std::to_string(rid));
        for (int p : it->second) free_.push(p);
        final_rows_[rid] = it->second;
        rows_.erase(it);
        journal_.push_back({rid, 0});
    }

    const std::vector<Event>& journal() const { return journal_; }
    // Page-table row a finished request held at its largest extent.
    const std::map<int, std::vector<int>>& final_rows() const { return final_rows_; }

private:
    long long n_pages_;
    std::priority_queue<int, std::vector<int>, std::greater<int>> free_;
    std::map<int, std::vector<int>> rows_;
    std::map<int, std::vector<int>> final_rows_;
    std::vector<Event> journal_;
};

}  // namespace sw
