// Plan cache compatible with the reference's `.fccplan` files (plan_cache.hpp).
#pragma once

#include <memory>
#include <mutex>
#include <string>

#include "plan.hpp"

namespace fcct {

class PlanStore {
public:
    explicit PlanStore(std::string dir);

    // PlanStore::load_or_build (plan_cache.cpp:222-282): valid files are
    // loaded (children resolved recursively), missing ones built, corrupt or
    // mismatched ones rebuilt in place with a warning on stderr.
    std::shared_ptr<const PlanNode> load_or_build(int n, const Params& p);

    struct Stats {
        int hits = 0, misses = 0, rebuilt = 0;
    };
    Stats stats() const {
        std::lock_guard<std::mutex> lock(mu_);
        return stats_;
    }
    const std::string& directory() const { return dir_; }
    std::string path_for(int n, const Params& p) const;
    static std::string cache_key(int n, const Params& p);

private:
    std::string dir_;
    Stats stats_;
    mutable std::mutex mu_;
};

}  // namespace fcct
