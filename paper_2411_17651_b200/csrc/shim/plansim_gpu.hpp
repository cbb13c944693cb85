// plansim_gpu.hpp — drop-in replacement for the reference's evaluate-all-plans
// entry points, over the reference's own C++ types.  A plansim build adds
// plansim_gpu.cpp and links libpsg.so; callers switch
//     plansim::search(...)  ->  plansim_gpu::search(...)
// (same arguments, same RankedPlans result, same exceptions).  See
// INTEGRATION.md.
//
// Replaces: plansim::search          include/plansim/simulator.hpp:99-103
//           plansim::simulate_plan   include/plansim/simulator.hpp:80-82
//                                    (emit_iterations included)
//           plansim::sweep_max_batch include/plansim/simulator.hpp:117-122
#pragma once

#include <vector>

#include "plansim/simulator.hpp"

namespace plansim_gpu {

// `jobs` maps to devices (the reference's worker threads,
// simulator.cpp:251-275): with jobs > 1 the entries are sharded longest-first
// over min(jobs, visible devices) contexts starting at `device` and ranked
// together; the result is identical for every jobs value.  `device` selects
// the (first) CUDA device; contexts are cached per device and locked per call,
// so concurrent callers are safe.
plansim::RankedPlans search(const std::vector<plansim::ExecutionPlan>& plans,
                            const plansim::ModelSpec& model,
                            const plansim::ClusterSpec& cluster,
                            const plansim::Trace& trace,
                            const plansim::ProfileStore& store,
                            plansim::Objective objective,
                            const std::vector<double>& frequencies,
                            const plansim::SimConfig& cfg, int jobs = 1, int device = 0);

plansim::SimulationReport simulate_plan(const plansim::ExecutionPlan& plan,
                                        const plansim::ModelSpec& model,
                                        const plansim::ClusterSpec& cluster,
                                        const plansim::Trace& trace,
                                        const plansim::ProfileStore& store,
                                        const plansim::SimConfig& cfg, int device = 0);

// All `segments` capped simulations run in one launch.
plansim::SweepTable sweep_max_batch(const plansim::ExecutionPlan& plan,
                                    const plansim::ModelSpec& model,
                                    const plansim::ClusterSpec& cluster,
                                    const plansim::Trace& trace,
                                    const plansim::ProfileStore& store,
                                    const plansim::SimConfig& cfg, int segments,
                                    int64_t subset_size = 256, int device = 0);

}  // namespace plansim_gpu
