// NSGA-II baseline: device-resident generational loop (nsga2.cu).
#pragma once
#include <vector>

#include "internal.h"
#include "run.h"

namespace temo_b200 {

struct SortScratch {
    uint64_t cap = 0;
    uint32_t *count = nullptr, *rank = nullptr, *front = nullptr, *n_front = nullptr;
    void alloc(uint64_t rows);
    void release();
};

// nondominated_sort (selection.hpp:251-283) of n x m device-resident objectives; returns the number of fronts.
uint64_t device_nondominated_sort(const double* f, uint64_t n, uint64_t m, SortScratch& sc, uint32_t* rank_host, cudaStream_t s);
// nsga2_select (selection.hpp:316-346) given the ranks; f is a host copy of the objectives.
void nsga2_select_host(const double* f, const uint32_t* rank, uint64_t n, uint64_t m, uint64_t target, uint32_t* selected);

struct Nsga2Run {  // reference: nsga2_run, algorithms.hpp:301-369 (track_archive = false)
    explicit Nsga2Run(const RunConfig& c);
    ~Nsga2Run();
    Nsga2Run(const Nsga2Run&) = delete;
    Nsga2Run& operator=(const Nsga2Run&) = delete;

    void step(const double* f_off_inject = nullptr);
    void inject(const double* x_in, const double* f_in, uint64_t counter_in, uint64_t t_in);
    void download(double* x_out, double* f_out);
    void last_generation(double* offspring, double* f_off, uint64_t* sel, uint64_t* pool);

    RunConfig cfg;
    uint64_t n = 0, d = 0, m = 0, counter = 0, t = 0;
    Rng rng{};
    cudaStream_t stream = nullptr;
    double* x[2] = {nullptr, nullptr};  // parents (current) / next parents, n x d
    int cur = 0;
    double* off = nullptr;              // offspring, n x d
    double* fm = nullptr;               // merged objectives, 2n x m (parents first, algorithms.hpp:351)
    double *lower = nullptr, *upper = nullptr;
    BoundSegments bound_seg;
    uint32_t* idx_dev = nullptr;        // tournament winners, then the selected merged rows
    SortScratch sort;
    std::vector<double> f_host, f_off_device;  // host mirror of fm; the device's own offspring objectives
    std::vector<uint32_t> rank_host, sel_host, pool_idx;
};

}  // namespace temo_b200
