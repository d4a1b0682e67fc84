// Hierarchical direction index over the reference vectors (see vecindex.cu).
#pragma once

#include <vector>

#include "internal.h"

namespace temo_b200 {

struct VecIndex {
    static constexpr int kMaxLevels = 4;  // 32^4 = 1M vectors below one top node; more just widens the top loop
    uint64_t r = 0, m = 0;
    int levels = 0;
    uint32_t* orig = nullptr;  // [r] original index of the vector at permuted position p
    double* vp = nullptr;      // [r x (m+1)] permuted vectors with their norms
    uint64_t count[kMaxLevels + 1] = {0, 0, 0, 0, 0};
    double* node[kMaxLevels + 1] = {nullptr, nullptr, nullptr, nullptr, nullptr};      // [count x (m+3)]
    uint32_t* centre[kMaxLevels + 1] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // [count] centre position
    uint32_t* flags = nullptr;  // device: bit0 = some component of V is negative / NaN (no pruning)
    bool ordered = false, built = false;

    void alloc(uint64_t r_, uint64_t m_);
    void release();
    void set_order(const double* v_host, cudaStream_t s);  // Morton order of the (initial) vectors
    void build(const double* v, const double* vn, cudaStream_t s);
};

std::vector<uint32_t> morton_order(const double* v, uint64_t r, uint64_t m);

void launch_assoc_indexed(const double* f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m, const double* z,
                          VecIndex& index, const double* gamma, double penalty, uint32_t* assoc, double* theta,
                          double* apd, unsigned long long* best_key, uint32_t* first_row, cudaStream_t s,
                          uint32_t row0 = 0);
void launch_gamma_indexed(const double* v, const double* vn, uint64_t r, uint64_t m, VecIndex& index, double* gamma,
                          uint32_t* err_flag, const uint32_t* skip_flag, cudaStream_t s);

}  // namespace temo_b200
