// decomp.hpp -- host-side load model and k-d tree spatial decomposition
// (§4: "Load costs" P:206-234 and "Tree-based decomposition"
// P:236-252).  Pure host C++; exposed through the C ABI so the multi-GPU
// engine and the tests share one implementation.
#pragma once
#include <cmath>
#include <cstdint>
#include <vector>

namespace mdd {

// Eq. 6: n_d(i) ~ N_i/2 (N_i + sum_{j in neigh(i)} N_j), neigh = the
// 26 adjacent cells (periodic).  counts/cost are x-fastest arrays.
inline void cell_cost(const int32_t* counts, int nx, int ny, int nz, double* cost)
{
    auto at = [&](int x, int y, int z) {
        x = (x + nx) % nx; y = (y + ny) % ny; z = (z + nz) % nz;
        return (double)counts[x + nx * (y + ny * z)];
    };
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                double Ni = at(x, y, z), s = 0.0;
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx)
                            if (dx || dy || dz) s += at(x + dx, y + dy, z + dz);
                cost[x + nx * (y + ny * z)] = 0.5 * Ni * (Ni + s);
            }
}

struct Box {
    int lo[3], hi[3];       // half-open cell ranges
};

// Minimum-imbalance plane along `axis` inside `b` for a (pl, pr) process
// split: minimise |load_l / pl - load_r / pr| over the planes that
// leave >= 2 cells on each side; ties go to the more central plane.
// Returns the plane index (first cell of the right part) or -1.
inline int best_plane(const double* cost, int nx, int ny, const Box& b, int axis, int pl, int pr,
                      double* imbalance)
{
    const int n = b.hi[axis] - b.lo[axis];
    if (n < 4) return -1;
    std::vector<double> prof(n, 0.0);
    for (int z = b.lo[2]; z < b.hi[2]; ++z)
        for (int y = b.lo[1]; y < b.hi[1]; ++y)
            for (int x = b.lo[0]; x < b.hi[0]; ++x) {
                const int c[3] = {x, y, z};
                prof[c[axis] - b.lo[axis]] += cost[x + nx * (y + ny * z)];
            }
    double total = 0.0;
    for (double v : prof) total += v;
    int best = -1;
    double bimb = 0.0, bcen = 0.0;
    double left = 0.0;
    for (int k = 1; k < n; ++k) {
        left += prof[k - 1];
        if (k < 2 || n - k < 2) continue;
        const double imb = std::fabs(left / pl - (total - left) / pr);
        const double cen = std::fabs(k - 0.5 * n);
        if (best < 0 || imb < bimb || (imb == bimb && cen < bcen)) {
            best = k; bimb = imb; bcen = cen;
        }
    }
    if (imbalance) *imbalance = bimb;
    return best < 0 ? -1 : b.lo[axis] + best;
}

// Recursive bisection with alternating axes x -> y -> z by depth (P:248,
// reading A18); if the depth's axis cannot be cut, the next axes are tried.
// Child process counts ceil(p/2), floor(p/2).  Leaves are appended in
// depth-first order (left first) = rank order.  Returns false if the 2-cell
// constraint cannot be met.
inline bool kd_split(const double* cost, int nx, int ny, const Box& b, int p, int depth,
                     std::vector<Box>& leaves)
{
    if (p == 1) {
        leaves.push_back(b);
        return true;
    }
    const int pl = (p + 1) / 2, pr = p / 2;
    for (int t = 0; t < 3; ++t) {
        const int axis = (depth + t) % 3;
        const int k = best_plane(cost, nx, ny, b, axis, pl, pr, nullptr);
        if (k < 0) continue;
        Box L = b, R = b;
        L.hi[axis] = k;
        R.lo[axis] = k;
        return kd_split(cost, nx, ny, L, pl, depth + 1, leaves) && kd_split(cost, nx, ny, R, pr, depth + 1, leaves);
    }
    return false;
}

}  // namespace mdd
