// Host-side (CPU, C++) pieces of the tree build: Chebyshev tables, per-level
// order selection, M2M/L2L shift operators, and the crosswell ray tracer.
// All of it is O(orders^4) or O(nnz(H)) setup work; the O(m k) hot path is on
// the GPU.  Compiled with -ffp-contract=off so the op order mirrors numpy.
#pragma once

#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace hikf {

constexpr int kMaxDepth = 20;         // fmm.py:35
constexpr int kMaxBoostedOrder = 16;  // fmm.py:204

std::vector<double> cheb_nodes(int n);                                  // fmm.py:57-60
// rows = evaluation points, cols = nodes (fmm.py:63-78)
std::vector<double> cheb_weights(const std::vector<double>& x, int n);  // len(x) x n
// Tn[k][j] = T_j(node_k), the node-side table used by the device interp kernel
std::vector<double> cheb_node_table(int n);

double interp_error_estimate(const KParams& k, int n, double h);        // fmm.py:206-225
// orders[lev] for lev in [2, depth] (0 elsewhere), fmm.py:227-244
void select_orders(const KParams& k, int n_cheb, int depth, double root_size, int orders[kMaxDepth + 1]);
// kron(Bx, By) for child parity (cx, cy): (n_child^2 x n_par^2) row-major (fmm.py:264-278)
std::vector<double> shift_operator(int n_par, int n_child, int cx, int cy);

// Straight-ray cell intersection lengths (tomography.py:76-133); CSR with
// sorted column indices and duplicates summed.
int ray_operator(int64_t nx, int64_t ny, double dx, double dy, double x0, double y0, int64_t n, const double* src,
                 const double* rcv, std::vector<int32_t>& indptr, std::vector<int32_t>& indices,
                 std::vector<double>& data);

// 3D extension (no reference; oracle/hikf_oracle3d.py trace_3d): cells x-fastest,
// breakpoints at x / y / z planes, midpoint rule with planes going low,
// length = sqrt((dx dx + dy dy) + dz dz).  n3 / d3 / o3 = cells / spacing / origin.
int ray_operator_3d(const int64_t n3[3], const double d3[3], const double o3[3], int64_t n, const double* src,
                    const double* rcv, std::vector<int32_t>& indptr, std::vector<int32_t>& indices,
                    std::vector<double>& data);
double ray_length_3d(const double* p0, const double* p1);

}  // namespace hikf
