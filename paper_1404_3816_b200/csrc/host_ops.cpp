// Host setup math for the tree build and the ray operator (see host_ops.h).
#include "host_ops.h"

#include <math.h>

#include <algorithm>
#include <cfloat>
#include <cstdarg>
#include <cstdio>

namespace hikf {

std::vector<double> cheb_nodes(int n) {
  std::vector<double> x(n);
  for (int k = 0; k < n; ++k) x[k] = cos(((double)(2 * k + 1) * M_PI) / (double)(2 * n));
  return x;
}

// T_0..T_{n-1} at each point: T_j = (2 x) T_{j-1} - T_{j-2} (numpy's left-to-right order)
static std::vector<double> cheb_table(const std::vector<double>& x, int n) {
  size_t p = x.size();
  std::vector<double> T(p * n);
  for (size_t i = 0; i < p; ++i) {
    double* row = &T[i * n];
    row[0] = 1.0;
    if (n > 1) row[1] = x[i];
    double two_x = 2.0 * x[i];
    for (int j = 2; j < n; ++j) row[j] = two_x * row[j - 1] - row[j - 2];
  }
  return T;
}

std::vector<double> cheb_node_table(int n) { return cheb_table(cheb_nodes(n), n); }

std::vector<double> cheb_weights(const std::vector<double>& x, int n) {
  std::vector<double> tx = cheb_table(x, n), tn = cheb_node_table(n);
  std::vector<double> W(x.size() * n);
  for (size_t i = 0; i < x.size(); ++i)
    for (int k = 0; k < n; ++k) {
      double dot = 0.0;
      for (int j = 1; j < n; ++j) dot += tx[i * n + j] * tn[(size_t)k * n + j];
      W[i * n + k] = (1.0 + 2.0 * dot) / n;
    }
  return W;
}

static double host_dist(double ax, double ay, double bx, double by) {
  double dx = ax - bx, dy = ay - by;
  return sqrt(dx * dx + dy * dy);
}

double interp_error_estimate(const KParams& k, int n, double h) {
  // 9x9 sample grid of the target box and the box two widths to the right
  std::vector<double> u(9), p1(9);
  for (int i = 0; i < 9; ++i) {
    u[i] = (((double)i + 0.5) / 9.0) * 2.0 - 1.0;
    p1[i] = u[i] * (h / 2.0);
  }
  std::vector<double> nd = cheb_nodes(n);
  int q = n * n;
  std::vector<double> w1 = cheb_weights(u, n);  // 9 x n
  // S[(p, r), (i, j)] = w1[p, i] w1[r, j]
  std::vector<double> S(81 * (size_t)q);
  for (int p = 0; p < 9; ++p)
    for (int r = 0; r < 9; ++r)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) S[(size_t)(p * 9 + r) * q + i * n + j] = w1[p * n + i] * w1[r * n + j];
  // node kernel block K(tn_a, tn_b + (2h, 0))
  std::vector<double> Kn((size_t)q * q);
  double shift = 2.0 * h;
  for (int a = 0; a < q; ++a) {
    double ax = nd[a / n] * (h / 2.0), ay = nd[a % n] * (h / 2.0);
    for (int b = 0; b < q; ++b) {
      double bx = nd[b / n] * (h / 2.0) + shift, by = nd[b % n] * (h / 2.0) + 0.0;
      Kn[(size_t)a * q + b] = kernel_of_r(k, host_dist(ax, ay, bx, by));
    }
  }
  // approx = (S Kn) S^T
  std::vector<double> SK(81 * (size_t)q, 0.0);
  for (int r = 0; r < 81; ++r)
    for (int a = 0; a < q; ++a) {
      double s = S[(size_t)r * q + a];
      const double* krow = &Kn[(size_t)a * q];
      double* out = &SK[(size_t)r * q];
      for (int b = 0; b < q; ++b) out[b] += s * krow[b];
    }
  double worst = 0.0;
  for (int r = 0; r < 81; ++r)
    for (int c = 0; c < 81; ++c) {
      double acc = 0.0;
      for (int b = 0; b < q; ++b) acc += SK[(size_t)r * q + b] * S[(size_t)c * q + b];
      double ex = kernel_of_r(k, host_dist(p1[r / 9], p1[r % 9], p1[c / 9] + shift, p1[c % 9] + 0.0));
      worst = std::max(worst, fabs(acc - ex));
    }
  return worst / std::max(k.variance, DBL_MIN);
}

void select_orders(const KParams& k, int n_cheb, int depth, double root_size, int orders[kMaxDepth + 1]) {
  for (int i = 0; i <= kMaxDepth; ++i) orders[i] = 0;
  if (depth < 2) return;
  orders[depth] = n_cheb;
  if (k.family == HIKF_LOGARITHM) {  // scale-free kernel: fixed order
    for (int lev = 2; lev < depth; ++lev) orders[lev] = n_cheb;
    return;
  }
  double base = std::max(interp_error_estimate(k, n_cheb, root_size / (double)(1LL << depth)), 1e-16);
  for (int lev = 2; lev < depth; ++lev) {
    double h = root_size / (double)(1LL << lev);
    int n = n_cheb;
    while (n < kMaxBoostedOrder && interp_error_estimate(k, n, h) > base) ++n;
    orders[lev] = n;
  }
}

std::vector<double> shift_operator(int n_par, int n_child, int cx, int cy) {
  std::vector<double> cn = cheb_nodes(n_child), xs(n_child), ys(n_child);
  for (int i = 0; i < n_child; ++i) {
    xs[i] = (cn[i] + (double)(2 * cx - 1)) / 2.0;
    ys[i] = (cn[i] + (double)(2 * cy - 1)) / 2.0;
  }
  std::vector<double> Bx = cheb_weights(xs, n_par), By = cheb_weights(ys, n_par);
  int qc = n_child * n_child, qp = n_par * n_par;
  std::vector<double> K((size_t)qc * qp);
  for (int i = 0; i < n_child; ++i)
    for (int j = 0; j < n_child; ++j)
      for (int a = 0; a < n_par; ++a)
        for (int b = 0; b < n_par; ++b)
          K[(size_t)(i * n_child + j) * qp + a * n_par + b] = Bx[i * n_par + a] * By[j * n_par + b];
  return K;
}

// ---------------------------------------------------------------------------
// crosswell ray operator
// ---------------------------------------------------------------------------
int ray_operator(int64_t nx, int64_t ny, double dx, double dy, double x0, double y0, int64_t n, const double* src,
                 const double* rcv, std::vector<int32_t>& indptr, std::vector<int32_t>& indices,
                 std::vector<double>& data) {
  if (nx < 1 || ny < 1 || !(dx > 0) || !(dy > 0) || n < 0) {
    set_error("ray_operator: bad grid");
    return HIKF_BAD_ARGUMENT;
  }
  double xmax = x0 + nx * dx, ymax = y0 + ny * dy;
  for (int64_t r = 0; r < n; ++r)
    for (const double* p : {src + 2 * r, rcv + 2 * r})
      if (!(p[0] >= x0 && p[0] <= xmax && p[1] >= y0 && p[1] <= ymax)) {
        set_error("sources/receivers must lie within the grid bounding box");
        return HIKF_BAD_ARGUMENT;
      }
  indptr.assign(n + 1, 0);
  indices.clear();
  data.clear();
  std::vector<double> t;
  std::vector<std::pair<int32_t, double>> row;
  for (int64_t r = 0; r < n; ++r) {
    const double *p0 = src + 2 * r, *p1 = rcv + 2 * r;
    double d0 = p1[0] - p0[0], d1 = p1[1] - p0[1];
    double length = hypot(d0, d1);
    if (length == 0.0) {
      set_error("source coincides with receiver (zero-length ray)");
      return HIKF_BAD_ARGUMENT;
    }
    t.assign({0.0, 1.0});
    if (d0 != 0.0)
      for (int64_t i = 1; i < nx; ++i) {
        double tt = ((x0 + (double)i * dx) - p0[0]) / d0;
        if (tt > 0.0 && tt < 1.0) t.push_back(tt);
      }
    if (d1 != 0.0)
      for (int64_t j = 1; j < ny; ++j) {
        double tt = ((y0 + (double)j * dy) - p0[1]) / d1;
        if (tt > 0.0 && tt < 1.0) t.push_back(tt);
      }
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    row.clear();
    for (size_t s = 0; s + 1 < t.size(); ++s) {
      double seg = (t[s + 1] - t[s]) * length;
      if (!(seg > 0.0)) continue;
      double tm = 0.5 * (t[s] + t[s + 1]);
      double u = ((p0[0] + tm * d0) - x0) / dx, w = ((p0[1] + tm * d1) - y0) / dy;
      int64_t i = (int64_t)floor(u), j = (int64_t)floor(w);
      if ((double)i == u && i > 0) --i;  // grazing: lower/left cell
      if ((double)j == w && j > 0) --j;
      i = std::min<int64_t>(std::max<int64_t>(i, 0), nx - 1);
      j = std::min<int64_t>(std::max<int64_t>(j, 0), ny - 1);
      row.push_back({(int32_t)(j * nx + i), seg});
    }
    std::stable_sort(row.begin(), row.end(),
                     [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) {
                       return a.first < b.first;
                     });
    for (size_t s = 0; s < row.size(); ++s) {
      if (s > 0 && row[s].first == row[s - 1].first) {
        data.back() += row[s].second;
      } else {
        indices.push_back(row[s].first);
        data.push_back(row[s].second);
      }
    }
    indptr[r + 1] = (int32_t)indices.size();
  }
  return HIKF_OK;
}

double ray_length_3d(const double* p0, const double* p1) {
  const double d0 = p1[0] - p0[0], d1 = p1[1] - p0[1], d2 = p1[2] - p0[2];
  return sqrt((d0 * d0 + d1 * d1) + d2 * d2);
}

int ray_operator_3d(const int64_t n3[3], const double d3[3], const double o3[3], int64_t n, const double* src,
                    const double* rcv, std::vector<int32_t>& indptr, std::vector<int32_t>& indices,
                    std::vector<double>& data) {
  for (int a = 0; a < 3; ++a)
    if (n3[a] < 1 || !(d3[a] > 0)) {
      set_error("ray_operator_3d: bad grid");
      return HIKF_BAD_ARGUMENT;
    }
  if (n < 0 || (n3[0] * n3[1] * n3[2]) > INT32_MAX) {
    set_error("ray_operator_3d: bad sizes");
    return HIKF_BAD_ARGUMENT;
  }
  for (int64_t r = 0; r < n; ++r)
    for (const double* p : {src + 3 * r, rcv + 3 * r})
      for (int a = 0; a < 3; ++a)
        if (!(p[a] >= o3[a] && p[a] <= o3[a] + n3[a] * d3[a])) {
          set_error("sources/receivers must lie within the grid bounding box");
          return HIKF_BAD_ARGUMENT;
        }
  indptr.assign(n + 1, 0);
  indices.clear();
  data.clear();
  std::vector<double> t;
  std::vector<std::pair<int32_t, double>> row;
  for (int64_t r = 0; r < n; ++r) {
    const double *p0 = src + 3 * r, *p1 = rcv + 3 * r;
    const double d[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
    const double length = ray_length_3d(p0, p1);
    if (length == 0.0) {
      set_error("source coincides with receiver (zero-length ray)");
      return HIKF_BAD_ARGUMENT;
    }
    t.assign({0.0, 1.0});
    for (int a = 0; a < 3; ++a)
      if (d[a] != 0.0)
        for (int64_t i = 1; i < n3[a]; ++i) {
          const double tt = ((o3[a] + (double)i * d3[a]) - p0[a]) / d[a];
          if (tt > 0.0 && tt < 1.0) t.push_back(tt);
        }
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    row.clear();
    for (size_t s = 0; s + 1 < t.size(); ++s) {
      const double seg = (t[s + 1] - t[s]) * length;
      if (!(seg > 0.0)) continue;
      const double tm = 0.5 * (t[s] + t[s + 1]);
      int64_t c[3];
      for (int a = 0; a < 3; ++a) {
        const double u = ((p0[a] + tm * d[a]) - o3[a]) / d3[a];
        int64_t i = (int64_t)floor(u);
        if ((double)i == u && i > 0) --i;  // on a plane: lower cell
        c[a] = std::min<int64_t>(std::max<int64_t>(i, 0), n3[a] - 1);
      }
      row.push_back({(int32_t)((c[2] * n3[1] + c[1]) * n3[0] + c[0]), seg});
    }
    std::stable_sort(row.begin(), row.end(),
                     [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) {
                       return a.first < b.first;
                     });
    for (size_t s = 0; s < row.size(); ++s) {
      if (s > 0 && row[s].first == row[s - 1].first) {
        data.back() += row[s].second;
      } else {
        indices.push_back(row[s].first);
        data.push_back(row[s].second);
      }
    }
    indptr[r + 1] = (int32_t)indices.size();
  }
  return HIKF_OK;
}

}  // namespace hikf
