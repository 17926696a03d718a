// Straight-ray operator H on the GPU (tomography.py:76-133).
//
// One CTA per ray.  The gridline crossings t_i = ((x0 + i dx) - p0x) / d
// are generated with the reference's operation order (no FMA contraction),
// block-sorted (CUB BlockRadixSort on the IEEE bit patterns: t is in (0, 1),
// so the bits order like the values) and de-duplicated (np.unique).  Each
// positive-length segment is assigned the cell of its midpoint with the
// grazing rule (on a gridline -> lower/left cell), the (cell, length) pairs
// are stably sorted by cell and duplicates summed in ray order.  The result is
// bit-identical to the host restatement (host_ops.cpp) and to the reference's
// CSR; ray lengths come from the host's hypot so they round like numpy's.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "host_ops.h"
#include "rays.h"

namespace hikf {

namespace {

constexpr int RT = 512;  // threads per ray CTA
constexpr int RIPT = 8;  // items per thread: nx + ny <= 4096 breakpoint candidates per ray

struct RayGrid {
  int64_t n[3];
  double d[3], o[3];
};

// DIM = 2: tomography.py:76-108; DIM = 3: its extension (oracle/hikf_oracle3d.py trace_3d)
template <int DIM>
__global__ void __launch_bounds__(RT) ray_cells_kernel(RayGrid gr, const double* __restrict__ src,
                                                       const double* __restrict__ rcv, const double* __restrict__ len,
                                                       int64_t cap, int32_t* __restrict__ cells,
                                                       double* __restrict__ segs, int32_t* __restrict__ counts) {
  typedef cub::BlockRadixSort<unsigned long long, RT, RIPT> TSort;
  typedef cub::BlockRadixSort<int32_t, RT, RIPT, double> CSort;
  typedef cub::BlockScan<int, RT> Scan;
  // the sorts' temp storage and the breakpoint / cell staging arrays are
  // never live at the same time: alias them (keeps static smem < 48 KB)
  __shared__ union {
    typename TSort::TempStorage ts;
    typename CSort::TempStorage cs;
    double t[RT * RIPT];
    int32_t c[RT * RIPT];
  } u;
  __shared__ typename Scan::TempStorage sc;
  __shared__ int nt;
  double* tsh = u.t;

  const int64_t r = blockIdx.x;
  double p0[DIM], dv[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    p0[a] = src[DIM * r + a];
    dv[a] = __dsub_rn(rcv[DIM * r + a], p0[a]);
  }
  const double length = len[r];
  const int tid = threadIdx.x;

  // ---- candidate breakpoints: 0, 1 and the plane crossings inside (0, 1) ----
  unsigned long long key[RIPT];
  int64_t ncand = 2;
#pragma unroll
  for (int a = 0; a < DIM; ++a) ncand += dv[a] != 0.0 ? gr.n[a] - 1 : 0;
#pragma unroll
  for (int q = 0; q < RIPT; ++q) {
    const int64_t c = (int64_t)tid * RIPT + q;
    double t = 2.0;  // sentinel (sorted last, dropped)
    if (c == 0) {
      t = 0.0;
    } else if (c == 1) {
      t = 1.0;
    } else if (c < ncand) {
      int64_t k = c - 2;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        if (dv[a] == 0.0) continue;
        if (k < gr.n[a] - 1) {
          t = __ddiv_rn(__dsub_rn(__dadd_rn(gr.o[a], __dmul_rn((double)(k + 1), gr.d[a])), p0[a]), dv[a]);
          break;
        }
        k -= gr.n[a] - 1;
      }
      if (!(t > 0.0 && t < 1.0)) t = 2.0;
    }
    key[q] = (unsigned long long)__double_as_longlong(t);  // t >= 0: bit order == value order
  }
  TSort(u.ts).SortBlockedToStriped(key);
  __syncthreads();
  // striped: item q of thread tid is element q * RT + tid
#pragma unroll
  for (int q = 0; q < RIPT; ++q) tsh[q * RT + tid] = __longlong_as_double((long long)key[q]);
  __syncthreads();
  // unique (np.unique) with a block scan: keep t[i] if i == 0 or t[i] != t[i-1]
  int keep[RIPT], tot = 0;
#pragma unroll
  for (int q = 0; q < RIPT; ++q) {
    const int i = tid * RIPT + q;
    const double t = tsh[i];
    keep[q] = (t <= 1.0) && (i == 0 || t != tsh[i - 1]);
    tot += keep[q];
  }
  int off;
  Scan(sc).ExclusiveSum(tot, off);
  __syncthreads();
  double tv[RIPT];
#pragma unroll
  for (int q = 0; q < RIPT; ++q) tv[q] = tsh[tid * RIPT + q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RIPT; ++q)
    if (keep[q]) tsh[off++] = tv[q];
  if (tid == RT - 1) nt = off;
  __syncthreads();
  const int nuniq = nt;

  // ---- segments -> (cell, length) ----
  int32_t ck[RIPT];
  double sv[RIPT];
#pragma unroll
  for (int q = 0; q < RIPT; ++q) {
    const int s = tid * RIPT + q;
    ck[q] = INT32_MAX;
    sv[q] = 0.0;
    if (s + 1 < nuniq) {
      const double ta = tsh[s], tb = tsh[s + 1];
      const double seg = __dmul_rn(__dsub_rn(tb, ta), length);
      if (seg > 0.0) {
        const double tm = __dmul_rn(0.5, __dadd_rn(ta, tb));
        int64_t cell = 0;
#pragma unroll
        for (int a = DIM - 1; a >= 0; --a) {
          const double u = __ddiv_rn(__dsub_rn(__dadd_rn(p0[a], __dmul_rn(tm, dv[a])), gr.o[a]), gr.d[a]);
          int64_t i = (int64_t)floor(u);
          if ((double)i == u && i > 0) --i;  // grazing: lower cell
          i = i < 0 ? 0 : (i > gr.n[a] - 1 ? gr.n[a] - 1 : i);
          cell = cell * gr.n[a] + i;  // x fastest
        }
        ck[q] = (int32_t)cell;
        sv[q] = seg;
      }
    }
  }
  __syncthreads();  // every thread has read the breakpoints out of the aliased buffer
  CSort(u.cs).SortBlockedToStriped(ck, sv);  // stable: equal cells keep ray order
  __syncthreads();
  // sum duplicates in order: stage striped results in shared memory
  int32_t* csh = u.c;
#pragma unroll
  for (int q = 0; q < RIPT; ++q) csh[q * RT + tid] = ck[q];
  __syncthreads();
  double* seg_out = segs + r * cap;  // also the staging area of the sorted lengths
  int32_t* cell_out = cells + r * cap;
  int head[RIPT], nh = 0;
#pragma unroll
  for (int q = 0; q < RIPT; ++q) {
    const int i = tid * RIPT + q;
    const int32_t c = csh[i];
    head[q] = (c != INT32_MAX) && (i == 0 || csh[i - 1] != c);
    nh += head[q];
  }
  // stage the sorted lengths (striped -> blocked) through global scratch
#pragma unroll
  for (int q = 0; q < RIPT; ++q) seg_out[q * RT + tid] = sv[q];
  __syncthreads();
  int hoff;
  Scan(sc).ExclusiveSum(nh, hoff);
  __syncthreads();
  double merged[RIPT];
  int32_t mcell[RIPT];
  int mslot[RIPT];
#pragma unroll
  for (int q = 0; q < RIPT; ++q) {
    mslot[q] = -1;
    const int i = tid * RIPT + q;
    if (!head[q]) continue;
    double s = seg_out[i];
    for (int k = i + 1; k < RT * RIPT && csh[k] == csh[i]; ++k) s += seg_out[k];
    merged[q] = s;
    mcell[q] = csh[i];
    mslot[q] = hoff++;
  }
  __syncthreads();  // all reads of the scratch done before it is overwritten
#pragma unroll
  for (int q = 0; q < RIPT; ++q)
    if (mslot[q] >= 0) {
      seg_out[mslot[q]] = merged[q];
      cell_out[mslot[q]] = mcell[q];
    }
  if (tid == RT - 1) counts[r] = hoff;
}

__global__ void compact_kernel(int64_t n, int64_t cap, const int32_t* __restrict__ cells,
                               const double* __restrict__ segs, const int32_t* __restrict__ indptr,
                               int32_t* __restrict__ indices, double* __restrict__ data) {
  const int64_t r = blockIdx.x;
  const int32_t b = indptr[r], e = indptr[r + 1];
  for (int32_t k = threadIdx.x; k < e - b; k += blockDim.x) {
    indices[b + k] = cells[r * cap + k];
    data[b + k] = segs[r * cap + k];
  }
}

}  // namespace

// shared driver: DIM-D rays with host-computed lengths (validated by the caller)
template <int DIM>
static int ray_driver(const RayGrid& gr, int64_t n, const double* src_host, const double* rcv_host,
                      const std::vector<double>& len, int32_t* indptr_dev, int32_t* indices_dev, double* data_dev,
                      int64_t capacity, int64_t* nnz_out, cudaStream_t st) {
  if (n == 0) {
    HIKF_CHECK_CUDA(cudaMemsetAsync(indptr_dev, 0, sizeof(int32_t), st));
    *nnz_out = 0;
    return HIKF_OK;
  }
  const int64_t cap = RT * RIPT;
  double *d_src, *d_rcv, *d_len, *segs;
  int32_t *cells, *counts;
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&d_src, sizeof(double) * DIM * n, st));
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&d_rcv, sizeof(double) * DIM * n, st));
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&d_len, sizeof(double) * n, st));
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&segs, sizeof(double) * n * cap, st));
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&cells, sizeof(int32_t) * n * cap, st));
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&counts, sizeof(int32_t) * (n + 1), st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(d_src, src_host, sizeof(double) * DIM * n, cudaMemcpyHostToDevice, st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(d_rcv, rcv_host, sizeof(double) * DIM * n, cudaMemcpyHostToDevice, st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(d_len, len.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  ray_cells_kernel<DIM><<<(unsigned)n, RT, 0, st>>>(gr, d_src, d_rcv, d_len, cap, cells, segs, counts);
  HIKF_CHECK_LAUNCH();
  // indptr = exclusive scan of the per-ray counts
  HIKF_CHECK_CUDA(cudaMemsetAsync(indptr_dev, 0, sizeof(int32_t), st));
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, counts, indptr_dev + 1, (int)n, st);
  void* tmp = nullptr;
  HIKF_CHECK_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), st));
  cub::DeviceScan::InclusiveSum(tmp, tb, counts, indptr_dev + 1, (int)n, st);
  int32_t nnz = 0;
  HIKF_CHECK_CUDA(cudaMemcpyAsync(&nnz, indptr_dev + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
  *nnz_out = nnz;
  int s = HIKF_OK;
  if (indices_dev && data_dev) {
    if (nnz > capacity) {
      set_error("ray operator needs %d entries, capacity %lld", nnz, (long long)capacity);
      s = HIKF_BAD_ARGUMENT;
    } else {
      compact_kernel<<<(unsigned)n, 256, 0, st>>>(n, cap, cells, segs, indptr_dev, indices_dev, data_dev);
      HIKF_CHECK_LAUNCH();
    }
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(d_src, st);
  cudaFreeAsync(d_rcv, st);
  cudaFreeAsync(d_len, st);
  cudaFreeAsync(segs, st);
  cudaFreeAsync(cells, st);
  cudaFreeAsync(counts, st);
  return s;
}

int ray_operator_device(int64_t nx, int64_t ny, double dx, double dy, double x0, double y0, int64_t n,
                        const double* src_host, const double* rcv_host, int32_t* indptr_dev, int32_t* indices_dev,
                        double* data_dev, int64_t capacity, int64_t* nnz_out, cudaStream_t st) {
  if (nx < 1 || ny < 1 || !(dx > 0) || !(dy > 0) || n < 0) {
    set_error("ray_operator: bad grid");
    return HIKF_BAD_ARGUMENT;
  }
  if (nx + ny > (int64_t)RT * RIPT) {
    set_error("device ray operator supports nx + ny <= %d", RT * RIPT);
    return HIKF_BAD_ARGUMENT;
  }
  const double xmax = x0 + nx * dx, ymax = y0 + ny * dy;
  std::vector<double> len(std::max<int64_t>(n, 1));
  for (int64_t r = 0; r < n; ++r) {
    for (const double* p : {src_host + 2 * r, rcv_host + 2 * r})
      if (!(p[0] >= x0 && p[0] <= xmax && p[1] >= y0 && p[1] <= ymax)) {
        set_error("sources/receivers must lie within the grid bounding box");
        return HIKF_BAD_ARGUMENT;
      }
    len[r] = hypot(rcv_host[2 * r] - src_host[2 * r], rcv_host[2 * r + 1] - src_host[2 * r + 1]);
    if (len[r] == 0.0) {
      set_error("source coincides with receiver (zero-length ray)");
      return HIKF_BAD_ARGUMENT;
    }
  }
  RayGrid gr{{nx, ny, 1}, {dx, dy, 1.0}, {x0, y0, 0.0}};
  return ray_driver<2>(gr, n, src_host, rcv_host, len, indptr_dev, indices_dev, data_dev, capacity, nnz_out, st);
}

int ray_operator_3d_device(const int64_t n3[3], const double d3[3], const double o3[3], int64_t n,
                           const double* src_host, const double* rcv_host, int32_t* indptr_dev, int32_t* indices_dev,
                           double* data_dev, int64_t capacity, int64_t* nnz_out, cudaStream_t st) {
  for (int a = 0; a < 3; ++a)
    if (n3[a] < 1 || !(d3[a] > 0)) {
      set_error("ray_operator_3d: bad grid");
      return HIKF_BAD_ARGUMENT;
    }
  if (n < 0 || n3[0] + n3[1] + n3[2] > (int64_t)RT * RIPT + 1 || n3[0] * n3[1] * n3[2] > INT32_MAX) {
    set_error("device 3D ray operator supports nx + ny + nz <= %d", RT * RIPT + 1);
    return HIKF_BAD_ARGUMENT;
  }
  std::vector<double> len(std::max<int64_t>(n, 1));
  for (int64_t r = 0; r < n; ++r) {
    for (const double* p : {src_host + 3 * r, rcv_host + 3 * r})
      for (int a = 0; a < 3; ++a)
        if (!(p[a] >= o3[a] && p[a] <= o3[a] + n3[a] * d3[a])) {
          set_error("sources/receivers must lie within the grid bounding box");
          return HIKF_BAD_ARGUMENT;
        }
    len[r] = ray_length_3d(src_host + 3 * r, rcv_host + 3 * r);
    if (len[r] == 0.0) {
      set_error("source coincides with receiver (zero-length ray)");
      return HIKF_BAD_ARGUMENT;
    }
  }
  RayGrid gr{{n3[0], n3[1], n3[2]}, {d3[0], d3[1], d3[2]}, {o3[0], o3[1], o3[2]}};
  return ray_driver<3>(gr, n, src_host, rcv_host, len, indptr_dev, indices_dev, data_dev, capacity, nnz_out, st);
}

}  // namespace hikf
