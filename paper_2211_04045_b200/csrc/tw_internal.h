// Host-side launchers of the engine kernels (defined in tw_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "tw_engine.cuh"

namespace tw {

// k_unpack + k_edges_init
void launch_setup(cudaStream_t s, int nv, const double* xs, const double* ys, const double* inv_mass,
                  double4* x, double4* yk1, double* r, unsigned long long* dmin, int* voff, int* vcnt,
                  double4* imp, int* nonfinite, int ne, const int2* edges, double* ly, uint8_t* is_er,
                  double* edge_lambda, int* er_color, const int* edge_color, int edge_rows,
                  int device_coloring);

void launch_pack(cudaStream_t s, int nv, const double4* x, double* out);

// LBVH build for one primitive class; tmp must hold cub temp + 4 arrays of n
size_t bvh_tmp_bytes(int n);
void launch_bvh_build(cudaStream_t s, int cls, const Bvh& B, const int4* tris, const int2* edges,
                      const int* iso, const double4* x, int nv, void* tmp, size_t tmp_bytes,
                      unsigned long long* box /* 6, device */);

int launch_count_last();  // kernels launched by the last launcher call
void launch_vertex_order(cudaStream_t s, int nv, const double4* x, void* tmp, size_t tmp_bytes,
                         unsigned long long* box, int* vperm);
// packet compactness of a query class in mesh order vs Morton order (spread[0..1], summed)
void launch_packet_spread(cudaStream_t s, int n, int cls, const int2* edges, const double4* x, const int* perm,
                          double* spread);
void launch_bounds(cudaStream_t s, int nv, const double4* x, unsigned long long* box);

// cooperative kernels
cudaError_t coop_resolve(cudaStream_t s, const Params& P, int nblocks, int minb);
cudaError_t coop_search(cudaStream_t s, const Params& P, int nblocks);
cudaError_t coop_refresh(cudaStream_t s, const Params& P, int nblocks, double bound);
cudaError_t launch_advance(cudaStream_t s, const Params& P, int nblocks);
// stage kernels for stage-by-stage parity (tw_stage_linearize/color/backward)
cudaError_t coop_stage_linearize(cudaStream_t s, const Params& P, int nblocks);
cudaError_t coop_ccd(cudaStream_t s, const Params& P, int nblocks);  // certification of x -> ccd_x1
cudaError_t coop_stage_color(cudaStream_t s, const Params& P, int nblocks, long long nc);
cudaError_t coop_stage_backward(cudaStream_t s, const Params& P, int nblocks, long long nc, int ncol, int mode);
// row stage entries (tw_stage_build_rows / constraint_value / fill_diag)
void launch_build_rows(cudaStream_t s, const double4* x, long long n, const int* kinds, const int* verts,
                       const double* closest, double delta, int gap, int* kind, int* nverts, int* rv, double* value,
                       double* jac, int* flavor, double* ref_volume, double* gw, double* denom);
void launch_value_at(cudaStream_t s, const double4* x, long long n, const int* flavor, const int* nverts,
                     const int* rv, const double* ref_volume, const double* gw, const double* denom,
                     const double* sigma, double* out);
void launch_fill_diag(cudaStream_t s, const double* inv_mass, long long n, const int* nverts, const int* rv,
                      const double* jac, double* diag);
cudaError_t launch_closest(cudaStream_t s, int nv, const double4* x, long long n, const int* kinds,
                           const int* verts, double* out, int* has);
// blocks per SM the resolve kernel instance built for `minb` CTAs/SM keeps resident
int resolve_blocks_per_sm(int minb);

// device-mode edge precoloring: one Jones-Plassmann round; returns via
// *colored the number of edges colored so far (device counter)
void launch_edge_color_round(cudaStream_t s, int ne, const int2* edges, const double* inv_mass,
                             const int* vedge_off, const int* vedge, int* color, int* stamp, int round,
                             int* colored);

}  // namespace tw
