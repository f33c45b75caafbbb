// Launchers of the frame-level / consensus-ADMM kernels (admm.cu).
#pragma once

#include "kernels.hpp"
#include "scene.hpp"

namespace dabd_gpu {

void launch_gather(int n, const int* ibody, const double* q, double* iq, cudaStream_t s);
// x[6 n_rows], p2[6 n_rows] from prev = (x_old, p2_old) through map (-1: zero).
void launch_warm_remap(int n_rows, const int* map, const double* prev, int r_old, double* x,
                       double* p2, cudaStream_t s);
void launch_predict(const SceneView& sc, int n, const int* ibody, const double* iq,
                    const double* qd, double h, double gx, double gy, const double* ifs,
                    double* iqt, cudaStream_t s);
void launch_delta_inf(int n_rows, const int* rinst, const int* rpart, int part_base,
                      const double* a, const double* b, double* out, cudaStream_t s);
void launch_masks(const SceneView& sc, const double* q, const double* planes, int np, double w,
                  uint32_t all, uint32_t* masks, int* err, cudaStream_t s);
void launch_vmax(const SceneView& sc, const double* qd, double* out, cudaStream_t s);
// Halo packet of one replica: q[6], u[6], rho.
constexpr int kHaloStride = 13;

void launch_consensus(int ns, const int* sh, const int* ipart, int part_base, const double* iq,
                      double* iu, const double* irho, const double* iz, const double* remote_lo,
                      const double* remote_hi, int n_lo, double* iznext, double* rb, double* sb,
                      double* rloc, double* sloc, int* err, cudaStream_t s);
void launch_pack_halo(int n, const int* inst, const double* iq, const double* iu,
                      const double* irho, double* out, cudaStream_t s);
void launch_select_commit(const SceneView& sc, const uint32_t* bmask, const int* part_rank,
                          const double* gath, size_t stride, double* q, double* qd,
                          cudaStream_t s);
void launch_merged(int n, const int* ianc, const double* iq, const double* iznext, double* out,
                   cudaStream_t s);
void launch_adapt(int n, const int* ianc, double* irho, const double* irho0, const double* rb,
                  const double* sb, const AdaptParams& a, double* iz, const double* iznext,
                  cudaStream_t s);
void launch_commit(const SceneView& sc, int n, const int* ibody, const int* ipart, const int* ianc,
                   const uint32_t* bmask, double* iq, const double* iznext, const double* q_start,
                   double h, double* q, double* qd, cudaStream_t s);
void launch_accept_copy(int n, const int* ipart, int part_base, const PartState* ps,
                        const double* src, double* dst, cudaStream_t s);

} // namespace dabd_gpu
