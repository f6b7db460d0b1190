/*
 * spc_oracle.h -- CPU oracle for the Spira SpC hot path (arXiv 2511.20834).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2511_20834_b200/), and it is
 * written from the paper's DEFINITIONS, not from its algorithm:
 *
 *   - canonical order        : lexicographic order of integer tuples (b,x,y,z)   (§5.2)
 *   - packed key (A1)        : the biased-field encoding of DESIGN.md §2 reading R3
 *                              (§5.3 field order; bias = reading A3)
 *   - downsampling Eq. (1)   : V_q = floor(V_p / s_q) * s_q, unique             (§2.1)
 *   - offsets Delta(K,s_p)   : K^3 offsets, lexicographic (dx,dy,dz)             (§2.1)
 *   - kernel map             : M[i,k] = j iff p_j = q_i + delta_k (hash-set lookup, the
 *                              indicator of Eq. (2))                             (§2.2)
 *   - features Eq. (2)       : f_i = sum_k sum_j 1[p_j = q_i + delta_k] f_j W_k  in fp64
 *                                                                                (§2.1)
 *   - voxelization           : v = floor(p_raw / g), unique, mean feature        (§2.1)
 *
 * Coordinates are int32 rows (b, x, y, z).  Index spaces are positions in the
 * canonical (sorted) order of each coordinate set.  All functions are
 * single-threaded and allocate with malloc; negative return = error.
 */
#ifndef SPC_ORACLE_H
#define SPC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Canonical order: sorted[pos] = coords[perm[pos]], lexicographic (b,x,y,z),
 * stable.  Returns the number of adjacent duplicate rows after sorting. */
int64_t orc_sort_coords(const int32_t *coords, int64_t n, int32_t *sorted_out, int32_t *perm_out);

/* A1 key (R3): key = b<<(Bx+By+Bz) | (x+2^(Bx-1))<<(By+Bz) | (y+2^(By-1))<<Bz | (z+2^(Bz-1)).
 * Returns the number of rows whose fields do not fit (those keys are set to 0). */
int64_t orc_pack(const int32_t *coords, int64_t n, int bits_b, int bits_x, int bits_y, int bits_z,
                 uint64_t *keys_out);

/* floor(v / s) * s, floor toward -infinity (P:96 floor, Eq. 1). */
int32_t orc_round_down(int32_t v, int32_t s);

/* Eq. (1): V_s = sorted unique { (b, floor(x/s)s, floor(y/s)s, floor(z/s)s) }.
 * out has room for n rows.  Returns |V_s|. */
int64_t orc_downsample(const int32_t *coords, int64_t n, int32_t s, int32_t *out);

/* Delta(K, spacing) in lexicographic (dx,dy,dz) order, dz fastest:
 * off[k] = (ex,ey,ez)*spacing with e in {-(K-1)/2 .. (K-1)/2}.  l1_units[k] = |ex|+|ey|+|ez|.
 * Returns K^3, or -1 for even / non-positive K. */
int orc_offsets(int K, int spacing, int32_t *off_out, int32_t *l1_units_out);

/* Kernel map by hash-set lookup.  Normal layer: triple (k, i, j) iff
 * in[j] = out[i] + delta_k.  Transposed layer (out = fine, in = coarse; same weight
 * index as the strided layer it inverts): triple iff in[j] = out[i] - delta_k.
 * Both coordinate sets must be canonical (sorted, unique).  Triples are written in
 * (k, i, j) lexicographic order, at most cap of them.  Returns nnz (may exceed cap). */
int64_t orc_kmap(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                 int K, int spacing, int transposed, int32_t *triples, int64_t cap);

/* Eq. (2) in fp64.  F_in [n_in][c_in], W [K^3][c_in][c_out], F_out [n_out][c_out].
 * order = 0: output-stationary loop order (i -> k -> j); order = 1: weight-stationary
 * loop order (k -> i -> j).  Returns nnz or -1. */
int64_t orc_conv(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                 int K, int spacing, int transposed, const double *F_in, int c_in,
                 const double *W, int c_out, double *F_out, int order);

/* Eq. (2) for a subset of output rows only (sampled parity at full sizes):
 * F_out[r] = f_{rows[r]}.  Returns the number of (row, k) matches. */
int64_t orc_conv_rows(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords,
                      const int64_t *rows, int64_t n_rows, int K, int spacing, int transposed,
                      const double *F_in, int c_in, const double *W, int c_out, double *F_out);

/* the generalised offset box -- K_a offsets per axis, odd K_a centred as
 * in Delta(K, s_p), even K_a = {0 .. K_a-1} (reading E1) -- and the
 * kernel map / Eq. (2) over it (same semantics as the cubic odd functions above). */
int orc_offsets3(int kx, int ky, int kz, int spacing, int32_t *off_out, int32_t *l1_units_out);
int64_t orc_kmap3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                  int kx, int ky, int kz, int spacing, int transposed, int32_t *triples, int64_t cap);
int64_t orc_conv3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                  int kx, int ky, int kz, int spacing, int transposed, const double *F_in, int c_in,
                  const double *W, int c_out, double *F_out, int order);
int64_t orc_conv_rows3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords,
                       const int64_t *rows, int64_t n_rows, int kx, int ky, int kz, int spacing, int transposed,
                       const double *F_in, int c_in, const double *W, int c_out, double *F_out);
/* spconv "regular" output sites: sorted unique { (b, p - delta) on the out_stride lattice }. */
int64_t orc_regular_outputs(const int32_t *in_coords, int64_t n, int kx, int ky, int kz, int spacing,
                            int out_stride, int32_t *out);

/* Voxelization: v = floor(p_raw / g) per axis (§2.1), the
 * quotient taken in float32 (the points are float32; reading V1) and floored
 * toward -infinity.  Point i: coordinates pts[i*ld + 0..2], batch b_i = batch[i] (batch
 * NULL: 0).  The voxel set is the canonical (sorted, unique) set of rows (b_i, v_i)
 * written to coords_out [n][4]; point_voxel[i] = the position of point i's row in it;
 * feats_out[v][0..c) = the mean of feats[i*ld_f + 0..c) over the points of voxel v
 * (duplicate voxels averaged), summed in fp64 in ascending point index.  feats /
 * feats_out / point_voxel may be NULL.  Returns the voxel count, or -(1 + i) for the
 * first point i whose coordinates are not finite or whose quotient leaves int32. */
int64_t orc_voxelize(const float *pts, int64_t ld, const int32_t *batch, int64_t n, const float *g,
                     const float *feats, int64_t ld_f, int c, int32_t *coords_out, int32_t *point_voxel,
                     double *feats_out);

/* SURVEY NEXT-4 training path (beyond the paper's inference scope): the gradients of
 * Eq. (2) (§2.1), f_out_i = sum_k sum_j 1[p_j = q_i + delta_k] f_j W_k, written
 * as their definitions with the same map semantics (box, spacing, transposed) as orc_conv3:
 *   dgrad : dF_in[j][c]    = sum over matches (i, j, k) of sum_o dF_out[i][o] * W[k][c][o]
 *   wgrad : dW[k][c][o]    = sum over matches (i, j, k) of F_in[j][c] * dF_out[i][o]
 * dgrad loops over outputs and scatters into dF_in (hash on the input set);
 * dgrad_rows computes chosen input rows by GATHER instead (hash on the output set: output
 * q_i = p_j - delta_k, or p_j + delta_k for a transposed map) -- the two loop orders meet
 * only in the definition.  dW / dF_in are overwritten.  Return nnz or -1. */
int64_t orc_conv_dgrad3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                        int kx, int ky, int kz, int spacing, int transposed, const double *dF_out, int c_out,
                        const double *W, int c_in, double *dF_in);
int64_t orc_conv_dgrad_rows3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                             const int64_t *rows, int64_t n_rows, int kx, int ky, int kz, int spacing,
                             int transposed, const double *dF_out, int c_out, const double *W, int c_in,
                             double *dF_in_rows);
int64_t orc_conv_wgrad3(const int32_t *in_coords, int64_t n_in, const int32_t *out_coords, int64_t n_out,
                        int kx, int ky, int kz, int spacing, int transposed, const double *F_in, int c_in,
                        const double *dF_out, int c_out, double *dW);

/* SURVEY NEXT-4 fused epilogue: inference batch normalisation, residual add and ReLU in
 * the order of the networks' residual blocks (TorchSparse / MinkowskiEngine
 * ResidualBlock: relu(bn(conv(x)) + shortcut)):
 *   y[i][c] = (x[i][c] - mean[c]) / sqrt(var[c] + eps) * gamma[c] + beta[c]
 *             (+ residual[i][c] if residual != NULL),   then max(y, 0) if relu != 0.
 * gamma == NULL skips the normalisation (y = x).  x and y may alias. */
void orc_bn_relu(const double *x, int64_t n, int c, const double *gamma, const double *beta, const double *mean,
                 const double *var, double eps, const double *residual, int relu, double *y);

/* Threads the Eq. (2) row loops use: 1 in the plain build (liboracle.so), the OpenMP
 * thread count in liboracle_omp.so (same arithmetic per row, rows in parallel). */
int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
