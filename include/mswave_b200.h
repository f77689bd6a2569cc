/*
 * mswave_b200.h -- C ABI of the B200-native on-line multiscale S-fraction ROM
 * stepper (arXiv 1604.06750) and its companion fine-grid leapfrog.
 *
 * This is the drop-in boundary.  Every entry point replaces one function of
 * the reference's Eigen-typed C++ API (namespace mswave, /root/reference/proj)
 * and is declared with plain pointers and sizes so any host (the C++ mirror in
 * include/mswave/, ctypes, cgo, JNI) can bind it.  All host arrays are fp64 and
 * little-endian; matrices are column-major exactly like the reference's
 * Eigen::MatrixXd storage, so an archived or in-memory SubdomainROM can be
 * handed over with m.data() pointers and no repacking.
 *
 * Batched sources: the reference API is single-source (step(..., double
 * source_value), msolver.hpp:66).  Here S independent sources are advanced in
 * one pass; the source index is ALWAYS the fastest-varying dimension of every
 * batched host array ([row][s]).  With S = 1 every array degenerates to the
 * reference layout.
 *
 * Return codes mirror the reference's exception classes and CLI exit codes
 * (types.hpp:23-34):
 *   MSW_OK               0
 *   MSW_CONFIG_ERROR     2  -> mswave::ConfigError
 *   MSW_NUMERICAL_ERROR  3  -> mswave::NumericalError
 *   MSW_CUDA_ERROR       4  -> device/runtime failure (no reference analogue)
 * msw_last_error() returns the message of the last failure on this thread;
 * instability messages keep the reference wording
 * "multiscale step: instability at step N" (msolver.cpp:149) and
 * "fine_leapfrog: instability at step N" (reference.cpp:75).
 */
#ifndef MSWAVE_B200_H
#define MSWAVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSW_OK 0
#define MSW_CONFIG_ERROR 2
#define MSW_NUMERICAL_ERROR 3
#define MSW_CUDA_ERROR 4

#define MSW_ABI_VERSION 3

/* ------------------------------------------------------------------------ */
/* Coupled ROM system description (MultiscaleSystem, msolver.hpp:38-46)      */
/* ------------------------------------------------------------------------ */

/*
 * Cells are the reference's SubdomainROM (romgen.hpp:23-45); interfaces are
 * its CoupledInterface (msolver.hpp:16-25).
 *
 * cell_iface_ptr is a CSR row pointer (n_cells + 1 entries) into
 * cell_iface_ids / cell_iface_offsets: for cell c the local interfaces are
 * entries [ptr[c], ptr[c+1]) -- iface_ids ascending as in romgen.cpp:404-412
 * and their block offsets (SubdomainROM::iface_offsets without the trailing
 * total, which is cell_ktilde[c]).
 *
 * ladders: for cell c, starting at cell_ladder_off[c] (in doubles):
 *   ladder[0..m-1]     (L^1..L^m,   SubdomainROM::ladder)      then
 *   ladder_hat[0..m-1] (Lhat^1..Lhat^m, SubdomainROM::ladder_hat),
 * each ktilde x ktilde column-major.
 *
 * iface_cj = -1 marks a single-sided interface (the reference's test
 * fixtures, msolver.hpp:13-15); iface_lj is ignored then.
 *
 * iface_mass: concatenation of the M_f x M_f column-major shared masses
 * (CoupledInterface::mass).  If NULL, msw_create computes them exactly as
 * assemble_system does (msolver.cpp:66-74): mass_form = inv(Lhat^1_i[f,f]) +
 * inv(Lhat^1_j[f,f]) via Cholesky, symmetrised, mass = inv(mass_form),
 * symmetrised.
 */
typedef struct msw_system_desc {
  int32_t n_cells;
  int32_t n_ifaces;
  const int32_t* cell_m;
  const int32_t* cell_ktilde;
  const int32_t* cell_iface_ptr;
  const int32_t* cell_iface_ids;
  const int32_t* cell_iface_offsets;
  const int64_t* cell_ladder_off;
  const double* ladders;
  const int32_t* iface_ci;
  const int32_t* iface_cj;
  const int32_t* iface_li;
  const int32_t* iface_lj;
  const int32_t* iface_size;
  const double* iface_mass; /* may be NULL */
} msw_system_desc;

/* Informational sizes (MultiscaleSystem::reduced_dof / flops_per_step,
 * msolver.cpp:14-29, plus the unique on-line DOF count n_flat, the same as
 * FlatOps::n, msolver.cpp:237-240). */
typedef struct msw_info {
  int64_t n_cells;
  int64_t n_ifaces;
  int64_t n_flat;          /* sum_f M_f + sum_c (m-1) ktilde_c            */
  int64_t reduced_dof;     /* sum_c m ktilde_c (reference definition)       */
  int64_t flops_per_step;  /* reference count, single source (1+3(m-1))    */
  int64_t dense_entries;   /* sum_c (2m-1) kt^2 + sum_f M_f^2 (used/step)   */
  int64_t sources;         /* S currently configured                        */
  int64_t receivers;       /* R currently configured                        */
  int64_t device_bytes;    /* device memory held by the handle              */
  int64_t k1_variant;      /* cell-kernel template instance in use          */
  int64_t k1_source_tile;  /* sources per cell work item                    */
  int64_t k1_panel;        /* ladder columns per smem panel                 */
  int64_t k1_rings;        /* state ring depth * 100 + ladder ring depth    */
  int64_t k1_tune_cached;  /* 1: geometry reused from the tuning cache      */
  double k1_fuse_kappa;    /* re-association sensitivity of the ladders:   *
                            * max ||Lhat|| ||L|| / ||Lhat L|| (Frobenius);  *
                            * the fused cell-kernel family is used only     *
                            * when it is <= 1e3 (well-conditioned ladders)  */
} msw_info;

typedef struct msw_system* msw_handle;

/* ABI version, for loaders. */
int msw_abi_version(void);

/* Last error message of the calling thread ("" if none). */
const char* msw_last_error(void);

/* assemble_system (msolver.cpp:31-106) + one-time upload of the ladders to
 * device-resident storage on `device`.  Validates matching block sizes
 * (msolver.cpp:58-60) and that every cell lists the interface
 * (msolver.cpp:45-52).  The handle starts with S = 1 zero source, R = 0
 * receivers and no state (call msw_make_state). */
int msw_create(const msw_system_desc* desc, int device, msw_handle* out);

/* read_rom_archive (rom_archive.cpp:110-190: manifest.json + cell_%04d.bin
 * containers, same checks and messages) + the on-line load of cmd_simulate
 * (cli_commands.cpp:111-116) without a partition: interface topology from
 * the cells' ascending interface lists, masses from the Lhat^1 blocks
 * (msolver.cpp:66-74), and the archive's own projected source / receiver as
 * S = 1, R = 1 (msolver.cpp:58-64 checks both sides agree bitwise).  Other
 * sources / receivers: project with the archived S_f and call
 * msw_set_sources / msw_set_receivers.  Corner groups need the partition
 * (msw_set_corners). */
int msw_create_from_archive(const char* dir, int device, msw_handle* out);
void msw_destroy(msw_handle h);
int msw_get_info(msw_handle h, msw_info* out);

/* Copies the shared masses / mass forms (concatenated M_f x M_f col-major). */
int msw_get_masses(msw_handle h, double* mass, double* mass_form);

/* Projected sources g~_f (CoupledInterface::g_proj) for S sources:
 * g_proj is [sum_f M_f][S], interface-major (interface f occupies rows
 * [off_f, off_f + M_f) with off_f the prefix sum of M).  Resets the state. */
int msw_set_sources(msw_handle h, int32_t S, const double* g_proj);

/* Receivers: R receivers, receiver r = sum over its terms t in
 * [rcv_ptr[r], rcv_ptr[r+1]) of q_t . ubar_{term_iface[t]}, q_t of length
 * M_{term_iface[t]} stored consecutively in term_q.  This is the sample()
 * of run_simulation (msolver.cpp:405-411) with q_proj nonzero only on the
 * listed interfaces (a skeleton node belongs to one interface after corner
 * removal).  Terms of one receiver are summed in ascending interface order. */
int msw_set_receivers(msw_handle h, int32_t R, const int32_t* rcv_ptr,
                      const int32_t* term_iface, const double* term_q);

/* Corner groups for corner_correct (msolver.cpp:196-227, CornerGroup
 * msolver.hpp:28-36).  grp_ptr: CSR over copies; copy_iface / copy_row /
 * copy_mass per copy.  basis: the interface bases S_f (K_f x M_f col-major,
 * concatenated in interface order), iface_K: K_f per interface. */
int msw_set_corners(msw_handle h, int32_t n_groups, const int32_t* grp_ptr,
                    const int32_t* copy_iface, const int32_t* copy_row,
                    const double* copy_mass, const int32_t* iface_K,
                    const double* basis);

/* make_state (msolver.cpp:108-121): zero state, t = 0, step_index = 0.
 * dt <= 0 -> MSW_CONFIG_ERROR "dt must be positive".
 * The first make_state of a handle also fixes the cell kernel's geometry
 * (template instance, source tile, panel, ring depths): by a device timing of
 * the candidates (a few seconds at the BASELINE sizes), or from the tuning
 * cache when a system of the same shape was tuned before -- in this process,
 * or in any process sharing the file named by the MSW_TUNE_CACHE environment
 * variable.  Every candidate gives the same result bits. */
int msw_make_state(msw_handle h, double dt);

/* One step (msolver.cpp:154-194).  source_values holds w_stride values
 * (1: one wavelet sample shared by all sources, S: one per source).  The
 * instability guard (max|u| > 1e12 or non-finite) returns
 * MSW_NUMERICAL_ERROR with the reference message. */
int msw_step(msw_handle h, const double* source_values, int32_t w_stride);

/* corner_correct (msolver.cpp:196-227) on the current state. */
int msw_corner_correct(msw_handle h);

/* WaveState access (msolver.hpp:53-59).  Layout, S fastest:
 *   u_cur/u_prev  : per cell, m*ktilde rows (layer k at offset (k-1) kt),
 *                   cells concatenated -> [sum_c m kt][S]
 *   ubar_cur/prev : per interface M_f rows -> [sum_f M_f][S]
 * get: any pointer may be NULL.  set: all four arrays required; the
 * layer-1 blocks of u_* are ignored and rebuilt from ubar_* (the
 * conjugation invariant, msolver.hpp:51-52). */
int msw_get_state(msw_handle h, double* u_cur, double* u_prev, double* ubar_cur,
                  double* ubar_prev, double* t, int64_t* step_index);
int msw_set_state(msw_handle h, const double* u_cur, const double* u_prev,
                  const double* ubar_cur, const double* ubar_prev, double t,
                  int64_t step_index);

/* The loop body of run_simulation (msolver.cpp:405-422) from the current
 * state: sample, then `steps` times {step(w[n]); corner_correct if asked;
 * sample}.  w: [steps][w_stride] wavelet samples (the caller evaluates the
 * wavelet at the accumulated time, msolver.cpp:191,415).  traces:
 * [(steps+1)][R][S]; times: steps+1 accumulated times (may be NULL).
 * Host buffers: the copies in and out are part of the call (the e2e path).
 * On instability returns MSW_NUMERICAL_ERROR and *bad_step = first bad step;
 * t and step_index then stand at that step (as the reference's state when it
 * throws), but the device state has run past it, so it is invalidated
 * (MSW_CONFIG_ERROR "wave state ran past an instability" from the calls that
 * read or advance it) until msw_make_state or msw_set_state. */
int msw_run(msw_handle h, int64_t steps, const double* w, int32_t w_stride,
            int32_t corner_correction, double* traces, double* times,
            int64_t* bad_step);

/* Same loop with device-resident w / traces (pointers from cudaMalloc or
 * torch) on the handle's stream or `stream` (a cudaStream_t, may be NULL),
 * asynchronous: no host synchronisation, no instability check (query it
 * with msw_check_instability after synchronising). */
int msw_run_device(msw_handle h, int64_t steps, const double* w_dev,
                   int32_t w_stride, int32_t corner_correction,
                   double* traces_dev, void* stream);
int msw_check_instability(msw_handle h, int64_t* bad_step);

/* estimate_dt (msolver.cpp:349-385) on the device: power iteration on the
 * acceleration operator from the reference's start vector (same stopping
 * rule), Gershgorin row-sum fallback with the operator's columns applied S at
 * a time; returns safety * 2 / sqrt(lambda).  An existing state is kept. */
int msw_estimate_dt(msw_handle h, double safety, double* dt_out);

/* energy (msolver.cpp:387-395) of the current state, one value per source:
 * 0.5 d.M d / dt^2 - 0.5 u_prev.M acc(u_cur), d = u_cur - u_prev, M =
 * mass_form (interfaces) and Lhat^k^-1 (interior layers).  energy_out[S]. */
int msw_energy(msw_handle h, double* energy_out);

/* Instantiate the CUDA graph msw_run / msw_run_device replay (normally done
 * lazily on the first run of >= 16 steps), so that setup cost stays out of a
 * timed region.  Needs a state (msw_make_state). */
int msw_prepare(msw_handle h, int32_t corner_correction);

/* Launch statistics of the last msw_run / msw_run_device call: number of
 * kernel launches this library issued (graph nodes count once per replay). */
int msw_last_launch_count(msw_handle h, int64_t* launches);

/* Profiling aid for the roofline: times `reps` back-to-back launches of
 * each step kernel alone with CUDA events on the handle's stream (after one
 * warm-up launch each).  ms[0] = cell kernel (K1), ms[1] = interface kernel
 * (K2) average per launch.  Leaves the state scrambled: call msw_make_state
 * afterwards. */
int msw_time_kernels(msw_handle h, int32_t reps, double* ms);

/* ------------------------------------------------------------------------ */
/* Fine-grid companion (fine_grid.cpp:58-112, reference.cpp:24-80)           */
/* ------------------------------------------------------------------------ */

typedef struct msw_fine* msw_fine_handle;

/* GridMedium (fine_grid.hpp:14-23): ndim 1..3, dims with the Dirichlet
 * ring, sigma/rho one value per node row-major (axis 0 slowest).  The
 * 3/5/7-point pencil of assemble_nd is applied matrix-free from sigma and
 * rho on the device (same coefficients, bit for bit). */
int msw_fine_create(int32_t ndim, const int32_t* dims, double h,
                    const double* sigma, const double* rho, int device,
                    msw_fine_handle* out);
void msw_fine_destroy(msw_fine_handle f);
/* interior node count n = prod(dims-2) */
int msw_fine_size(msw_fine_handle f, int64_t* n);

/* fine_leapfrog (reference.cpp:49-80) for S sources / R receivers.
 * Sources and receivers are sparse over interior rows (SparsePencil
 * numbering, fine_grid.cpp:29-36): src_ptr CSR over (src_row, src_val);
 * rcv likewise.  w: [steps][w_stride] samples at t_s = s*dt (reference.cpp:67,
 * NOT accumulated).  traces: [(steps+1)][R][S]. */
int msw_fine_leapfrog(msw_fine_handle f, int32_t S, const int32_t* src_ptr,
                      const int64_t* src_row, const double* src_val, int32_t R,
                      const int32_t* rcv_ptr, const int64_t* rcv_row,
                      const double* rcv_val, double dt, int64_t steps,
                      const double* w, int32_t w_stride, double* traces,
                      int64_t* bad_step);

/* Device-resident variant for throughput measurement: w_dev/traces_dev are
 * device pointers, asynchronous on `stream`.  Keeps the wavefield of the
 * previous call unless reset != 0. */
int msw_fine_leapfrog_device(msw_fine_handle f, int32_t S,
                             const int32_t* src_ptr, const int64_t* src_row,
                             const double* src_val, int32_t R,
                             const int32_t* rcv_ptr, const int64_t* rcv_row,
                             const double* rcv_val, double dt, int64_t steps,
                             const double* w_dev, int32_t w_stride,
                             double* traces_dev, int32_t reset, void* stream);
int msw_fine_check_instability(msw_fine_handle f, int64_t* bad_step);

/* A general fine pencil (SparsePencil, fine_grid.hpp:31-41) as the reference
 * holds it: A (n x n) in Eigen's compressed column storage -- outer = the n + 1
 * column pointers, inner = row indices, values (SpMat::outerIndexPtr /
 * innerIndexPtr / valuePtr) -- and the diagonal mass B.  Any sparsity (the
 * corner-modified pencil with hanging copies included).  msw_fine_leapfrog on
 * such a handle sums each row in ascending column order, the order of the
 * reference's A * u (reference.cpp:68), so traces are bit-identical to it;
 * sources / receivers index the pencil's rows. */
int msw_fine_create_csc(int64_t n, const int32_t* outer, const int32_t* inner,
                        const double* values, const double* B, int device,
                        msw_fine_handle* out);

/* fine_cfl (reference.cpp:24-47): largest stable leapfrog step
 * 2 / sqrt(lambda_max(B^-1 (-A))) by power iteration on the device from the
 * reference's start vector sin(0.7 i + 0.3) + 1e-3, stopping when the
 * eigenvalue estimate moves by <= 1e-7 relative after iteration 32 (at most
 * 5000 iterations); Gershgorin row-sum bound if the iteration yields no
 * positive eigenvalue, MSW_NUMERICAL_ERROR "fine_cfl: could not bound the
 * spectrum" if neither does.  Works on either kind of fine handle. */
int msw_fine_cfl(msw_fine_handle f, double* dt_out);

#ifdef __cplusplus
}
#endif

#endif /* MSWAVE_B200_H */
