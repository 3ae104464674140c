/*
 * qfb200.h -- C ABI of the B200 batched state-vector engine (libqfb200.so).
 *
 * The reference (qcflow, pure Python) has no FFI; its operator API is a set of
 * Python functions.  This header is the C boundary those functions are rebuilt
 * on: every entry point is extern "C", takes plain device pointers / sizes and
 * a cudaStream_t (as void*), is stream-ordered, never allocates persistent
 * device memory and never frees caller memory.  Status: 0 = ok, otherwise an
 * error code; qf_last_error() returns a thread-local message that the Python
 * host maps onto the reference's exception classes (ValueError / KeyError /
 * MemoryError / AssertionError).
 *
 * Which reference interface each entry replaces:
 *   qf_build_ops      gate_matrix + fuse_resolved   qcflow/circuit.py:281-309, fusion.py:78-176
 *   qf_run_passes     run_ops / apply_matrix / simulate / expectation
 *                                                   qcflow/sim.py:88-150, :177-213
 *   qf_adjoint_passes (new) adjoint differentiator; oracle = parameter_shift_grad
 *                                                   qcflow/gradients.py:158-165, 241-326
 *   qf_reduce_slots   _pairwise_sum over terms / PS accumulation
 *                                                   qcflow/sim.py:162-174, gradients.py:321
 *   qf_pauli_expect   pauli_term_values + expectation  qcflow/sim.py:177-213
 *   qf_pauli_apply    (H|psi>, adjoint seed)        index/phase form of qcflow/sim.py:183-196
 *   qf_sample         _draw_bits / sample            qcflow/sim.py:216-227, rng.py:14-19
 *   qf_frame_walk     per-row Pauli-frame re-factorisation of the gate_matrix products
 *                                                   qcflow/circuit.py:281-309 (exact, see planner.py)
 *   qf_reduce_slots_scaled  _pairwise_sum with per-row frame scales  qcflow/sim.py:162-174
 *   qf_jit_*          compile / load / launch the plan-specialised pass kernels (jit.py)
 */
#ifndef QFB200_H
#define QFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- device program descriptors (all-int32 layouts, mirrored in planner.py) ---- */

#define QF_MAX_R 8
#define QF_LANE_Q 4   /* qubits 0..3 are lane bits at every load/store */
#define QF_MAX_T 16
#define QF_MAX_Q 40

enum {
  QF_OP_DENSE1 = 1,   /* 2x2 unitary on register slot s0 */
  QF_OP_DENSE2 = 2,   /* 4x4 unitary on register slots (s0 = MSB, s1), s0 < s1 */
  QF_OP_DIAG = 3,     /* phase polynomial exp(-i sum_k theta_k Z-string_k) */
  QF_OP_OBS = 4,      /* diagonal observable: expectation slot (and lambda = H psi in adjoint) */
};

enum { QF_INIT_LOAD = 0, QF_INIT_ZERO = 1, QF_INIT_PRODUCT = 2, QF_INIT_LOAD_PSI = 3 };

typedef struct QfStage {
  int32_t reg_glob[QF_MAX_R];   /* global bit position of register slot j */
  int32_t thr_glob[QF_MAX_T];   /* global bit position of thread slot i (lane bits first) */
  int32_t reg_phys[QF_MAX_R];   /* swizzled smem offset contributed by register slot j */
  int32_t thr_phys[QF_MAX_T];   /* swizzled smem offset contributed by thread slot i */
  int32_t op_begin, op_end;
  int32_t pad[14];
} QfStage;                       /* 64 x int32 */

typedef struct QfOp {
  int32_t kind, s0, s1;
  int32_t mat;                   /* DENSE: offset (complex units) into the row's matrix slab */
  int32_t term_begin, term_end;  /* DIAG/OBS: term range (sorted by register subset) */
  int32_t grp;                   /* DIAG/OBS: offset of the 2^R+1 subset-boundary table */
  int32_t slot;                  /* gradient / expectation slot, -1 = none */
  int32_t gen;                   /* ADJ dense gradient: generator matrix offset (complex units) */
  int32_t cls;                   /* DENSE1 matrix class: 0 general, 1 [[a,ib],[ic,d]], 2 real */
  int32_t gkind;                 /* ADJ DENSE1 generator: 0 matrix, 1 X, 2 Y, 3 Z (scale = complex genmats[gen + 4].x) */
  int32_t pad[5];
} QfOp;                          /* 16 x int32 */

typedef struct QfPass {
  int32_t stage_begin, stage_end;
  int32_t init, store;
  int32_t mat_begin, mat_end;    /* matrix slab range used by this pass (complex units) */
  int32_t ang_begin, ang_end;    /* angle columns used by this pass */
  int32_t slot_begin, slot_end;  /* slots written by this pass */
  int32_t n_outer;
  int32_t coef_begin, coef_end;  /* observable coefficient columns */
  int32_t L;
  int32_t term_begin, term_end;  /* phase-polynomial / observable terms of this pass */
  int32_t outer_pos[32];         /* global positions of the n-L non-tile bits */
  int32_t init_mat[32];          /* product init: matrix offset of qubit q's leading 2x2, -1 = |0> */
  int32_t grp_begin, grp_end;    /* subset-boundary tables of this pass */
  int32_t op_begin, op_end;      /* ops of this pass */
  int32_t store_pos[16];         /* relabelled passes: physical bit local tile bit i is stored to */
  int32_t pad1[26];
  int32_t relabelled;            /* 1: the pass stores its tile permuted (plan-specialised kernels only) */
  int32_t pad2;
} QfPass;                        /* 128 x int32 */

/* Everything one pass launch needs; pointers are device pointers. */
typedef struct QfProgram {
  const QfPass* passes;
  const QfStage* stages;
  const QfOp* ops;
  const uint32_t* term_mask;     /* Z-string masks (global bits, n <= 32) */
  const int32_t* term_idx;       /* angle column (DIAG) or coefficient column (OBS) */
  const float* term_w;           /* ADJ: gradient weight 2*coeff*beta_k per term */
  const int32_t* grp;            /* subset-boundary tables */
  const float* genmats;          /* ADJ: generator matrices (interleaved complex64) */
  int32_t n_passes;
  int32_t n_slots;               /* total slots (gradient + expectation) */
  int32_t n_mat;                 /* complex entries per row in the matrix slab */
  int32_t n_ang;                 /* angle columns per row */
  int32_t n_coef;                /* observable coefficient columns per row */
  int32_t L, R;                  /* tile bits / register bits used by every pass */
  int32_t coef_row_stride;       /* 0 = coefficients broadcast over rows */
  const QfPass* host_passes;     /* host copy of `passes` (launch geometry / smem sizing) */
} QfProgram;

/* Recipe for per-row matrices / angles (qf_build_ops). */
typedef struct QfBuildRecipe {
  int32_t n_gen;                 /* symbolic generator-exponential gates */
  const int32_t* gen_sym;        /* [n_gen] symbol column */
  const double* gen_coeff;       /* [n_gen] exponent coeff */
  const double* gen_const;       /* [n_gen] exponent const */
  const int32_t* gen_dim;        /* [n_gen] 2 or 4 */
  const double* gen_eval;        /* [n_gen*4] eigenvalues of the generator (incl. identity part) */
  const double* gen_evec;        /* [n_gen*16*2] eigenvectors, row-major complex (re,im) */
  int32_t n_fixed;               /* concrete gates */
  const double* fixed;           /* [fixed_rows, n_fixed, 16, 2] complex128 */
  int32_t fixed_rows;            /* 1 (broadcast) or rows */
  int32_t n_dense;               /* dense ops to build */
  const int32_t* dense_mat;      /* [n_dense] output offset (complex units) */
  const int32_t* dense_dim;      /* [n_dense] 2 or 4 */
  const int32_t* dense_fbeg;     /* [n_dense+1] factor range */
  const int32_t* factor;         /* [n_factors*3]: (src_kind 0=gen 1=fixed, src index, embed) */
  int32_t n_terms;               /* diagonal angle columns */
  const int32_t* term_src;       /* [n_terms*2]: (src_kind 0=gen 1=const, index) */
  const double* term_beta;       /* [n_terms] beta (gen) */
  const double* term_const;      /* [const_rows, n_const] constant angles */
  int32_t const_rows;            /* 1 or rows */
  int32_t n_const;
  int32_t max_dim;               /* largest dense_dim (threads per op in the build); 0 = 4 */
} QfBuildRecipe;

const char* qf_last_error(void);
int qf_version(void);
int qf_device_sm_count(int device);

/* Per-row op matrices (complex64 slab [rows, n_mat]) and angles (int32 turns [rows, n_ang])
 * from symbol values theta [rows, n_sym] (float32, row stride theta_stride). */
int qf_build_ops(const QfBuildRecipe* recipe, const float* theta, int64_t theta_stride, int rows,
                 float* mats, int n_mat, int32_t* angles, int n_ang, void* stream);

/* Forward passes [pass_begin, pass_end) over psi [rows, 2^n] (complex64 interleaved). */
int qf_run_passes(const QfProgram* prog, int pass_begin, int pass_end, float* psi, int n,
                  int rows, const float* mats, const int32_t* angles, const float* coefs,
                  double* partials, int tiles_per_row, void* stream);

/* Adjoint backward passes, executed in order pass_begin..pass_end-1 of the backward program. */
int qf_adjoint_passes(const QfProgram* prog, int pass_begin, int pass_end, float* psi, float* lam,
                      int n, int rows, const float* mats, const int32_t* angles,
                      const float* coefs, double* partials, int tiles_per_row, void* stream);

/* out[row, col] (+)= sum over slots of column col (CSR col_ptr/slot_list) of sum_tile partials. */
int qf_reduce_slots(const double* partials, int rows, int n_slots, int tiles,
                    const int32_t* col_ptr, const int32_t* slot_list, int n_cols, double* out,
                    int accumulate, void* stream);

/* As qf_reduce_slots, each slot's sum multiplied by slot_scale[row, slot] (the Pauli-frame
 * scale written by qf_frame_walk).  Same reference role as qf_reduce_slots. */
int qf_reduce_slots_scaled(const double* partials, int rows, int n_slots, int tiles,
                           const int32_t* col_ptr, const int32_t* slot_list, int n_cols, double* out,
                           int accumulate, const double* slot_scale, void* stream);

/* As qf_reduce_slots_scaled, plus col_offset[col] (nullable) added to every row's column:
 * the identity terms of an observable (exact constants, qcflow/sim.py:203-213) folded into
 * the reduction, so out needs no zero-fill or separate add. */
int qf_reduce_slots_offset(const double* partials, int rows, int n_slots, int tiles,
                           const int32_t* col_ptr, const int32_t* slot_list, int n_cols, double* out,
                           int accumulate, const double* slot_scale, const double* col_offset, void* stream);

/* Per-row Pauli frame of a normalised program: true state = sqrt(m) X^x Z^z stored state
 * (up to a global phase). */
typedef struct QfFrame {
  uint32_t x;
  uint32_t z;
  double m;
} QfFrame;

/* Pauli-frame walk over a program's events [n_events, 8] (planner.build_program frame=True),
 * in execution order, one thread per row: rewrites normalised rotation matrices to their
 * tau form, folds the frame into general dense matrices, writes the frame x-masks into the
 * angle table and the slot scales [rows, n_slots].  frame_in (nullable) = the forward
 * program's frame_out for the adjoint sweep.  Part of gate_matrix/fuse per row
 * (qcflow/circuit.py:281-309, fusion.py:78-176): an exact re-factorisation, not a new op. */
int qf_frame_walk(const int32_t* events, int n_events, int adjoint, int rows, float* mats, int n_mat,
                  int32_t* angles, int n_ang, double* slot_scale, int n_slots, const QfFrame* frame_in,
                  QfFrame* frame_out, void* stream);

/* qf_frame_walk for checkpointed adjoint sweeps: pass-boundary events record the stored
 * state's scale per forward pass into pass_m [rows, n_pass] (forward) or reload it from there
 * (adjoint, whose passes read psi from the forward's pass outputs).  n_stage (0 = n_mat): the
 * prefix of each row's slab the events touch, staged in shared memory (a block-fused adjoint's
 * per-factor matrices follow it). */
int qf_frame_walk_ckpt(const int32_t* events, int n_events, int adjoint, int rows, float* mats, int n_mat,
                       int32_t* angles, int n_ang, double* slot_scale, int n_slots, const QfFrame* frame_in,
                       QfFrame* frame_out, double* pass_m, int n_pass, int n_stage, void* stream);

/* Block-fused adjoint (planner.build_program(block=True)): per (row, block) the gradient
 * value Tr(W_f^dag G_f W_f A) of every factor f of a fused dense block from the block's
 * two-point matrix A (slots of ``a`` [rows, n_a], reduced from the adjoint's partials).
 * blocks [n_blocks, 4] = (factor begin, factor end, D, first A slot); factors [n_factors, 3]
 * = (matrix offset in mats, generator offset in gens or -1, symbol column); gens: complex
 * D x D generators (interleaved fp64); out [rows, n_factors].  Replaces the per-gate
 * Im<lambda|G|psi> loop of the adjoint differentiator for fused blocks. */
int qf_block_grads(const int32_t* blocks, int n_blocks, const int32_t* factors, int n_factors, const double* gens,
                   const float* mats, int n_mat, const double* a, int n_a, double* out, int rows, void* stream);

/* Generic Pauli-sum expectation partials: partials[row, k, chunk] = coef[row, k] *
 * sum_{x in chunk} Re(conj(psi[x ^ xm_k]) i^{ny_k} (-1)^{popc(x & zm_k)} psi[x]);
 * chunks = ceil(2^n / 2048).  Sum with qf_reduce_slots (slots = terms, tiles = chunks).
 * coef_stride 0 = coefficients broadcast over rows. */
int qf_pauli_expect(const float* psi, int n, int rows, int n_terms, const uint32_t* xmask,
                    const uint32_t* zmask, const int32_t* ny, const float* coefs,
                    int64_t coef_stride, double* partials, void* stream);

/* lam = H psi for a per-row weighted Pauli sum (adjoint seed for non-diagonal H). */
int qf_pauli_apply(const float* psi, float* lam, int n, int rows, int n_terms,
                   const uint32_t* xmask, const uint32_t* zmask, const int32_t* ny,
                   const float* coefs, int64_t coef_stride, void* stream);

/* Shot sampler: numpy Generator(Philox).choice(2^n, shots, p=|a|^2/sum) semantics.
 * keys [rows*2] uint64 Philox keys, ctr0 [rows] counter of the first block used (numpy's
 * Philox starts at counter 1), out_idx [rows, shots] int64.  scratch: >= rows*(2^n/1024+2) doubles. */
int qf_sample(const float* psi, int n, int rows, int shots, const uint64_t* keys,
              double* scratch, int64_t* out_idx, int32_t* near_boundary, void* stream);

/* qf_sample with keys_per_row substreams per state row: keys [rows*keys_per_row*2],
 * out_idx [rows, keys_per_row, shots], near_boundary [rows*keys_per_row].  One CDF per row
 * serves every key: sampled_expectation draws each Pauli term k of a basis with
 * substream(seed, k) from the same state (qcflow/sim.py:245-272). */
int qf_sample_multi(const float* psi, int n, int rows, int keys_per_row, int shots, const uint64_t* keys,
                    double* scratch, int64_t* out_idx, int32_t* near_boundary, void* stream);

/* State of a relabelled program (planner.plan_passes_remap: qubit q on physical bit pos[q],
 * host array [n]) back to the logical layout: out[row, j] = in[row, i], bit pos[q] of i = bit q
 * of j.  The StateVector the reference's simulate returns (qcflow/sim.py:139-150) is logical. */
int qf_permute_bits(const float* in, float* out, int n, int rows, const int32_t* pos, void* stream);

/* ---- tensor-core dense blocks (prototype, csrc/qf_tc.cu) ----
 * A 16 x 16 complex unitary on qubits 0..3 of a [rows, 2^n] complex64 state (n in [11, 32]) on
 * the tcgen05 tensor cores: kind::tf32 MMAs (M=128, N=32, K=32 in real form) with 3xTF32 error
 * compensation, TMEM accumulators.  The gate-apply of sim.apply_matrix (qcflow/sim.py:88-105)
 * for a dense 4-qubit block.  qf_dense4_tc_prepare (host) builds the B operand image
 * [2][32][32] floats (tf32 hi, lo parts) from U as (re, im) doubles, row-major; the caller
 * copies it to the device.  in == out is allowed. */
int qf_dense4_tc_prepare(const double* u, float* out);
int qf_dense4_tc(const float* in, float* out, int n, int rows, const float* bmat, void* stream);

/* Tensor-core stages of a forward program (planner tc_blocks): per (row, block) the 16 x 16
 * product of the stage's dense ops from the row's matrix slab, as the MMA B image (tf32 hi, lo).
 * ops [n_ops, 4] = (kind 1 = 2x2 / 2 = 4x4, matrix offset, slot 0, slot 1), bptr [n_blocks+1],
 * out [rows, n_blocks, 2048] floats.  Part of run_ops / fusion (qcflow/sim.py:122-136,
 * fusion.py:78-176): the products the tile passes apply with tcgen05 MMAs. */
int qf_tc_build(const float* mats, int n_mat, int rows, const int32_t* ops, const int32_t* bptr, int n_blocks,
                float* out, void* stream);

/* ---- plan-specialised kernels (jit.py generates CUDA source from the descriptors above) ---- */

/* NVRTC-compile `src` (libnvrtc.so.12 loaded at run time) into a cubin; free with qf_jit_free. */
int qf_jit_compile(const char* src, const char* name, const char* const* opts, int nopts, void** image,
                   size_t* size);
void qf_jit_free(void* p);
/* Load a cubin into the current (primary) context; look up a kernel; unload. */
int qf_jit_load(const void* image, void** module);
int qf_jit_function(void* module, const char* name, int max_dyn_smem, void** func);
int qf_jit_unload(void* module);
/* Resident CTAs per SM of a loaded pass kernel (grid size of the persistent kernels). */
int qf_jit_occupancy(void* func, int block, int dyn_smem, int* blocks_per_sm);
/* Device address / size of a loaded module's __constant__ symbol (jit.py constant slabs). */
int qf_jit_global(void* module, const char* name, void** dptr, size_t* bytes);
/* Stage one pass's rotation coefficients into its module's constant slab on `stream`:
 * staging[row][j] = (x, x), x = Re mats[row * n_mat + cols[j]], then a device copy into
 * `symbol` (rows * k * 8 bytes <= symbol_bytes).  Replaces nothing in the reference (the
 * reference has no native code; this feeds the kernels that replace qcflow sim.py:88-105). */
int qf_jit_cm_stage(const void* mats, int n_mat, int rows, const int* cols, int k, void* staging, void* symbol,
                    size_t symbol_bytes, void* stream);
/* Launch n generated pass kernels in order on `stream` with one packed argument struct
 * (QfJitArgs in csrc/qf_jit_prelude.cuh). */
int qf_jit_run(void* const* funcs, const uint32_t* grid, const uint32_t* block, const uint32_t* smem, int n,
               void* stream, const void* args, size_t args_size);

#ifdef __cplusplus
}
#endif
#endif
