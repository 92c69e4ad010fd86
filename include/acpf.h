/*
 * acpf.h — C-ABI of libacpf.so, the B200 (sm_100a) batched AC power-flow engine.
 *
 * This is the drop-in boundary for the reference's batched-solve hot path
 * (arxiv 2605.14103 reference package `acpflow`, pkg/src/acpflow/):
 *
 *   acpf_nr_*    replaces the per-scenario Newton solve the reference batch
 *                driver calls, `newton_solve` -> `_newton_loop`
 *                (transmission.py:306-330, 333-380), including its mismatch
 *                map (transmission.py:194-215) and its GMRES/FD step solve
 *                (transmission.py:259-298, sparse.py:219-338), which this
 *                engine replaces with an exact sparse LU step.
 *   acpf_zbus_*  replaces `zbus_iterate` -> `_zbus_loop` and
 *                `batch_zbus_solve` (distribution.py:633-711), including
 *                `current_injection` (:573-610), `ZBusModel.z_apply`
 *                (:423-425) and `fixed_point_residual` (:613-621).
 *
 * The reference's own binding for this path is the Python callable passed to
 * `run_batch(solver, scenarios, ...)` (batch.py:280-344); INTEGRATION.md
 * shows the ctypes stub that binds these symbols behind that callable.
 *
 * Conventions
 *  - Plain pointers and sizes only. All scenario arrays are row-major per
 *    scenario ([batch][...]); complex values are interleaved (re, im) doubles.
 *  - `flags` selects where batch buffers live: ACPF_HOST_PTRS (pageable or
 *    pinned host memory; the library stages through device memory) or
 *    ACPF_DEVICE_PTRS (device memory on the plan's device).
 *  - Numerical outcomes are per-scenario status codes, never errors:
 *    a call returns ACPF_OK even when scenarios diverge.
 *  - Setup/usage errors return a negative acpf_status; the message is
 *    available from acpf_last_error() (thread-local).
 *  - Ownership: a plan owns device copies of the model (made at create,
 *    released at destroy). The caller owns every batch buffer.
 *  - Threading: calls on one plan must be serialised by the caller; distinct
 *    plans (e.g. one per GPU) may be driven from different host threads.
 *  - Determinism: each scenario's outputs are bitwise independent of the
 *    batch size, its position in the batch and the chunking.
 */
#ifndef ACPF_H
#define ACPF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t acpf_status;

#define ACPF_OK 0
#define ACPF_EINVAL (-1)  /* bad argument / inconsistent sizes            */
#define ACPF_ECUDA (-2)   /* CUDA runtime error (message has details)     */
#define ACPF_ENOMEM (-3)  /* device or host allocation failed             */
#define ACPF_ESTRUCT (-4) /* structural problem: singular pattern/matrix, */
                          /* or a network beyond the kernels' limits     */

#define ACPF_HOST_PTRS 0u
#define ACPF_DEVICE_PTRS 1u

#define ACPF_ABI_VERSION 1

/* Per-scenario Newton status (acpf_nr_solve `status`). Mirrors the exit
 * branches of _newton_loop (transmission.py:347-359) in their check order. */
#define ACPF_NR_CONVERGED 0  /* ||F||inf <= tol                          */
#define ACPF_NR_MAX_ITER 1   /* k == max_newton, not converged           */
#define ACPF_NR_NONFINITE 2  /* mismatch became non-finite               */
#define ACPF_NR_VMAG_LE0 3   /* min V <= 0                               */
#define ACPF_NR_ZERO_PIVOT 4 /* exact zero pivot in the static-pivot LU  */

/* Per-scenario Z-Bus status (acpf_zbus_solve `status`), _zbus_loop :653-687. */
#define ACPF_ZB_CONVERGED 0
#define ACPF_ZB_MAX_ITER 1
#define ACPF_ZB_FLOOR 2 /* VoltageFloorError mid-iteration; see floor_slot */

const char* acpf_last_error(void);
int32_t acpf_abi_version(void);
int32_t acpf_device_count(void);

/* ------------------------------------------------------------------------
 * Transmission Newton-Raphson
 * ------------------------------------------------------------------------ */
typedef struct acpf_nr_plan* acpf_nr_plan_t;

typedef struct acpf_nr_plan_info {
  int32_t n_bus;        /* buses                                        */
  int32_t n_theta;      /* |PV| + |PQ|  (angle unknowns)                */
  int32_t n_q;          /* |PQ|         (magnitude unknowns)            */
  int32_t n_j;          /* block rows (= n_theta, one 2x2 block per     */
                        /* non-slack bus; PV buses padded)              */
  int32_t nnz_y;        /* Ybus nonzeros                                */
  int32_t nnz_j;        /* Jacobian 2x2 blocks (Ybus pattern, no slack) */
  int64_t nnz_lu;       /* static-pivot L+U 2x2 blocks (incl. fill)     */
  int64_t n_pairs;      /* 2x2-block Crout updates of one refactorisation */
  int32_t group;        /* scenarios interleaved per warp (8)           */
  int32_t etree_height; /* informational                                */
  int64_t workspace_bytes_per_group;
} acpf_nr_plan_info;

/* Build the device plan for one network (reference model build
 * transmission.py:146-160 + the symbolic LU this engine needs).
 *   y_*           complex CSR Ybus, n_bus rows, sorted column indices
 *                 (network.py:450-496 / AdmittanceMatrix.complex_csr).
 *   theta_block   bus indices of the angle unknowns, PV then PQ (len n_theta)
 *   q_block       bus indices of the magnitude unknowns, PQ   (len n_q)
 *                 (network.py:499-516)
 *   theta_init, vmag_init   flat start incl. pinned slack/PV values
 *                 (transmission.py:169-177), len n_bus.
 *   perm          fill-reducing ordering of the n_theta block rows (one
 *                 2x2 block per non-slack bus): perm[k] = index into
 *                 theta_block of the bus eliminated k-th; NULL for the
 *                 built-in minimum-fill ordering (acpf_nr_ordering with
 *                 ACPF_ORDER_MIN_FILL). Rows are then
 *                 level-sorted (a topological order of the elimination tree,
 *                 same fill).                                              */
acpf_status acpf_nr_plan_create(int32_t device, int32_t n_bus, const int32_t* y_rowptr,
                                const int32_t* y_col, const double* y_re, const double* y_im,
                                int32_t n_theta, const int32_t* theta_block, int32_t n_q,
                                const int32_t* q_block, const double* theta_init,
                                const double* vmag_init, const int32_t* perm,
                                acpf_nr_plan_t* out);

/* Host-only: native report emission, byte-identical to
 * the reference's json.dumps(doc, indent=1) of the `solve` command's
 * acpflow-solve-result/1 document (cli.py:141-180, embedding
 * report_to_dict, batch.py:352-376) and to report_to_csv (batch.py:379-387).
 * Written to `path` when non-NULL, else into out[capacity] with the byte
 * count in *length (a first call with capacity 0 sizes the buffer).
 *   errors[i]        NULL or the record's error text (UTF-8)
 *   state_a/state_b  [count][n_state]: theta/vmag (kind "tx") or
 *                    v_re/v_im (kind "dist"); has_solution[i] == 0 (or a
 *                    NULL state) writes null lists (errored records)
 *   node_phase_ids   dist only: the reduced node-phase labels            */
typedef struct {
  const char* case_name; /* "case": file name of the network             */
  const char* kind;      /* "tx" | "dist"                                  */
  int64_t seed;
  double spread;
  int64_t batch;
  int64_t worker_count;
  double total_wall_time;
  double throughput;
} acpf_result_meta;

acpf_status acpf_solve_result_json(const acpf_result_meta* meta, int64_t count, const uint8_t* converged,
                                   const int32_t* iterations, const double* residual, const double* wall_time,
                                   const char* const* errors, int32_t n_state, const double* state_a,
                                   const double* state_b, const uint8_t* has_solution, int32_t n_ids,
                                   const char* const* node_phase_ids, const char* path, char* out,
                                   int64_t capacity, int64_t* length);

acpf_status acpf_report_csv(int64_t count, const uint8_t* converged, const int32_t* iterations,
                            const double* residual, const double* wall_time, const char* const* errors,
                            const char* path, char* out, int64_t capacity, int64_t* length);

/* Host-only (no device): native model build, bit-identical
 * to the reference's NumPy/SciPy assembly: CSR with sorted columns, exact
 * 0+0j entries absent, duplicates summed in the reference's order. Call
 * with capacity 0 (arrays may be NULL) to get *nnz, then again with
 * capacity >= *nnz and rowptr[n+1], col/re/im[capacity].
 *
 * acpf_ybus_build: pi-model Ybus (network.py:450-496). Per branch k (bus
 * INDICES from_idx/to_idx, in_service 0/1): series 1/(r + jx), charging
 * b_ch, tap ratio and shift (rad); stamps (f,f) (y + j b/2)/tap^2,
 * (t,t) y + j b/2, (f,t) -y/conj(a), (t,f) -y/a, a = tap e^{j shift}; then
 * bus shunts gs + j bs. Zero parts are +0.0 (the reference's G + jB).
 * ACPF_EINVAL for an in-service branch with r = x = 0 or tap = 0.           */
acpf_status acpf_ybus_build(int32_t n_bus, int32_t n_branch, const int32_t* from_idx, const int32_t* to_idx,
                            const double* r, const double* x, const double* b_ch, const double* tap,
                            const double* shift, const uint8_t* in_service, const double* gs, const double* bs,
                            int64_t capacity, int32_t* rowptr, int32_t* col, double* re, double* im,
                            int64_t* nnz);

/* acpf_y3_build: node-phase Y of a three-phase feeder (distribution.py:
 * 356-391) from its primitive blocks in stamp order (per line y_ff, y_ft,
 * y_tf, y_tt, then the shunts). Block b is k x k, k = block_ptr[b+1] -
 * block_ptr[b]; its row node-phases are idx[2 block_ptr[b] ..][0..k), its
 * column node-phases the next k; its values row-major complex (re, im
 * interleaved) consecutively in val.                                        */
acpf_status acpf_y3_build(int32_t n, int32_t n_blocks, const int32_t* block_ptr, const int32_t* idx,
                          const double* val, int64_t capacity, int32_t* rowptr, int32_t* col, double* re,
                          double* im, int64_t* nnz);

/* Host-only (no device): a fill-reducing elimination order of the n_theta
 * block rows for acpf_nr_plan_create's `perm` (replaces the SciPy/SuperLU
 * MMD ordering a NumPy host would take; the reference factors dense,
 * sparse.py:159-176). Greedy on the 2x2-block bus graph, lowest index
 * breaking ties:
 *   ACPF_ORDER_MIN_DEGREE  fewest remaining neighbours;
 *   ACPF_ORDER_MIN_FILL    fewest fill edges, then degree (fewer block
 *                          updates, hence a shorter factor gather stream).
 * perm_out: len n_theta, perm_out[k] = index into theta_block.             */
#define ACPF_ORDER_MIN_DEGREE 1
#define ACPF_ORDER_MIN_FILL 2
acpf_status acpf_nr_ordering(int32_t n_bus, const int32_t* y_rowptr, const int32_t* y_col,
                             int32_t n_theta, const int32_t* theta_block, int32_t kind,
                             int32_t* perm_out);

/* Host-only symbolic analysis (no device needed): fills the structural
 * fields of `info` (workspace_bytes_per_group included) for the same inputs
 * acpf_nr_plan_create takes. Used to inspect orderings offline.          */
acpf_status acpf_nr_analyze(int32_t n_bus, const int32_t* y_rowptr, const int32_t* y_col,
                            int32_t n_theta, const int32_t* theta_block, int32_t n_q,
                            const int32_t* q_block, const int32_t* perm, acpf_nr_plan_info* info);

/* Host-only (no GPU): solve J(x0) x = rhs with the LU of the flat-start
 * Jacobian that every scenario's first Newton step shares (the factor
 * acpf_nr_plan_create builds). rhs, x_out: len n_theta + n_q in the
 * reference's unknown order [theta_block; q_block]. ACPF_ESTRUCT on a zero
 * pivot. For checking the shared factor against a dense Jacobian.          */
acpf_status acpf_nr_flat_start_solve(int32_t n_bus, const int32_t* y_rowptr, const int32_t* y_col,
                                     const double* y_re, const double* y_im, int32_t n_theta,
                                     const int32_t* theta_block, int32_t n_q, const int32_t* q_block,
                                     const double* theta_init, const double* vmag_init,
                                     const int32_t* perm, const double* rhs, double* x_out);

acpf_status acpf_nr_plan_info_get(acpf_nr_plan_t plan, acpf_nr_plan_info* info);

/* Export the plan's ordering (len n_j) and LU row pointers (len n_j+1). */
acpf_status acpf_nr_plan_structure(acpf_nr_plan_t plan, int32_t* perm_out, int64_t* lu_rowptr_out);

/* Solve `batch` scenarios (each = newton_solve(model, scenario, opts) from the
 * flat start).
 *   p_spec [batch][n_theta], q_spec [batch][n_q]   (TransmissionScenario)
 *   theta_out, vmag_out [batch][n_bus]             (NewtonResult.state)
 *   converged [batch] u8, iterations [batch], final_mismatch_inf [batch],
 *   status [batch] (ACPF_NR_*).
 * Any output pointer except theta_out/vmag_out may be NULL.
 * The first Newton step of every scenario uses the LU of the flat-start
 * Jacobian, which does not depend on the scenario (factored once at plan
 * create; ACPF_NR_SHARED0=0 factors it per scenario instead).
 * ACPF_HOST_PTRS: the batch is copied in chunks solved on two concurrent
 * lanes (streams); the call drives the second lane from an internal host
 * thread that is joined before it returns (ACPF_NR_PIPELINE=1: one stream
 * plus a copy stream, 0: serial chunks); results are complete on return.
 * ACPF_DEVICE_PTRS: the solve is enqueued on cuda_stream and the call returns
 * without waiting (stream-ordered, like a CUDA library call): synchronise the
 * stream (or call acpf_nr_last_timing) before reading the results on the
 * host; consecutive device-pointer solves of one plan must use one stream.
 * The Newton loop runs on the device (one CUDA graph with conditional nodes
 * per solve; ACPF_NR_DEVLOOP=0 steps it from the host).                      */
acpf_status acpf_nr_solve(acpf_nr_plan_t plan, int64_t batch, const double* p_spec,
                          const double* q_spec, double tol_mismatch, int32_t max_newton,
                          double* theta_out, double* vmag_out, uint8_t* converged,
                          int32_t* iterations, double* final_mismatch_inf, int32_t* status,
                          uint32_t flags, void* cuda_stream);

/* acpf_nr_solve from a given start state instead of the plan's flat start
 * (reference newton_solve(..., start=PolarState), transmission.py:306-330):
 * theta_start, vmag_start [batch][n_bus] (host or device per flags, like the
 * other batch buffers). The first Newton step is then factored per scenario
 * (the shared flat-start LU does not apply); slack and PV entries keep the
 * start's values, as in the reference's PolarState.with_packed (:70-78). */
acpf_status acpf_nr_solve_start(acpf_nr_plan_t plan, int64_t batch, const double* p_spec,
                                const double* q_spec, const double* theta_start,
                                const double* vmag_start, double tol_mismatch, int32_t max_newton,
                                double* theta_out, double* vmag_out, uint8_t* converged,
                                int32_t* iterations, double* final_mismatch_inf, int32_t* status,
                                uint32_t flags, void* cuda_stream);

/* Time (ms) of the last acpf_nr_solve, measured with CUDA events, and the
 * number of kernel launches it made. Device pointers (and the host-pointer
 * serial / copy-stream pipelines, ACPF_NR_PIPELINE=0/1): the device time of
 * the Newton kernel launches on the solve stream. Host pointers on the
 * default two-lane pipeline: the wall time of the whole call on the device,
 * from the first H2D to the last D2H (copies included), since the two lanes'
 * kernels overlap each other and the copies. */
acpf_status acpf_nr_last_timing(acpf_nr_plan_t plan, double* kernel_ms, int32_t* launches);

acpf_status acpf_nr_plan_destroy(acpf_nr_plan_t plan);

/* ------------------------------------------------------------------------
 * Distribution Z-Bus fixed point
 * ------------------------------------------------------------------------ */
typedef struct acpf_zbus_plan* acpf_zbus_plan_t;

/* Build the device plan (reference ZBusModel, distribution.py:394-517).
 *   n            non-slack node-phases
 *   n_l, l_index load-touched reduced indices (sorted, unique)
 *   zl           Z[:, l] as [n][n_l] interleaved complex (row-major)
 *   v0           no-load profile [n] complex
 *   wye_idx      [n_wye] reduced index per wye load
 *   delta_p/q    [n_delta] reduced indices of each delta pair
 *   voltage_floor  division guard (default 1e-6 in the reference)       */
acpf_status acpf_zbus_plan_create(int32_t device, int32_t n, int32_t n_l, const int32_t* l_index,
                                  const double* zl, const double* v0, int32_t n_wye,
                                  const int32_t* wye_idx, int32_t n_delta, const int32_t* delta_p,
                                  const int32_t* delta_q, double voltage_floor,
                                  acpf_zbus_plan_t* out);

/* Solve `batch` scenarios (each = zbus_iterate(model, scenario, opts)).
 *   s_wye [batch][n_wye] complex, s_delta [batch][n_delta] complex
 *   v_out [batch][n] complex (FixedPointResult.v)
 *   converged u8, iterations, final_delta, residual_inf, status (ACPF_ZB_*)
 *   floor_slot: for ACPF_ZB_FLOOR, which check failed first, in the
 *   reference's order: k (wye k), n_wye+k (delta k, phase p),
 *   n_wye+n_delta+k (delta k, phase q), n_wye+2*n_delta+k (delta k, p-q);
 *   -1 otherwise. Any output pointer except v_out may be NULL.
 * ACPF_DEVICE_PTRS: enqueued on cuda_stream, returns without waiting (as
 * acpf_nr_solve); ACPF_HOST_PTRS: results complete on return.            */
acpf_status acpf_zbus_solve(acpf_zbus_plan_t plan, int64_t batch, const double* s_wye,
                            const double* s_delta, double tol, int32_t max_iter, double* v_out,
                            uint8_t* converged, int32_t* iterations, double* final_delta,
                            double* residual_inf, int32_t* status, int32_t* floor_slot,
                            uint32_t flags, void* cuda_stream);

acpf_status acpf_zbus_last_timing(acpf_zbus_plan_t plan, double* kernel_ms, int32_t* launches);

acpf_status acpf_zbus_plan_destroy(acpf_zbus_plan_t plan);

/* ------------------------------------------------------------------------
 * Seeded scenario inputs generated on the device (bitwise the reference
 * generator, batch.py:45-60 Philox4x64-10 keyed (seed, i), and its load
 * scaling batch.py:121-151). Rows start..start+count-1 of the batch.
 * ------------------------------------------------------------------------ */

/* Multiplier table [count][n_elem] (generate_load_multipliers). */
acpf_status acpf_philox_multipliers(uint64_t seed, int64_t start, int64_t count, int32_t n_elem,
                                    double spread, double* out, uint32_t flags, void* cuda_stream);

/* Transmission scenarios for a plan: element_bus [n_elem] = buses with a
 * nonzero base load (transmission_base.load_elements); p_load, q_load,
 * p_gen, q_gen [n_bus] host arrays (per unit). Writes p_spec [count][n_theta]
 * and q_spec [count][n_q] (host or device per flags). */
acpf_status acpf_nr_scenarios(acpf_nr_plan_t plan, uint64_t seed, int64_t start, int64_t count,
                              double spread, int32_t n_elem, const int32_t* element_bus,
                              const double* p_load, const double* q_load, const double* p_gen,
                              const double* q_gen, double* p_spec, double* q_spec, uint32_t flags,
                              void* cuda_stream);

/* Distribution scenarios: multiplier k scales wye load elem_target[k] (>= 0)
 * or delta load -elem_target[k]-1 (the reference load order); wye_s, delta_s
 * host base powers (interleaved complex). Writes s_wye [count][n_wye] and
 * s_delta [count][n_delta] complex. */
acpf_status acpf_zbus_scenarios(acpf_zbus_plan_t plan, uint64_t seed, int64_t start, int64_t count,
                                double spread, int32_t n_elem, const int32_t* elem_target,
                                const double* wye_s, const double* delta_s, double* s_wye,
                                double* s_delta, uint32_t flags, void* cuda_stream);

/* ------------------------------------------------------------------------
 * On-device certificates. Replace the host certificate
 * helpers the reference's tests call per scenario.
 * ------------------------------------------------------------------------ */

/* Attach the branch table of the network to an NR plan (needed by
 * acpf_nr_certify): per in-service branch its end buses and the four
 * admittances yff, yft, ytf, ytt (interleaved complex, [n_br][4]) of the
 * pi model, as branch_flows (transmission.py:453-481) forms them; bus_gs
 * [n_bus] the bus shunt conductances. Copied to the device. */
acpf_status acpf_nr_plan_set_branches(acpf_nr_plan_t plan, int32_t n_br, const int32_t* from_bus,
                                      const int32_t* to_bus, const double* y4, const double* bus_gs);

/* Per scenario of a solved batch (theta, vmag [batch][n_bus]; p_spec
 * [batch][n_theta]; q_spec [batch][n_q]):
 *   mismatch_inf  = ||F||inf at the state (mismatch, transmission.py:202-215;
 *                   NaN if any mismatch is NaN),
 *   slack_balance = sum over slack buses of P_calc
 *                   - (-sum p_spec + branch loss + shunt loss)
 *                   (test_transmission.py:398-416 for every scenario),
 *   branch_loss   = sum over branches of Re(s_from + s_to).
 * Any output pointer may be NULL. */
acpf_status acpf_nr_certify(acpf_nr_plan_t plan, int64_t batch, const double* theta,
                            const double* vmag, const double* p_spec, const double* q_spec,
                            double* mismatch_inf, double* slack_balance, double* branch_loss,
                            uint32_t flags, void* cuda_stream);

/* Attach the reduced network to a Z-Bus plan (needed by
 * acpf_zbus_kirchhoff): Y_NN in CSR (interleaved complex values, nnz =
 * rowptr[n]) and inj = Y_NS v_slack [n] (interleaved complex). */
acpf_status acpf_zbus_plan_set_network(acpf_zbus_plan_t plan, const int32_t* ynn_rowptr,
                                       const int32_t* ynn_col, const double* ynn_val,
                                       const double* inj);

/* Kirchhoff residual per scenario (kirchhoff_residual, distribution.py:
 * 624-630): max_k |(Y_NN v + Y_NS v_slack)_k - i_loads(v)_k| for v
 * [batch][n] complex; +inf where a load voltage is at the voltage floor
 * (the reference raises VoltageFloorError there). */
acpf_status acpf_zbus_kirchhoff(acpf_zbus_plan_t plan, int64_t batch, const double* v,
                                const double* s_wye, const double* s_delta, double* kcl,
                                uint32_t flags, void* cuda_stream);

/* ------------------------------------------------------------------------
 * Network reduction on the device (reference reduce_zbus,
 * distribution.py:431-517): factor Y_NN (CSR, interleaved complex values)
 * with partial pivoting and solve for the load columns and v0:
 *   zl_out [n][n_l] = (Y_NN^-1)[:, l_index]   (interleaved complex, row-major)
 *   v0_out [n]      = Y_NN^-1 rhs0,  rhs0 = -(Y_NS v_slack)
 * ACPF_ESTRUCT when Y_NN is numerically singular by the reference's test
 * (non-finite factor or min |U_ii| <= n eps max |Y_NN|). The outputs feed
 * acpf_zbus_plan_create.
 * ------------------------------------------------------------------------ */
acpf_status acpf_zbus_reduce(int32_t device, int32_t n, const int32_t* ynn_rowptr, const int32_t* ynn_col,
                             const double* ynn_val, const double* rhs0, int32_t n_l, const int32_t* l_index,
                             double* zl_out, double* v0_out);

/* ------------------------------------------------------------------------
 * The reference's own Newton step on the GPU (an ablation of
 * the exact sparse-LU step): matrix-free J v (_jvp_operator,
 * transmission.py:218-236) inside left-preconditioned restarted GMRES
 * (sparse.py:219-338) with the fast-decoupled preconditioner
 * (transmission.py:259-298).
 * ------------------------------------------------------------------------ */

/* FD data of the network: bprime_inv = (B' + eps I)^-1 [n_theta][n_theta]
 * and bdprime_inv = (B'' + eps I)^-1 [n_q][n_q] (row-major; B' = -Im Y over
 * the theta block, B'' = -Im Y over the q block, network.py:519-543), and
 * G = -Re Y[q, theta] in CSR (n_q rows, columns index the theta block). */
acpf_status acpf_nr_plan_set_fd(acpf_nr_plan_t plan, const double* bprime_inv, const double* bdprime_inv,
                                const int32_t* g_rowptr, const int32_t* g_col, const double* g_val);

/* Batched GMRES-Newton (reference _newton_loop semantics, statuses 0-3 as
 * acpf_nr_solve). precond: 1 = FD, 0 = none. Extra outputs (each may be
 * NULL): gmres_steps [batch][max_newton] GMRES iterations of each Newton step
 * (NewtonResult.per_iteration_gmres, entries past `iterations` are 0);
 * gmres_diag [batch]: 0 none, 1 breakdown, 2 stagnation (transmission.py:
 * 371-376) at Newton step gmres_diag_k with relres gmres_diag_relres. */
acpf_status acpf_nr_solve_gmres(acpf_nr_plan_t plan, int64_t batch, const double* p_spec, const double* q_spec,
                                double tol_mismatch, int32_t max_newton, double gmres_tol, int32_t restart,
                                int32_t max_outer, int32_t precond, double* theta_out, double* vmag_out,
                                uint8_t* converged, int32_t* iterations, double* final_mismatch_inf,
                                int32_t* status, int32_t* gmres_steps, int32_t* gmres_diag, int32_t* gmres_diag_k,
                                double* gmres_diag_relres, uint32_t flags, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* ACPF_H */
