/*
 * fgadmm_b200.h — C-ABI of the B200 engine for the five-phase factor-graph
 * ADMM iteration (x, m, z, u, n) of the reference package `fgadmm`.
 *
 * The reference is pure Python/NumPy; its "FFI" for this path is the
 * Python engine API.  Each entry point below replaces one reference
 * interface (file:line relative to /root/reference/pkg/src/fgadmm):
 *
 *   fg_plan_create        engine.py:166-210  _GraphOps/_plan (per-graph plan,
 *                                            kind batching, CSR-by-variable)
 *                         graph.py:151-214   flat layout it consumes
 *   fg_plan_sync_params   graph.py:232-246   set_edge_params (rho/alpha and
 *                                            z_weights re-read each entry)
 *   fg_state_upload       engine.py:468-471  run(..., state=prior)
 *   fg_state_download     engine.py:521-522  state mutated in place / solution
 *   fg_run                engine.py:454-531  run (five phases, residuals, stop)
 *   fg_phase_*            engine.py:353-385  update_x .. update_n (unfused)
 *   fg_residuals          engine.py:398-406  residuals
 *   fg_prox_eval          prox.py:60-78      ProxFactor.batch_eval per kind
 *                         operators.py       (11 closed forms)
 *   fg_wproj              operators.py:86-96, 606-623  weighted null-space
 *                                            projection (mpc_dyn_prox with
 *                                            three weights)
 *   fg_last_error         engine.py:145-149, 333-350 (error text source)
 *
 * All arrays are HOST pointers in the reference's own order (edge-creation
 * order for payload arrays, variable order for z).  Device memory, streams
 * and CUDA graphs are owned by the plan.  Every function returns 0 on
 * success or a negative FG_ERR_* code; fg_last_error() gives the text.
 * Calls on one plan must be serialized by the caller (as in the reference,
 * no phase may run concurrently with set_edge_params).
 */
#ifndef FGADMM_B200_H
#define FGADMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FG_ABI_VERSION 1
#define FG_MAX_SLOTS 8

/* error codes */
#define FG_OK 0
#define FG_ERR_INVALID (-1)   /* bad argument / shape -> ValueError      */
#define FG_ERR_CUDA (-2)      /* CUDA runtime failure -> RuntimeError    */
#define FG_ERR_UNSUPPORTED (-3) /* kind without a device kernel          */
#define FG_ERR_NONFINITE (-4) /* non-finite value detected (see result)  */

/* operator kinds (registry names in operators.py) */
#define FG_KIND_QUADRATIC 1   /* operators.py:99-149  */
#define FG_KIND_COLLISION 2   /* operators.py:152-200 */
#define FG_KIND_WALL 3        /* operators.py:203-246 */
#define FG_KIND_RADIUS 4      /* operators.py:249-287 */
#define FG_KIND_MPC_COST 5    /* operators.py:290-326 */
#define FG_KIND_MPC_INIT 6    /* operators.py:329-365 */
#define FG_KIND_MPC_DYN 7     /* operators.py:368-417 */
#define FG_KIND_SVM_SLACK 8   /* operators.py:420-454 */
#define FG_KIND_SVM_NORM 9    /* operators.py:457-490 */
#define FG_KIND_SVM_MARGIN 10 /* operators.py:493-539 */
#define FG_KIND_EQUALITY 11   /* operators.py:542-572 */
#define FG_KIND_NAN_TEST 12   /* device fault injector (replaces tests' _Rogue) */

/* phases, engine.py:25 */
#define FG_PHASE_X 0
#define FG_PHASE_M 1
#define FG_PHASE_Z 2
#define FG_PHASE_U 3
#define FG_PHASE_N 4

/* buffers addressable by fg_debug_download */
#define FG_BUF_X 0
#define FG_BUF_U0 1
#define FG_BUF_U1 2
#define FG_BUF_AUX 3
#define FG_BUF_Z0 4   /* z ping-pong slots (Z doubles, variable order):     */
#define FG_BUF_Z1 5   /* iteration j of a run reads slot (j-1)&1, writes j&1 */

typedef struct fg_plan fg_plan;

/* The frozen graph's flat layout (graph.py:171-197). */
typedef struct {
    int64_t num_vars;            /* V                                    */
    int64_t num_edges;           /* E                                    */
    int64_t payload;             /* P = total_edge_payload               */
    int64_t z_dim;               /* Z                                    */
    const int32_t* var_dim;      /* [V] variable dims                    */
    const int64_t* var_offsets;  /* [V+1] z offsets (graph.var_offsets)  */
    const int32_t* edge_var;     /* [E] graph.edge_var                   */
    const int64_t* edge_offsets; /* [E+1] graph.edge_offsets             */
    int32_t chunk;               /* items per one-CTA pairwise subtree
                                    (128..8192; 0 = 8192)               */
    int32_t small_degree;        /* max degree summed by one thread
                                    (1..32; 0 = 32)                     */
    /* Multi-GPU partitions.  For a rank's LOCAL graph:
     * z_cut_index[k] is the position of local z component k in the
     * all-gathered cut vector (-1: variable not cut), ncut its length.
     * NULL / 0 for a whole graph. */
    const int32_t* z_cut_index;
    int64_t ncut;
} fg_graph_desc;

/* One homogeneous factor batch: one (kind, slot dims) group, as
 * engine.py:113-129 (_Group) builds it.  Edges of a factor are
 * consecutive (graph.py:161-167), so slot j of factor i is reference edge
 * first_edge[i] + j.  Parameters come from the kind's stack_params. */
typedef struct {
    int32_t kind;                  /* FG_KIND_*                           */
    int32_t nslots;
    int32_t slot_dim[FG_MAX_SLOTS];
    int64_t count;                 /* factors in the group                */
    const int64_t* first_edge;     /* [count]                             */
    const double* fparams;         /* [count * fstride] per-factor params */
    int32_t fstride;
    int32_t tstride;               /* doubles per shared table entry      */
    const double* tables;          /* [ntables * tstride]                 */
    int64_t ntables;
    const int32_t* fsys;           /* [count] table index, or NULL        */
    int32_t iparam;                /* kind integer param (mpc_dyn: state
                                      dim d; tables hold M (d x cols),
                                      Q (d x d), L (d) per system)        */
    int32_t reserved;
} fg_group_desc;

typedef struct {
    int64_t max_iterations;        /* RunConfig.max_iterations            */
    double primal_tol;             /* 0 disables (engine.py:473)          */
    double dual_tol;
    int32_t first_reads_n;         /* 1: first x-phase reads uploaded n   */
    int32_t timing;                /* 1: per-pass CUDA-event timing,
                                      direct launches (no CUDA graph);
                                      2: phase profile -- the five phases
                                      as separate kernels with events
                                      (engine.py:489-500), times from
                                      fg_run_phase_ms                     */
    int32_t graph_chunk;           /* iterations per CUDA-graph launch    */
    int32_t reserved;
} fg_run_config;

typedef struct {
    int64_t iterations;            /* executed (RunReport.iterations)     */
    int32_t converged;
    int32_t error_phase;           /* -1, or FG_PHASE_* of first failure  */
    int64_t error_iteration;       /* run-local iteration of the failure  */
    double primal;                 /* residuals of the last iteration     */
    double dual;
    double ms_total;               /* device time of the iteration loop   */
    double ms_edge_pass;           /* x-phase kernels (fused n); timing=1:
                                      summed over all iterations, else
                                      iteration 1 only (gives the shares) */
    double ms_var_pass;            /* z-phase kernels (fused m, u)        */
    double ms_reduce;              /* residual/stop kernel                */
    int64_t launches;              /* kernels launched by the loop        */
} fg_run_result;

/* ---- plan lifecycle ---------------------------------------------------- */
int fg_plan_create(const fg_graph_desc* graph, const fg_group_desc* groups,
                   int32_t ngroups, int32_t device, fg_plan** out);
void fg_plan_destroy(fg_plan* plan);
/* out[0..11]: V, E, P, Z, small / large / giant components, giant chunks,
 * launches of iteration 1, launches of later iterations, fused SVM chain on,
 * chain form (0 off, 1 generic, 2 fast, 3 unit-weight; the unit form is
 * re-decided at every fg_plan_sync_params) */
int fg_plan_info(const fg_plan* plan, int64_t* out12);
/* Kernel forms the next run uses (decided at plan creation and at every
 * fg_plan_sync_params): out[0] fused SVM chain (0 off, 1 generic, 2 fast,
 * 3 unit-weight), out[1] collision tiles in unit-weight form, out[2..5]
 * class-L rows of dim 1..4 in unit-weight form, out[6] mpc_dyn matrix
 * form, out[7] giant top/reduce fused, out[8] iterations per launch of the
 * temporally blocked MPC chain in fixed-budget runs (0: not blocked). */
int fg_plan_forms(const fg_plan* plan, int32_t* out9);
int fg_plan_sync_params(fg_plan* plan, const double* edge_rho,
                        const double* edge_alpha, const double* z_weights);

/* ---- fused run (the hot path) ------------------------------------------ */
/* z and u are on the device when fg_state_upload returns; n may still be in
 * flight (it is compared with z[zmap] - u on a copy stream while the next
 * fg_run starts from n = z - u, and fg_run repeats the run from the
 * uploaded state if they differ), so the n buffer must stay valid and
 * unchanged until the next call on the plan.  Plans attached to NCCL or
 * peer memory (and FGADMM_SPEC_UPLOAD=0) upload all three synchronously. */
int fg_state_upload(fg_plan* plan, const double* z, const double* u,
                    const double* n);
int fg_run(fg_plan* plan, const fg_run_config* cfg, double* history,
           fg_run_result* out);
int fg_state_download(fg_plan* plan, double* x, double* m, double* z,
                      double* u, double* n);
/* Per-iteration device milliseconds of the five phases (x, m, z, u, n) of
 * the last fg_run with timing == 2 (RunReport.phase_seconds and the
 * history rows, engine.py:489-514): out[5*i + k] for iteration i < *count,
 * *count = min(max_iterations, iterations executed); 0 after other runs. */
int fg_run_phase_ms(const fg_plan* plan, int64_t max_iterations, double* out,
                    int64_t* count);
/* First non-finite entry (reference edge order) of the payload arrays the
 * last fg_state_download wrote: out4[0..3] for x, m, u, n, -1 when all
 * finite or not downloaded.  Replaces the host scan behind the reference's
 * final n check (engine.py:333-350, 519). */
int fg_state_nonfinite(const fg_plan* plan, int64_t* out4);
/* x/u/aux buffers are P doubles in reference edge order; FG_BUF_Z0/1 are Z
 * doubles.  After a failed fg_run, FG_BUF_X holds x of the failing
 * iteration (materialized when that iteration ran fused kernels). */
int fg_debug_download(fg_plan* plan, int32_t buffer, double* out_ref);
/* Per-kernel device time of `iterations` fused iterations (after
 * fg_state_upload): labels[32*i], ms[i], counts[i] for each kernel slot of
 * one iteration (edge_<kind>..., var_*, reduce).  The first iteration of
 * the timed sequence runs untimed when more follow (kernel loading), so
 * counts[i] = iterations - 1 (generic) or - 2 (fused chain).  Profiling
 * aid; the arithmetic is exactly fg_run's. */
int fg_profile_kernels(fg_plan* plan, int64_t iterations, int32_t max_slots,
                       char* labels, double* ms, int64_t* counts,
                       int32_t* nslots);

/* ---- unfused per-phase API (update_x .. update_n) ----------------------- */
int fg_phase_upload(fg_plan* plan, const double* x, const double* m,
                    const double* z, const double* u, const double* n);
int fg_phase(fg_plan* plan, int32_t phase);
int fg_phase_download(fg_plan* plan, double* x, double* m, double* z,
                      double* u, double* n);
int fg_residuals(fg_plan* plan, const double* x, const double* z,
                 const double* z_prev, double* primal, double* dual);
/* Objective sum and largest constraint violation at z (graph.py:253-263);
 * z == NULL evaluates the plan's current device z.  out2 = {obj, viol}. */
int fg_evaluate(fg_plan* plan, const double* z, double* out2);

/* ---- standalone batched prox (ProxFactor.batch_eval) -------------------- */
/* values: per slot j a (count, slot_dim[j]) row-major array, concatenated
 * slot after slot; rhos: (nslots, count); out like values. */
int fg_prox_eval(const fg_group_desc* group, const double* values,
                 const double* rhos, double* out, int32_t device);
/* Weighted projection of each row of nv (rows x D) onto {v : M v = 0}
 * (M is r x D, row-major, shared by all rows) minimizing sum w (v - nv)^2,
 * operators.py:86-96.  Weights must be positive (FG_ERR_INVALID);
 * a singular M W^-1 M^T gives FG_ERR_NONFINITE ("Singular matrix"). */
int fg_wproj(const double* M, int32_t r, int32_t D, const double* nv,
             const double* w, int64_t rows, double* out, int32_t device);

/* ---- self-test --------------------------------------------------------- */
/* q[i] = the engine's inline division x[i] / y[i] (fg_device.cuh qdiv),
 * ref[i] = the CUDA runtime's x[i] / y[i]; the two must agree bitwise. */
int fg_selftest_div(const double* x, const double* y, int64_t n, double* q,
                    double* ref, int32_t device);

/* ---- multi-GPU exchange of cut-variable partial sums ------------------- */
/* NCCL (one process per GPU): rank 0 calls fg_nccl_unique_id, the id is
 * broadcast by the caller (e.g. torch.distributed), every rank attaches it
 * to its plan; fg_run then all-gathers the cut partials and the residual
 * partials inside the iteration (captured in the CUDA graph).  `nccl_lib`
 * is the libnccl.so.2 to dlopen (NULL: default search path). */
int fg_nccl_unique_id(const char* nccl_lib, char* out128);
int fg_plan_attach_nccl(fg_plan* plan, const char* nccl_lib, const char* id128,
                        int32_t rank, int32_t world);
/* Peer memory (one process per GPU, no collective library): every rank
 * calls fg_p2p_export (allocates its receive buffer and flag array for
 * `world` ranks; out128 = their two CUDA IPC handles), the caller
 * all-gathers the handles (rank-major, world x 128 bytes), then every rank
 * calls fg_plan_attach_p2p with them and the graph's global payload size.
 * fg_run then stores each rank's cut and residual partials straight into
 * every peer's receive buffer over NVLink and synchronises on per-rank
 * epoch flags, inside the captured iteration -- fused with the kernels that
 * consume the gathered values (k_cut_p2p, k_reduce_p2p); the rank-order sum
 * is the same as the NCCL path's.  A rank that stops answering for 10 s
 * fails the run with FG_ERR_CUDA instead of hanging.  A plan attaches to
 * one exchange once (NCCL or peer memory); FG_ERR_INVALID otherwise. */
int fg_p2p_export(fg_plan* plan, int32_t world, char* out128);
int fg_plan_attach_p2p(fg_plan* plan, int32_t rank, int32_t world, const char* handles,
                       int64_t payload_global);
/* Local group: the G partition plans of one graph on ONE device, exchanged
 * by device copies (single-GPU validation of the partitioned algorithm).
 * Results are those of rank 0 (identical on all ranks). */
int fg_group_run(fg_plan** plans, int32_t nplans, const fg_run_config* cfg,
                 double* history, fg_run_result* out);

/* ---- pinned host memory (state arrays that stream at full PCIe rate) --- */
int fg_host_alloc(int64_t bytes, void** out);
int fg_host_free(void* ptr);

/* ---- misc --------------------------------------------------------------- */
const char* fg_last_error(void);
int fg_abi_version(void);
int fg_device_count(int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* FGADMM_B200_H */
