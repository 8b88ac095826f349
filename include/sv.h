/*
 * sv.h -- C-ABI of the B200 state-vector gate-application engine (libsv.so).
 *
 * The path: load a circuit (IR text) -> classify, fuse and plan passes ->
 * initialise a 2^n complex state in HBM -> apply the passes with sm_100a kernels ->
 * read out amplitudes, marginal probabilities or the norm.  Optionally the state is
 * sharded across P GPUs by its top log2(P) qubits, and dense gates on those "global"
 * qubits trigger NCCL all-to-all qubit swaps.
 *
 * Passages that define the operations (P:n = PAPER.md line n, S:n = SPEC.md line n):
 *   - P:38 (Background): the state of an n-qubit circuit is a 2^n complex vector of
 *     amplitudes; each moment is a 2^n x 2^n matrix; a Schroedinger simulator stores all
 *     amplitudes and its time grows linearly with the number of gates.
 *   - P:55 (Methods, assumption a): "a quantum circuit simulator is a matrix vector
 *     multiplication software"; memory and communication dominate at large n.
 *   - P:123: multi-GPU simulation is the stated future work (implemented here).
 *   - S:72-120 (qcore), S:167-206 (kernels), S:542-557 (bindings): operation semantics.
 *
 * Conventions (all entry points):
 *   - extern "C"; every function except sv_memory_estimate / sv_last_error returns an
 *     sv_status (SV_OK = 0).  No C++ exception crosses the boundary.
 *   - Little-endian: qubit q is bit q of the basis index.  Inside a
 *     k-qubit matrix, row/column bit j <-> targets[j] (reading R2).  A gate applies U
 *     when every control qubit is 1.
 *   - Amplitudes are interleaved (re, im): SV_C64 = 2 x float32 (8 B per amplitude),
 *     SV_C128 = 2 x float64 (16 B per amplitude).
 *   - Pointers named host* are host memory borrowed for the duration of the call only.
 *     Device memory of a state is owned by the handle (sv_create) or borrowed from the
 *     caller (sv_wrap); the handle never frees a borrowed buffer.
 *   - Calls that launch work are asynchronous on the handle's CUDA stream; calls that
 *     return data to the host (sv_amplitudes, sv_probabilities, sv_norm) synchronise it.
 *     Asynchronous CUDA/NCCL faults surface at the next synchronising call as SV_ERR_CUDA
 *     / SV_ERR_NCCL.  An error detected before any launch leaves the handle unchanged.
 *   - sv_last_error() returns a thread-local message for the last failing call.
 *   - A state handle is single-writer; a plan may be applied to different states
 *     from several threads (applies of one plan are serialised internally), and
 *     sv_apply_circuit's process-wide plan cache is thread-safe.  Sharded handles are collective: every rank
 *     makes the same calls in the same order.
 */
#ifndef SV_H_
#define SV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sv_state_s* sv_state;   /* opaque state handle */
typedef struct sv_plan_s* sv_plan;     /* opaque compiled circuit (parse + fuse + plan) */

typedef enum { SV_C64 = 1, SV_C128 = 2 } sv_dtype;

typedef enum {
    SV_OK = 0,
    SV_ERR_ARG = 1,       /* bad argument: null pointer, k > 5, bad dtype, bad option */
    SV_ERR_RANGE = 2,     /* qubit >= n, duplicate qubits across targets and controls, index range */
    SV_ERR_RESOURCE = 3,  /* allocation failed; message carries sv_memory_estimate(n) */
    SV_ERR_PARSE = 4,     /* IR text error; message carries the 1-based line number */
    SV_ERR_CUDA = 5,      /* CUDA runtime error (possibly from an earlier async launch) */
    SV_ERR_NCCL = 6,      /* NCCL error */
    SV_ERR_STATE = 7      /* handle/plan mismatch (e.g. plan compiled for another width) */
} sv_status;

/* Kernel selection for ablations (sv_run_opts.force_kernel). */
typedef enum {
    SV_KERNEL_AUTO = 0,       /* fused tile passes, each compiled to a specialised sm_100a kernel (default) */
    SV_KERNEL_PER_GATE = 1,   /* one single-stage pass per gate (no fusion), precompiled interpreter kernel */
    SV_KERNEL_DENSE = 2,      /* one pass per gate, every gate as a generic dense block (K4) */
    SV_KERNEL_INTERP = 3      /* fused tile passes run by the precompiled interpreter kernel (ablation) */
} sv_kernel;

typedef struct {
    int fuse;            /* 1 (default) = fuse gates into multi-stage tile passes */
    int tile_qubits;     /* m, qubits per tile pass; 0 = auto */
    int max_fused_k;     /* unused (ABI slot): the planner fuses by stages and passes, never by
                            pre-multiplying blocks; must be 0 */
    int force_kernel;    /* sv_kernel */
    int check_unitary;   /* 1 = reject matrices with |U^dagger U - I| > 1e-9 */
    int use_graph;       /* 1 = record the plan's launches into a CUDA graph on first use */
    int profile;         /* 1 = bracket every pass with CUDA events (sv_plan_pass_times) */
    int exchange;        /* sharded global<->local swaps: 0 (default) = fused into the preceding
                            pass, whose stores go straight to the peers' second buffers over
                            NVLink peer memory (CUDA IPC; needs a second shard
                            buffer, falls back to 1 if it cannot be allocated or mapped on every
                            rank); 1 = NCCL send/recv through a staging chunk */
} sv_run_opts;

typedef struct {
    uint64_t gates;              /* IR gates applied (= gate count) */
    uint64_t passes;             /* kernel passes launched */
    uint64_t stages;             /* register stages across all passes */
    uint64_t swaps;              /* global<->local qubit swap steps (sharded only) */
    uint64_t launches;           /* kernels launched by this call */
    uint64_t hbm_bytes;          /* algorithmic HBM bytes (read + write) of the passes */
    uint64_t nvlink_bytes;       /* bytes sent per rank in swap steps */
    double plan_ms;              /* host time spent parsing + planning (sv_apply_circuit) */
} sv_run_stats;

/* 2^n * bytes-per-amplitude of dtype; saturates at UINT64_MAX (reading R20).
 * Returns 0 for a bad dtype or n < 0. */
uint64_t sv_memory_estimate(int n, sv_dtype dtype);

/* Allocate a 2^n-amplitude state on the current CUDA device, initialised to |0...0>
 * (S:72-80).  1 <= n <= 40.  stream: a cudaStream_t to launch on, or NULL to create a
 * private non-blocking stream.  SV_ERR_RESOURCE if the allocation fails. */
sv_status sv_create(int n, sv_dtype dtype, void* stream, sv_state* out);

/* Wrap a caller-owned device buffer of 2^n amplitudes (e.g. a torch tensor; the
 * state is the 2^n amplitude vector in index order).  The buffer contents are left as they
 * are; the handle never frees it.  Every call that changes the state leaves the buffer in
 * logical index order once its work on the stream completes (a relabelling plan's final
 * layout is undone inside sv_plan_apply / sv_apply_circuit for borrowed buffers), so the
 * caller may read the tensor after synchronising the stream (sv_sync or its own sync). */
sv_status sv_wrap(int n, sv_dtype dtype, void* dev_ptr, void* stream, sv_state* out);

/* NCCL bootstrap for sharded states: rank 0 writes a 128-byte unique id into out_128B;
 * the caller broadcasts it (torch.distributed) to every rank. */
sv_status sv_nccl_unique_id(void* out_128B);

/* Collective: create a state of n qubits sharded over `world` GPUs (world a power of two
 * >= 2, one process per GPU).  Rank r holds the 2^(n-g) amplitudes whose top g = log2(world)
 * physical qubits equal r.  State = |0...0>. */
sv_status sv_create_sharded(int n, sv_dtype dtype, const void* uid_128B, int world, int rank,
                            void* stream, sv_state* out);

/* Host control plane for sharded states (alternative to NCCL's): the library needs only an
 * all-gather of small host messages and a barrier across the ranks.  Each callback returns
 * 0 on success and is called collectively (every rank, same order) from the thread making
 * the sv_* call.  allgather: every rank contributes `bytes` bytes from `in`; `out` receives
 * world * bytes bytes in rank order.  barrier: returns when every rank has entered it.
 * With a host control plane the library synchronises the state's stream before each
 * barrier, and every global<->local exchange goes through peer memory (CUDA IPC mappings of
 * every rank's buffer pair: remote stores fused into the preceding pass, or a peer-copy
 * kernel); there is no NCCL communicator.  This is how several ranks can share one GPU. */
typedef struct {
    void* user;
    int (*allgather)(void* user, const void* in, size_t bytes, void* out);
    int (*barrier)(void* user);
} sv_control;

/* Collective: a sharded state as sv_create_sharded, with either an NCCL unique id
 * (uid_128B != NULL, ctl == NULL) or a host control plane (ctl != NULL, uid_128B == NULL).
 * dev_ptr: NULL = allocate the local shard of 2^(n-g) amplitudes; else a caller-owned
 * device buffer of that size, borrowed (never freed), which holds the local shard in
 * logical order whenever a call's work completes.  The peer-memory exchange
 * allocates a second shard buffer; SV_ERR_RESOURCE if that fails with a host control plane
 * (there is no NCCL fallback there).  Errors as sv_create_sharded; SV_ERR_ARG if both or
 * neither of uid_128B and ctl are given. */
sv_status sv_create_sharded_ex(int n, sv_dtype dtype, const void* uid_128B, const sv_control* ctl, int world,
                               int rank, void* dev_ptr, void* stream, sv_state* out);

/* Single-process emulation of a `world`-way sharded state on one GPU (tests): the shards
 * are slices of one allocation and the all-to-all is device-to-device copies.  Runs the
 * same planner, qubit map and swap schedule as sv_create_sharded. */
sv_status sv_create_virtual_sharded(int n, sv_dtype dtype, int world, void* stream, sv_state* out);

sv_status sv_destroy(sv_state s);

/* Initialisation (basis state, or the uniform superposition).  On a single-GPU state that
 * owns its buffer the write is deferred: the next sv_plan_apply / sv_apply_circuit whose
 * first pass is a generated tile pass synthesises |k> (or 2^(-n/2) everywhere) inside that
 * pass (init fused into pass 0, no read of the buffer);
 * every other call (readouts, sv_apply_gate, sv_sync, sv_device_ptr, ...) writes it first.
 * Code that reads the buffer through a pointer obtained earlier calls sv_sync first. */
sv_status sv_init_zero(sv_state s);
sv_status sv_init_basis(sv_state s, uint64_t k);        /* |k>, SV_ERR_RANGE if k >= 2^n */
sv_status sv_init_uniform(sv_state s);                  /* every amplitude 2^(-n/2) */

/* Copy `count` amplitudes (interleaved, state dtype) from host memory into logical
 * indices [first, first+count).  Sharded: each rank writes the part it holds. */
sv_status sv_set_amplitudes(sv_state s, uint64_t first, uint64_t count, const void* host);

/* Apply one gate.  mat: 2^k x 2^k complex matrix, row-major, interleaved
 * (re, im) doubles, rounded to the state dtype before use and copied before return; an
 * entry component within 2^-52 of 0, +1 or -1 is taken as exactly that value (as in the IR's
 * custom matrices), e.g. cos(pi/2) = 6.1e-17.
 * 1 <= k <= 5; targets[k]; controls[ncontrols] (may be NULL when ncontrols == 0).
 * SV_ERR_RANGE on qubit >= n or duplicates across targets and controls. */
sv_status sv_apply_gate(sv_state s, const double* mat, int k, const int* targets,
                        const int* controls, int ncontrols);

/* Compile IR text for an n-qubit state of dtype: parse (SV_ERR_PARSE with line number),
 * classify, fuse, plan.  opts NULL = defaults.  The plan is independent of the state's
 * contents and can be applied many times. */
sv_status sv_plan_compile(const char* ir_text, sv_dtype dtype, const sv_run_opts* opts,
                          sv_plan* out);
sv_status sv_plan_info(sv_plan p, int* n, uint64_t* gates, uint64_t* passes, uint64_t* stages);
/* Generated CUDA source of tile pass `pass` of the single-GPU schedule (inspection and
 * profiling).  Writes at most cap bytes (NUL-terminated) and the full length to *len.
 * Returns SV_ERR_RANGE for a bad pass index; an empty string for a non-tile pass.  With the
 * environment variable SV_SOURCE_VARIANT=basis (uniform), pass 0 is returned in its variant
 * that synthesises a basis state (the uniform superposition) instead of loading its input. */
sv_status sv_plan_source(sv_plan p, int pass, char* buf, size_t cap, size_t* len);
sv_status sv_plan_destroy(sv_plan p);
/* Logical -> physical qubit map the single-GPU schedule leaves (a relabelling schedule stores
 * its final tiles permuted; readouts undo it).  phys_out: n ints, caller-owned. */
sv_status sv_plan_qubit_map(sv_plan p, int* phys_out);

/* Host-only dry run of the sharded schedule of a plan over `world` GPUs (power of two >= 2),
 * starting from the identity qubit map: number of global<->local exchange steps, of pass
 * batches, and of passes rank 0 launches.  No GPU needed. */
sv_status sv_plan_shard_info(sv_plan p, int world, uint64_t* swaps, uint64_t* batches, uint64_t* passes);

/* Apply a compiled plan to a state (asynchronous).  stats may be NULL. */
sv_status sv_plan_apply(sv_state s, sv_plan p, sv_run_stats* stats);

/* Device time of every pass of the last sv_plan_apply of a plan compiled with
 * opts.profile = 1 (CUDA events on the state's stream; synchronises).  Writes up to cap
 * values (ms) and the pass count to *n. */
sv_status sv_plan_pass_times(sv_plan p, float* ms_out, int cap, int* n);

/* Parse + plan + apply every gate of every moment in order.  opts and stats
 * may be NULL; stats->gates equals the IR gate count. */
sv_status sv_apply_circuit(sv_state s, const char* ir_text, const sv_run_opts* opts,
                           sv_run_stats* stats);

/* Read amplitudes [first, first+count) of the logical state into host_out (interleaved,
 * state dtype).  P:38 (the state is the 2^n amplitude vector), S:112-120 (amplitude
 * readout).  A relabelled layout (sv_qubit_map not the identity) is first made canonical on
 * the device.  Synchronises.  SV_ERR_RANGE if the range exceeds 2^n.  Sharded: each rank receives the part of the range it holds
 * (after the qubit map is made canonical) at host_out + (index - first). */
sv_status sv_amplitudes(sv_state s, uint64_t first, uint64_t count, void* host_out);

/* P:38 (|a_i|^2 are the outcome probabilities of the 2^n basis states), S:92-100,
 * reading R11.  Marginal probabilities of the qubit subset: host_out[k] = sum over basis states whose
 * bit qubits[j] equals bit j of k of |a|^2, accumulated in fp64 in a fixed order
 * (deterministic), 2^nq doubles.  0 <= nq <= min(n, 28).  Sharded: global value on every rank. */
sv_status sv_probabilities(sv_state s, const int* qubits, int nq, double* host_out);

/* sqrt(sum |a_i|^2) accumulated in fp64 with a fixed-order tree. */
sv_status sv_norm(sv_state s, double* out);

/* Wait for every launched call on the handle's stream (calls are asynchronous,
 * readouts synchronise).  A deferred initialisation (sv_init_*) is written first.  Does NOT
 * change the layout: an owned state may be left relabelled by its last plan (sv_qubit_map);
 * use sv_device_ptr or the readouts for index order.  Borrowed buffers are always in index
 * order (sv_wrap).  Returns SV_ERR_CUDA for an asynchronous fault of an earlier launch. */
sv_status sv_sync(sv_state s);

/* Introspection for the bindings and the bench. */
sv_status sv_info(sv_state s, int* n, int* n_local, int* world, int* rank, sv_dtype* dtype);
/* Device pointer of the (local) state buffer and its amplitude count.  Makes the layout
 * canonical first (logical index order; on the stream, asynchronous).  The pointer is valid
 * until the next call that applies gates: a permutation (gather) pass of an owned state
 * writes the other buffer of a pair and swaps them, so re-query after every apply. */
sv_status sv_device_ptr(sv_state s, void** dev_ptr, uint64_t* local_amps);
sv_status sv_stream(sv_state s, void** stream);
/* Current physical position of every logical qubit (phys[q]).  Not the identity after a
 * relabelling single-GPU plan (owned states) or sharded exchange steps; readouts,
 * sv_device_ptr and sv_set_amplitudes restore the identity. */
sv_status sv_qubit_map(sv_state s, int* phys_out);

const char* sv_last_error(void);
const char* sv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SV_H_ */
