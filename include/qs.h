/*
 * qs.h — C ABI of the B200-native state-vector gate engine (arXiv 2506.09198 hot path).
 *
 * The operation (§II-C1): a state of 2^n complex amplitudes, 16 B each,
 * updated IN PLACE by the matrix-vector product of a 1-qubit, controlled-1-qubit or 2-qubit gate
 * ("the core operation is a matrix-vector multiplication"; fig. `unitary6q` L264-L268 and
 * `control6q2` L269-L273).  Circuits (QFT PAPER.md:L295, RQC L327) are ordered gate lists.
 *
 * Conventions (binding for every function below; DESIGN.md "Readings" R1-R4):
 *  - amplitude i is stored at byte offset 16*i of its shard, real part first (AoS);
 *  - qubit t is bit t of i, qubit 0 the least significant (Alg. 1 "sizeHalfBlock <- 1<<t");
 *  - a 1q matrix u2[8] = {u00.re,u00.im, u01.re,u01.im, u10.re,u10.im, u11.re,u11.im} (row-major,
 *    complex interleaved) acts as (a0', a1') = U (a0, a1), a0 having the target bit 0;
 *  - a 2q matrix u4[32]: u4[2*(4r+c)] = Re U[r][c]; rows/cols indexed by k = bit_q0 + 2*bit_q1
 *    (q0 is the low sub-bit whether q0 < q1 or not);
 *  - controlled-1q: U is applied to the target where the control bit is 1.
 *
 * Sharding: P = 2^k shards; shard d holds global indices [d*2^m, (d+1)*2^m),
 * m = n - k.  Qubits >= m are "global": bit (g - m) of the shard rank.
 *
 * Ownership: the library owns all device memory.  Host matrices / gate arrays are read during
 * the call only.  `out`/`in` buffers of qs_read_amps / qs_write_amps are caller-owned.
 *
 * Synchronisation: qs_apply_*, qs_run_circuit, qs_init_* are stream-ordered and asynchronous;
 * qs_read_amps, qs_write_amps, qs_norm2, qs_sync, qs_destroy block.  Argument errors return
 * synchronously with no side effect.  A CUDA/NCCL failure is reported by the call that sees it
 * (at the latest the next blocking call) and makes the handle sticky: afterwards every call but
 * qs_destroy / qs_last_error returns QS_ERR_STATE.
 *
 * Threading: one host thread drives a handle at a time.
 */
#ifndef QS_H
#define QS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qs_state qs_state; /* opaque, owned by the library */

typedef enum {
    QS_OK = 0,
    QS_ERR_ARG = 1,         /* bad qubit, ctrl==target, q0==q1, bad n/P, NULL pointer, non-unitary */
    QS_ERR_RANGE = 2,       /* basis index or amplitude range outside [0, 2^n) or outside this rank */
    QS_ERR_OOM = 3,         /* device memory short; qs_last_error gives requested and free bytes   */
    QS_ERR_CUDA = 4,        /* CUDA runtime failure (sticky)                                       */
    QS_ERR_NCCL = 5,        /* NCCL failure (sticky)                                               */
    QS_ERR_STATE = 6,       /* handle already in a sticky error state                              */
    QS_ERR_UNSUPPORTED = 7  /* valid request this build does not implement                         */
} qs_status;

enum { QS_G_1Q = 0, QS_G_C1Q = 1, QS_G_2Q = 2 };

/* One gate of a circuit.  kind QS_G_1Q: q0 = target, m[0..7] = U2.
 * kind QS_G_C1Q: q0 = control, q1 = target, m[0..7] = U2.  kind QS_G_2Q: (q0, q1), m[0..31] = U4.
 * flags: reserved, must be 0.  sizeof(qs_gate) == 272. */
typedef struct {
    int32_t kind, q0, q1, flags;
    double m[32];
} qs_gate;

/* ---- lifetime --------------------------------------------------------------------------------
 * Defining passages: SPEC.md:L44-L52 (create_state: |0...0>, 16*2^n bytes, allocation failure reports
 * requested and free bytes), §I ("16 bytes per amplitude", 35 qubits ~ 0.5 TiB: why the
 * state is sharded), §III-B1 (the V2 "split" of one region over memory domains: here, P
 * GPUs each holding 2^m of the 2^n amplitudes).
 * qs_create: n_qubits >= 1 on n_gpus in {1,2,4,8} devices 0..n_gpus-1 driven by this one process
 * (NCCL communicator from ncclCommInitAll when n_gpus > 1).  The state starts as |0...0>.
 * Errors: QS_ERR_ARG (n < 1, bad P, P > device count, m < QS_MIN_LOCAL for P > 1, n > 40),
 * QS_ERR_OOM (16*2^m + exchange buffers do not fit), QS_ERR_CUDA / QS_ERR_NCCL.
 * On failure *out is NULL and qs_last_error(NULL) explains. */
qs_status qs_create(int n_qubits, int n_gpus, qs_state **out);

/* qs_create_virtual: P = n_shards shards of the SAME sharded algorithm placed on the current
 * device.  A global-qubit gate runs as the fused peer-memory kernels (option "p2p" = 1, default) or as
 * the buffered exchange pipeline of the multi-GPU path with device copies (option "vtransport" = 0) or
 * ncclSend/ncclRecv to self on a one-rank communicator ("vtransport" = 1) moving the chunks.  Exists to
 * exercise the global-qubit path (planner, pack/unpack, fused update, pipeline) on one GPU. */
qs_status qs_create_virtual(int n_qubits, int n_shards, qs_state **out);

/* Multi-process mode (one process per GPU, e.g. torchrun): every rank calls qs_create_rank with
 * the same n_qubits/world and a 128-byte NCCL unique id produced by qs_get_unique_id on rank 0
 * and broadcast by the caller (e.g. torch.distributed).  The handle owns shard `rank` only;
 * qs_read_amps / qs_write_amps accept ranges inside that shard (else QS_ERR_RANGE) and
 * qs_norm2 returns the global norm (all ranks must call it). */
qs_status qs_get_unique_id(void *id128);
qs_status qs_create_rank(int n_qubits, int world, int rank, int device, const void *id128, qs_state **out);

/* Frees every device buffer, stream, event and communicator.  NULL-safe.  Blocks.  Explicit, measurable
 * teardown: the paper's RQC timing includes "state destruction" (§IV-C). */
void qs_destroy(qs_state *s);

/* ---- initialisation (asynchronous) -----------------------------------------------------------
 * Defining passages: SPEC.md:L44-L52 (the |0...0> / basis state), BASELINE.json configs[0] ("seeded random
 * normalised vector (iid Gaussian re/im, then normalised)"); the generator is reading R9 of DESIGN.md.
 * qs_init_basis: |index>, index < 2^n else QS_ERR_RANGE.
 * qs_init_random: amplitude i = gauss2(seed, i) (SplitMix64 + Box-Muller by GLOBAL index, so it
 * is invariant under sharding), then multiplied by 1/sqrt(sum |a|^2) (deterministic pairwise sum).
 * Blocks once internally for the norm. */
qs_status qs_init_basis(qs_state *s, uint64_t index);
qs_status qs_init_random(qs_state *s, uint64_t seed);

/* ---- gates (asynchronous, in place) ----------------------------------------------------------
 * Defining passages: §II-C1 ("the core operation is a matrix-vector multiplication");
 * qs_apply_1q: Alg. 1 PAPER.md:L117-L154 (pair (indexUp, indexLo) at stride 2^t, L124-L134) and fig.
 * `unitary6q` L264-L268, SPEC.md:L218-L225 (apply_single_qubit_unitary, non-unitary rejected unless a flag
 * is set); qs_apply_ctrl_1q: fig. `control6q2` L269-L273 and L288 (only control-1 amplitudes updated),
 * SPEC.md:L236-L254 (CNOT, controlled phase); qs_apply_2q: BASELINE.json north_star (general 4x4 unitary;
 * the paper's only 2q gates are CNOT and the QFT's controlled phase / SWAP, L287, L295)
 * (SWAP).
 * Errors: QS_ERR_ARG for a qubit outside [0, n), ctrl == target, q0 == q1, NULL matrix, or a
 * matrix with max|U^H U - I| > 1e-10 (check disabled by qs_set_option("check_unitary", 0)). */
qs_status qs_apply_1q(qs_state *s, int target, const double u2[8]);
qs_status qs_apply_ctrl_1q(qs_state *s, int ctrl, int target, const double u2[8]);
qs_status qs_apply_2q(qs_state *s, int q0, int q1, const double u4[32]);

/* Defining passages: SPEC.md:L404-L412 (run_circuit: gates applied in order), §IV-B (QFT:
 * "a Hadamard gate followed by controlled phase shifts", ending SWAPs), L327 §IV-C (RQC), L84 (cache
 * blocking / fusion "traverse the state fewer times": the tile passes below).
 * Applies gates[0..n_gates): the state afterwards is M_G ... M_1 psi.  With option "fuse" = 1
 * (default) gates whose qubits fit one shared-memory tile are applied in one HBM pass; with the
 * defaults of "reorder", "ladder_min" and "factor" commuting gates may be applied in another order and
 * phase runs / scalar factors combined (results equal to rounding); with those three off, results are
 * bitwise identical to fuse = 0 (same per-gate arithmetic, same order).  All gates are validated
 * before any work is queued.  n_gates == 0 is a no-op. */
qs_status qs_run_circuit(qs_state *s, const qs_gate *gates, size_t n_gates);

/* ---- readback (blocking) -----------------------------------------------------------------------
 * Defining passages: SPEC.md:L54-L72 (total_probability = sum(re^2 + im^2), a pure read; get_amp / set_amp
 * with out-of-bounds errors); the pairwise (deterministic) sum is SURVEY.md §8(c) c.6.
 * out/in hold 2*count doubles (re, im interleaved) for global amplitudes [start, start+count). */
qs_status qs_read_amps(qs_state *s, uint64_t start, uint64_t count, double *out);
qs_status qs_write_amps(qs_state *s, uint64_t start, uint64_t count, const double *in);
/* Stream-ordered variants (return at once): the copy runs on the handle's stream after the work
 * queued before it and before the work queued after it; the host buffer must stay valid (and, for a
 * copy that overlaps other handles' work, be page-locked) until qs_sync.  Errors as above. */
qs_status qs_read_amps_async(qs_state *s, uint64_t start, uint64_t count, double *out);
qs_status qs_write_amps_async(qs_state *s, uint64_t start, uint64_t count, const double *in);
qs_status qs_norm2(qs_state *s, double *out);   /* sum |a|^2, deterministic order */
qs_status qs_sync(qs_state *s);                  /* waits for every shard; surfaces async errors */

/* ---- introspection / options -------------------------------------------------------------------*/
/* s == NULL: message of the last failed qs_create* on this thread. Never NULL. */
const char *qs_last_error(const qs_state *s);
/* n, shards P, local qubits m, shards owned by this handle, rank of the first owned shard. */
qs_status qs_info(const qs_state *s, int *n_qubits, int *n_shards, int *local_qubits, int *owned, int *first_rank);
/* Number of kernels this library has launched for the handle (all shards). */
uint64_t qs_launch_count(const qs_state *s);
/* cudaStream_t (as void*) on which owned shard `i` runs its compute kernels. */
void *qs_stream(const qs_state *s, int i);
/* Options: "fuse" (0/1, default 1), "tile_qubits" (6..12, default 12), "chunk_bytes" (a power of two
 * >= 4096; default 256 MiB: the global-qubit exchange moves 2^m or 2^(m-1) amplitudes in chunks of
 * chunk_bytes/16), "vtransport" (virtual shards with p2p = 0: 0 device copies, 1 ncclSend/ncclRecv to self on
 * a one-rank communicator — the NCCL path's calls on one GPU), "graph" (0/1, default 1: on a single-shard
 * handle, the second and later runs of the same circuit replay a captured CUDA graph of its passes; same
 * kernels and arguments, identical results), "jit_family" (0: pass kernels with every
 * entry code compiled in; 1, default: those when compiled, else a cached FAMILY kernel — a grid-RQC gate
 * sqrtX/sqrtY/sqrtW picked per op at run time, so a new seed compiles nothing — with the specialised kernel
 * compiled in the background; 2: family kernels only; all give identical bits), "check_unitary" (0/1, default 1), "jit" (0/1, default 1:
 * tile passes run as NVRTC-compiled straight-line kernels, cached by pass structure; 0 = the
 * precompiled interpreter kernel; both give bitwise-identical results), "tile_low" (1..8, default 4:
 * local qubits 0..tile_low-1 are in every tile, i.e. 2^tile_low-amplitude contiguous runs),
 * "ladder_min" (>= 0, default 4: inside a tile pass, runs of >= ladder_min consecutive pure-phase
 * gates sharing one qubit — the QFT's controlled-R_k ladder — are applied as ONE factor per amplitude;
 * 0 = off), "perm_low" (0..6, default 5: a run of disjoint local SWAPs whose qubits do not fit one tile
 * is ONE in-place permutation pass gathering 2^perm_low-amplitude runs; 0 = off), "perm_fuse" (0/1,
 * default 1: such a run joins the tile pass right before it when that pass's qubits and their images
 * fit one tile of <= 12 qubits — the pass stores each tile onto its image, one HBM pass fewer; the
 * permutation is data movement, so the result is bitwise the unfused one), "perm_hoist" (0/1, default
 * 1: a permutation pass that cannot join the pass before it is split over the tile passes before it —
 * each of its transpositions (a, b) joins the store of one of them and the gates in between act on b
 * for a — when that removes the permutation pass (QFT(32): the final bit reversal rides on two of the
 * four ladder passes); SWAP then G(a) equals G(b) then SWAP exactly, but the ladder products of the
 * relabelled passes multiply their factors in another order: results agree to rounding), "reorder" (0/1,
 * default 1: commutation-aware scheduling of the gates between exchanges into tile passes; 0 = gate
 * order), "factor" (0/1, default 1: circuits apply 1q gates U = c M with monomial M — entries 0, +-1,
 * +-i, or w(+-1+-i) — as M with one deferred global scalar), "remap" (0/1, default 1: sharded circuits
 * swap global qubits to local positions when that lowers the exchange volume), "p2p" (0/1, default 1:
 * global-qubit gates run as fused peer-memory kernels where every shard can address its partner —
 * virtual shards, single-process multi-GPU with peer access; 0 = buffered NCCL exchange), "jit_async"
 * (0/1, default 0: 1 = pass kernels not yet compiled run in the interpreter while NVRTC compiles them
 * in the background; 0 = compile first, in parallel, then run), "jit_wait" (action: wait for
 * background compilations).  With ladder_min = 0,
 * reorder = 0 and factor = 0 every fused path is bitwise identical to the unfused one and to any shard
 * count; with them on, results agree to rounding (reading R21).
 * Unknown key: QS_ERR_ARG. */
qs_status qs_set_option(qs_state *s, const char *key, int64_t value);
/* Plan statistics of the last qs_run_circuit: number of HBM passes (tile + single-gate kernels) and
 * number of exchange steps. */
qs_status qs_last_plan(const qs_state *s, uint64_t *passes, uint64_t *exchanges);
/* Process-wide JIT counters: tile kernels compiled, JIT launches, failed compilations (after a
 * failure the interpreter kernel runs the pass; the message is in qs_last_error). */
qs_status qs_jit_stats(const qs_state *s, uint64_t *compiled, uint64_t *launched, uint64_t *failed);

#define QS_MIN_LOCAL 8

#ifdef __cplusplus
}
#endif
#endif /* QS_H */
