/*
 * tilecast_b200.h -- C ABI of the B200-native batched environment step.
 *
 * This is the drop-in boundary for the reference's kernel plugin interface
 * (/root/reference/pkg/src/tilecast/backend/__init__.py:28-57 selects a
 * module exporting BACKEND_NAME / cast_ray / render_into / batch_kernel;
 * tables.py:251-266 is the one spelling of batch_kernel's argument order).
 * Every entry point below names the reference function it replaces.
 *
 * Conventions
 *   - Plain C types only: pointers, sizes, int status codes. No torch types.
 *   - "dev" pointers are CUDA device pointers (any allocator: torch, cudaMalloc);
 *     "host" pointers are ordinary host memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Functions return TC_OK (0) or a negative TC_E* error code; a message for
 *     the last error on the calling thread is available via tc_last_error().
 *   - Per-environment engine faults are NOT errors of the call: they are
 *     written as status codes (TC_ST_*) into out->statuses, exactly like the
 *     reference (tables.py:267-272 turns them into RuntimeError host-side).
 *   - The library never allocates on the step path; the caller owns every
 *     state/output buffer (tables.py:187-245 ownership rules).
 */
#ifndef TILECAST_B200_H
#define TILECAST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_ABI_VERSION 1

/* ---- call status (return values) -------------------------------------- */
#define TC_OK 0
#define TC_E_INVALID (-1)   /* bad argument / contract violation            */
#define TC_E_CUDA (-2)      /* CUDA runtime error (message in tc_last_error) */
#define TC_E_CAPACITY (-3)  /* exceeds MAX_ENTITIES / MAX_DOORS / obs size   */

/* ---- per-env kernel status codes (backend/layout.py:47-51) ------------- */
#define TC_ST_OK 0
#define TC_ST_ESCAPED 1      /* ray left the grid: map not sealed          */
#define TC_ST_STEP_BUDGET 2  /* ray exceeded 2*(w+h) boundary steps        */
#define TC_ST_BAD_ACTION 3   /* device-side action check (batch.py:92-106) */

/* ---- modes (layout.py:60-62) ------------------------------------------ */
#define TC_MODE_RESET 0
#define TC_MODE_STEP 1

/* ---- capacities (layout.py:64-66) ------------------------------------- */
#define TC_MAX_ENTITIES 64
#define TC_MAX_DOORS 32
#define TC_MAX_OBS_W 1024
#define TC_MAX_OBS_H 1024

/*
 * Read-only per-spec tables, field order = tables.py:257-261 (the order
 * batch_kernel receives them in), plus the array extents that the Cython
 * memoryviews carried implicitly. All pointers are HOST pointers when passed
 * to tc_spec_create (which packs and uploads them once per spec, like
 * build_tables, tables.py:92-184) and to the tc_host_* parity helpers.
 */
typedef struct tc_tables {
  /* map group */
  const uint8_t *kind;      /* u8  [h, w]   cell tags (C_FLOOR/C_WALL/C_DOOR)  */
  const uint8_t *wcol;      /* u8  [h, w]   wall palette index                  */
  const int16_t *didx;      /* i16 [h, w]   door index or -1                    */
  const int16_t *eat;       /* i16 [h, w]   entity index or -1                  */
  const uint8_t *dcol;      /* u8  [D]      door key colour                     */
  const uint8_t *dlock;     /* u8  [D]      door locked flag                    */
  const uint8_t *ekind;     /* u8  [E]      entity kind                         */
  const uint8_t *ecol;      /* u8  [E]      entity colour (keys)                */
  const double *epx;        /* f64 [E]      entity x (tile centre)              */
  const double *epy;        /* f64 [E]                                          */
  const double *spx;        /* f64 [S]      spawn x                             */
  const double *spy;        /* f64 [S]                                          */
  const int32_t *goal_ent;  /* i32 [G]      goal candidate entity indices       */
  const double *dirs;       /* f64 [4, 2]   E, S, W, N headings                 */
  /* render group */
  const uint8_t *pal;       /* u8  [P, 3]   wall palette                        */
  const uint8_t *door_rgb;  /* u8  [3, 3]                                       */
  const uint8_t *key_rgb;   /* u8  [3, 3]                                       */
  const uint8_t *goal_rgb;  /* u8  [3]                                          */
  const uint8_t *med_box;   /* u8  [3]                                          */
  const uint8_t *med_cross; /* u8  [3]                                          */
  const uint8_t *ceil_rgb;  /* u8  [3]                                          */
  const uint8_t *floor_rgb; /* u8  [3]                                          */
  const double *coef;       /* f64 [obs_w]  camera-plane coefficient per column */
  /* constants */
  const double *fc;         /* f64 [11]     layout.py:8-19                      */
  const int64_t *ic;        /* i64 [3]      layout.py:22-25                     */
  const uint8_t *legal;     /* u8  [7]      legal action tags (tables.py:165)   */
  /* extents */
  int32_t h, w;             /* map tiles                                        */
  int32_t n_doors, n_entities, n_spawns, n_goals, n_pal;
  int32_t obs_h, obs_w;
} tc_tables;

/* Mutable per-env state, env index first (StateBlock, tables.py:187-215). */
typedef struct tc_state {
  double *px, *py, *dx, *dy, *health; /* f64 [N]    */
  uint8_t *inv;                       /* u8  [N]    */
  int64_t *t;                         /* i64 [N]    */
  uint64_t *rkey, *rctr;              /* u64 [N]    */
  uint8_t *done;                      /* u8  [N]    */
  int32_t *agoal;                     /* i32 [N]    */
  uint8_t *dopen;                     /* u8  [N, D] */
  uint8_t *ealive;                    /* u8  [N, E] */
} tc_state;

/* Per-call outputs (OutBlock, tables.py:223-245) plus optional debug taps. */
typedef struct tc_out {
  uint8_t *frames;    /* u8  [N, obs_h, obs_w, 3] (required)                    */
  double *zbuf;       /* f64 [N, obs_w]   optional (NULL = not written)          */
  double *rewards;    /* f64 [N]          required in MODE_STEP                  */
  uint8_t *dones;     /* u8  [N]          required in MODE_STEP                  */
  uint8_t *truncs;    /* u8  [N]          required in MODE_STEP                  */
  uint32_t *events;   /* u32 [N]          required in MODE_STEP                  */
  int32_t *statuses;  /* i32 [N]          required                               */
  /* debug taps for the north-star per-item parity checks (NULL = off):        */
  int32_t *rayinfo;   /* i32 [N, obs_w, 4] (mapx, mapy, side, steps) per column  */
  uint64_t *spritevis;/* u64 [N]   bit e set = entity e drew >= 1 pixel column   */
} tc_out;

/* Device-side counters written by the step kernel (read lazily by the host;
 * no per-step synchronisation). Passing one also enables dynamic env
 * scheduling (warps pull env indices from next_env). One tc_counters must not
 * be used by two launches that may run concurrently. */
typedef struct tc_counters {
  uint64_t violations;   /* collision-invariant violations (batch.py:133)   */
  uint32_t bad_status;   /* OR of (1 << status) over all non-OK statuses    */
  uint32_t next_env;     /* env scheduler ticket: kernel-internal, must be  */
  uint32_t ctas_done;    /*   zero at first use; the kernel re-zeroes them  */
  uint32_t pad;
} tc_counters;           /* 24 bytes; allocate zeroed, reuse across calls   */

typedef struct tc_spec tc_spec; /* opaque, device-resident packed tables */

/* ABI / build info. */
int tc_abi_version(void);
const char *tc_last_error(void);
const char *tc_build_info(void);
/* Which step kernel a tc_batch_kernel / tc_batch_step_* call over n envs of
 * this spec launches (a description string; for reports). */
const char *tc_step_kernel(const tc_spec *spec, int64_t n);

/* Perf diagnostics (not part of the reference contract): per-env and
 * per-CTA timestamp buffers (TC_TRACE builds only; TC_E_INVALID otherwise),
 * and the mean host-side split of tc_batch_step_mapped (launch call, wait
 * for the results, call count) since the last reset (reset = 2: the split
 * of the released tc_batch_step_pipelined steps instead -- release call,
 * wait for the results, count -- then reset). */
int tc_debug_trace(void *dev_buf);
int tc_debug_trace_cta(void *dev_buf);
int tc_debug_mapped_timing(double *out3, int32_t reset);
/* The resident pipelined loop's device timeline (TILECAST_PIPE_TRACE=1):
 * u64 globaltimer [64 steps][3 stamps][grid CTAs], *grid = CTAs. */
int tc_debug_pipe_trace(uint64_t *host, int64_t cap, int32_t *grid);

/* Pack + upload a spec's tables once (replaces build_tables' device half,
 * tables.py:92-184). `host` points at host arrays. */
int tc_spec_create(const tc_tables *host, tc_spec **out);
int tc_spec_destroy(tc_spec *spec);

/* Reset (mode 0) or step (mode 1) envs [0, n) in place
 * (replaces backend.batch_kernel, _core.pyx:715-763 / _pycore.py:346-387).
 * `state`/`out` hold DEVICE pointers; `actions_dev` is i64[n] (ignored in
 * reset mode). `counters_dev` (device, may be NULL) accumulates violations
 * and status bits; the reference returns the violation count synchronously
 * instead (tc_host_batch_kernel below does). Asynchronous on `stream`. */
int tc_batch_kernel(const tc_spec *spec, const tc_state *state,
                    const int64_t *actions_dev, const tc_out *out, int64_t n,
                    int32_t mode, int32_t auto_reset, int32_t validate,
                    tc_counters *counters_dev, void *stream);

/* Out-of-place step: reads state_in, writes the stepped state to state_out
 * (both DEVICE pointers, may not overlap unless equal). This is batch_step's
 * "new BatchState from the old one" (batch.py:109-138) without the
 * reference's 13 per-step state copies (tables.py:217-220). */
int tc_batch_step_into(const tc_spec *spec, const tc_state *state_in,
                       const tc_state *state_out, const int64_t *actions_dev,
                       const tc_out *out, int64_t n, int32_t auto_reset,
                       int32_t validate, tc_counters *counters_dev, void *stream);

/* K consecutive steps (K x batch_step, batch.py:109-138, auto-reset) as K
 * launches of the lean kernel chained per env instead of by a grid-wide
 * wait between them: state ping-pongs a -> b -> a ..., step k reads
 * actions_dev[k * n .. k * n + n) and writes outs[k % ring]; the final state
 * is in b when k_steps is odd, else in a. flags_dev: device
 * u32[n + max(n, 64 * 2048)] zeroed once per batch; epoch0: a per-batch
 * counter the caller advances by k_steps per call (epochs are never reused).
 * One-wave batches (rings of up to 64 blocks): env i of step k waits only
 * for its own state from step k - 1 and for the CTA of the step that last
 * wrote outs[k % ring] (a row of done epochs per ring slot). Multi-wave batches (env
 * tickets): env i of step k waits for env i's whole step k - 1; each launch
 * draws its tickets from its own slot of flags_dev[n ..), zeroed by a
 * stream-ordered memset per run of n launches. The first step waits for all
 * prior work on the stream, so the action table may come from any earlier
 * kernel. Batches outside the lean kernels, and rings with debug taps, get
 * K ordinary launches, and so do multi-wave batches more than 4 waves deep
 * (their launch tails are negligible; the per-env epochs are not). */
int tc_batch_steps(const tc_spec *spec, const tc_state *state_a,
                   const tc_state *state_b, const int64_t *actions_dev,
                   const tc_out *outs, int32_t ring, int64_t n, int32_t k_steps,
                   int32_t auto_reset, int32_t validate,
                   tc_counters *counters_dev, uint32_t *flags_dev,
                   uint32_t epoch0, void *stream);

/* Heterogeneous-map step (the reference steps one
 * homogeneous batch per batch_kernel call, tables.py:251-273):
 * n_groups out-of-place steps, group g = counts[g] envs of specs[g] with
 * states_in[g] -> states_out[g], actions actions_dev[offset_g ..], outputs
 * outs[g] (typically views of one batch-wide block), counters[g] (one per
 * group), in ONE launch (up to 16 groups with a common frame shape; more
 * groups run as concurrent launches on library-owned side streams forked
 * from and joined back into `stream`); asynchronous like tc_batch_step_into. */
int tc_multi_step(const tc_spec *const *specs, const tc_state *states_in,
                  const tc_state *states_out, const int64_t *actions_dev,
                  const tc_out *outs, const int64_t *counts, int32_t n_groups,
                  int32_t auto_reset, int32_t validate, tc_counters *const *counters,
                  void *stream);

/* batch_step over HOST buffers in one call (batch.py:109-138 semantics, the
 * reference's numpy-in / numpy-out contract): H2D of actions_host into
 * actions_dev, one fused out-of-place step, D2H of rewards (f64[n]) and
 * dones (u8[n]) into host memory, stream synchronised on return. Any host
 * pointer may be pageable; rewards_host / dones_host may be NULL. */
int tc_batch_step_host(const tc_spec *spec, const tc_state *state_in,
                       const tc_state *state_out, const int64_t *actions_host,
                       int64_t *actions_dev, const tc_out *out, int64_t n,
                       int32_t auto_reset, int32_t validate,
                       tc_counters *counters_dev, double *rewards_host,
                       uint8_t *dones_host, void *stream);

/* batch_step over HOST buffers with no copy engine on the path: the
 * fused step kernel reads actions_host (i64[n]) straight from pinned host
 * memory, and its last CTA writes [rewards f64[n] | dones u8[n]] (9n bytes,
 * the out->rewards / out->dones device layout, 16-byte aligned) to
 * results_host with coalesced 16-byte stores, then raises flag_host[1]; the
 * call returns once flag_host[1] is set (the host spins on it instead of
 * synchronising the stream, which still sees the kernel's teardown). flag_host
 * is int32[2]: a contract-violating action sets flag_host[0] = 1 (the caller
 * zeroes it before the call; flag_host[1] is managed by the call) and leaves that env's state unchanged in state_out, so
 * the caller can raise the reference's ContractError (batch.py:92-106) with
 * state_in still valid. Same semantics as tc_batch_step_host otherwise. All
 * three host buffers must be page-locked and UVA-mapped (cudaHostAlloc /
 * torch pin_memory), else TC_E_INVALID. */
int tc_batch_step_mapped(const tc_spec *spec, const tc_state *state_in,
                         const tc_state *state_out, const int64_t *actions_host,
                         const tc_out *out, int64_t n, int32_t auto_reset,
                         int32_t validate, tc_counters *counters_dev,
                         uint8_t *results_host, int32_t *flag_host, void *stream);

/* tc_batch_step_mapped with its arguments in one struct, for bindings whose
 * per-argument marshalling dominates a ~30 us step (Python ctypes: ~3 us for
 * 12 arguments, ~0.5 us for one pointer). A step loop keeps one struct per
 * (state_in, state_out) pair and passes it every step. */
typedef struct tc_mapped_call {
  const tc_spec *spec;
  const tc_state *state_in;
  const tc_state *state_out;
  const int64_t *actions_host;
  const tc_out *out;
  int64_t n;
  int32_t auto_reset;
  int32_t validate;
  tc_counters *counters_dev;
  uint8_t *results_host;
  int32_t *flag_host;
  void *stream;
} tc_mapped_call;
int tc_batch_step_mapped_call(const tc_mapped_call *call);

/* Pipelined host step loop: batch_step(bs, actions, reuse=True)
 * (batch.py:109-138) over host buffers, one step per call, like
 * tc_batch_step_mapped_call -- plus, before waiting for this step's results,
 * it launches the NEXT step of the reuse=True ping-pong (input = this step's
 * state_out, output = this step's state_in, output block = next_out) behind
 * a gate: that launch stages its tables, waits for this step's grid, then
 * waits for the host. The next call whose arguments match releases it with
 * one store to host memory instead of launching (the caller has already
 * written that step's actions), so the launch call, the launch latency and
 * this step's frame rendering leave the host's per-step critical path.
 * flag_host is int32[8] (16-byte aligned): [0] bad action, [1] results
 * ready (as tc_batch_step_mapped), [4] / [5] the gate's go / cancel words,
 * [6] expired mark -- all managed by the call except [0]. gate_dev is a
 * zeroed device uint32[4096] per action stage (the gate's broadcast lines and
 * the result hand-off counters). A call that does not match the
 * pending launch (other buffers, another batch) cancels it first, as does
 * every other library launch; a watchdog thread cancels a launch nobody
 * released within TILECAST_PIPE_TIMEOUT_US (default 1000 us), so work queued
 * behind it waits at most that long. A cancelled launch exits without any
 * effect. speculate = 0 makes this exactly tc_batch_step_mapped_call.
 * (No reference counterpart: the reference's batch_step is synchronous CPU
 * code; this is the same step sequence with the launch moved earlier.) */
typedef struct tc_pipe_call {
  tc_mapped_call step;
  const tc_out *next_out;
  uint32_t *gate_dev;   /* zeroed device uint32[4096] per action stage */
  int32_t speculate;
  int32_t device;       /* the CUDA device of the batch (made current for the call) */
} tc_pipe_call;
int tc_batch_step_pipelined(const tc_pipe_call *call);
/* Cancel a pending pipelined launch (no-op if none). */
int tc_pipe_cancel(void);
/* Cancel a pending launch and clear the timeout back-off. */
int tc_pipe_reset(void);
/* Pipeline counters: [released, cancelled, of which timeouts, pending]. */
int tc_pipe_stats(uint64_t *out4);

/* K fused steps in one launch with on-device uniform-random actions drawn
 * exactly as batch.policy_actions (batch.py:141-153) would draw them for
 * steps [step0, step0+K) of an (n_total)-env rollout whose env 0 is global
 * env `base`. Frames of step k go to out->frames + (k % frame_ring) * N*H*W*3
 * (a ring of frame_ring >= 1 frame blocks, or K for a full rollout buffer).
 * rewards/dones/truncs/events (if non-NULL) are [K, N]. Auto-reset is on. */
int tc_rollout(const tc_spec *spec, const tc_state *state, const tc_out *out,
               int64_t n, int64_t base, int64_t n_total, uint64_t policy_key,
               int64_t step0, int32_t k_steps, int32_t frame_ring,
               tc_counters *counters_dev, void *stream);

/* Per-env RNG streams: rkey[i] = split(from_seed(seed), base+i).key,
 * rctr[i] = 0 (replaces the host loop batch.py:81-85; rng.py:96-99). */
int tc_seed_streams(uint64_t seed, int64_t base, int64_t n, uint64_t *rkey_dev,
                    uint64_t *rctr_dev, void *stream);

/* Uniform-random actions for one step of a seeded rollout
 * (batch.py:141-153, rng.py:102-129): actions[i] = action_tags[
 * mulhi(mix(key + (step*n_total + base + i)*GOLDEN), n_tags)]. */
int tc_policy_actions(uint64_t policy_key, int64_t step, int64_t n_total,
                      int64_t base, int64_t n, const int64_t *action_tags_host,
                      int32_t n_tags, int64_t *actions_dev, void *stream);

/* Host-pointer parity entry points (replace the module-level cast_ray /
 * render_into / batch_kernel, _core.pyx:683-763). They copy H2D, run the
 * SAME device code as the batch path, copy D2H and synchronise. */
int tc_host_cast_ray(const uint8_t *kind, const int16_t *didx,
                     const uint8_t *dopen, int32_t h, int32_t w, double ox,
                     double oy, double rx, double ry, int32_t *status,
                     int32_t *mapx, int32_t *mapy, int32_t *side, double *perp,
                     double *wall_u, int32_t *steps);
int tc_host_render_into(const tc_tables *host, double px, double py, double dx,
                        double dy, const uint8_t *dopen_row,
                        const uint8_t *ealive_row, int32_t agoal,
                        uint8_t *frame, double *zbuf, int32_t *status);
int tc_host_batch_kernel(const tc_tables *host, const tc_state *state_host,
                         const int64_t *actions_host, const tc_out *out_host,
                         int64_t n, int32_t mode, int32_t auto_reset,
                         int32_t validate, int64_t *violations);

#ifdef __cplusplus
}
#endif
#endif /* TILECAST_B200_H */
