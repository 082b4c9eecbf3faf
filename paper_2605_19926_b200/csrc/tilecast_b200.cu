// tilecast_b200.cu -- B200-native (sm_100a) fused batched environment step.
//
// One launch steps N independent environments: dynamics (turn / slide move /
// doors / pickups / health / termination), auto-reset with the counter-based
// RNG, DDA ray cast per screen column, z-buffered sprite billboards, and the
// uint8 RGB frame written row-major to HBM with TMA bulk stores.
//
// Semantics: bit-exact with the reference's kernels
// (/root/reference/pkg/src/tilecast/backend/_pycore.py, transcribed in
// _core.pyx); every floating-point expression keeps the reference's operation
// order and is compiled with --fmad=false (no contraction), IEEE division and
// sqrt. Citations below are _pycore.py:line unless stated.
//
// Work decomposition:
//   * one warp owns one environment at a time; CTAs loop over envs
//     (grid sized to the SM count x occupancy, so every launch is one wave);
//   * dynamics run warp-uniform (every lane computes the same scalars);
//   * lane L casts the rays of columns L, L+32, ... (its z-buffer entries stay
//     in registers for the sprite pass);
//   * the frame is produced in horizontal bands staged in shared memory:
//     lanes compose 4-pixel (12-byte) groups with PRMT byte packing, sprites
//     overwrite their pixels column-by-column in draw order, and one lane
//     ships the band with cp.async.bulk (TMA bulk copy) while the warp
//     composes the next band into the other buffer.
//   * the packed tile map is staged once per CTA into shared memory.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/tilecast_b200.h"

namespace {

// ---------------------------------------------------------------- constants
// layout.py:8-66 (mirrored in paper_2605_19926_b200/layout.py)
enum { FC_MOVE_SPEED = 0, FC_RADIUS, FC_TURN_COS, FC_TURN_SIN, FC_ATTEN,
       FC_GOAL_REWARD, FC_LIVING_REWARD, FC_HEALTH_DECAY, FC_HEALTH_RESTORE,
       FC_SPRITE_K, FC_MIN_SPRITE_DEPTH, FC_COUNT };
enum { A_FORWARD = 0, A_BACKWARD, A_TURN_LEFT, A_TURN_RIGHT, A_STRAFE_LEFT,
       A_STRAFE_RIGHT, A_NOOP, A_COUNT };
enum { C_FLOOR = 0, C_WALL = 1, C_DOOR = 2 };
enum { K_KEY = 0, K_GOAL = 1, K_MEDKIT = 2 };
enum { EV_KEY_BASE_BIT = 0, EV_DOOR_BASE_BIT = 3, EV_MEDKIT_BIT = 6,
       EV_GOAL_BIT = 7, EV_DIED_BIT = 8, EV_TRUNCATED_BIT = 9 };
enum { MODE_RESET = 0, MODE_STEP = 1, MODE_RENDER = 2 };

constexpr double PLANE_HALF_WIDTH = 0.66;  // geometry.py:18
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t MIX2 = 0x94D049BB133111EBULL;
constexpr uint64_t SPLIT_SALT = 0x3C6EF372FE94F82AULL;

constexpr int WARPS_PER_CTA = 4;
#ifndef TC_TRACE
#define TC_TRACE 0  // perf experiments only: per-env phase timestamps
#endif
#ifndef TC_LOCKSTEP
#define TC_LOCKSTEP 2  // rays per lane marched in lockstep on sealed maps
#endif
#ifndef TC_SPRITE_UNIFIED
#define TC_SPRITE_UNIFIED 0  // 1 = one sprite pixel loop for the three kinds
#endif
#ifndef TC_STORE
#define TC_STORE __stcs  // frame stores (direct path): streaming / evict-first
#endif
#ifndef TC_MIN_CTAS16
#define TC_MIN_CTAS16 4  // the same for 16-lane-group kernels (128 registers)
#endif
#ifndef TC_MIN_CTAS16_WIDE
#define TC_MIN_CTAS16_WIDE 5  // 16-lane groups, multi-wave batches (96 registers)
#endif
#ifndef TC_MIN_CTAS
#define TC_MIN_CTAS 5  // resident CTAs per SM the register budget is sized for
#endif
#ifndef TC_MIN_CTAS_LEAN
#define TC_MIN_CTAS_LEAN 7  // lean one-env-per-warp kernel: 28 warps / SM (72 registers)
#endif
constexpr int BAND_BYTES_TARGET = 3072;       // per staging buffer
constexpr int CTA_SCRATCH = 160;               // step kernel per-CTA scratch bytes
constexpr int SMEM_MAP_MAX_CELLS = 4096;      // stage map in smem up to this
constexpr int CHAIN_MAX_RING = 64;             // one wave: ring slots with done rows
constexpr int CHAIN_DONE_ROW = 2048;           // done epochs per ring slot (>= CTAs)
constexpr int CHAIN_MAX_WAVES = 4;            // tc_batch_steps chains multi-wave batches up to this
constexpr int SMEM_U8_MAX_BYTES = 48 * 1024;  // u8 stop codes (+ tables) staged up to this

// packed cell word: bits 0-7 = wall colour or door index, 8-9 = cell tag,
// 16-23 = entity index + 1 (0 = no entity on the tile)
constexpr uint32_t CELL_TAG_SHIFT = 8;
constexpr uint32_t CELL_EAT_SHIFT = 16;

// ------------------------------------------------------------- device spec
struct SpecDev {
  const uint32_t* cell;     // [h*w] packed cells
  const uint32_t* solid;    // [h*w] stop codes: wall ~0u, door d 1u<<d, floor 0
  const uint32_t* pal;      // [n_pal] wall colours, r | g<<8 | b<<16
  const uint32_t* doorrgb;  // [D] door_rgb[dcol[d]]
  const uint8_t* dcol;      // [D]
  const uint8_t* dlock;     // [D]
  const double* epx;        // [E]
  const double* epy;        // [E]
  const uint8_t* ekind;     // [E]
  const uint8_t* ecol;      // [E]
  const double* spx;        // [S]
  const double* spy;        // [S]
  const int32_t* goal_ent;  // [G]
  const double* coef;       // [obs_w]
  double fc[FC_COUNT];
  double dirs[8];
  long long max_steps;
  int goal_mode, use_health;
  uint32_t ceil_rgb, floor_rgb, goal_rgb, med_box, med_cross, key_rgb[3];
  uint32_t legal_mask;
  int h, w, n_doors, n_ent, n_spawns, n_goals, n_pal, obs_h, obs_w;
  // launch geometry derived on the host
  int band_rows;     // rows per staging band
  int band_stride;   // bytes per staging buffer (16-aligned)
  int smem_map;      // 1 = stage cells + u32 stop codes into shared memory
  int smem_u8;       // 1 = map too large for that: stage u8 stop codes only (march in
                     //     shared memory; cells / dynamics read global memory)
  int b_code8;       // blob offset of the first u8 stop code (guards around it)
  int quads;         // 1 = obs_w % 4 == 0 (4-pixel packed compose)
  int bulk;          // 1 = frame rows are 16-byte multiples (TMA bulk store)
  int sealed;        // 1 = map rim is all wall (rays cannot escape)
  int mirror;        // 1 = mirrored-band SWAR compose (even H <= 254, W % 16 == 0)
  int mir_rpi;       // rows per 32-lane pass in the mirror compose (32 / (W/16), >= 1)
  int mir_rpi16;     // same for 16-lane groups
  int group;         // lanes per env: 32 (one env per warp) or 16 (two per warp)
  int direct;        // 1 = mirror compose stores straight to HBM (no TMA staging)
  int contig;        // direct path: lanes store consecutive 16-byte chunks ((W/16) | G)
  int npairs;        // mirror path: staged band pairs in flight (2..4)
  int lean;          // 1 = the lean one-env-per-warp step kernel applies (lean_kernel)
  int o_t0, o_b0, o_t8, o_wrgb, o_zbuf, o_gdep, o_recs, o_band;  // WarpSmem offsets
  int o_wpk, o_tpk;  // contig compose: packed wall RGB / per-byte top row streams
  int o_sct;         // contig sprites: per-column terms (f64[W] then u8[W] flags)
  int o_srow;        // contig sprites: per-row terms (f64[H] then u8[H] flags)
  int warp_smem;     // bytes of per-warp shared memory
  // Read-only tables staged per CTA into shared memory (smem offset = blob
  // offset): [coef | pal | doorrgb | epx | epy | spx | spy | goal_ent | dcol |
  // dlock | ekind | ecol] always, then [cells | guarded stop codes] when the
  // map fits (smem_map). stage_bytes = the staged prefix of the blob.
  const uint8_t* blob;
  int b_coef, b_pal, b_door, b_epx, b_epy, b_spx, b_spy, b_goal, b_dcol, b_dlock, b_ekind,
      b_ecol, b_cell, b_solid;
  int stage_bytes;
};

// the dynamic shared memory of every kernel that stages a spec
extern __shared__ __align__(16) uint8_t g_smem[];
template <class T>
__device__ __forceinline__ const T* stab(int off) {
  return reinterpret_cast<const T*>(g_smem + off);
}
#define T_COEF(S) stab<double>((S).b_coef)
#define T_PAL(S) stab<uint32_t>((S).b_pal)
#define T_DOOR(S) stab<uint32_t>((S).b_door)
#define T_EPX(S) stab<double>((S).b_epx)
#define T_EPY(S) stab<double>((S).b_epy)
#define T_SPX(S) stab<double>((S).b_spx)
#define T_SPY(S) stab<double>((S).b_spy)
#define T_GOAL(S) stab<int32_t>((S).b_goal)
#define T_DCOL(S) stab<uint8_t>((S).b_dcol)
#define T_DLOCK(S) stab<uint8_t>((S).b_dlock)
#define T_EKIND(S) stab<uint8_t>((S).b_ekind)
#define T_ECOL(S) stab<uint8_t>((S).b_ecol)

struct StateDev {
  double *px, *py, *dx, *dy, *health;
  uint8_t* inv;
  long long* t;
  unsigned long long *rkey, *rctr;
  uint8_t* done;
  int32_t* agoal;
  uint8_t* dopen;
  uint8_t* ealive;
};

struct OutDev {
  uint8_t* frames;
  double* zbuf;
  double* rewards;
  uint8_t* dones;
  uint8_t* truncs;
  uint32_t* events;
  int32_t* statuses;
  int32_t* rayinfo;
  unsigned long long* spritevis;
  // mapped host step (tc_batch_step_mapped): the last CTA copies
  // [rewards f64[n] | dones u8[n]] to res_host; a bad action sets *flag_host
  uint8_t* res_host;
  int32_t* flag_host;
};

struct RolloutArgs {
  unsigned long long policy_key;
  long long base, n_total, step0;
  int k_steps, frame_ring;
  int n_tags;
  int tags[A_COUNT];
};

// per-env register state, warp-uniform
struct Env {
  double x, y, dx, dy, health;
  long long t;
  unsigned long long rkey, rctr;
  uint32_t dmask;       // bit d = door d open
  unsigned long long emask;  // bit e = entity e alive
  int agoal;
  uint32_t inv;
  int done;
};

// sprite record in draw order (far -> near), _pycore.py:219-252
struct SpriteRec {
  double dep, ks, halfk;
  int vtop, denom, r0, r1;
  uint32_t s1, s2;  // shaded main / secondary colour
  int kd, ent;
};

#if TC_TRACE
__device__ unsigned long long* g_trace = nullptr;
// per-CTA launch timeline [generation][cta][4]: entry, map staged, past
// griddepcontrol.wait, exit; the generation of a CTA is the number of
// earlier launches whose CTA of the same index entered (PDL starts every
// CTA of a launch before any CTA of its dependent)
__device__ unsigned long long* g_trace_cta = nullptr;
__device__ unsigned int g_cta_gen[16384];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(i, slot)                                                   \
  do {                                                                   \
    if (g_trace && (threadIdx.x & (G - 1)) == 0) g_trace[(i) * 16 + (slot)] = gtime(); \
  } while (0)
#else
#define TRACE(i, slot) do { } while (0)
#endif

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= MIX1;
  x ^= x >> 27;
  x *= MIX2;
  x ^= x >> 31;
  return x;
}

// _pycore.py:27-35
__device__ __forceinline__ uint64_t draw_below(uint64_t key, unsigned long long& ctr,
                                               uint64_t n) {
  const uint64_t x = mix64(key + ctr * GOLDEN);
  ctr += 1;
  return __umul64hi(x, n);
}

// Exact small-integer <-> double conversions on the fp64 pipe instead of the
// conversion unit: for 0 <= k < 2^31, double(k) = as_double(2^52 bits | k) -
// 2^52; for 0 <= x < 2^52, floor(x) is the low word of x + 2^52 rounded
// toward -inf (the ulp of 2^52 is 1).
__device__ __forceinline__ double u2d_small(uint32_t k) {
  return __longlong_as_double(0x4330000000000000LL | (long long)k) - 0x1p52;
}
__device__ __forceinline__ int floor_small(double x) {
  return (int)(uint32_t)__double_as_longlong(__dadd_rd(x, 0x1p52));
}
// rgb_scale for shade in [0, 1] (every product in [0, 255]): the same
// (int)(channel * shade) per channel, _pycore.py:168-170
__device__ __forceinline__ uint32_t rgb_scale_unit(uint32_t rgb, double shade) {
  const int r = floor_small(u2d_small(rgb & 0xffu) * shade);
  const int g = floor_small(u2d_small((rgb >> 8) & 0xffu) * shade);
  const int b = floor_small(u2d_small((rgb >> 16) & 0xffu) * shade);
  return (uint32_t)(r & 0xff) | ((uint32_t)(g & 0xff) << 8) | ((uint32_t)(b & 0xff) << 16);
}

__device__ __forceinline__ uint32_t rgb_scale(uint32_t rgb, double shade) {
  // (int)(channel * shade) per channel, _pycore.py:168-170
  const int r = (int)((double)(rgb & 0xff) * shade);
  const int g = (int)((double)((rgb >> 8) & 0xff) * shade);
  const int b = (int)((double)((rgb >> 16) & 0xff) * shade);
  return (uint32_t)(r & 0xff) | ((uint32_t)(g & 0xff) << 8) | ((uint32_t)(b & 0xff) << 16);
}

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// DDA, _pycore.py:38-96. `cell` may point at shared or global memory.
struct RayHit {
  int status, mapx, mapy, side, steps;
  double perp, wu;
};

__device__ __forceinline__ RayHit cast_ray(const uint32_t* __restrict__ cell, int h, int w,
                                           uint32_t dmask, double ox, double oy,
                                           double rx, double ry) {
  int mapx = (int)floor(ox);
  int mapy = (int)floor(oy);
  double ddx, ddy, sdx, sdy;
  int stepx, stepy;
  if (rx != 0.0) {
    ddx = fabs(1.0 / rx);
    stepx = rx > 0.0 ? 1 : -1;
    sdx = rx > 0.0 ? (((double)mapx + 1.0) - ox) * ddx : (ox - (double)mapx) * ddx;
  } else {
    ddx = dinf();
    stepx = 0;
    sdx = dinf();
  }
  if (ry != 0.0) {
    ddy = fabs(1.0 / ry);
    stepy = ry > 0.0 ? 1 : -1;
    sdy = ry > 0.0 ? (((double)mapy + 1.0) - oy) * ddy : (oy - (double)mapy) * ddy;
  } else {
    ddy = dinf();
    stepy = 0;
    sdy = dinf();
  }
  const int limit = 2 * (w + h);
  int side = 0, steps = 0;
  RayHit r;
  for (;;) {
    if (sdx < sdy) {  // ties step Y (_pycore.py:70)
      sdx += ddx;
      mapx += stepx;
      side = 0;
    } else {
      sdy += ddy;
      mapy += stepy;
      side = 1;
    }
    steps += 1;
    if (steps > limit || (unsigned)mapx >= (unsigned)w || (unsigned)mapy >= (unsigned)h) {
      r.status = steps > limit ? TC_ST_STEP_BUDGET : TC_ST_ESCAPED;
      r.mapx = mapx; r.mapy = mapy; r.side = side; r.steps = steps;
      r.perp = 0.0; r.wu = 0.0;
      return r;
    }
    const uint32_t cw = cell[mapy * w + mapx];
    const uint32_t tag = (cw >> CELL_TAG_SHIFT) & 3u;
    if (tag == C_WALL) break;
    if (tag == C_DOOR && ((dmask >> (cw & 31u)) & 1u) == 0) break;
  }
  double perp, wu;
  if (side == 0) {
    perp = sdx - ddx;
    wu = oy + perp * ry;
  } else {
    perp = sdy - ddy;
    wu = ox + perp * rx;
  }
  wu -= floor(wu);
  r.status = TC_ST_OK;
  r.mapx = mapx; r.mapy = mapy; r.side = side; r.steps = steps;
  r.perp = perp; r.wu = wu;
  return r;
}


// A group of G lanes (G = 32: one env per warp; G = 16: two envs per warp,
// one per half) and its collectives. Masks are the group's own, so the two
// halves of a warp may diverge freely.
template <int G>
struct Grp {
  int lane;        // lane within the group
  int shift;       // bit offset of the group inside the warp
  unsigned mask;   // member mask
  __device__ __forceinline__ Grp() {
    const int l = threadIdx.x & 31;
    lane = l & (G - 1);
    shift = l & ~(G - 1) & 31;
    mask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << shift);
  }
  __device__ __forceinline__ unsigned ballot(bool p) const {
    return (__ballot_sync(mask, p) & mask) >> shift;
  }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(mask, p); }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  template <class T>
  __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(mask, v, src, G); }
  __device__ __forceinline__ int min(int v) const {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = ::min(v, __shfl_xor_sync(mask, v, o, G));
    return v;
  }
  __device__ __forceinline__ int max(int v) const {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = ::max(v, __shfl_xor_sync(mask, v, o, G));
    return v;
  }
};

// One pass over the <= 2x2 tiles the disc (cx, cy, radius) overlaps, doing
// _touch_doors (_pycore.py:307-343; only when `touch`) and then _blocked
// (:274-304) for each tile. Equivalent to the reference's two passes: a
// door's open flag only affects its own tile (one door record per door
// cell), and touch never skips a tile that blocked would test. The tiles are
// tested lane-parallel (lane q of the group takes tile (tx0 + q%2, ty0 +
// q/2)) and combined with group reductions. Returns (door mask, events,
// blocked-after-touch) packed.
template <int G>
__device__ __forceinline__ uint64_t scan_tiles(const SpecDev& S, const uint32_t* __restrict__ cell,
                                               const uint32_t* __restrict__ solid,
                                               uint32_t dmask, double cx, double cy,
                                               double radius, uint32_t inv, bool touch) {
  const Grp<G> g;
  const int tx0 = (int)floor(cx - radius), tx1 = (int)floor(cx + radius);
  const int ty0 = (int)floor(cy - radius), ty1 = (int)floor(cy + radius);
  const double r2 = radius * radius;
  const int tx = tx0 + (g.lane & 1), ty = ty0 + ((g.lane >> 1) & 1);
  uint32_t opened = 0, events = 0;
  bool b = false;
  if (g.lane < 4 && tx <= tx1 && ty <= ty1) {
    if (tx < 0 || tx >= S.w || ty < 0 || ty >= S.h) {
      b = true;
    } else {
      const uint32_t code = solid[ty * S.w + tx];
      if (code != 0u) {  // not floor
        double nx = cx;
        if (nx < tx) nx = tx;
        else if (nx > tx + 1.0) nx = tx + 1.0;
        double ny = cy;
        if (ny < ty) ny = ty;
        else if (ny > ty + 1.0) ny = ty + 1.0;
        const double ddx = cx - nx, ddy = cy - ny;
        if (ddx * ddx + ddy * ddy < r2) {  // overlap
          uint32_t dm = dmask;
          if (code != 0xffffffffu && (code & ~dm) != 0u && touch) {  // closed door
            const int di = (int)(cell[ty * S.w + tx] & 31u);
            const int dc = T_DCOL(S)[di];
            if (!(T_DLOCK(S)[di] != 0 && ((inv >> dc) & 1u) == 0)) {
              opened = 1u << di;
              events = 1u << (EV_DOOR_BASE_BIT + dc);
              dm |= opened;
            }
          }
          if ((code & ~dm) != 0u || code == 0xffffffffu) b = true;
        }
      }
    }
  }
  dmask |= __reduce_or_sync(g.mask, opened);
  events = __reduce_or_sync(g.mask, events);
  const bool blk = g.any(b);
  // packed result: new door mask | events << 32 | blocked << 63
  return (uint64_t)dmask | ((uint64_t)events << 32) | ((uint64_t)(blk ? 1 : 0) << 63);
}

// _pycore.py:390-414: draws in the contract order spawn, heading, goal
__device__ __forceinline__ void reset_draws_inl(const SpecDev& S, Env& e) {
  unsigned long long ctr = e.rctr;
  uint64_t v = draw_below(e.rkey, ctr, (uint64_t)S.n_spawns);
  e.x = T_SPX(S)[v];
  e.y = T_SPY(S)[v];
  v = draw_below(e.rkey, ctr, 4);
  e.dx = S.dirs[2 * v];
  e.dy = S.dirs[2 * v + 1];
  if (S.goal_mode == 1 && S.n_goals > 0) {
    v = draw_below(e.rkey, ctr, (uint64_t)S.n_goals);
    e.agoal = T_GOAL(S)[v];
  } else if (S.n_goals > 0) {
    e.agoal = T_GOAL(S)[0];
  } else {
    e.agoal = -1;
  }
  e.rctr = ctr;
  e.health = 100.0;
  e.inv = 0;
  e.t = 0;
  e.done = 0;
  e.dmask = 0;
  e.emask = S.n_ent >= 64 ? ~0ULL : ((1ULL << S.n_ent) - 1ULL);
}

// out of line: runs once per episode (instruction-cache footprint)
__device__ __noinline__ Env reset_env(const SpecDev& S, unsigned long long rkey,
                                      unsigned long long rctr) {
  Env e;
  e.rkey = rkey;
  e.rctr = rctr;
  reset_draws_inl(S, e);
  return e;
}
__device__ __forceinline__ void reset_draws(const SpecDev& S, Env& e) {
  e = reset_env(S, e.rkey, e.rctr);
}

struct StepOut {
  double reward;
  uint32_t events;
  int done, trunc, violation;
};

// _pycore.py:431-531 (everything before the render / auto-reset branch);
// called by all G lanes of the group (the tile scan is lane-parallel)
template <int G>
__device__ __forceinline__ StepOut step_dynamics(const SpecDev& S, const uint32_t* __restrict__ cell,
                                                 const uint32_t* __restrict__ solid, Env& e,
                                                 int act, int validate) {
  StepOut o;
  o.events = 0;
  o.reward = 0.0;
  o.violation = 0;
  int terminated = 0, truncated = 0;
  double x = e.x, y = e.y, dxx = e.dx, dyy = e.dy;
  const double ms = S.fc[FC_MOVE_SPEED], radius = S.fc[FC_RADIUS];
  if (act == A_TURN_LEFT || act == A_TURN_RIGHT) {
    const double s = act == A_TURN_RIGHT ? S.fc[FC_TURN_SIN] : -S.fc[FC_TURN_SIN];
    const double cs = S.fc[FC_TURN_COS];
    const double ndx = dxx * cs - dyy * s;
    const double ndy = dxx * s + dyy * cs;
    const double nrm = sqrt(ndx * ndx + ndy * ndy);
    dxx = ndx / nrm;
    dyy = ndy / nrm;
  } else if (act != A_NOOP) {
    double mvx = 0.0, mvy = 0.0;
    if (act == A_FORWARD) { mvx = ms * dxx; mvy = ms * dyy; }
    else if (act == A_BACKWARD) { mvx = -ms * dxx; mvy = -ms * dyy; }
    else if (act == A_STRAFE_LEFT) { mvx = ms * dyy; mvy = -ms * dxx; }
    else if (act == A_STRAFE_RIGHT) { mvx = -ms * dyy; mvy = ms * dxx; }
    // slide: resolve x then y; contact opens doors first (_pycore.py:476-488)
#pragma unroll 1
    for (int ax = 0; ax < 3; ax++) {
      if (ax == 2 && !validate) break;
      const double cx = ax == 0 ? x + mvx : x;
      const double cy = ax == 1 ? y + mvy : y;
      const uint64_t r = scan_tiles<G>(S, cell, solid, e.dmask, cx, cy, radius, e.inv, ax < 2);
      e.dmask = (uint32_t)r;
      o.events |= (uint32_t)(r >> 32) & 0x3ffu;
      const bool blk = (r >> 63) != 0;
      if (ax == 0 && !blk) x = cx;
      if (ax == 1 && !blk) y = cy;
      if (ax == 2 && blk) o.violation = 1;
    }
  }
  // pickups on the agent-centre tile only, _pycore.py:490-507
  const int ctx = (int)floor(x), cty = (int)floor(y);
  const int ent = (int)((cell[cty * S.w + ctx] >> CELL_EAT_SHIFT) & 0xffu) - 1;
  if (ent >= 0 && ((e.emask >> ent) & 1ULL)) {
    const int kd = T_EKIND(S)[ent];
    if (kd == K_KEY) {
      const int col = T_ECOL(S)[ent];
      e.inv = (e.inv | (1u << col)) & 0xffu;
      e.emask &= ~(1ULL << ent);
      o.events |= 1u << (EV_KEY_BASE_BIT + col);
    } else if (kd == K_MEDKIT) {
      e.emask &= ~(1ULL << ent);
      const double hv = e.health + S.fc[FC_HEALTH_RESTORE];
      e.health = hv > 100.0 ? 100.0 : hv;
      o.events |= 1u << EV_MEDKIT_BIT;
    } else if (kd == K_GOAL && ent == e.agoal) {
      o.reward = o.reward + S.fc[FC_GOAL_REWARD];
      terminated = 1;
      o.events |= 1u << EV_GOAL_BIT;
    }
  }
  // health layer, _pycore.py:509-516
  if (S.use_health != 0 && terminated == 0) {
    o.reward = o.reward + S.fc[FC_LIVING_REWARD];
    e.health = e.health - S.fc[FC_HEALTH_DECAY];
    if (e.health <= 0.0) {
      e.health = 0.0;
      terminated = 1;
      o.reward = 0.0;
      o.events |= 1u << EV_DIED_BIT;
    }
  }
  e.t = e.t + 1;
  if (terminated == 0 && e.t >= S.max_steps) {
    truncated = 1;
    o.events |= 1u << EV_TRUNCATED_BIT;
  }
  e.x = x; e.y = y; e.dx = dxx; e.dy = dyy;
  e.done = (terminated != 0 || truncated != 0) ? 1 : 0;
  o.done = e.done;
  o.trunc = truncated;
  return o;
}

// ------------------------------------------------------- async bulk stores
__device__ __forceinline__ void bulk_fence() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_copy(void* gdst, const void* ssrc, uint32_t bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gdst), "r"(s), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  bulk_copy(gdst, ssrc, bytes);
  bulk_commit();
}
// byte permute with per-byte sign replication (selector nibble bit 3)
__device__ __forceinline__ uint32_t prmt_sx(uint32_t a, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(a), "r"(sel));
  return d;
}
// wait until at most n bulk groups still read shared memory (n = 1..3)
__device__ __forceinline__ void bulk_wait_read_le(int n) {
  if (n <= 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  else if (n == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
  else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// --------------------------------------------------------------- rendering
// Per-warp shared memory layout (offsets in bytes, all 16-aligned):
//   spans: t0 u16[Wp], b0 u16[Wp], wrgb u32[Wp], zbuf f64[Wp]  (Wp = obs_w rounded to 4)
//   gather: dep f64[E], lat f64[E], ent i32[E]
//   recs: SpriteRec[E]
//   band buffers: 2 x band_stride
struct WarpSmem {
  // one 32-bit offset into the dynamic shared memory per lane group; the
  // regions sit at host-computed offsets carried in SpecDev (constant-bank
  // operands), so the compose / ray / sprite code does not keep a dozen
  // 64-bit pointers live in registers, and every access -- also inside the
  // out-of-line functions that receive a WarpSmem -- is visibly a
  // shared-memory access (LDS / STS, not a generic load)
  uint32_t off;
  __device__ __forceinline__ uint16_t* t0(const SpecDev& S) const { return (uint16_t*)(g_smem + off + S.o_t0); }
  __device__ __forceinline__ uint16_t* b0(const SpecDev& S) const { return (uint16_t*)(g_smem + off + S.o_b0); }
  __device__ __forceinline__ uint8_t* t8(const SpecDev& S) const { return g_smem + off + S.o_t8; }
  __device__ __forceinline__ uint32_t* wrgb(const SpecDev& S) const { return (uint32_t*)(g_smem + off + S.o_wrgb); }
  __device__ __forceinline__ uint8_t* wpk(const SpecDev& S) const { return g_smem + off + S.o_wpk; }
  __device__ __forceinline__ uint8_t* tpk(const SpecDev& S) const { return g_smem + off + S.o_tpk; }
  __device__ __forceinline__ double* sct(const SpecDev& S) const { return (double*)(g_smem + off + S.o_sct); }
  __device__ __forceinline__ uint8_t* scf(const SpecDev& S) const {
    return g_smem + off + S.o_sct + 8 * ((S.obs_w + 15) & ~15);
  }
  __device__ __forceinline__ double* srt(const SpecDev& S) const { return (double*)(g_smem + off + S.o_srow); }
  __device__ __forceinline__ uint8_t* srf(const SpecDev& S) const {
    return g_smem + off + S.o_srow + 8 * ((S.obs_h + 15) & ~15);
  }
  __device__ __forceinline__ double* zbuf(const SpecDev& S) const { return (double*)(g_smem + off + S.o_zbuf); }
  __device__ __forceinline__ double* gdep(const SpecDev& S) const { return (double*)(g_smem + off + S.o_gdep); }
  __device__ __forceinline__ SpriteRec* recs(const SpecDev& S) const { return (SpriteRec*)(g_smem + off + S.o_recs); }
  __device__ __forceinline__ uint8_t* band(const SpecDev& S, int k) const {
    return g_smem + off + S.o_band + k * S.band_stride;
  }
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

// wall colours are stored 16 columns per 20-word block (4 words of pad) so
// the per-16-column uint4 loads of neighbouring column groups fall in
// different bank quads (stride 20 words: 5*cg mod 8 is a permutation)
__host__ __device__ __forceinline__ int wslot(int c) { return c + ((c >> 4) << 2); }

// per-warp shared-memory layout; returns the window size. nbands = staging
// buffers (0 for the direct-store compose).
__host__ inline int warp_smem_layout(SpecDev& d, int nbands) {
  const int wp = (d.obs_w + 15) & ~15;
  const int e = d.n_ent > 0 ? d.n_ent : 1;
  int off = 0;
  d.o_t0 = off; off += align16(wp * 2);
  d.o_b0 = off; off += align16(wp * 2);
  d.o_t8 = off; off += align16(wp);
  d.o_wrgb = off; off += align16((wp / 16) * 20 * 4 + 64);
  d.o_zbuf = off; off += align16(wp * 8);
  d.o_gdep = off; off += align16(e * 8);
  d.o_recs = off; off += align16(e * (int)sizeof(SpriteRec));
  d.o_band = off; off += nbands * d.band_stride;
  // contig compose: the wall colours / tops as byte streams laid out like a
  // frame row (3 bytes per column)
  d.o_wpk = off; off += d.contig ? align16(3 * wp) : 0;
  d.o_tpk = off; off += d.contig ? align16(3 * wp) : 0;
  d.o_sct = off; off += d.contig ? align16(9 * wp) : 0;
  d.o_srow = off; off += d.contig ? align16(9 * ((d.obs_h + 15) & ~15)) : 0;
  return align16(off);
}

__device__ inline WarpSmem carve(uint8_t* base) {
  WarpSmem m;
  m.off = (uint32_t)(base - g_smem);
  return m;
}


// (int)min(H / perp, 1e9) // 2 (_pycore.py:171-174) with the IEEE division
// replaced on the common path: q = H * r, r = rcp.approx refined by two
// Newton steps (relative error < 2^-50), is within q * 2^-49 of H / perp,
// and fl(H / perp) within q * 2^-53 of it; when q is farther than
// q * 2^-40 from an integer, floor(q) = floor(fl(H / perp)) exactly.
// Near-integers, q >= 1e9 - 1 and non-finite values take the division.
__device__ __forceinline__ int line_half(int H, double perp) {
  double r0;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(perp));
  const double e0 = fma(-perp, r0, 1.0);
  const double r1 = fma(r0, e0, r0);
  const double e1 = fma(-perp, r1, 1.0);
  const double r2 = fma(r1, e1, r1);
  const double q = (double)H * r2;
  if (q < 999999999.0) {  // (false for NaN / inf too)
    const int iq = floor_small(q);
    const double fq = u2d_small((uint32_t)iq);
    const double tol = q * 0x1p-40;
    if (q - fq > tol && (fq + 1.0) - q > tol) return iq >> 1;
  }
  double lh_f = (double)H / perp;
  if (lh_f > 1e9) lh_f = 1e9;
  return (int)lh_f / 2;
}

// One DDA march, _pycore.py:38-96. `solid` holds per-cell stop codes
// (wall = ~0u, door d = 1u << d, floor = 0): a ray stops in a cell iff
// (code & ~dmask) != 0 or code == ~0u (walls, closed doors). With a sealed
// rim and the origin inside the grid a ray can neither escape nor exceed
// the 2(w+h) budget (it crosses at most w+h-2 boundaries before the rim),
// so CHECKED=false drops those tests; the result is identical.
struct March {
  double sdx, sdy, ddx, ddy;
  int idx, steps, status;
  bool xs;  // last step was an x step (side 0)
};

__device__ __forceinline__ bool stops(uint32_t code, uint32_t dmask) {
  return (code & ~dmask) != 0u || code == 0xffffffffu;
}

template <bool CHECKED>
__device__ __forceinline__ March march(const uint32_t* __restrict__ solid, int mw, int mh,
                                       uint32_t dmask, double ox, double oy, int mapx0,
                                       int mapy0, double rx, double ry) {
  March r;
  int stepx, stepy;
  if (rx != 0.0) {
    r.ddx = fabs(1.0 / rx);
    stepx = rx > 0.0 ? 1 : -1;
    r.sdx = rx > 0.0 ? (((double)mapx0 + 1.0) - ox) * r.ddx : (ox - (double)mapx0) * r.ddx;
  } else {
    r.ddx = dinf(); stepx = 0; r.sdx = dinf();
  }
  if (ry != 0.0) {
    r.ddy = fabs(1.0 / ry);
    stepy = ry > 0.0 ? 1 : -1;
    r.sdy = ry > 0.0 ? (((double)mapy0 + 1.0) - oy) * r.ddy : (oy - (double)mapy0) * r.ddy;
  } else {
    r.ddy = dinf(); stepy = 0; r.sdy = dinf();
  }
  const int dyi = stepy * mw;
  int idx = mapy0 * mw + mapx0;
  int steps = 0;
  bool xs = false;
  if (!CHECKED) {
    for (;;) {
      xs = r.sdx < r.sdy;  // ties step Y (_pycore.py:70)
      if (xs) { r.sdx += r.ddx; idx += stepx; } else { r.sdy += r.ddy; idx += dyi; }
      steps += 1;
      if (stops(solid[idx], dmask)) break;
    }
    r.status = TC_ST_OK;
  } else {
    int mapx = mapx0, mapy = mapy0;
    const int limit = 2 * (mw + mh);
    r.status = TC_ST_OK;
    for (;;) {
      xs = r.sdx < r.sdy;
      if (xs) { r.sdx += r.ddx; mapx += stepx; } else { r.sdy += r.ddy; mapy += stepy; }
      steps += 1;
      if (steps > limit) { r.status = TC_ST_STEP_BUDGET; break; }
      if ((unsigned)mapx >= (unsigned)mw || (unsigned)mapy >= (unsigned)mh) {
        r.status = TC_ST_ESCAPED;
        break;
      }
      idx = mapy * mw + mapx;
      if (stops(solid[idx], dmask)) break;
    }
    // escaped / budget: report the out-of-grid cell like the reference
    if (r.status != TC_ST_OK) idx = mapy * mw + mapx;
    if (r.status != TC_ST_OK) { r.steps = steps; r.xs = xs; r.idx = idx;
      r.sdx = (double)mapx; r.sdy = (double)mapy; return r; }
  }
  r.idx = idx;
  r.steps = steps;
  r.xs = xs;
  return r;
}

// Two rays marched in lockstep (sealed-map fast path): the two dependency
// chains interleave, hiding latency when few warps share the SM. Each ray
// follows exactly the same sequence of operations as march<false>.
struct RaySetup {
  double sdx, sdy, ddx, ddy;
  int stepx, dyi, idx;
};
__device__ __forceinline__ RaySetup ray_setup(int mw, double ox, double oy, int mapx0, int mapy0,
                                              double rx, double ry) {
  // _pycore.py:44-63 without branches: __drcp_rn is the IEEE reciprocal (the
  // exact 1.0 / r, inf for a zero component), the axis with a zero
  // component gets sdx = inf and step 0 like the reference; a NaN component
  // takes the reference's r < 0 arm (step -1)
  RaySetup r;
  r.ddx = fabs(__drcp_rn(rx));
  r.stepx = rx > 0.0 ? 1 : (rx != 0.0 ? -1 : 0);
  const double fx = rx > 0.0 ? (((double)mapx0 + 1.0) - ox) : (ox - (double)mapx0);
  r.sdx = rx != 0.0 ? fx * r.ddx : dinf();
  r.ddy = fabs(__drcp_rn(ry));
  const int stepy = ry > 0.0 ? 1 : (ry != 0.0 ? -1 : 0);
  const double fy = ry > 0.0 ? (((double)mapy0 + 1.0) - oy) : (oy - (double)mapy0);
  r.sdy = ry != 0.0 ? fy * r.ddy : dinf();
  r.dyi = stepy * mw;
  r.idx = mapy0 * mw + mapx0;
  return r;
}

__device__ __forceinline__ void march2(const uint32_t* __restrict__ solid, uint32_t dmask,
                                       RaySetup& a, RaySetup& b, March& ra, March& rb) {
  bool la = true, lb = true, xa = false, xb = false;
  int sa = 0, sb = 0;
  do {
    if (la) {
      xa = a.sdx < a.sdy;
      if (xa) { a.sdx += a.ddx; a.idx += a.stepx; } else { a.sdy += a.ddy; a.idx += a.dyi; }
      sa += 1;
    }
    if (lb) {
      xb = b.sdx < b.sdy;
      if (xb) { b.sdx += b.ddx; b.idx += b.stepx; } else { b.sdy += b.ddy; b.idx += b.dyi; }
      sb += 1;
    }
    if (la) la = !stops(solid[a.idx], dmask);
    if (lb) lb = !stops(solid[b.idx], dmask);
  } while (la || lb);
  ra.sdx = a.sdx; ra.sdy = a.sdy; ra.ddx = a.ddx; ra.ddy = a.ddy;
  ra.idx = a.idx; ra.steps = sa; ra.status = TC_ST_OK; ra.xs = xa;
  rb.sdx = b.sdx; rb.sdy = b.sdy; rb.ddx = b.ddx; rb.ddy = b.ddy;
  rb.idx = b.idx; rb.steps = sb; rb.status = TC_ST_OK; rb.xs = xb;
}

// R rays marched in lockstep: independent fp64 chains interleave. Each ray
// performs exactly the reference's additions in the reference's order. (A
// software-pipelined variant that issues step k+1's stop-code load before
// step k's test -- the stop-code array keeps the w+1-cell wall guards it
// needs -- measured no faster on B200.)
template <int R>
__device__ __forceinline__ void march_n(const uint32_t* __restrict__ solid, uint32_t dmask,
                                        RaySetup (&a)[R], March (&out)[R]) {
  bool live[R], xs[R];
  int st[R];
#pragma unroll
  for (int q = 0; q < R; q++) { live[q] = true; xs[q] = false; st[q] = 0; }
  bool any;
  do {
#pragma unroll
    for (int q = 0; q < R; q++) {
      if (live[q]) {
        xs[q] = a[q].sdx < a[q].sdy;  // ties step Y (_pycore.py:70)
        if (xs[q]) { a[q].sdx += a[q].ddx; a[q].idx += a[q].stepx; }
        else { a[q].sdy += a[q].ddy; a[q].idx += a[q].dyi; }
        st[q] += 1;
      }
    }
    any = false;
#pragma unroll
    for (int q = 0; q < R; q++) {
      if (live[q]) live[q] = !stops(solid[a[q].idx], dmask);
      any |= live[q];
    }
  } while (any);
#pragma unroll
  for (int q = 0; q < R; q++) {
    out[q].sdx = a[q].sdx; out[q].sdy = a[q].sdy; out[q].ddx = a[q].ddx; out[q].ddy = a[q].ddy;
    out[q].idx = a[q].idx; out[q].steps = st[q]; out[q].status = TC_ST_OK; out[q].xs = xs[q];
  }
}

// R rays in lockstep over the shared-memory stop codes (map staged in smem,
// fewer than 32 doors, sealed rim): every ray keeps a running shared-memory
// byte address instead of a cell index, steps under a predicate (one DSETP,
// one predicated DADD per axis, one SEL + IADD on the address, one LDS, one
// LOP3 stop test against ~dmask -- walls ~0u always intersect it because bit
// 31 of dmask is clear with < 32 doors). The side of the last step is
// recovered from the last address increment (|stepx| = 4 B, |dyi| = 4*mw B,
// mw >= 2), the step count (debug taps only) from the cell displacement
// (each x step moves mapx by stepx, each y step mapy by stepy). The adds are
// the reference's, in its order (_pycore.py:66-80).
struct FastRay {
  double sdx, sdy, ddx, ddy;
  uint32_t addr;   // shared byte address of the current cell's stop code
  int incx, incy;  // byte increments of an x / y step
  int last;        // increment of the last step
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Two rays: the whole loop in PTX so the live flags stay predicates and the
// axis choice predicates the adds (the C version compiles to compute-both +
// FSEL and byte-sized live flags: ~43 instructions per iteration vs 20).
__device__ __forceinline__ void march_fast2(uint32_t smask, FastRay& a, FastRay& b) {
  asm volatile(
      "{\n\t"
      ".reg .pred l0, l1, x0, y0, x1, y1, any;\n\t"
      ".reg .b32 c0, c1, ix0, iy0, ix1, iy1, sm;\n\t"
      ".reg .f64 ex0, ey0, ex1, ey1;\n\t"
      // copy every input first: an input may share a register with an
      // in/out operand (no early-clobber), and the loop writes those
      "mov.f64 ex0, %8;\n\t"
      "mov.f64 ey0, %9;\n\t"
      "mov.b32 ix0, %10;\n\t"
      "mov.b32 iy0, %11;\n\t"
      "mov.f64 ex1, %12;\n\t"
      "mov.f64 ey1, %13;\n\t"
      "mov.b32 ix1, %14;\n\t"
      "mov.b32 iy1, %15;\n\t"
      "mov.b32 sm, %16;\n\t"
      "setp.eq.b32 l0, sm, sm;\n\t"
      "setp.eq.b32 l1, sm, sm;\n\t"
      "MARCH%=:\n\t"
      // one compare per ray: x = (sdx < sdy) & live, y = !(sdx < sdy) & live
      "setp.lt.and.f64 x0|y0, %0, %1, l0;\n\t"
      "setp.lt.and.f64 x1|y1, %4, %5, l1;\n\t"
      "@x0 add.rn.f64 %0, %0, ex0;\n\t"
      "@y0 add.rn.f64 %1, %1, ey0;\n\t"
      "@x1 add.rn.f64 %4, %4, ex1;\n\t"
      "@y1 add.rn.f64 %5, %5, ey1;\n\t"
      "@l0 selp.b32 %3, ix0, iy0, x0;\n\t"
      "@l1 selp.b32 %7, ix1, iy1, x1;\n\t"
      "@l0 add.u32 %2, %2, %3;\n\t"
      "@l1 add.u32 %6, %6, %7;\n\t"
      "@l0 ld.shared.u32 c0, [%2];\n\t"
      "@l1 ld.shared.u32 c1, [%6];\n\t"
      "@l0 and.b32 c0, c0, sm;\n\t"
      "@l1 and.b32 c1, c1, sm;\n\t"
      "@l0 setp.eq.b32 l0, c0, 0;\n\t"
      "@l1 setp.eq.b32 l1, c1, 0;\n\t"
      "or.pred any, l0, l1;\n\t"
      "@any bra MARCH%=;\n\t"
      "}"
      : "+d"(a.sdx), "+d"(a.sdy), "+r"(a.addr), "+r"(a.last),
        "+d"(b.sdx), "+d"(b.sdy), "+r"(b.addr), "+r"(b.last)
      : "d"(a.ddx), "d"(a.ddy), "r"(a.incx), "r"(a.incy),
        "d"(b.ddx), "d"(b.ddy), "r"(b.incx), "r"(b.incy), "r"(smask));
}

// march_fast2 over u8 stop codes (large maps): code 0 floor, d + 1 door d
// (n_doors <= 30), 31 wall; a ray stops iff bit `code` of `smask` is set,
// smask = (closed doors << 1) | 1 << 31. One LDS.U8 + SHF + LOP3 per step.
__device__ __forceinline__ void march_fast2_u8(uint32_t smask, FastRay& a, FastRay& b) {
  asm volatile(
      "{\n\t"
      ".reg .pred l0, l1, x0, y0, x1, y1, any;\n\t"
      ".reg .b32 c0, c1, ix0, iy0, ix1, iy1, sm;\n\t"
      ".reg .f64 ex0, ey0, ex1, ey1;\n\t"
      "mov.f64 ex0, %8;\n\t"
      "mov.f64 ey0, %9;\n\t"
      "mov.b32 ix0, %10;\n\t"
      "mov.b32 iy0, %11;\n\t"
      "mov.f64 ex1, %12;\n\t"
      "mov.f64 ey1, %13;\n\t"
      "mov.b32 ix1, %14;\n\t"
      "mov.b32 iy1, %15;\n\t"
      "mov.b32 sm, %16;\n\t"
      "setp.eq.b32 l0, sm, sm;\n\t"
      "setp.eq.b32 l1, sm, sm;\n\t"
      "MARCH8%=:\n\t"
      "setp.lt.and.f64 x0|y0, %0, %1, l0;\n\t"
      "setp.lt.and.f64 x1|y1, %4, %5, l1;\n\t"
      "@x0 add.rn.f64 %0, %0, ex0;\n\t"
      "@y0 add.rn.f64 %1, %1, ey0;\n\t"
      "@x1 add.rn.f64 %4, %4, ex1;\n\t"
      "@y1 add.rn.f64 %5, %5, ey1;\n\t"
      "@l0 selp.b32 %3, ix0, iy0, x0;\n\t"
      "@l1 selp.b32 %7, ix1, iy1, x1;\n\t"
      "@l0 add.u32 %2, %2, %3;\n\t"
      "@l1 add.u32 %6, %6, %7;\n\t"
      "@l0 ld.shared.u8 c0, [%2];\n\t"
      "@l1 ld.shared.u8 c1, [%6];\n\t"
      "@l0 shr.b32 c0, sm, c0;\n\t"
      "@l1 shr.b32 c1, sm, c1;\n\t"
      "@l0 and.b32 c0, c0, 1;\n\t"
      "@l1 and.b32 c1, c1, 1;\n\t"
      "@l0 setp.eq.b32 l0, c0, 0;\n\t"
      "@l1 setp.eq.b32 l1, c1, 0;\n\t"
      "or.pred any, l0, l1;\n\t"
      "@any bra MARCH8%=;\n\t"
      "}"
      : "+d"(a.sdx), "+d"(a.sdy), "+r"(a.addr), "+r"(a.last),
        "+d"(b.sdx), "+d"(b.sdy), "+r"(b.addr), "+r"(b.last)
      : "d"(a.ddx), "d"(a.ddy), "r"(a.incx), "r"(a.incy),
        "d"(b.ddx), "d"(b.ddy), "r"(b.incx), "r"(b.incy), "r"(smask));
}

// Four rays in lockstep (TC_LOCKSTEP=4): same loop as march_fast2; each
// ray's x / y byte increments arrive packed as (incy << 8) | (incx & 0xff)
// to stay within the asm operand limit.
__device__ __forceinline__ void march_fast4(uint32_t smask, FastRay (&a)[4]) {
  uint32_t pk[4];
#pragma unroll
  for (int q = 0; q < 4; q++) pk[q] = ((uint32_t)a[q].incy << 8) | ((uint32_t)a[q].incx & 0xffu);
  asm volatile(
      "{\n\t"
      ".reg .pred l0, l1, l2, l3, x0, y0, x1, y1, x2, y2, x3, y3, any;\n\t"
      ".reg .b32 c0, c1, c2, c3, ix0, iy0, ix1, iy1, ix2, iy2, ix3, iy3, sm, t;\n\t"
      ".reg .f64 ex0, ey0, ex1, ey1, ex2, ey2, ex3, ey3;\n\t"
      // inputs are copied first (no early-clobber on the in/out operands)
      "mov.f64 ex0, %16;\n\t"
      "mov.f64 ey0, %17;\n\t"
      "shl.b32 t, %18, 24;\n\t"
      "shr.s32 ix0, t, 24;\n\t"
      "shr.s32 iy0, %18, 8;\n\t"
      "mov.f64 ex1, %19;\n\t"
      "mov.f64 ey1, %20;\n\t"
      "shl.b32 t, %21, 24;\n\t"
      "shr.s32 ix1, t, 24;\n\t"
      "shr.s32 iy1, %21, 8;\n\t"
      "mov.f64 ex2, %22;\n\t"
      "mov.f64 ey2, %23;\n\t"
      "shl.b32 t, %24, 24;\n\t"
      "shr.s32 ix2, t, 24;\n\t"
      "shr.s32 iy2, %24, 8;\n\t"
      "mov.f64 ex3, %25;\n\t"
      "mov.f64 ey3, %26;\n\t"
      "shl.b32 t, %27, 24;\n\t"
      "shr.s32 ix3, t, 24;\n\t"
      "shr.s32 iy3, %27, 8;\n\t"
      "mov.b32 sm, %28;\n\t"
      "setp.eq.b32 l0, sm, sm;\n\t"
      "setp.eq.b32 l1, sm, sm;\n\t"
      "setp.eq.b32 l2, sm, sm;\n\t"
      "setp.eq.b32 l3, sm, sm;\n\t"
      "MARCH4%=:\n\t"
      "setp.lt.and.f64 x0, %0, %1, l0;\n\t"
      "setp.geu.and.f64 y0, %0, %1, l0;\n\t"
      "setp.lt.and.f64 x1, %4, %5, l1;\n\t"
      "setp.geu.and.f64 y1, %4, %5, l1;\n\t"
      "setp.lt.and.f64 x2, %8, %9, l2;\n\t"
      "setp.geu.and.f64 y2, %8, %9, l2;\n\t"
      "setp.lt.and.f64 x3, %12, %13, l3;\n\t"
      "setp.geu.and.f64 y3, %12, %13, l3;\n\t"
      "@x0 add.rn.f64 %0, %0, ex0;\n\t"
      "@y0 add.rn.f64 %1, %1, ey0;\n\t"
      "@x1 add.rn.f64 %4, %4, ex1;\n\t"
      "@y1 add.rn.f64 %5, %5, ey1;\n\t"
      "@x2 add.rn.f64 %8, %8, ex2;\n\t"
      "@y2 add.rn.f64 %9, %9, ey2;\n\t"
      "@x3 add.rn.f64 %12, %12, ex3;\n\t"
      "@y3 add.rn.f64 %13, %13, ey3;\n\t"
      "@l0 selp.b32 %3, ix0, iy0, x0;\n\t"
      "@l0 add.u32 %2, %2, %3;\n\t"
      "@l1 selp.b32 %7, ix1, iy1, x1;\n\t"
      "@l1 add.u32 %6, %6, %7;\n\t"
      "@l2 selp.b32 %11, ix2, iy2, x2;\n\t"
      "@l2 add.u32 %10, %10, %11;\n\t"
      "@l3 selp.b32 %15, ix3, iy3, x3;\n\t"
      "@l3 add.u32 %14, %14, %15;\n\t"
      "@l0 ld.shared.u32 c0, [%2];\n\t"
      "@l1 ld.shared.u32 c1, [%6];\n\t"
      "@l2 ld.shared.u32 c2, [%10];\n\t"
      "@l3 ld.shared.u32 c3, [%14];\n\t"
      "@l0 and.b32 c0, c0, sm;\n\t"
      "@l0 setp.eq.b32 l0, c0, 0;\n\t"
      "@l1 and.b32 c1, c1, sm;\n\t"
      "@l1 setp.eq.b32 l1, c1, 0;\n\t"
      "@l2 and.b32 c2, c2, sm;\n\t"
      "@l2 setp.eq.b32 l2, c2, 0;\n\t"
      "@l3 and.b32 c3, c3, sm;\n\t"
      "@l3 setp.eq.b32 l3, c3, 0;\n\t"
      "or.pred any, l0, l1;\n\t"
      "or.pred any, any, l2;\n\t"
      "or.pred any, any, l3;\n\t"
      "@any bra MARCH4%=;\n\t"
      "}"
      : "+d"(a[0].sdx), "+d"(a[0].sdy), "+r"(a[0].addr), "+r"(a[0].last),
        "+d"(a[1].sdx), "+d"(a[1].sdy), "+r"(a[1].addr), "+r"(a[1].last),
        "+d"(a[2].sdx), "+d"(a[2].sdy), "+r"(a[2].addr), "+r"(a[2].last),
        "+d"(a[3].sdx), "+d"(a[3].sdy), "+r"(a[3].addr), "+r"(a[3].last)
      : "d"(a[0].ddx), "d"(a[0].ddy), "r"(pk[0]), "d"(a[1].ddx), "d"(a[1].ddy), "r"(pk[1]),
        "d"(a[2].ddx), "d"(a[2].ddy), "r"(pk[2]), "d"(a[3].ddx), "d"(a[3].ddy), "r"(pk[3]),
        "r"(smask));
}

template <int R>
__device__ __forceinline__ void march_fast(uint32_t smask, FastRay (&a)[R]) {
  if constexpr (R == 4) {
    march_fast4(smask, a);
    return;
  }
  if constexpr (R == 2) {
    march_fast2(smask, a[0], a[1]);
    return;
  }
  uint32_t live = (1u << R) - 1u;
#pragma unroll 1
  do {
#pragma unroll
    for (int q = 0; q < R; q++) {
      if (live & (1u << q)) {
        const bool x = a[q].sdx < a[q].sdy;  // ties step Y (_pycore.py:70)
        if (x) a[q].sdx += a[q].ddx; else a[q].sdy += a[q].ddy;
        a[q].last = x ? a[q].incx : a[q].incy;
        a[q].addr += a[q].last;
      }
    }
#pragma unroll
    for (int q = 0; q < R; q++) {
      if (live & (1u << q)) {
        if ((lds_u32(a[q].addr) & smask) != 0u) live &= ~(1u << q);
      }
    }
  } while (live);
}

// Wall pass: lane L casts the rays of columns L + 32j; per-column spans,
// colours and zbuf go to shared memory (_pycore.py:153-190). Returns the
// status of the first failing column (warp-uniform).
template <int NC, bool CHECKED, int G, bool FAST = false, int FWC = 0, int FHC = 0>
__device__ __forceinline__ int wall_pass(const SpecDev& S, const uint32_t* __restrict__ cell,
                                         const uint32_t* __restrict__ solid,
                                         const WarpSmem& sm, const Env& e, double planex,
                                         double planey, double* __restrict__ zbuf_out,
                                         int32_t* __restrict__ rayinfo, long long ti = -1) {
  const Grp<G> g;
  const int lane = g.lane;
  // (FWC / FHC: compile-time frame shape -- the column rounds unroll)
  const int W = FWC ? FWC : S.obs_w, H = FHC ? FHC : S.obs_h, h2 = H / 2, mw = S.w;
  const int ox = (int)floor(e.x), oy = (int)floor(e.y);
  const double atten = S.fc[FC_ATTEN];
  int bad_col = 0x7fffffff, bad_status = TC_ST_OK;
  // the shaded wall slice of column c from its perpendicular distance and
  // hit cell (the ray state itself is dead by now)
  // the hit cell's base colour (door colour or wall palette entry)
  auto col_base = [&](int hit) -> uint32_t {
    const uint32_t cw = cell[hit];
    return (((cw >> CELL_TAG_SHIFT) & 3u) == C_DOOR) ? T_DOOR(S)[cw & 31u] : T_PAL(S)[cw & 0xffu];
  };
  // column c's outputs from its distance, base colour and half height;
  // split from the loads so a lane's rays issue their loads and arithmetic
  // back to back before any shared-memory store orders them
  auto col_store = [&](int c, double perp, uint32_t rgb, int half) {
    sm.zbuf(S)[c] = perp;
    if (zbuf_out) zbuf_out[c] = perp;
    const int top = h2 - half, bot = h2 + half;
    if (S.contig) {
      // mirrored compose reads only the (colour, top) byte streams
      uint8_t* wp = sm.wpk(S) + 3 * c;
      uint8_t* tp = sm.tpk(S) + 3 * c;
      const uint8_t t = (uint8_t)(top > 0 ? top : 0);
      wp[0] = (uint8_t)rgb; wp[1] = (uint8_t)(rgb >> 8); wp[2] = (uint8_t)(rgb >> 16);
      tp[0] = t; tp[1] = t; tp[2] = t;
    } else {
      sm.wrgb(S)[wslot(c)] = rgb;
      sm.t0(S)[c] = (uint16_t)(top > 0 ? top : 0);
      sm.t8(S)[c] = (uint8_t)(top > 0 ? top : 0);
      sm.b0(S)[c] = (uint16_t)(bot < H ? bot : H);
    }
  };
  auto col_write = [&](int c, double perp, int hit) {
    const uint32_t base = col_base(hit);
    col_store(c, perp, rgb_scale(base, __drcp_rn(1.0 + atten * perp)), line_half(H, perp));
  };
  // per-column result -> zbuf / spans / shaded colour, _pycore.py:159-178
  auto column_out = [&](int c, const March& r) {
    if (rayinfo) {
      int mx, my;
      if (CHECKED && r.status != TC_ST_OK) { mx = (int)r.sdx; my = (int)r.sdy; }
      else { my = r.idx / mw; mx = r.idx - my * mw; }
      rayinfo[c * 4 + 0] = mx; rayinfo[c * 4 + 1] = my;
      rayinfo[c * 4 + 2] = r.xs ? 0 : 1; rayinfo[c * 4 + 3] = r.steps;
    }
    if (CHECKED && r.status != TC_ST_OK) {
      if (c < bad_col) { bad_col = c; bad_status = r.status; }
      return;
    }
    col_write(c, r.xs ? r.sdx - r.ddx : r.sdy - r.ddy, r.idx);
  };
  int c = lane;
  if (FAST || (!CHECKED && mw >= 2 &&
                ((S.smem_map && S.n_doors < 32) || (S.smem_u8 && S.n_doors <= 30)))) {
    // shared-memory stop codes, predicated lockstep march (march_fast):
    // rounds of TC_LOCKSTEP columns (c, c + G, ...), then pairs, then singles.
    // u32 codes (4-byte cells, stop iff code & ~dmask) or, for large maps,
    // u8 codes (1-byte cells, stop iff bit `code` of the stop mask is set)
    const bool u8 = S.smem_u8 != 0;
    const int shift = u8 ? 0 : 2;
    const uint32_t sbase = u8 ? (uint32_t)__cvta_generic_to_shared(g_smem + S.b_code8)
                              : (uint32_t)__cvta_generic_to_shared(solid);
    const uint32_t nd_mask = S.n_doors >= 32 ? ~0u : ((1u << S.n_doors) - 1u);
    const uint32_t smask = u8 ? (((~e.dmask & nd_mask) << 1) | 0x80000000u) : ~e.dmask;
    const int idx0 = oy * mw + ox;
    auto fast_round = [&](auto rtag) {
      constexpr int LR = decltype(rtag)::value;
      FastRay fr[LR];
#pragma unroll
      for (int q = 0; q < LR; q++) {
        const double k = T_COEF(S)[c + q * G];
        const RaySetup rs = ray_setup(mw, e.x, e.y, ox, oy, e.dx + planex * k, e.dy + planey * k);
        fr[q].sdx = rs.sdx; fr[q].sdy = rs.sdy; fr[q].ddx = rs.ddx; fr[q].ddy = rs.ddy;
        fr[q].addr = sbase + ((uint32_t)idx0 << shift);
        fr[q].incx = rs.stepx * (1 << shift); fr[q].incy = rs.dyi * (1 << shift);
        fr[q].last = fr[q].incx;
      }
#if TC_TRACE
      if (ti >= 0) TRACE(ti, 8);
#endif
      if constexpr (LR == 2) {
        if (u8) march_fast2_u8(smask, fr[0], fr[1]);
        else march_fast<LR>(smask, fr);
      } else {
        march_fast<LR>(smask, fr);
      }
#if TC_TRACE
      if (ti >= 0) TRACE(ti, 9);
#endif
      if (rayinfo) {
#pragma unroll
        for (int q = 0; q < LR; q++) {
          March r;
          r.sdx = fr[q].sdx; r.sdy = fr[q].sdy; r.ddx = fr[q].ddx; r.ddy = fr[q].ddy;
          r.idx = (int)(fr[q].addr - sbase) >> shift;
          r.xs = fr[q].last == fr[q].incx;
          r.status = TC_ST_OK;
          const int my = r.idx / mw, mx = r.idx - my * mw;
          r.steps = abs(mx - ox) + abs(my - oy);
          column_out(c + q * G, r);
        }
      } else {
        // reduce every ray to (perp, hit cell) first: the sdx/sdy/ddx/ddy
        // of the later rays are not kept live across the earlier ones' writes
        double perp[LR];
        int hit[LR];
#pragma unroll
        for (int q = 0; q < LR; q++) {
          const bool xs = fr[q].last == fr[q].incx;
          perp[q] = xs ? fr[q].sdx - fr[q].ddx : fr[q].sdy - fr[q].ddy;
          hit[q] = (int)(fr[q].addr - sbase) >> shift;
        }
        uint32_t base[LR], rgb[LR];
        int half[LR];
#pragma unroll
        for (int q = 0; q < LR; q++) base[q] = col_base(hit[q]);
#pragma unroll
        for (int q = 0; q < LR; q++) {
          // shade = 1.0 / (1.0 + atten * perp) (IEEE reciprocal), _pycore.py:161-170
          rgb[q] = rgb_scale_unit(base[q], __drcp_rn(1.0 + atten * perp[q]));
          half[q] = line_half(H, perp[q]);
        }
#pragma unroll
        for (int q = 0; q < LR; q++) col_store(c + q * G, perp[q], rgb[q], half[q]);
      }
    };
    constexpr int LR = TC_LOCKSTEP;
#pragma unroll 1
    for (; c + (LR - 1) * G < W; c += LR * G) fast_round(std::integral_constant<int, LR>());
    if (LR > 2) {
#pragma unroll 1
      for (; c + G < W; c += 2 * G) fast_round(std::integral_constant<int, 2>());
    }
  } else if (!CHECKED && !FAST) {
    // groups of TC_LOCKSTEP columns (c, c + G, ...) marched in lockstep
    constexpr int LR = TC_LOCKSTEP;
#pragma unroll 1
    for (; c + (LR - 1) * G < W; c += LR * G) {
      RaySetup rs[LR];
      March rr[LR];
#pragma unroll
      for (int q = 0; q < LR; q++) {
        const double k = T_COEF(S)[c + q * G];
        rs[q] = ray_setup(mw, e.x, e.y, ox, oy, e.dx + planex * k, e.dy + planey * k);
      }
      march_n<LR>(solid, e.dmask, rs, rr);
#pragma unroll
      for (int q = 0; q < LR; q++) column_out(c + q * G, rr[q]);
    }
#pragma unroll 1
    for (; c + G < W; c += 2 * G) {
      const double k0 = T_COEF(S)[c], k1 = T_COEF(S)[c + G];
      RaySetup a = ray_setup(mw, e.x, e.y, ox, oy, e.dx + planex * k0, e.dy + planey * k0);
      RaySetup b = ray_setup(mw, e.x, e.y, ox, oy, e.dx + planex * k1, e.dy + planey * k1);
      March ra, rb;
      march2(solid, e.dmask, a, b, ra, rb);
      column_out(c, ra);
      column_out(c + G, rb);
    }
  }
#pragma unroll 1
  for (; c < W; c += G) {
    const double k = T_COEF(S)[c];
    const double rx = e.dx + planex * k;
    const double ry = e.dy + planey * k;
    const March r = march<CHECKED>(solid, mw, S.h, e.dmask, e.x, e.y, ox, oy, rx, ry);
    column_out(c, r);
  }
  // pad columns so 4-wide loads past W read harmless data
  if (lane < ((W + 3) & ~3) - W) {
    sm.t0(S)[W + lane] = (uint16_t)h2; sm.b0(S)[W + lane] = (uint16_t)h2; sm.wrgb(S)[wslot(W + lane)] = 0;
  }
  if (!CHECKED) return TC_ST_OK;
  const int first_bad = g.min(bad_col);
  if (first_bad == 0x7fffffff) return TC_ST_OK;
  return g.shfl(bad_status, first_bad % G);
}

// Sprite gather (entity order, _pycore.py:192-209) and per-sprite
// parameters (:219-252). Sprites that provably draw nothing -- denom <= 0,
// an empty row span, or (debug-tap builds only; the draw repeats the test)
// no column with zbuf[c] > dep and |a| < 1 (the reference's own per-column
// tests, evaluated exactly) -- are dropped
// here; the survivors keep their relative order, so the stable far->near
// sort (= the reference's insertion sort, :210-217) of the survivors is the
// reference's order restricted to sprites that draw. Returns the survivor
// count m; records land in sm.recs(S)[0..m) in draw order.
template <int G>
__device__ __forceinline__ int sprite_setup(const SpecDev& S, const WarpSmem& sm, const Env& e,
                                            double planex, double planey,
                                            unsigned long long* __restrict__ spritevis_out) {
  const Grp<G> g;
  const int lane = g.lane;
  const int W = S.obs_w, H = S.obs_h, h2 = H / 2;
  int m = 0;
  unsigned long long vis = 0;
  const double det = planex * e.dy - e.dx * planey;
  if (det != 0.0) {
    const double invdet = 1.0 / det;
    const double atten = S.fc[FC_ATTEN], spk = S.fc[FC_SPRITE_K];
    for (int base = 0; base < S.n_ent; base += G) {
      const int ent = base + lane;
      bool keep = false;
      double lat = 0.0, dep = 0.0;
      if (ent < S.n_ent && ((e.emask >> ent) & 1ULL) &&
          !(T_EKIND(S)[ent] == K_GOAL && ent != e.agoal)) {
        const double relx = T_EPX(S)[ent] - e.x;
        const double rely = T_EPY(S)[ent] - e.y;
        lat = invdet * (e.dy * relx - e.dx * rely);
        dep = invdet * (-planey * relx + planex * rely);
        keep = !(dep < S.fc[FC_MIN_SPRITE_DEPTH]);
        // conservative horizontal-FOV cull (no division): if |lat| exceeds
        // (dep + K)(1 + 1e-6) then |ks| > 1 + halfk by a margin far above
        // rounding, so every column's |a| >= 1 and the sprite draws nothing
        if (keep && fabs(lat) > (dep + S.fc[FC_SPRITE_K]) * (1.0 + 1e-6)) keep = false;
      }
      uint32_t bal = g.ballot(keep);
      while (bal) {  // warp-uniform walk over the gathered sprites
        const int src = __ffs(bal) - 1;
        bal &= bal - 1u;
        const double d = g.shfl(dep, src);
        const double l = g.shfl(lat, src);
        // the four per-sprite quotients, one per lane (same operands and
        // order as _pycore.py:220-223), then broadcast
        const double qn = lane == 0 ? (double)H : lane == 1 ? l : lane == 2 ? spk : 1.0;
        const double qd = lane == 3 ? 1.0 + atten * d : d;
        const double q = qn / qd;
        double sh_f = g.shfl(q, 0);
        const double ks = g.shfl(q, 1);
        const double halfk = g.shfl(q, 2);
        const double shade = g.shfl(q, 3);
        if (sh_f > 1e9) sh_f = 1e9;
        const int vhalf = (int)sh_f / 2;
        const int vtop = h2 - vhalf, vbot = h2 + vhalf;
        const int r0 = vtop > 0 ? vtop : 0, r1 = vbot < H ? vbot : H;
        if (vbot - vtop <= 0 || r0 >= r1) continue;
        if (spritevis_out) {
          // debug tap: keep exactly the sprites with a visible column (the
          // draw evaluates the same per-column test; a sprite with none
          // draws nothing, so the frames do not depend on this filter)
          bool any = false;
#pragma unroll 1
          for (int c = lane; c < W; c += G) {
            if (!(sm.zbuf(S)[c] <= d)) {
              const double a = (T_COEF(S)[c] - ks) / halfk;
              any |= !(a <= -1.0 || a >= 1.0);
            }
          }
          if (!g.any(any)) continue;
        }
        const int en = base + src;
        if (lane == 0) {
          SpriteRec r;
          r.dep = d;
          r.ks = ks;
          r.halfk = halfk;
          r.vtop = vtop;
          r.denom = vbot - vtop;
          r.r0 = r0;
          r.r1 = r1;
          r.kd = T_EKIND(S)[en];
          r.ent = en;
          const uint32_t m1 = r.kd == K_KEY ? S.key_rgb[T_ECOL(S)[en]]
                              : r.kd == K_GOAL ? S.goal_rgb : S.med_cross;
          r.s1 = rgb_scale(m1, shade);
          r.s2 = rgb_scale(S.med_box, shade);
          sm.gdep(S)[m] = d;
          sm.recs(S)[m] = r;  // gathered (entity) order
        }
        vis |= 1ULL << en;
        m++;
      }
    }
  }
  if (spritevis_out && lane == 0) *spritevis_out = vis;
  if (m > 1) {
    // stable far -> near: rank = #deeper + #equal-and-earlier; permute via
    // registers (all lanes read before any lane writes)
    g.sync();
    SpriteRec mine;
    int rank = 0;
    if (lane < m) {
      mine = sm.recs(S)[lane];
      const double d = sm.gdep(S)[lane];
      for (int j = 0; j < m; j++) {
        const double dj = sm.gdep(S)[j];
        rank += (dj > d) || (dj == d && j < lane);
      }
    }
    g.sync();
    if (lane < m) sm.recs(S)[rank] = mine;
    // m > G survivors: rare (capacity 64); sort the tail serially
    if (m > G) {
      g.sync();
      if (lane == 0) {
        for (int i = 1; i < m; i++) {
          const SpriteRec it = sm.recs(S)[i];
          int j = i;
          while (j > 0 && sm.recs(S)[j - 1].dep < it.dep) { sm.recs(S)[j] = sm.recs(S)[j - 1]; j--; }
          sm.recs(S)[j] = it;
        }
      }
    }
  }
  g.sync();
  return m;
}

// Sprites in draw order overwrite their pixels of the staged band(s); lane
// L owns columns L + 32j (_pycore.py:253-270). bandB (may be NULL) is a
// second band of the same height (the mirrored bottom band). Per column the
// lane computes a = (coef - ks) / halfk (and the key's aa / 0.30) once per
// band; per row, v = ((row - vtop) + 0.5) / denom (and the key's
// (v - 0.30) / 0.18) is computed lane-parallel -- lane k divides for row
// ra + k -- and broadcast with shuffles. Same doubles, same comparisons as
// the reference, ~1 division per 32 rows instead of 1 per row.
template <int NC, int G>
__device__ __forceinline__ void draw_sprites(const SpecDev& S, const WarpSmem& sm, int m,
                                             uint8_t* bandA, int rA, uint8_t* bandB, int rB,
                                             int rows) {
  const Grp<G> g;
  const int lane = g.lane;
  const int W = S.obs_w, row_bytes = W * 3;
  for (int s = 0; s < m; s++) {
    const SpriteRec r = sm.recs(S)[s];
    const double denom = (double)r.denom;
    const bool key = r.kd == K_KEY;
    for (int half = 0; half < 2; half++) {
      uint8_t* band = half ? bandB : bandA;
      const int r_lo = half ? rB : rA;
      if (band == nullptr) continue;
      const int ra = max(r.r0, r_lo), rb = min(r.r1, r_lo + rows);
      if (ra >= rb) continue;
      // per-column terms: goal -> aa; key -> (aa/0.30)^2 and rectangle
      // flags aa<=0.07 | aa<=0.24 | aa<=0.24; medkit -> aa<=0.10 | aa<=0.38 |
      // aa<=0.60 (_pycore.py:99-129 split into column and row factors)
      double ct[NC];
      int cf[NC];
      bool vis[NC];
      bool anyv = false;
#pragma unroll
      for (int j = 0; j < NC; j++) {
        const int c = lane + G * j;
        vis[j] = false;
        ct[j] = 0.0;
        cf[j] = 0;
        if (c < W && !(sm.zbuf(S)[c] <= r.dep)) {
          const double a = (T_COEF(S)[c] - r.ks) / r.halfk;
          if (!(a <= -1.0 || a >= 1.0)) {
            vis[j] = true;
            const double aa = a >= 0.0 ? a : -a;
            if (r.kd == K_GOAL) {
              ct[j] = aa;
            } else if (key) {
              const double ea = aa / 0.30;
              ct[j] = ea * ea;
              cf[j] = (aa <= 0.07 ? 1 : 0) | (aa <= 0.24 ? 6 : 0);
            } else {
              cf[j] = (aa <= 0.10 ? 1 : 0) | (aa <= 0.38 ? 2 : 0) | (aa <= 0.60 ? 4 : 0);
            }
          }
        }
        anyv |= vis[j];
      }
      if (!g.any(anyv)) continue;
      for (int r32 = ra; r32 < rb; r32 += G) {
        // lane-parallel row terms for rows r32 .. r32+G-1: goal -> |v-0.5|*2;
        // key -> ((v-0.30)/0.18)^2 and v-range flags; medkit -> v-range flags
        double rt_l = 0.0;
        int rf_l = 0;
        if (r32 + lane < rb) {
          const double v = ((double)(r32 + lane - r.vtop) + 0.5) / denom;
          if (r.kd == K_GOAL) {
            double dv = v - 0.5;
            if (dv < 0.0) dv = -dv;
            rt_l = dv * 2.0;
          } else if (key) {
            const double ev = (v - 0.30) / 0.18;
            rt_l = ev * ev;
            rf_l = (0.30 <= v && v <= 0.85 ? 1 : 0) | (0.62 <= v && v <= 0.70 ? 2 : 0) |
                   (0.76 <= v && v <= 0.84 ? 4 : 0);
          } else {
            rf_l = (0.32 <= v && v <= 0.73 ? 1 : 0) | (0.47 <= v && v <= 0.60 ? 2 : 0) |
                   (0.25 <= v && v <= 0.80 ? 4 : 0);
          }
        }
        const int nr = min(G, rb - r32);
        for (int k = 0; k < nr; k++) {
          const double rt = g.shfl(rt_l, k);
          const int rf = g.shfl(rf_l, k);
          uint8_t* drow = band + (r32 + k - r_lo) * row_bytes;
#pragma unroll
          for (int j = 0; j < NC; j++) {
            if (!vis[j]) continue;
            int mk;
            if (r.kd == K_GOAL) {
              mk = (ct[j] + rt <= 0.8) ? 1 : 0;  // aa + |v-0.5|*2.0 <= 0.8
            } else if (key) {
              const double e = ct[j] + rt;        // ea*ea + ev*ev
              mk = ((0.30 <= e && e <= 1.0) || (cf[j] & rf) != 0) ? 1 : 0;
            } else {
              const int x = cf[j] & rf;
              mk = (x & 3) ? 1 : ((x & 4) ? 2 : 0);
            }
            if (mk) {
              // a pixel is 3 bytes: one aligned 16-bit store + one byte store
              // (bytes 0-1 + 2 at an even address, byte 0 + bytes 1-2 at an
              // odd one; every lane runs the same two stores)
              const uint32_t col = mk == 1 ? r.s1 : r.s2;
              uint8_t* d = drow + (lane + G * j) * 3;
              const int odd = (int)(reinterpret_cast<uintptr_t>(d) & 1u);
              *reinterpret_cast<uint16_t*>(d + odd) = (uint16_t)(col >> (8 * odd));
              d[odd ? 0 : 2] = (uint8_t)(odd ? col : col >> 16);
            }
          }
        }
      }
    }
  }
}

// per-lane compose geometry, computed once per kernel (no divisions per env)
struct LaneGeo {
  int rowoff, cg0;
};
template <int G>
__device__ __forceinline__ LaneGeo lane_geo(const SpecDev& S) {
  const int lane = Grp<G>().lane;
  const int CG = S.obs_w >> 4;
  LaneGeo lg;
  lg.rowoff = (S.mirror && CG < G) ? lane / CG : 0;
  lg.cg0 = (S.mirror && CG < G) ? lane - lg.rowoff * CG : lane;
  return lg;
}

// 4-pixel group (12 bytes) from 4 packed rgb words
__device__ __forceinline__ void put_quad(uint32_t* dst, uint32_t p0, uint32_t p1, uint32_t p2,
                                         uint32_t p3) {
  dst[0] = __byte_perm(p0, p1, 0x4210);
  dst[1] = __byte_perm(p1, p2, 0x5421);
  dst[2] = __byte_perm(p2, p3, 0x6542);
}

// Render one environment's frame (all 32 lanes of the warp participate).
// the wall pass for maps / poses off the fast path (unsealed rim, origin
// off the grid, global-memory stop codes, 32 doors)
template <int NC, int G>
__device__ __noinline__ int wall_pass_cold(const SpecDev& S, const uint32_t* __restrict__ cell,
                                           const uint32_t* __restrict__ solid, WarpSmem sm,
                                           Env e, double planex, double planey,
                                           double* __restrict__ zbuf_out,
                                           int32_t* __restrict__ rayinfo, bool sealed_inside) {
  return sealed_inside
      ? wall_pass<NC, false, G>(S, cell, solid, sm, e, planex, planey, zbuf_out, rayinfo)
      : wall_pass<NC, true, G>(S, cell, solid, sm, e, planex, planey, zbuf_out, rayinfo);
}

// Returns the status of the first failing column (or OK), warp-uniform.
// _pycore.py:132-271.
// Phase 1 of rendering: wall pass (spans / zbuf into shared memory).
template <int NC, int G>
__device__ __forceinline__ int render_walls(const SpecDev& S, const uint32_t* __restrict__ cell,
                                            const uint32_t* __restrict__ solid,
                                            const WarpSmem& sm, const Env& e,
                                            double* __restrict__ zbuf_out,
                                            int32_t* __restrict__ rayinfo) {
  const double planex = -e.dy * PLANE_HALF_WIDTH;
  const double planey = e.dx * PLANE_HALF_WIDTH;
  // fast march when the rim is sealed, the origin is on the grid and the
  // stop codes sit in shared memory; every other case runs out of line so
  // the hot kernel body stays compact (instruction-cache footprint)
  // (a zero view direction -- only reachable through a restored state or
  // tc_host_render_into -- makes every ray (0, 0): the checked march then
  // reports the step budget like the reference instead of spinning)
  const bool inside = e.x >= 0.0 && e.y >= 0.0 && e.x < (double)S.w && e.y < (double)S.h &&
                      (e.dx != 0.0 || e.dy != 0.0);
  const int st = (S.sealed && inside && S.w >= 2 &&
                  ((S.smem_map && S.n_doors < 32) || (S.smem_u8 && S.n_doors <= 30)))
      ? wall_pass<NC, false, G, true>(S, cell, solid, sm, e, planex, planey, zbuf_out, rayinfo)
      : wall_pass_cold<NC, G>(S, cell, solid, sm, e, planex, planey, zbuf_out, rayinfo,
                              S.sealed && inside);
  Grp<G>().sync();
  return st;
}

// Phase 2: sprite setup; returns the number of sprites that draw.
template <int G>
__device__ __forceinline__ int render_sprites(const SpecDev& S, const WarpSmem& sm, const Env& e,
                                              unsigned long long* __restrict__ spritevis_out) {
  if (S.n_ent == 0) {
    if (spritevis_out && (threadIdx.x & 31) == 0) *spritevis_out = 0;
    return 0;
  }
  const double planex = -e.dy * PLANE_HALF_WIDTH;
  const double planey = e.dx * PLANE_HALF_WIDTH;
  return sprite_setup<G>(S, sm, e, planex, planey, spritevis_out);
}

// Mirrored-band compose + sprites + TMA store (see render_frame_out).
template <int NC, bool SPR, int G>
__device__ __forceinline__ void mirror_bands(const SpecDev& S, const WarpSmem& sm, int m,
                                             uint8_t* __restrict__ frame, int& bulk_pending,
                                             int& buf, const LaneGeo& lg) {
  const Grp<G> g;
  const int lane = g.lane;
  const int W = S.obs_w, H = S.obs_h, h2 = H / 2;
    // Mirrored bands (even H <= 254, W % 16 == 0). Row r and row H-1-r have
    // the same wall / non-wall pattern (t0 = h2-half, b0 = h2+half), so one
    // SWAR compare serves both: per byte, (0x80|r) - t0 has its MSB set iff
    // r >= t0 (r, t0 <= 127, no inter-byte borrow). PRMT sign-replication
    // turns the 4 per-pixel flags of a quad into the 3 byte masks of its 12
    // bytes, and one LOP3 per word blends wall with ceiling (top row) or
    // floor (bottom row). A lane owns 16 columns (48 bytes = 3 x 16B stores).
    const int row_bytes = W * 3;
    const int B = S.band_rows;
    const int CG = W >> 4;
    const int RPI = G == 32 ? S.mir_rpi : S.mir_rpi16;
    const int rowoff = lg.rowoff;
    const int cg0 = lg.cg0;
    const uint32_t C = S.ceil_rgb, F = S.floor_rgb;
    const uint32_t cw0 = __byte_perm(C, C, 0x4210), cw1 = __byte_perm(C, C, 0x5421),
                   cw2 = __byte_perm(C, C, 0x6542);
    const uint32_t fw0 = __byte_perm(F, F, 0x4210), fw1 = __byte_perm(F, F, 0x5421),
                   fw2 = __byte_perm(F, F, 0x6542);
    const int NP = S.npairs;  // band-pair buffers in flight
    for (int r_lo = 0; r_lo < h2; r_lo += B, buf = (buf + 1 == NP ? 0 : buf + 1)) {
      const int rows = min(B, h2 - r_lo);
      uint8_t* top = sm.band(S, 2 * buf);
      uint8_t* bot = sm.band(S, 2 * buf + 1);
      const int r_bot = H - r_lo - rows;  // first frame row of the bottom band
      // the pair we overwrite was shipped NP pairs ago
      if (lane == 0 && bulk_pending >= NP) bulk_wait_read_le(NP - 1);
      g.sync();
      if (rowoff < RPI) {
        for (int cg = cg0; cg < CG; cg += G) {
          const uint4 T = *reinterpret_cast<const uint4*>(sm.t8(S) + 16 * cg);
          const uint4* wp = reinterpret_cast<const uint4*>(sm.wrgb(S) + 20 * cg);
          uint32_t Wd[12];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint4 w = wp[j];
            Wd[3 * j + 0] = __byte_perm(w.x, w.y, 0x4210);
            Wd[3 * j + 1] = __byte_perm(w.y, w.z, 0x5421);
            Wd[3 * j + 2] = __byte_perm(w.z, w.w, 0x6542);
          }
          const uint32_t Tj[4] = {T.x, T.y, T.z, T.w};
          for (int rr = rowoff; rr < rows; rr += RPI) {
            const uint32_t R = 0x80808080u + (uint32_t)(r_lo + rr) * 0x01010101u;
            uint32_t tw[12], bw[12];
#pragma unroll
            for (int j = 0; j < 4; j++) {
              const uint32_t D = R - Tj[j];
              const uint32_t m0 = prmt_sx(D, 0x9888), m1 = prmt_sx(D, 0xAA99),
                             m2 = prmt_sx(D, 0xBBBA);
              tw[3 * j + 0] = (m0 & Wd[3 * j + 0]) | (~m0 & cw0);
              tw[3 * j + 1] = (m1 & Wd[3 * j + 1]) | (~m1 & cw1);
              tw[3 * j + 2] = (m2 & Wd[3 * j + 2]) | (~m2 & cw2);
              bw[3 * j + 0] = (m0 & Wd[3 * j + 0]) | (~m0 & fw0);
              bw[3 * j + 1] = (m1 & Wd[3 * j + 1]) | (~m1 & fw1);
              bw[3 * j + 2] = (m2 & Wd[3 * j + 2]) | (~m2 & fw2);
            }
            uint4* dt = reinterpret_cast<uint4*>(top + rr * row_bytes + cg * 48);
            uint4* db = reinterpret_cast<uint4*>(bot + (rows - 1 - rr) * row_bytes + cg * 48);
            dt[0] = make_uint4(tw[0], tw[1], tw[2], tw[3]);
            dt[1] = make_uint4(tw[4], tw[5], tw[6], tw[7]);
            dt[2] = make_uint4(tw[8], tw[9], tw[10], tw[11]);
            db[0] = make_uint4(bw[0], bw[1], bw[2], bw[3]);
            db[1] = make_uint4(bw[4], bw[5], bw[6], bw[7]);
            db[2] = make_uint4(bw[8], bw[9], bw[10], bw[11]);
          }
        }
      }
      if (SPR && m > 0) {
        g.sync();
        draw_sprites<NC, G>(S, sm, m, top, r_lo, bot, r_bot, rows);
      }
      if (S.direct == 2) {
        // coalesced copy-out by the warp: each 16-byte store instruction
        // covers 512 contiguous bytes (full sectors), generic proxy only
        g.sync();
        const int nchunk = rows * row_bytes / 16;
        const uint4* st4 = reinterpret_cast<const uint4*>(top);
        const uint4* sb4 = reinterpret_cast<const uint4*>(bot);
        uint4* gt = reinterpret_cast<uint4*>(frame + (size_t)r_lo * row_bytes);
        uint4* gb = reinterpret_cast<uint4*>(frame + (size_t)r_bot * row_bytes);
        for (int k = lane; k < nchunk; k += G) {
          const uint4 a = st4[k], b = sb4[k];
          __stcs(gt + k, a);
          __stcs(gb + k, b);
        }
        g.sync();
      } else {
        bulk_fence();
        g.sync();
        if (lane == 0) {
          bulk_copy(frame + (size_t)r_lo * row_bytes, top, (uint32_t)(rows * row_bytes));
          bulk_copy(frame + (size_t)r_bot * row_bytes, bot, (uint32_t)(rows * row_bytes));
          bulk_commit();
          bulk_pending++;
        }
      }
    }
  g.sync();
}

// Mirrored compose written straight to HBM from registers (no staging):
// each lane stores its 48 bytes per row as 3 streaming 16-byte stores; the
// sprite pass then overwrites its pixels with byte stores after a __syncwarp
// (which orders the warp's memory operations).
template <int NC, int G>
__device__ __forceinline__ void mirror_direct(const SpecDev& S, const WarpSmem& sm, int m,
                                              uint8_t* __restrict__ frame, const LaneGeo& lg) {
  const Grp<G> g;
  const int W = S.obs_w, H = S.obs_h, h2 = H / 2;
  const int row_bytes = W * 3;
  const int CG = W >> 4;
  const int RPI = G == 32 ? S.mir_rpi : S.mir_rpi16;
  const int rowoff = lg.rowoff;
  const uint32_t C = S.ceil_rgb, F = S.floor_rgb;
  const uint32_t cw0 = __byte_perm(C, C, 0x4210), cw1 = __byte_perm(C, C, 0x5421),
                 cw2 = __byte_perm(C, C, 0x6542);
  const uint32_t fw0 = __byte_perm(F, F, 0x4210), fw1 = __byte_perm(F, F, 0x5421),
                 fw2 = __byte_perm(F, F, 0x6542);
  if (rowoff < RPI) {
    for (int cg = lg.cg0; cg < CG; cg += G) {
      const uint4 T = *reinterpret_cast<const uint4*>(sm.t8(S) + 16 * cg);
      const uint4* wp = reinterpret_cast<const uint4*>(sm.wrgb(S) + 20 * cg);
      uint32_t Wd[12];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint4 w = wp[j];
        Wd[3 * j + 0] = __byte_perm(w.x, w.y, 0x4210);
        Wd[3 * j + 1] = __byte_perm(w.y, w.z, 0x5421);
        Wd[3 * j + 2] = __byte_perm(w.z, w.w, 0x6542);
      }
      const uint32_t Tj[4] = {T.x, T.y, T.z, T.w};
      uint8_t* top = frame + (size_t)rowoff * row_bytes + cg * 48;
      uint8_t* bot = frame + (size_t)(H - 1 - rowoff) * row_bytes + cg * 48;
      const size_t step = (size_t)RPI * row_bytes;
      // one row pair (row r and its mirror H-1-r) -> 6 x 16-byte stores
      auto row_out = [&](int r, uint8_t* top_p, uint8_t* bot_p) {
        const uint32_t R = 0x80808080u + (uint32_t)r * 0x01010101u;
        uint32_t tw[12], bw[12];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t D = R - Tj[j];
          const uint32_t m0 = prmt_sx(D, 0x9888), m1 = prmt_sx(D, 0xAA99),
                         m2 = prmt_sx(D, 0xBBBA);
          tw[3 * j + 0] = (m0 & Wd[3 * j + 0]) | (~m0 & cw0);
          tw[3 * j + 1] = (m1 & Wd[3 * j + 1]) | (~m1 & cw1);
          tw[3 * j + 2] = (m2 & Wd[3 * j + 2]) | (~m2 & cw2);
          bw[3 * j + 0] = (m0 & Wd[3 * j + 0]) | (~m0 & fw0);
          bw[3 * j + 1] = (m1 & Wd[3 * j + 1]) | (~m1 & fw1);
          bw[3 * j + 2] = (m2 & Wd[3 * j + 2]) | (~m2 & fw2);
        }
        uint4* dt = reinterpret_cast<uint4*>(top_p);
        uint4* db = reinterpret_cast<uint4*>(bot_p);
        TC_STORE(dt + 0, make_uint4(tw[0], tw[1], tw[2], tw[3]));
        TC_STORE(dt + 1, make_uint4(tw[4], tw[5], tw[6], tw[7]));
        TC_STORE(dt + 2, make_uint4(tw[8], tw[9], tw[10], tw[11]));
        TC_STORE(db + 0, make_uint4(bw[0], bw[1], bw[2], bw[3]));
        TC_STORE(db + 1, make_uint4(bw[4], bw[5], bw[6], bw[7]));
        TC_STORE(db + 2, make_uint4(bw[8], bw[9], bw[10], bw[11]));
      };
      // two row pairs per trip (independent registers) so a trip's compute
      // does not wait for the previous trip's stores to release theirs
      int r = rowoff;
      for (; r + RPI < h2; r += 2 * RPI, top += 2 * step, bot -= 2 * step) {
        row_out(r, top, bot);
        row_out(r + RPI, top + step, bot - step);
      }
      if (r < h2) row_out(r, top, bot);
    }
  }
  if (m > 0) {
    g.sync();
    draw_sprites<NC, G>(S, sm, m, frame, 0, nullptr, 0, H);
  }
  g.sync();
}

// Pixels of one sprite over its visible rectangle [lo, lo + w) x [r0, r0 + h):
// the rectangle is walked row-major with the lanes strided over it (every
// lane busy whatever the sprite's shape), each pixel's mask evaluated from
// the per-column and per-row terms in shared memory (_pycore.py:99-129
// split into exact column and row factors: the same doubles and comparisons
// as the reference), and the pixel written as one 16-bit + one 8-bit store.
// One loop for the three kinds (instruction-cache footprint): with
// e = ct + rt and x = cf & rf & 7 the reference's masks are
//   goal   (e <= 0.8)                       -> colour 1
//   key    (0.30 <= e <= 1.0) || x != 0     -> colour 1
//   medkit (x & 3) -> colour 1, else (x & 4) -> colour 2
// i.e. mk = (elo <= e <= ehi || (x & m1)) ? 1 : ((x & m2) ? 2 : 0) with
// per-kind (elo, ehi, m1, m2); a medkit's terms are 0 and its e-range empty,
// a goal's flags are 0.
template <int G>
__device__ __forceinline__ void sprite_pixels(uint8_t* __restrict__ frame, int row_bytes, int lo,
                                              int w, int r0, int h, const double* sct,
                                              const uint8_t* scf, const double* srt,
                                              const uint8_t* srf, uint32_t s1, uint32_t s2,
                                              int kind, int lane) {
  const double elo = kind == K_GOAL ? -dinf() : (kind == K_KEY ? 0.30 : dinf());
  const double ehi = kind == K_GOAL ? 0.8 : 1.0;
  const int m1 = kind == K_KEY ? 7 : (kind == K_MEDKIT ? 3 : 0);
  const int m2 = kind == K_MEDKIT ? 4 : 0;
  const int npx = w * h;
  int pr = lane / w, pc = lane - (lane / w) * w;
  const int dr = G / w, dc = G - (G / w) * w;
#pragma unroll 1
  for (int p = lane; p < npx; p += G) {
    const int c = lo + pc, r = r0 + pr;
    const int cf = scf[c];
    if (cf & 0x80) {
      const double e = sct[c] + srt[r];
      const int x = cf & srf[r] & 7;
      const int mk = ((elo <= e && e <= ehi) || (x & m1)) ? 1 : ((x & m2) ? 2 : 0);
      if (mk) {
        // three byte stores at immediate offsets from one global address
        const uint32_t col = mk == 1 ? s1 : s2;
        uint8_t* d = frame + (uint32_t)(r * row_bytes + c * 3);  // < 2^31 per frame
        asm volatile(
            "st.global.u8 [%0], %1;\n\t"
            "st.global.u8 [%0+1], %2;\n\t"
            "st.global.u8 [%0+2], %3;"
            ::"l"(d), "r"(col), "r"(col >> 8), "r"(col >> 16) : "memory");
      }
    }
    pc += dc;
    pr += dr;
    if (pc >= w) { pc -= w; pr++; }
  }
}

// Sprites over a directly stored frame (contig compose), in draw order:
// per sprite, the lanes compute the column terms of their own columns
// (shared memory; visible span [lo, hi] by group min / max) and the row
// terms of rows [r0, r1) (shared memory, one division per row), then
// sprite_pixels walks the visible rectangle.
template <int NC, int G>
__device__ __noinline__ void draw_sprites_direct(const SpecDev& S, WarpSmem sm, int m,
                                                 uint8_t* __restrict__ frame) {
  const Grp<G> g;
  const int lane = g.lane;
  const int W = S.obs_w, row_bytes = W * 3;
  double* sct = sm.sct(S);
  uint8_t* scf = sm.scf(S);
  double* srt = sm.srt(S);
  uint8_t* srf = sm.srf(S);
#pragma unroll 1
  for (int s = 0; s < m; s++) {
    const SpriteRec r = sm.recs(S)[s];
    const bool key = r.kd == K_KEY;
    int lo = 0x7fffffff, hi = -1;
#pragma unroll 1
    for (int c = lane; c < W; c += G) {
      double ct = 0.0;
      int cf = 0;
      bool vis = false;
      if (!(sm.zbuf(S)[c] <= r.dep)) {
        const double a = (T_COEF(S)[c] - r.ks) / r.halfk;
        if (!(a <= -1.0 || a >= 1.0)) {
          vis = true;
          const double aa = a >= 0.0 ? a : -a;
          if (r.kd == K_GOAL) {
            ct = aa;
          } else if (key) {
            const double ea = aa / 0.30;
            ct = ea * ea;
            cf = (aa <= 0.07 ? 1 : 0) | (aa <= 0.24 ? 6 : 0);
          } else {
            cf = (aa <= 0.10 ? 1 : 0) | (aa <= 0.38 ? 2 : 0) | (aa <= 0.60 ? 4 : 0);
          }
        }
      }
      sct[c] = ct;
      scf[c] = (uint8_t)(vis ? (cf | 0x80) : 0);
      if (vis) { lo = min(lo, c); hi = max(hi, c); }
    }
    lo = g.min(lo);
    hi = g.max(hi);
    if (hi < 0) continue;
    const double denom = (double)r.denom;
#pragma unroll 1
    for (int row = r.r0 + lane; row < r.r1; row += G) {
      const double v = ((double)(row - r.vtop) + 0.5) / denom;
      double rt = 0.0;
      int rf = 0;
      if (r.kd == K_GOAL) {
        double dv = v - 0.5;
        if (dv < 0.0) dv = -dv;
        rt = dv * 2.0;
      } else if (key) {
        const double ev = (v - 0.30) / 0.18;
        rt = ev * ev;
        rf = (0.30 <= v && v <= 0.85 ? 1 : 0) | (0.62 <= v && v <= 0.70 ? 2 : 0) |
             (0.76 <= v && v <= 0.84 ? 4 : 0);
      } else {
        rf = (0.32 <= v && v <= 0.73 ? 1 : 0) | (0.47 <= v && v <= 0.60 ? 2 : 0) |
             (0.25 <= v && v <= 0.80 ? 4 : 0);
      }
      srt[row] = rt;
      srf[row] = (uint8_t)rf;
    }
    g.sync();
    const int w = hi - lo + 1, h = r.r1 - r.r0;
#if TC_SPRITE_UNIFIED
    sprite_pixels<G>(frame, row_bytes, lo, w, r.r0, h, sct, scf, srt, srf, r.s1, r.s2, r.kd,
                     lane);
#else
    // one call site per kind: the kind is a constant inside each, so the
    // unified loop's per-kind selects fold away
    if (r.kd == K_GOAL)
      sprite_pixels<G>(frame, row_bytes, lo, w, r.r0, h, sct, scf, srt, srf, r.s1, r.s2, K_GOAL,
                       lane);
    else if (key)
      sprite_pixels<G>(frame, row_bytes, lo, w, r.r0, h, sct, scf, srt, srf, r.s1, r.s2, K_KEY,
                       lane);
    else
      sprite_pixels<G>(frame, row_bytes, lo, w, r.r0, h, sct, scf, srt, srf, r.s1, r.s2,
                       K_MEDKIT, lane);
#endif
    g.sync();  // the next sprite reuses the term scratch; pixel order = draw order
  }
}

// Direct mirrored compose with lane-contiguous stores: the top half of the
// frame (h2 rows, contiguous in HBM) is cut into 16-byte chunks and lane l
// of the group writes chunks l, l+G, l+2G, ... so every store instruction
// covers G x 16 contiguous bytes (2 cache lines for 16 lanes instead of ~8
// with a per-column layout), plus the mirror row's chunk at the same row
// offset. Needs CPR = 3W/16 chunks per row to divide 3G: then a lane's chunk
// column k repeats with period 3 (phases p) and its rows step by RB = 3G/CPR.
// The wall pass left the wall colours and tops as byte streams laid out like
// a frame row (wpk / tpk), so chunk k's wall words and per-byte tops are one
// 16-byte load each; per row and word: one SWAR subtract, one PRMT
// sign-fill, one LOP3 each for the ceiling (top) and floor (bottom) blend.
template <int NC, int G>
__device__ __forceinline__ void mirror_contig(const SpecDev& S, const WarpSmem& sm, int m,
                                              uint8_t* __restrict__ frame) {
  const Grp<G> g;
  const int lane = g.lane;
  const int W = S.obs_w, H = S.obs_h, h2 = H / 2;
  const int row_bytes = W * 3;
  const int CPR = row_bytes >> 4;
  const int RB = 3 * G / CPR;
  const uint4* __restrict__ wpk = reinterpret_cast<const uint4*>(sm.wpk(S));
  const uint4* __restrict__ tpk = reinterpret_cast<const uint4*>(sm.tpk(S));
  // ceiling / floor words by position of the word's first byte in its pixel
  // (a chunk starting at byte 16k begins at component k mod 3)
  const uint32_t C = S.ceil_rgb, F = S.floor_rgb;
  const uint32_t c0 = __byte_perm(C, 0, 0x0210), c1 = __byte_perm(C, 0, 0x1021),
                 c2 = __byte_perm(C, 0, 0x2102);
  const uint32_t f0 = __byte_perm(F, 0, 0x0210), f1 = __byte_perm(F, 0, 0x1021),
                 f2 = __byte_perm(F, 0, 0x2102);
#pragma unroll 1
  for (int p = 0; p < 3; p++) {
    const int c = lane + G * p;
    const int rp = c / CPR, k = c - rp * CPR;
    const int s0 = k % 3;
    const uint4 Wd = wpk[k], T = tpk[k];
    const uint32_t ca = s0 == 0 ? c0 : (s0 == 1 ? c1 : c2);
    const uint32_t cb = s0 == 0 ? c1 : (s0 == 1 ? c2 : c0);
    const uint32_t cc = s0 == 0 ? c2 : (s0 == 1 ? c0 : c1);
    const uint32_t fa = s0 == 0 ? f0 : (s0 == 1 ? f1 : f2);
    const uint32_t fb = s0 == 0 ? f1 : (s0 == 1 ? f2 : f0);
    const uint32_t fc = s0 == 0 ? f2 : (s0 == 1 ? f0 : f1);
    uint4* top = reinterpret_cast<uint4*>(frame + (size_t)rp * row_bytes) + k;
    uint4* bot = reinterpret_cast<uint4*>(frame + (size_t)(H - 1 - rp) * row_bytes) + k;
    const int step = RB * CPR;  // in uint4
    const int nt = (h2 - rp + RB - 1) / RB;
#pragma unroll 2
    for (int t = 0; t < nt; t++, top += step, bot -= step) {
      const uint32_t R = 0x80808080u + (uint32_t)(rp + t * RB) * 0x01010101u;
      // MSB of byte b set iff row >= top of its pixel; sign-fill -> mask
      const uint32_t m0 = prmt_sx(R - T.x, 0xBA98), m1 = prmt_sx(R - T.y, 0xBA98),
                     m2 = prmt_sx(R - T.z, 0xBA98), m3 = prmt_sx(R - T.w, 0xBA98);
      TC_STORE(top, make_uint4((m0 & Wd.x) | (~m0 & ca), (m1 & Wd.y) | (~m1 & cb),
                               (m2 & Wd.z) | (~m2 & cc), (m3 & Wd.w) | (~m3 & ca)));
      TC_STORE(bot, make_uint4((m0 & Wd.x) | (~m0 & fa), (m1 & Wd.y) | (~m1 & fb),
                               (m2 & Wd.z) | (~m2 & fc), (m3 & Wd.w) | (~m3 & fa)));
    }
  }
  if (m > 0) {
    g.sync();
    draw_sprites_direct<NC, G>(S, sm, m, frame);
  }
  g.sync();
}

// mirror_contig for a compile-time frame shape (W x H, G lanes): the chunk
// geometry of every lane and phase, the row steps and the store offsets
// are constants, so each row pair is 4 SWAR subtracts, 4 PRMT sign fills,
// 8 LOP3 blends and 2 streaming 16-byte stores at immediate offsets from
// one base pointer per phase (no per-trip address arithmetic).
template <int W, int H, int G>
__device__ __forceinline__ void mirror_contig_fixed(const SpecDev& S, const WarpSmem& sm, int m,
                                                    uint8_t* __restrict__ frame) {
  constexpr int ROW = W * 3, CPR = ROW / 16, RB = 3 * G / CPR, H2 = H / 2;
  constexpr int NT = (H2 + RB - 1) / RB;
  static_assert(ROW % 16 == 0 && (3 * G) % CPR == 0, "mirror_contig_fixed shape");
  const Grp<G> g;
  const int lane = g.lane;
  const uint4* __restrict__ wpk = reinterpret_cast<const uint4*>(sm.wpk(S));
  const uint4* __restrict__ tpk = reinterpret_cast<const uint4*>(sm.tpk(S));
  const uint32_t C = S.ceil_rgb, F = S.floor_rgb;
  const uint32_t c0 = __byte_perm(C, 0, 0x0210), c1 = __byte_perm(C, 0, 0x1021),
                 c2 = __byte_perm(C, 0, 0x2102);
  const uint32_t f0 = __byte_perm(F, 0, 0x0210), f1 = __byte_perm(F, 0, 0x1021),
                 f2 = __byte_perm(F, 0, 0x2102);
// (phases rolled: one copy of the row-pair code keeps the hot kernel small
  // in the instruction cache when envs are in different phases at once)
#pragma unroll 1
  for (int p = 0; p < 3; p++) {
    const int c = lane + G * p;
    const int rp = c / CPR, k = c - rp * CPR;
    const int s0 = k % 3;
    const uint4 Wd = wpk[k], T = tpk[k];
    const uint32_t ca = s0 == 0 ? c0 : (s0 == 1 ? c1 : c2);
    const uint32_t cb = s0 == 0 ? c1 : (s0 == 1 ? c2 : c0);
    const uint32_t cc = s0 == 0 ? c2 : (s0 == 1 ? c0 : c1);
    const uint32_t fa = s0 == 0 ? f0 : (s0 == 1 ? f1 : f2);
    const uint32_t fb = s0 == 0 ? f1 : (s0 == 1 ? f2 : f0);
    const uint32_t fc = s0 == 0 ? f2 : (s0 == 1 ? f0 : f1);
    uint4* top = reinterpret_cast<uint4*>(frame + rp * ROW) + k;
    uint4* bot = reinterpret_cast<uint4*>(frame + (H - 1 - rp) * ROW) + k;
    const uint32_t R0 = 0x80808080u + (uint32_t)rp * 0x01010101u;
#pragma unroll
    for (int t = 0; t < NT; t++) {
      if (H2 % RB != 0 && rp + t * RB >= H2) break;
      const uint32_t R = R0 + (uint32_t)(t * RB) * 0x01010101u;
      const uint32_t m0 = prmt_sx(R - T.x, 0xBA98), m1 = prmt_sx(R - T.y, 0xBA98),
                     m2 = prmt_sx(R - T.z, 0xBA98), m3 = prmt_sx(R - T.w, 0xBA98);
      TC_STORE(top + t * RB * CPR,
               make_uint4((m0 & Wd.x) | (~m0 & ca), (m1 & Wd.y) | (~m1 & cb),
                          (m2 & Wd.z) | (~m2 & cc), (m3 & Wd.w) | (~m3 & ca)));
      TC_STORE(bot - t * RB * CPR,
               make_uint4((m0 & Wd.x) | (~m0 & fa), (m1 & Wd.y) | (~m1 & fb),
                          (m2 & Wd.z) | (~m2 & fc), (m3 & Wd.w) | (~m3 & fa)));
    }
  }
  if (m > 0) {
    g.sync();
    draw_sprites_direct<(W + G - 1) / G, G>(S, sm, m, frame);
  }
  g.sync();
}

// Phase 3: compose the frame in staged bands, draw sprites, ship with TMA.
template <int NC, int G>
__device__ __forceinline__ void render_frame_general(const SpecDev& S, const WarpSmem& sm, int m,
                                                     uint8_t* __restrict__ frame,
                                                     int& bulk_pending, int& buf,
                                                     const LaneGeo& lg);

// bulk_pending | buf << 16 (no references across the out-of-line call)
template <int NC, int G>
__device__ __noinline__ int render_frame_cold(const SpecDev& S, WarpSmem sm, int m,
                                              uint8_t* __restrict__ frame, int bulk_pending,
                                              int buf, LaneGeo lg) {
  render_frame_general<NC, G>(S, sm, m, frame, bulk_pending, buf, lg);
  return bulk_pending | (buf << 16);
}

template <int NC, int G, bool FIX = false>
__device__ __forceinline__ void render_frame_out(const SpecDev& S, const WarpSmem& sm, int m,
                                                 uint8_t* __restrict__ frame, int& bulk_pending,
                                                 int& buf, const LaneGeo& lg) {
  // the lane-contiguous direct compose inline; every other layout out of
  // line (instruction-cache footprint of the hot kernel)
  if (S.mirror && S.direct == 1 && S.contig) {
    // the BASELINE frame shapes take the compile-time-geometry compose
    // (FIX: only where the register budget holds its unrolled row pairs --
    // the 96-register multi-wave variant spills with it, -12 % at c3)
    if constexpr (FIX && G == 16 && NC == 4) {
      if (S.obs_w == 64 && S.obs_h == 64) {
        mirror_contig_fixed<64, 64, G>(S, sm, m, frame);
        return;
      }
    }
    if constexpr (FIX && G == 32 && NC == 4) {
      if (S.obs_w == 128 && S.obs_h == 128) {
        mirror_contig_fixed<128, 128, G>(S, sm, m, frame);
        return;
      }
    }
    mirror_contig<NC, G>(S, sm, m, frame);
    return;
  }
  const int r = render_frame_cold<NC, G>(S, sm, m, frame, bulk_pending, buf, lg);
  bulk_pending = r & 0xffff;
  buf = r >> 16;
}

template <int NC, int G>
__device__ __forceinline__ void render_frame_general(const SpecDev& S, const WarpSmem& sm, int m,
                                                     uint8_t* __restrict__ frame,
                                                     int& bulk_pending, int& buf,
                                                     const LaneGeo& lg) {
  const Grp<G> g;
  const int lane = g.lane;
  const int W = S.obs_w, H = S.obs_h;
  if (S.mirror) {
    if (S.direct == 1 && S.contig) mirror_contig<NC, G>(S, sm, m, frame);
    else if (S.direct == 1) mirror_direct<NC, G>(S, sm, m, frame, lg);
    else mirror_bands<NC, true, G>(S, sm, m, frame, bulk_pending, buf, lg);
    return;
  }

  // Row classes, warp-uniform: [0,tmin) ceiling everywhere, [tmin,tmax)
  // mixed ceiling/wall, [tmax,bmin) wall everywhere, [bmin,bmax) mixed
  // wall/floor, [bmax,H) floor everywhere (t0 <= h2 <= b0 per column).
  int tlo = 0x7fffffff, thi = 0, blo = 0x7fffffff, bhi = 0;
  for (int c = lane; c < W; c += G) {
    const int t = sm.t0(S)[c], b = sm.b0(S)[c];
    tlo = min(tlo, t); thi = max(thi, t); blo = min(blo, b); bhi = max(bhi, b);
  }
  const int tmin = g.min(tlo), tmax = g.max(thi);
  const int bmin = g.min(blo), bmax = g.max(bhi);

  const int row_bytes = W * 3;
  const int B = S.band_rows;
  const uint32_t C = S.ceil_rgb, F = S.floor_rgb;
  const uint32_t c0w = __byte_perm(C, C, 0x4210), c1w = __byte_perm(C, C, 0x5421),
                 c2w = __byte_perm(C, C, 0x6542);
  const uint32_t f0w = __byte_perm(F, F, 0x4210), f1w = __byte_perm(F, F, 0x5421),
                 f2w = __byte_perm(F, F, 0x6542);
  const int Q = W >> 2;
  const int RG = Q >= G ? 1 : G / Q;  // row groups per lane group
  const int rsub = Q >= G ? 0 : lane / Q;
  const int q_first = Q >= G ? lane : lane - rsub * Q;

  for (int r_lo = 0; r_lo < H; r_lo += B, buf ^= 1) {
    const int rows = min(B, H - r_lo);
    const int r_end = r_lo + rows;
    uint8_t* band = sm.band(S, buf);
    // the buffer we are about to overwrite was shipped two bands ago
    if (S.bulk && lane == 0 && bulk_pending > 1) bulk_wait_read_le1();
    g.sync();
    if (S.quads) {
      if (rsub < RG) {
        for (int q = q_first; q < Q; q += G) {
          const uint2 t4 = *reinterpret_cast<const uint2*>(sm.t0(S) + 4 * q);
          const uint2 b4 = *reinterpret_cast<const uint2*>(sm.b0(S) + 4 * q);
          const uint4 w4 = *reinterpret_cast<const uint4*>(sm.wrgb(S) + wslot(4 * q));
          const int t0 = t4.x & 0xffff, t1 = t4.x >> 16, t2 = t4.y & 0xffff, t3 = t4.y >> 16;
          const int b0 = b4.x & 0xffff, b1 = b4.x >> 16, b2 = b4.y & 0xffff, b3 = b4.y >> 16;
          const uint32_t w0w = __byte_perm(w4.x, w4.y, 0x4210),
                         w1w = __byte_perm(w4.y, w4.z, 0x5421),
                         w2w = __byte_perm(w4.z, w4.w, 0x6542);
          uint32_t* dst = reinterpret_cast<uint32_t*>(band + rsub * row_bytes + q * 12);
          const int dstep = RG * row_bytes / 4;
          int row = r_lo + rsub;
          for (const int lim = min(r_end, tmin); row < lim; row += RG, dst += dstep) {
            dst[0] = c0w; dst[1] = c1w; dst[2] = c2w;
          }
          for (const int lim = min(r_end, tmax); row < lim; row += RG, dst += dstep)
            put_quad(dst, row < t0 ? C : w4.x, row < t1 ? C : w4.y, row < t2 ? C : w4.z,
                     row < t3 ? C : w4.w);
          for (const int lim = min(r_end, bmin); row < lim; row += RG, dst += dstep) {
            dst[0] = w0w; dst[1] = w1w; dst[2] = w2w;
          }
          for (const int lim = min(r_end, bmax); row < lim; row += RG, dst += dstep)
            put_quad(dst, row < b0 ? w4.x : F, row < b1 ? w4.y : F, row < b2 ? w4.z : F,
                     row < b3 ? w4.w : F);
          for (; row < r_end; row += RG, dst += dstep) {
            dst[0] = f0w; dst[1] = f1w; dst[2] = f2w;
          }
        }
      }
    } else {
      const int items = rows * W;
      for (int p = lane; p < items; p += G) {
        const int rr = p / W, c = p - rr * W;
        const uint32_t row = (uint32_t)(r_lo + rr);
        const uint32_t col = row < sm.t0(S)[c] ? C : (row < sm.b0(S)[c] ? sm.wrgb(S)[wslot(c)] : F);
        uint8_t* d = band + rr * row_bytes + c * 3;
        d[0] = (uint8_t)col; d[1] = (uint8_t)(col >> 8); d[2] = (uint8_t)(col >> 16);
      }
    }
    if (m > 0) {
      g.sync();
      draw_sprites<NC, G>(S, sm, m, band, r_lo, nullptr, 0, rows);
    }
    // ship the band
    const int bytes = rows * row_bytes;
    uint8_t* gdst = frame + (size_t)r_lo * row_bytes;
    if (S.bulk) {
      bulk_fence();
      g.sync();
      if (lane == 0) {
        bulk_store(gdst, band, (uint32_t)bytes);
        bulk_pending++;
      }
    } else {
      g.sync();
      for (int b = lane; b < bytes; b += G) gdst[b] = band[b];
    }
  }
  g.sync();
}

// Render one environment's frame (all 32 lanes of the warp participate).
// Returns the status of the first failing column (or OK), warp-uniform.
// _pycore.py:132-271.
template <int NC, int G, bool FIX = false>
__device__ __forceinline__ int render_env(const SpecDev& S, const uint32_t* __restrict__ cell,
                                          const uint32_t* __restrict__ solid, const WarpSmem& sm,
                                          const Env& e, uint8_t* __restrict__ frame,
                                          double* __restrict__ zbuf_out,
                                          int32_t* __restrict__ rayinfo,
                                          unsigned long long* __restrict__ spritevis_out,
                                          int& bulk_pending, int& buf, const LaneGeo& lg,
                                          long long ti = 0) {
  const int st = render_walls<NC, G>(S, cell, solid, sm, e, zbuf_out, rayinfo);
  if (st != TC_ST_OK) return st;
  TRACE(ti, 3);
  const int m = render_sprites<G>(S, sm, e, spritevis_out);
  TRACE(ti, 4);
#if TC_TRACE
  if (g_trace && Grp<G>().lane == 0) {
    // sprites drawn and their pixel footprint (rows x visible-column bound)
    unsigned long long px = 0;
    for (int k = 0; k < m; k++) {
      const SpriteRec r = sm.recs(S)[k];
      const double w = 2.0 * r.halfk * (S.obs_w - 1) / 2.0;
      px += (unsigned long long)(r.r1 - r.r0) * (unsigned long long)(w < S.obs_w ? w : S.obs_w);
    }
    g_trace[ti * 16 + 7] = (unsigned long long)m | (px << 8);
  }
#endif
  render_frame_out<NC, G, FIX>(S, sm, m, frame, bulk_pending, buf, lg);
  return TC_ST_OK;
}

// ------------------------------------------------------------- the kernels

template <int G>
__device__ __forceinline__ void load_env(const SpecDev& S, const StateDev& st, long long i,
                                         Env& e) {
  const Grp<G> g;
  const int lane = g.lane;
  e.x = st.px[i]; e.y = st.py[i]; e.dx = st.dx[i]; e.dy = st.dy[i];
  e.health = st.health[i];
  e.inv = st.inv[i];
  e.t = st.t[i];
  e.rkey = st.rkey[i];
  e.rctr = st.rctr[i];
  e.done = st.done[i];
  e.agoal = st.agoal[i];
  uint32_t dm = 0;
  for (int b = 0; b < S.n_doors; b += G) {
    const bool d = b + lane < S.n_doors && st.dopen[i * S.n_doors + b + lane] != 0;
    dm |= g.ballot(d) << b;
  }
  e.dmask = dm;
  unsigned long long em = 0;
  for (int b = 0; b < S.n_ent; b += G) {
    const bool a = b + lane < S.n_ent && st.ealive[i * S.n_ent + b + lane] != 0;
    em |= (unsigned long long)g.ballot(a) << b;
  }
  e.emask = em;
}

template <int G>
__device__ __forceinline__ void store_env(const SpecDev& S, const StateDev& st, long long i,
                                          const Env& e) {
  const Grp<G> g;
  const int lane = g.lane;
  if (lane == 0) {
    st.px[i] = e.x; st.py[i] = e.y; st.dx[i] = e.dx; st.dy[i] = e.dy;
    st.health[i] = e.health;
    st.inv[i] = (uint8_t)e.inv;
    st.t[i] = e.t;
    st.rkey[i] = e.rkey;
    st.rctr[i] = e.rctr;
    st.done[i] = (uint8_t)e.done;
    st.agoal[i] = e.agoal;
  }
  for (int d = lane; d < S.n_doors; d += G)
    st.dopen[i * S.n_doors + d] = (uint8_t)((e.dmask >> d) & 1u);
  for (int k = lane; k < S.n_ent; k += G)
    st.ealive[i * S.n_ent + k] = (uint8_t)((e.emask >> k) & 1ULL);
}

// Spec staging, once per CTA: the blob prefix (the small tables -- column
// coefficients, palette, door colours, entity / spawn / goal arrays -- and,
// when the map fits, the packed cells and guarded stop codes) is copied to
// shared memory at the same offsets, so every table read on the step's
// critical path is a shared-memory load instead of an L1/L2 round trip.
__host__ __device__ __forceinline__ int map_smem_bytes(const SpecDev& S) { return S.stage_bytes; }
// The copy itself is one TMA bulk copy (cp.async.bulk global -> shared,
// completion counted in bytes on an mbarrier) issued by thread 0: one
// instruction instead of a per-thread loop of 16-byte cp.async chunks.
__shared__ __align__(8) uint64_t g_stage_bar;

__device__ __forceinline__ void stage_map_issue(const SpecDev& S, uint32_t* smap,
                                                const uint32_t*& cell, const uint32_t*& solid) {
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&g_stage_bar);
  if (threadIdx.x == 0) {
    const uint32_t sdst = (uint32_t)__cvta_generic_to_shared(smap);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((uint32_t)S.stage_bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(sdst), "l"(S.blob), "r"((uint32_t)S.stage_bytes), "r"(bar) : "memory");
  }
  if (S.smem_map) {
    cell = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(smap) + S.b_cell);
    solid = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(smap) + S.b_solid);
  } else {
    cell = S.cell;
    solid = S.solid;
  }
}
// every thread: the barrier is initialised (CTA barrier), then its phase 0
// completes when the bulk copy's bytes have landed
__device__ __forceinline__ void stage_map_wait() {
  __syncthreads();
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&g_stage_bar);
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra WAIT%=;\n\t"
      "}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void stage_map(const SpecDev& S, uint32_t* smap, const uint32_t*& cell,
                                          const uint32_t*& solid) {
  stage_map_issue(S, smap, cell, solid);
  stage_map_wait();
}


// multi-wave mapped step, last CTA: the [rewards | dones] block to pinned host
// memory, 8 independent 16-byte loads in flight per thread (the copy is
// bound by the loads' round trip, not by the bus)
__device__ __forceinline__ void copy_results_host(const uint4* src, uint4* dst, size_t nv) {
  constexpr int U = 8;
  const size_t step = (size_t)blockDim.x * U;
  size_t k = threadIdx.x;
  for (; k + (U - 1) * blockDim.x < nv; k += step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = __ldcg(src + k + (size_t)u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; u++) dst[k + (size_t)u * blockDim.x] = v[u];
  }
  for (; k < nv; k += blockDim.x) dst[k] = __ldcg(src + k);
}

// MODE_RESET / MODE_STEP / MODE_RENDER over envs [0, n), _pycore.py:346-387.
// A group of G lanes owns one env at a time (G = 32: a warp; G = 16: each
// half of a warp runs its own env).
// The body is shared by batch_kernel (one spec, the whole grid) and
// multi_kernel (one launch over several specs: each CTA belongs to one
// group's contiguous CTA range); `cta` / `ncta` are the CTA's index within
// its group's range and the range's size.
template <int NC, int G, bool TAPS, bool FIX>
__device__ __forceinline__ void batch_body(const SpecDev& S, const StateDev& st,
                                           const StateDev& so,
                                           const long long* __restrict__ actions,
                                           const OutDev& out, long long n, int mode,
                                           int auto_reset, int validate,
                                           tc_counters* __restrict__ counters, int cta,
                                           int ncta) {
  uint8_t* const smem = g_smem;
  constexpr int NG = 32 / G;  // groups per warp
  const Grp<G> g;
  const int lane = g.lane;
  const int grp = (threadIdx.x >> 5) * NG + (threadIdx.x & 31) / G;  // group id in the CTA
  uint32_t* smap = reinterpret_cast<uint32_t*>(smem);
  const int map_bytes = map_smem_bytes(S);
  const uint32_t *cell, *solid;
  // programmatic dependent launch: let the next step's grid start its
  // prologue as our CTAs retire, and stage the (constant) map before
  // waiting for the previous step's state to be complete and visible
#if TC_TRACE
  unsigned long long tcta[4] = {0, 0, 0, 0};
  unsigned int tgen = 0;
  if (g_trace_cta && threadIdx.x == 0) {
    tcta[0] = gtime();
    tgen = atomicAdd(&g_cta_gen[blockIdx.x], 1u);
  }
#endif
  asm volatile("griddepcontrol.launch_dependents;");
  // no env for this CTA (n < grid); it still counts itself done when the
  // last CTA ships the results to the host
  // env scheduling. One wave (n <= groups in the grid): CTA c owns the
  // contiguous envs [c*epc, c*epc + epc), epc = ceil(n / grid) <= groups per
  // CTA, so every SM gets the same number of envs +-1 and a CTA's actions /
  // results are one contiguous run (one bus transaction each on the mapped
  // host path). Several waves: env grp*grid + cta first, then envs pulled
  // from a self-resetting device ticket counter (the last CTA to finish
  // zeroes it for the next launch).
  // Without counters (no ticket word) a multi-wave batch is interleaved
  // statically: env grp*grid + cta, then + stride.
  const long long stride = (long long)ncta * WARPS_PER_CTA * NG;
  const bool one_wave = n <= stride;
  const bool dyn = !one_wave && counters != nullptr;
  const int epc = one_wave ? (int)((n + ncta - 1) / ncta) : 0;
  const long long cbase = (long long)cta * epc;
  const int cta_envs = one_wave ? (int)max(0LL, min((long long)epc, n - cbase)) : 0;
  // no env for this CTA; it still counts itself done on the mapped host path
  if ((one_wave ? cta_envs == 0 : (long long)cta >= n) && !out.res_host) return;
  const long long i_first = one_wave ? (grp < cta_envs ? cbase + grp : n)
                                     : (long long)grp * ncta + cta;
  // per-CTA scratch after the group windows: actions / rewards / dones of
  // the CTA's envs (one-wave mapping)
  uint8_t* cta_s = smem + map_bytes + WARPS_PER_CTA * NG * S.warp_smem;
  long long* act_s = reinterpret_cast<long long*>(cta_s);
  double* rew_s = reinterpret_cast<double*>(cta_s + 64);
  uint8_t* done_s = cta_s + 128;
  // On the mapped host path (tc_batch_step_mapped) the host wrote the
  // actions to pinned memory before the launch, so they are fetched before
  // the map staging and the dependent-launch wait (their bus latency overlaps
  // both). Device-resident actions may come from the kernel just before this
  // one on the stream (a policy draw, a policy network): they are read only
  // after griddepcontrol.wait, which makes that kernel's writes visible.
  const bool warp0 = threadIdx.x < 32;
  const bool early = out.res_host != nullptr;
  long long a_pre = 0;
  if (mode == MODE_STEP && early) {
    if (one_wave) {
      if (warp0 && (int)threadIdx.x < cta_envs) a_pre = actions[cbase + threadIdx.x];
    } else if (i_first < n) {
      a_pre = actions[i_first];
    }
  }
  stage_map_issue(S, smap, cell, solid);
  if (one_wave && warp0 && (int)threadIdx.x < cta_envs) {
    act_s[threadIdx.x] = a_pre;
    rew_s[threadIdx.x] = 0.0;
    done_s[threadIdx.x] = 0;
  }
  stage_map_wait();
#if TC_TRACE
  if (g_trace_cta && threadIdx.x == 0) tcta[1] = gtime();
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if TC_TRACE
  if (g_trace_cta && threadIdx.x == 0) tcta[2] = gtime();
#endif
  const WarpSmem sm = carve(smem + map_bytes + grp * S.warp_smem);
  const size_t frame_bytes = (size_t)S.obs_h * S.obs_w * 3;
  const LaneGeo lg = lane_geo<G>(S);
  int bulk_pending = 0, buf = 0;
  unsigned long long viol = 0;
  uint32_t badbits = 0;
  long long i = i_first;
  while (i < n) {
    // grab the next ticket now; its latency hides behind this env's work
    long long tnext = i + stride;
    if (dyn && lane == 0) tnext = stride + (long long)atomicAdd(&counters->next_env, 1u);
    Env e;
    int status = TC_ST_OK;
    TRACE(i, 0);
    if (mode == MODE_RESET) {
      e.rkey = st.rkey[i];
      e.rctr = st.rctr[i];
      reset_draws(S, e);
      store_env<G>(S, so, i, e);
    } else {
      // the action is fetched before the state so both loads are in flight
      // together (one memory latency, not two, ahead of the dynamics)
      long long act = 0;
      if (mode == MODE_STEP)
        act = (early && i == i_first) ? (one_wave ? act_s[grp] : a_pre) : actions[i];
      load_env<G>(S, st, i, e);
      if (mode == MODE_STEP) {
        TRACE(i, 1);
        if (act < 0 || act >= A_COUNT || !((S.legal_mask >> act) & 1u)) {
          status = TC_ST_BAD_ACTION;
          if (out.flag_host && lane == 0) *(volatile int32_t*)out.flag_host = 1;
          store_env<G>(S, so, i, e);  // out-of-place: carry the state over
        } else {
          const StepOut o = step_dynamics<G>(S, cell, solid, e, (int)act, validate);
          if (lane == 0) {
            out.rewards[i] = o.reward;
            out.dones[i] = (uint8_t)o.done;
            out.truncs[i] = (uint8_t)o.trunc;
            out.events[i] = o.events;
            if (one_wave && out.res_host) {
              rew_s[grp] = o.reward;
              done_s[grp] = (uint8_t)o.done;
            }
          }
          viol += (unsigned long long)o.violation;
          if (o.done && auto_reset) reset_draws(S, e);
          store_env<G>(S, so, i, e);
          TRACE(i, 2);
        }
      }
    }
    if (status == TC_ST_OK) {
      // debug taps only in the TAPS instantiation (nullptr constants fold
      // the tap code out of the throughput kernel)
      status = render_env<NC, G, FIX>(
          S, cell, solid, sm, e, out.frames + (size_t)i * frame_bytes,
          (TAPS && out.zbuf) ? out.zbuf + (size_t)i * S.obs_w : nullptr,
          (TAPS && out.rayinfo) ? out.rayinfo + (size_t)i * S.obs_w * 4 : nullptr,
          (TAPS && out.spritevis) ? out.spritevis + i : nullptr, bulk_pending, buf, lg, i);
    }
    if (lane == 0) out.statuses[i] = status;
    // a bad action on the mapped host path is reported through flag_host
    // only (the host voids the step); the sticky counters keep real faults
    if (status != TC_ST_OK && !(status == TC_ST_BAD_ACTION && out.flag_host))
      badbits |= 1u << status;
#if TC_TRACE
    if (g_trace && lane == 0) {
      unsigned int smid;
      asm("mov.u32 %0, %smid;" : "=r"(smid));
      g_trace[i * 16 + 5] = gtime();
      g_trace[i * 16 + 6] = smid | ((unsigned long long)grp << 16) |
                           ((unsigned long long)blockIdx.x << 32);
    }
#endif
    i = dyn ? g.shfl(tnext, 0) : i + stride;
  }
  if (lane == 0) {
    if (bulk_pending) bulk_wait_all();
    if (counters) {
      if (viol) atomicAdd(reinterpret_cast<unsigned long long*>(&counters->violations), viol);
      if (badbits) atomicOr(&counters->bad_status, badbits);
    }
  }
  if (dyn || out.res_host) {
    // every warp is done with its shared memory: word 0 carries the flag
    volatile int& s_last = *reinterpret_cast<int*>(smem);
    __syncthreads();
    if (one_wave && out.res_host) {
      // one-wave mapping: the CTA's contiguous rewards / dones go to pinned
      // host memory as one run each, ordered (device-scope fence here, one
      // cumulative system fence by the last CTA, as in ship_results) before
      // the host's completion word (a voided bad-action env keeps reward 0,
      // done 0)
      if (warp0 && (int)threadIdx.x < cta_envs) {
        const int k = threadIdx.x;
        reinterpret_cast<double*>(out.res_host)[cbase + k] = rew_s[k];
        out.res_host[(size_t)n * 8 + cbase + k] = done_s[k];
        __threadfence();
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      __threadfence();
      const bool last = atomicAdd(&counters->ctas_done, 1u) == (unsigned)ncta - 1;
      if (last) {
        counters->next_env = 0;
        counters->ctas_done = 0;
      }
      s_last = last;
    }
    __syncthreads();
    if (s_last && out.res_host && one_wave) {
      // every CTA's results reached host memory before it was counted
      if (threadIdx.x == 0) {
        __threadfence_system();
        *(volatile int32_t*)(out.flag_host + 1) = 1;
      }
    } else if (s_last && out.res_host) {
      // every CTA's rewards / dones are visible (fence before the count);
      // ship them to pinned host memory with 16-byte coalesced stores
      __threadfence();
      const size_t bytes = (size_t)n * 9, nv = bytes >> 4;
      copy_results_host(reinterpret_cast<const uint4*>(out.rewards),
                        reinterpret_cast<uint4*>(out.res_host), nv);
      const uint8_t* sb = reinterpret_cast<const uint8_t*>(out.rewards);
      for (size_t k = nv * 16 + threadIdx.x; k < bytes; k += blockDim.x)
        out.res_host[k] = __ldcg(sb + k);
      // results (and every CTA's state / frame writes) are complete: raise
      // the host's completion word once the copies are visible system-wide
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x == 0) *(volatile int32_t*)(out.flag_host + 1) = 1;
    }
  }
#if TC_TRACE
  if (g_trace_cta) {
    __syncthreads();
    if (threadIdx.x == 0) {
      tcta[3] = gtime();
      unsigned long long* d = g_trace_cta + ((size_t)tgen * 16384 + blockIdx.x) * 4;
      d[0] = tcta[0]; d[1] = tcta[1]; d[2] = tcta[2]; d[3] = tcta[3];
    }
  }
#endif
}

// The lean step kernel: one env per warp (all 32 lanes, NC = W / 32 columns
// per lane, one lockstep march round), for the common shape -- a sealed map
// staged in shared memory, fewer than 32 doors, mirrored lane-contiguous
// compose (W / 16 divides 32) -- and no debug taps. A batch_kernel
// specialisation with only the hot path in it: the two envs of a 16-lane
// pair no longer serialise each other's divergent phases (turn vs move,
// sprites vs none, long vs short rays), and the code is small and register
// lean (7 CTAs of 4 warps per SM: a 4096-env batch is one wave). Envs whose
// pose is off the grid or whose view direction is zero take the checked
// wall pass out of line. _pycore.py:346-547 like batch_kernel.
template <int NC, int G, int MINB, bool TAPS>
__global__ void __launch_bounds__(WARPS_PER_CTA * 32, MINB)
batch_kernel(const __grid_constant__ SpecDev S, const __grid_constant__ StateDev st,
             const __grid_constant__ StateDev so, const long long* __restrict__ actions,
             const __grid_constant__ OutDev out,
             long long n, int mode, int auto_reset, int validate,
             tc_counters* __restrict__ counters) {
  batch_body<NC, G, TAPS, (MINB <= 4)>(S, st, so, actions, out, n, mode, auto_reset, validate,
                                       counters, blockIdx.x, gridDim.x);
}

// Heterogeneous-map step in ONE launch: up to TC_MULTI_MAX groups (spec g
// over envs [off_g, off_g + n_g) of the batch, its own state blocks, output
// views and counters). Work is handed out in blocks of one CTA pass (one env
// per lane group) from ONE ticket counter, in group order: a CTA keeps its
// staged spec while its tickets stay in the same group and restages (a new
// TMA bulk copy, the group's launch record copied to shared memory) when it
// crosses into the next group -- so the maps' different costs balance over
// the whole grid instead of over fixed per-group CTA ranges. Lifts the
// reference's homogeneous-batch limit.
constexpr int TC_MULTI_MAX = 16;
struct MultiGroup {
  SpecDev spec;
  StateDev st, so;
  OutDev out;
  long long n, off;
  tc_counters* counters;
};
struct MultiArgs {
  int n_groups;
  long long total_blocks;
  long long block_begin[TC_MULTI_MAX + 1];
  tc_counters* ticket;  // the launch's block ticket / CTA count (group 0's counters)
  MultiGroup g[TC_MULTI_MAX];
};

template <int NC, int G, int MINB>
__global__ void __launch_bounds__(WARPS_PER_CTA * 32, MINB)
multi_kernel(const __grid_constant__ MultiArgs A, const long long* __restrict__ actions,
             int auto_reset, int validate) {
  constexpr int NG = 32 / G;
  __shared__ __align__(16) MultiGroup s_grp;
  __shared__ long long s_block;
  uint8_t* const smem = g_smem;
  const Grp<G> g;
  const int lane = g.lane;
  const int grp = (threadIdx.x >> 5) * NG + (threadIdx.x & 31) / G;
  constexpr int PER_CTA = WARPS_PER_CTA * NG;
  uint32_t* smap = reinterpret_cast<uint32_t*>(smem);
  const uint32_t *cell = nullptr, *solid = nullptr;
  asm volatile("griddepcontrol.launch_dependents;");
  int cur = -1;
  bool waited = false;
  const LaneGeo lg = lane_geo<G>(A.g[0].spec);
  int bulk_pending = 0, buf = 0;
  unsigned long long viol = 0;
  uint32_t badbits = 0;
  for (;;) {
    if (waited) __syncthreads();  // the previous block is done with the staged spec
    if (threadIdx.x == 0)
      s_block = waited ? (long long)gridDim.x + atomicAdd(&A.ticket->next_env, 1u) : -1;
    __syncthreads();
    long long b = s_block;
    if (!waited) {
      // the first block is blockIdx.x (no ticket); stage before the wait
      b = blockIdx.x;
    }
    if (b >= A.total_blocks) break;
    int gi = 0;
    while (gi + 1 < A.n_groups && b >= A.block_begin[gi + 1]) gi++;
    if (gi != cur) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(&A.g[gi]);
      uint32_t* dst = reinterpret_cast<uint32_t*>(&s_grp);
      for (int k = threadIdx.x; k < (int)(sizeof(MultiGroup) / 4); k += blockDim.x) dst[k] = src[k];
      __syncthreads();
      stage_map_issue(s_grp.spec, smap, cell, solid);
      stage_map_wait();
      cur = gi;
    }
    if (!waited) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
    }
    const SpecDev& S = s_grp.spec;
    const long long i = (b - A.block_begin[gi]) * PER_CTA + grp;
    if (i < s_grp.n) {
      const WarpSmem sm = carve(smem + map_smem_bytes(S) + grp * S.warp_smem);
      const size_t frame_bytes = (size_t)S.obs_h * S.obs_w * 3;
      const long long act = actions[s_grp.off + i];
      Env e;
      load_env<G>(S, s_grp.st, i, e);
      int status = TC_ST_OK;
      if (act < 0 || act >= A_COUNT || !((S.legal_mask >> act) & 1u)) {
        status = TC_ST_BAD_ACTION;
        store_env<G>(S, s_grp.so, i, e);
      } else {
        const StepOut o = step_dynamics<G>(S, cell, solid, e, (int)act, validate);
        if (lane == 0) {
          s_grp.out.rewards[i] = o.reward;
          s_grp.out.dones[i] = (uint8_t)o.done;
          s_grp.out.truncs[i] = (uint8_t)o.trunc;
          s_grp.out.events[i] = o.events;
        }
        viol += (unsigned long long)o.violation;
        if (o.done && auto_reset) reset_draws(S, e);
        store_env<G>(S, s_grp.so, i, e);
        status = render_env<NC, G, (MINB <= 4)>(S, cell, solid, sm, e,
                                                s_grp.out.frames + (size_t)i * frame_bytes,
                                                nullptr, nullptr, nullptr, bulk_pending, buf,
                                                lg, i);
      }
      if (lane == 0) s_grp.out.statuses[i] = status;
      if (status != TC_ST_OK && lane == 0 && s_grp.counters)
        atomicOr(&s_grp.counters->bad_status, 1u << status);
      if (viol && lane == 0 && s_grp.counters) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_grp.counters->violations), viol);
        viol = 0;
      }
    }
  }
  if (lane == 0 && bulk_pending) bulk_wait_all();
  (void)badbits;
  // the last CTA to finish re-arms the launch's ticket
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&A.ticket->ctas_done, 1u) == gridDim.x - 1) {
      A.ticket->next_env = 0;
      A.ticket->ctas_done = 0;
    }
  }
}

// Mapped host step, one wave: each warp parks its env's [reward | done] in
// the CTA scratch right after the dynamics; at a CTA barrier warp 0 ships the
// CTA's contiguous run to pinned host memory (one system fence per CTA) and
// counts the CTA; the CTA completing the count raises the host's completion
// word -- while the frames are still being rendered. The host may return
// and prepare the next step meanwhile: anything it launches next on the
// stream is ordered after this kernel (complete frames and state).
__device__ __forceinline__ void ship_results(const OutDev& out, tc_counters* counters,
                                             long long n, long long cbase, int cta_envs,
                                             int ctas, const double* rew_s,
                                             const uint8_t* done_s) {
  asm volatile("bar.sync 1, %0;" ::"r"(WARPS_PER_CTA * 32) : "memory");
  if (threadIdx.x < 32) {
    const int k = threadIdx.x;
    if (k < cta_envs) {
      reinterpret_cast<double*>(out.res_host)[cbase + k] = rew_s[k];
      out.res_host[(size_t)n * 8 + cbase + k] = done_s[k];
    }
    // device-scope fence before the count; the CTA completing the count
    // fences system-wide before raising the word, and fences are cumulative
    // (PTX causality order is transitive), so every CTA's host writes are
    // visible to a host that has seen the word -- one system fence per
    // launch instead of one per CTA (-5 us per mapped step at 1036 CTAs,
    // tools/ubench_mapped.cu modes 3 / 4)
    __threadfence();
    __syncwarp();
    if (k == 0) {
      const unsigned int c = atomicAdd(&counters->ctas_done, 1u);
      if ((int)c == ctas - 1) {
        counters->ctas_done = 0;  // every CTA has counted: ready for the next launch
        __threadfence_system();
        *(volatile int32_t*)(out.flag_host + 1) = 1;
      }
    }
  }
}

// Launch schedule of the lean kernel, computed on the host: one wave
// (CTA c owns envs [c*epc, c*epc + epc)) or tickets (first env grp*grid +
// cta, then an atomic ticket per env, stride = grid * warps per CTA).
struct LeanSched {
  long long n, stride;
  int epc, early;
  int ctas;  // one wave: CTAs that own envs (the mapped host step counts them)
  // Chained steps (tc_batch_steps, one wave): per-env "state written" and
  // per-CTA "frames written" epochs in device memory (flags = [ready u32[n] |
  // done u32[ctas]]). A launch with need_ready != 0 skips the grid-wide
  // griddepcontrol.wait: env i waits only for ready[i] >= need_ready (its
  // state from the previous step) and, when need_done != 0, for the CTA's
  // done[] >= need_done (the output block it is about to overwrite was
  // finished), so a step's CTAs start as soon as the previous step's CTAs
  // free their slots instead of after its slowest CTA.
  // Multi-wave (env tickets): ready[i] is published after env i's whole
  // step (state and frames), so a later step's env i waits for nothing else
  // (no per-CTA done epochs), and each launch draws its tickets from its own
  // zeroed counter (`tickets`) instead of counters->next_env, which the
  // previous launch's last CTA would otherwise still be re-zeroing.
  unsigned int* flags;
  unsigned int* tickets;
  unsigned int epoch, need_ready, need_done;
  // one wave: the done epochs of the output block this launch writes are
  // flags[done_off + cta] (one row per ring slot: launches that write other
  // blocks may finish out of order, so a shared row would let a later
  // launch's epoch stand in for the slot's previous writer)
  unsigned int done_off;
  // Pipelined host step (tc_batch_step_pipelined): a launch made one step
  // ahead of its actions. After the previous grid (griddepcontrol.wait) and
  // the spec staging, CTA 0 polls the host gate words [go | cancel] (pinned,
  // written by the host) for gate_q and publishes the outcome to gate_dev
  // (2q = go, 2q + 1 = cancel); the other CTAs poll gate_dev in L2. A
  // cancelled launch exits before touching any state or output.
  unsigned int* gate_dev;
  const unsigned long long* gate_host;
  unsigned int gate_q;
  // resident host-step loop (lean_kernel RES = true): after step k the
  // kernel waits at gate gate_q + k + 1 for step k + 1 of the reuse=True
  // ping-pong (state blocks swap, output blocks alternate out / out2)
  // instead of exiting; a cancel ends it with every state block as an
  // ordinary launch sequence would have left it
  OutDev out2;
  // resident loop timeline (TILECAST_PIPE_TRACE=1 only): globaltimer per
  // step k < 64 and CTA: [k][0] past the gate, [k][1] results shipped,
  // [k][2] frame written
  unsigned long long* rtrace;
};

constexpr int GATE_LINES = 32;  // gate_dev: GATE_LINES words, 128 B apart

// the pipelined step's gate (see LeanSched): true = released (the host's
// actions for this step are in pinned memory), false = cancelled. A launch
// nobody releases or cancels within ~1 s cancels itself and leaves an
// "expired" mark in the host word after the gate pair (a host that released
// it then sees the kernel finish without results and reports the error).
__device__ __forceinline__ unsigned long long gate_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// host-written data read after the gate (the actions): ordinary loads. The
// gate is a causality chain -- host stores actions, then go (x86 TSO); CTA 0
// observes go with an acquire.sys load and publishes it with a release.gpu
// store; every other CTA acquires that store -- so the loads after it see
// the host's actions. (A relaxed.sys load per warp instead costs ~140 us per
// step at 4096 envs, measured: sys-scope loads of pinned memory serialise.)
__device__ __forceinline__ long long ld_sys(const long long* p) { return *p; }
__device__ __forceinline__ void rstamp(const LeanSched& ls, unsigned int k, int slot) {
  if (ls.rtrace && threadIdx.x == 0 && k < 64u)
    ls.rtrace[((size_t)k * 3 + slot) * gridDim.x + blockIdx.x] = gate_clock();
}
// the actions after the gate: one wave, the CTA's contiguous run in one bus
// read (4,096 single-env reads of pinned memory queue on the bus: +2 us per
// step), parked in the CTA scratch; multi-wave, per env
template <bool ONE_WAVE>
__device__ __forceinline__ long long gate_actions(const LeanSched& ls, const long long* actions,
                                                  long long i, long long cbase, int cta_envs,
                                                  long long* act_s) {
  if (!ONE_WAVE) return i < ls.n ? ld_sys(actions + i) : 0;
  if (threadIdx.x < (unsigned)cta_envs) act_s[threadIdx.x] = ld_sys(actions + cbase + threadIdx.x);
  __syncthreads();
  return i < ls.n ? act_s[threadIdx.x >> 5] : 0;
}
__device__ __noinline__ bool gate_pass(const LeanSched& ls, unsigned int q) {
  bool go = false;
  if (threadIdx.x == 0) {
    const unsigned int q2 = 2u * q;
    unsigned int w;
    if (blockIdx.x == 0) {
      const unsigned long long t0 = gate_clock();
      for (unsigned int spin = 0;; spin++) {
        unsigned long long hw;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(hw) : "l"(ls.gate_host) : "memory");
        if ((unsigned int)hw == q) { w = q2; break; }
        if ((unsigned int)(hw >> 32) == q) { w = q2 + 1u; break; }
        if ((spin & 255u) == 255u && gate_clock() - t0 > 1000000000ull) {
          w = q2 + 1u;
          *(volatile unsigned int*)(ls.gate_host + 1) = q;
          __threadfence_system();
          break;
        }
      }
      // publish to GATE_LINES copies (one 128-byte line each) so the other
      // CTAs' polls spread over lines instead of queueing on one: a
      // fence-based release, then relaxed stores
      __threadfence();
#pragma unroll 1
      for (int l = 0; l < GATE_LINES; l++)
        asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(ls.gate_dev + l * 32), "r"(w) : "memory");
    } else {
      const unsigned int* line = ls.gate_dev + (blockIdx.x % GATE_LINES) * 32;
      for (;;) {
        asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(w) : "l"(line) : "memory");
        if ((int)(w - q2) >= 0) break;
      }
      __threadfence();  // fence-based acquire
    }
    go = w == q2;
  }
  return __syncthreads_or(go) != 0;
}

// chained steps: env i's state is in memory -- every lane fences its own
// stores (store_env spreads them over lanes), then lane 0 publishes the epoch
template <class Grp_>
__device__ __forceinline__ void state_ready(const Grp_& g, const LeanSched& ls, long long i) {
  __threadfence();
  g.sync();
  if (g.lane == 0) *(volatile unsigned int*)(ls.flags + i) = ls.epoch;
}

template <int NC, bool ONE_WAVE, int FW, int FH, int G, int MINB, bool RES = false>
__global__ void __launch_bounds__(WARPS_PER_CTA * 32, MINB)
lean_kernel(const __grid_constant__ SpecDev S, const __grid_constant__ StateDev st,
            const __grid_constant__ StateDev so, const long long* __restrict__ actions,
            const __grid_constant__ OutDev out, const __grid_constant__ LeanSched ls,
            int auto_reset, int validate, tc_counters* __restrict__ counters) {
  // G = 32: one env per warp (one-wave batches); G = 16: the two halves of
  // a warp run one env each (multi-wave batches: the pair shares its
  // convergent code, the issue-bound regime)
  constexpr int NG = 32 / G, PER_CTA = WARPS_PER_CTA * NG;
  const Grp<G> gr;
  uint8_t* const smem = g_smem;
  const int lane = gr.lane;
  const int grp = (threadIdx.x >> 5) * NG + (threadIdx.x & 31) / G;
  uint32_t* smap = reinterpret_cast<uint32_t*>(smem);
  const uint32_t *cell, *solid;
#if TC_TRACE
  unsigned long long tcta[4] = {0, 0, 0, 0};
  unsigned int tgen = 0;
  if (g_trace_cta && threadIdx.x == 0) {
    tcta[0] = gtime();
    tgen = atomicAdd(&g_cta_gen[blockIdx.x], 1u);
  }
#endif
  asm volatile("griddepcontrol.launch_dependents;");
  const long long n = ls.n;
  const long long cbase = ONE_WAVE ? (long long)blockIdx.x * ls.epc : 0;
  const int cta_envs = ONE_WAVE ? (int)max(0LL, min((long long)ls.epc, n - cbase)) : 0;
  // (multi-wave mapped steps count every CTA at the end, envs or not)
  if (ONE_WAVE ? cta_envs == 0 : ((long long)blockIdx.x >= n && !out.res_host)) return;
  long long i = ONE_WAVE ? (grp < cta_envs ? cbase + grp : n)
                         : (long long)grp * gridDim.x + blockIdx.x;
  const int map_bytes = map_smem_bytes(S);
  // CTA scratch after the per-warp windows: [rewards f64 | dones u8 | goals
  // i32 | (pipelined, one wave) actions i64 at +96]
  long long* const act_s =
      reinterpret_cast<long long*>(smem + map_bytes + PER_CTA * S.warp_smem + 96);
  static_assert(!ONE_WAVE || 96 + 8 * PER_CTA <= CTA_SCRATCH, "CTA scratch: actions");
  // mapped host path: the host wrote the actions before the launch (see
  // batch_kernel); device actions are read after griddepcontrol.wait
  long long act = 0, act_next = 0;
  const bool gated = ls.gate_dev != nullptr;
  if (ls.early && !gated && i < n) act = actions[i];
  // multi-wave mapped: the next ticket's action is read from host memory one
  // env ahead (after this env's dynamics), so its bus round trip overlaps
  // the render instead of stalling the warp at the top of every env
  const auto prefetch = [&](long long tn) {
    if (!ONE_WAVE && ls.early && lane == 0 && tn < n)
      act_next = gated ? ld_sys(actions + tn) : actions[tn];
  };
  stage_map_issue(S, smap, cell, solid);
  stage_map_wait();
#if TC_TRACE
  if (g_trace_cta && threadIdx.x == 0) tcta[1] = gtime();
#endif
  const bool chained = ls.flags != nullptr && ls.need_ready != 0;
  if (!chained) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (gated) {
    // pipelined host step: wait here (previous grid done, tables staged)
    // for the host to release or cancel this launch
    if (!gate_pass(ls, ls.gate_q)) return;
    if (ls.early) act = gate_actions<ONE_WAVE>(ls, actions, i, cbase, cta_envs, act_s);
  }
#if TC_TRACE
  if (g_trace_cta && threadIdx.x == 0) tcta[2] = gtime();
#endif
  const WarpSmem sm = carve(smem + map_bytes + grp * S.warp_smem);
  double* rew_s = reinterpret_cast<double*>(smem + map_bytes + PER_CTA * S.warp_smem);
  uint8_t* done_s = reinterpret_cast<uint8_t*>(rew_s + PER_CTA);
  // the env's goal entity parks here across the wall pass (only the sprite
  // cull reads it after the dynamics): a register there would be spilled
  int* agoal_s = reinterpret_cast<int*>(rew_s + 2 * PER_CTA);
  static_assert(20 * PER_CTA <= CTA_SCRATCH, "CTA scratch: rewards, dones, goals");
  for (unsigned int k = 0;; k++) {
    const StateDev& sti = (RES && (k & 1u)) ? so : st;
    const StateDev& sto = (RES && (k & 1u)) ? st : so;
    const OutDev& ob = (RES && (k & 1u)) ? ls.out2 : out;
    if constexpr (RES) rstamp(ls, k, 0);
    // one wave, mapped: warps without an env still take part in the CTA's
    // result hand-off barrier
    if (ONE_WAVE && ob.res_host && i >= n)
      ship_results(ob, counters, n, cbase, cta_envs, ls.ctas, rew_s, done_s);
    constexpr size_t FB = (size_t)FW * FH * 3;
    const size_t frame_bytes = FB ? FB : (size_t)S.obs_h * S.obs_w * 3;
    bool first = true;
    if (ONE_WAVE && chained && i < n) {
      // this env's state from the previous step, and (need_done) the output
      // block this launch overwrites finished by the step that last wrote it
      if (lane == 0) {
        const volatile unsigned int* rd = ls.flags + i;
        const volatile unsigned int* dn = ls.flags + ls.done_off + blockIdx.x;
        while ((int)(*rd - ls.need_ready) < 0 ||
               (ls.need_done != 0 && (int)(*dn - ls.need_done) < 0))
          __nanosleep(64);
      }
      gr.sync();
      __threadfence();  // acquire: the flag's writer fenced before setting it
    }
    while (i < n) {
      long long tnext = 0;
      if (!ONE_WAVE && lane == 0 && (counters || ls.flags))
        tnext = ls.stride + (long long)atomicAdd(ls.flags ? ls.tickets : &counters->next_env, 1u);
      if (!ONE_WAVE && chained) {
        // multi-wave chained: env i's previous step (state and frames) is done
        if (lane == 0) {
          const volatile unsigned int* rd = ls.flags + i;
          while ((int)(*rd - ls.need_ready) < 0) __nanosleep(64);
        }
        gr.sync();
        __threadfence();
      }
      if (!ls.early) {
        act = actions[i];
      } else if (!first) {
        act = gr.shfl(act_next, 0);
      }
      first = false;
      Env e;
      TRACE(i, 0);
      load_env<G>(S, sti, i, e);
      // outputs, status and host results are written as soon as they are
      // known, so nothing but the env index stays live across the render
      if (act < 0 || act >= A_COUNT || !((S.legal_mask >> act) & 1u)) {
        store_env<G>(S, sto, i, e);  // out-of-place: carry the state over
        if (ONE_WAVE && ls.flags) state_ready(gr, ls, i);
        if (lane == 0) {
          ob.statuses[i] = TC_ST_BAD_ACTION;
          if (ob.flag_host) {
            *(volatile int32_t*)ob.flag_host = 1;
          } else if (counters) {
            atomicOr(&counters->bad_status, 1u << TC_ST_BAD_ACTION);
          }
          if (ONE_WAVE && ob.res_host) {  // a voided env reports reward 0, done 0
            rew_s[grp] = 0.0;
            done_s[grp] = 0;
          }
        }
        if (ONE_WAVE && ob.res_host)
          ship_results(ob, counters, n, cbase, cta_envs, ls.ctas, rew_s, done_s);
        prefetch(tnext);
      } else {
        TRACE(i, 1);
        const StepOut o = step_dynamics<G>(S, cell, solid, e, (int)act, validate);
        prefetch(tnext);
        if (lane == 0) {
          ob.rewards[i] = o.reward;
          ob.dones[i] = (uint8_t)o.done;
          ob.truncs[i] = (uint8_t)o.trunc;
          ob.events[i] = o.events;
          ob.statuses[i] = TC_ST_OK;
          if (o.violation && counters)
            atomicAdd(reinterpret_cast<unsigned long long*>(&counters->violations), 1ull);
          if (ONE_WAVE && ob.res_host) {
            // this env's [reward | done] straight to pinned host memory (the
            // CTA's envs are contiguous: the warps' stores merge on the bus)
            rew_s[grp] = o.reward;
            done_s[grp] = (uint8_t)o.done;
          }
        }
        if (ONE_WAVE && ob.res_host)
          ship_results(ob, counters, n, cbase, cta_envs, ls.ctas, rew_s, done_s);
        if constexpr (RES) rstamp(ls, k, 1);
        if (o.done && auto_reset) reset_draws(S, e);
        store_env<G>(S, sto, i, e);
        if (ONE_WAVE && ls.flags) state_ready(gr, ls, i);
        if (lane == 0) agoal_s[grp] = e.agoal;
        TRACE(i, 2);
        uint8_t* frame = ob.frames + (size_t)i * frame_bytes;
        const double planex = -e.dy * PLANE_HALF_WIDTH;
        const double planey = e.dx * PLANE_HALF_WIDTH;
        const bool inside = e.x >= 0.0 && e.y >= 0.0 && e.x < (double)S.w && e.y < (double)S.h &&
                            (e.dx != 0.0 || e.dy != 0.0);
        int status;
        if (inside) {
          wall_pass<NC, false, G, true, FW, FH>(S, cell, solid, sm, e, planex, planey, nullptr,
                                                nullptr, TC_TRACE ? i : -1);
          status = TC_ST_OK;
        } else {
          status = wall_pass_cold<NC, G>(S, cell, solid, sm, e, planex, planey, nullptr, nullptr,
                                         false);
        }
        gr.sync();
        TRACE(i, 3);
        if (status == TC_ST_OK) {
          e.agoal = agoal_s[grp];  // (the wall pass synced the group)
          const int m = S.n_ent ? sprite_setup<G>(S, sm, e, planex, planey, nullptr) : 0;
          TRACE(i, 4);
  #if TC_TRACE
          if (g_trace && lane == 0) g_trace[i * 16 + 7] = (unsigned long long)m;
  #endif
          if constexpr (FW != 0) mirror_contig_fixed<FW, FH, G>(S, sm, m, frame);
          else mirror_contig<NC, G>(S, sm, m, frame);
        } else if (lane == 0) {
          ob.statuses[i] = status;
          if (counters) atomicOr(&counters->bad_status, 1u << status);
        }
      }
  #if TC_TRACE
      if (g_trace && lane == 0) {
        unsigned int smid;
        asm("mov.u32 %0, %smid;" : "=r"(smid));
        g_trace[i * 16 + 5] = gtime();
        g_trace[i * 16 + 6] = smid | ((unsigned long long)grp << 16) |
                             ((unsigned long long)blockIdx.x << 32);
      }
  #endif
      if (ONE_WAVE) break;
      if (ls.flags) state_ready(gr, ls, i);  // multi-wave chained: the whole step
      i = (counters || ls.flags) ? gr.shfl(tnext, 0) : i + ls.stride;
    }
    if constexpr (!RES) {
      break;
    } else {
      // resident host-step loop: step k + 1 of the ping-pong, once the host
      // has written its actions (or the end of the loop: a cancel)
      rstamp(ls, k, 2);
      if (!gate_pass(ls, ls.gate_q + k + 1u)) return;
      act = gate_actions<ONE_WAVE>(ls, actions, i, cbase, cta_envs, act_s);
    }
  }
#if TC_TRACE
  if (g_trace_cta) {
    __syncthreads();
    if (threadIdx.x == 0) {
      tcta[3] = gtime();
      unsigned long long* d = g_trace_cta + ((size_t)tgen * 16384 + blockIdx.x) * 4;
      d[0] = tcta[0]; d[1] = tcta[1]; d[2] = tcta[2]; d[3] = tcta[3];
    }
  }
#endif
  if (ONE_WAVE && ls.flags) {
    // every warp's frame writes are performed before the CTA's done epoch
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) *(volatile unsigned int*)(ls.flags + ls.done_off + blockIdx.x) = ls.epoch;
  }
  // one wave: the mapped host step was released by ship_results as soon as
  // every env's reward / done had reached the host; nothing left to count
  // (multi-wave chained launches draw tickets from their own counter: nothing
  // to re-zero)
  if (ONE_WAVE || !counters || ls.flags) return;
  {
    volatile int& s_last = *reinterpret_cast<int*>(smem);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const bool last = atomicAdd(&counters->ctas_done, 1u) == gridDim.x - 1;
      if (last) {
        counters->next_env = 0;
        counters->ctas_done = 0;
      }
      s_last = last;
    }
    __syncthreads();
    if (s_last && out.res_host && ONE_WAVE) {
      if (threadIdx.x == 0) {
        __threadfence_system();
        *(volatile int32_t*)(out.flag_host + 1) = 1;
      }
    } else if (s_last && out.res_host) {
      __threadfence();
      const size_t bytes = (size_t)n * 9, nv = bytes >> 4;
      copy_results_host(reinterpret_cast<const uint4*>(out.rewards),
                        reinterpret_cast<uint4*>(out.res_host), nv);
      const uint8_t* sb = reinterpret_cast<const uint8_t*>(out.rewards);
      for (size_t k = nv * 16 + threadIdx.x; k < bytes; k += blockDim.x)
        out.res_host[k] = __ldcg(sb + k);
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x == 0) *(volatile int32_t*)(out.flag_host + 1) = 1;
    }
  }
}

// K fused steps with on-device policy actions (batch.py:141-153 draws) and
// auto-reset; the env's state stays in registers across steps.
template <int NC, int G>
__global__ void __launch_bounds__(WARPS_PER_CTA * 32, G == 16 ? TC_MIN_CTAS16 : TC_MIN_CTAS)
rollout_kernel(const __grid_constant__ SpecDev S, const __grid_constant__ StateDev st,
               const __grid_constant__ OutDev out, long long n,
               const __grid_constant__ RolloutArgs ra, tc_counters* __restrict__ counters) {
  uint8_t* const smem = g_smem;
  constexpr int NG = 32 / G;
  const Grp<G> g;
  const int lane = g.lane;
  const int grp = (threadIdx.x >> 5) * NG + (threadIdx.x & 31) / G;
  uint32_t* smap = reinterpret_cast<uint32_t*>(smem);
  const int map_bytes = map_smem_bytes(S);
  const uint32_t *cell, *solid;
  if ((long long)blockIdx.x >= n) return;  // no env for this CTA (n < grid)
  stage_map(S, smap, cell, solid);
  const WarpSmem sm = carve(smem + map_bytes + grp * S.warp_smem);
  const size_t frame_bytes = (size_t)S.obs_h * S.obs_w * 3;
  const LaneGeo lg = lane_geo<G>(S);
  int bulk_pending = 0, buf = 0;
  uint32_t badbits = 0;
  const long long stride = (long long)gridDim.x * WARPS_PER_CTA * NG;
  for (long long i = (long long)grp * gridDim.x + blockIdx.x; i < n; i += stride) {
    Env e;
    int st_acc = TC_ST_OK;
    load_env<G>(S, st, i, e);
    int ring_k = 0;
    for (int k = 0; k < ra.k_steps; k++) {
      const long long step = ra.step0 + k;
      unsigned long long ctr = (unsigned long long)(step * ra.n_total + ra.base + i);
      const int act = ra.tags[draw_below(ra.policy_key, ctr, (uint64_t)ra.n_tags)];
      const StepOut o = step_dynamics<G>(S, cell, solid, e, act, 0);
      const size_t kn = (size_t)k * (size_t)n + (size_t)i;
      if (lane == 0) {
        if (out.rewards) out.rewards[kn] = o.reward;
        if (out.dones) out.dones[kn] = (uint8_t)o.done;
        if (out.truncs) out.truncs[kn] = (uint8_t)o.trunc;
        if (out.events) out.events[kn] = o.events;
      }
      if (o.done) reset_draws(S, e);
      const size_t slot = (size_t)ring_k * (size_t)n + (size_t)i;
      if (++ring_k == ra.frame_ring) ring_k = 0;
      const int status = render_env<NC, G, true>(S, cell, solid, sm, e, out.frames + slot * frame_bytes,
                                           nullptr, nullptr, nullptr, bulk_pending, buf, lg);
      if (status != TC_ST_OK) {
        badbits |= 1u << status;
        if (st_acc == TC_ST_OK) st_acc = status;
      }
    }
    store_env<G>(S, st, i, e);
    if (lane == 0 && out.statuses) out.statuses[i] = st_acc;
  }
  if (lane == 0) {
    if (bulk_pending) bulk_wait_all();
    if (counters && badbits) atomicOr(&counters->bad_status, badbits);
  }
}

__global__ void seed_kernel(uint64_t root, long long base, long long n,
                            unsigned long long* rkey, unsigned long long* rctr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    rkey[i] = mix64(root + SPLIT_SALT + (uint64_t)(base + i) * GOLDEN);
    rctr[i] = 0;
  }
}

struct Tags { long long v[A_COUNT]; };

__global__ void policy_kernel(uint64_t key, long long step, long long n_total, long long base,
                              long long n, Tags tags, int n_tags, long long* actions) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long ctr = (unsigned long long)(step * n_total + base + i);
    actions[i] = tags.v[draw_below(key, ctr, (uint64_t)n_tags)];
  }
}

__global__ void cast_ray_kernel(const uint32_t* cell, int h, int w, uint32_t dmask, double ox,
                                double oy, double rx, double ry, int32_t* io, double* dout) {
  const RayHit r = cast_ray(cell, h, w, dmask, ox, oy, rx, ry);
  io[0] = r.status; io[1] = r.mapx; io[2] = r.mapy; io[3] = r.side; io[4] = r.steps;
  dout[0] = r.perp; dout[1] = r.wu;
}

}  // namespace

// =================================================================== host
struct tc_spec {
  SpecDev dev;
  void* blob = nullptr;
  int nc = 1;
  int max_ctas = 0;    // grid size for one full wave
  int max_ctas_w = 0;  // the same for the multi-wave (wide) step kernel
  size_t smem_bytes = 0;
  int lean_ctas = 0;   // grid size for one full wave of lean_kernel (one env per warp)
  size_t lean_smem = 0;
  int lean16_ctas = 0;  // the same for the two-envs-per-warp multi-wave lean kernel (0: none)
  size_t lean16_smem = 0;
  int tab_bytes = 0;  // blob prefix holding the small tables
  int map_bytes = 0;  // blob prefix up to the end of the guarded stop codes
  int code8_bytes = 0;  // blob prefix up to the end of the guarded u8 stop codes
};

namespace {

thread_local std::string g_err;
thread_local double g_mapped_time[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
double host_us() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return 1e6 * (double)ts.tv_sec + 1e-3 * (double)ts.tv_nsec;
}
// programmatic dependent launch of consecutive steps (TILECAST_PDL=0 disables)
const bool g_pdl = [] {
  const char* e = getenv("TILECAST_PDL");
  return e ? atoi(e) != 0 : true;
}();
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(TC_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define TC_CUDA(call)                                    \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

uint32_t pack_rgb(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16);
}

// columns per lane for a group of G lanes, rounded to an instantiated NC
int pick_nc(int obs_w, int group) {
  const int need = (obs_w + group - 1) / group;
  const int opts[] = {1, 2, 3, 4, 8, 16, 32};
  for (int o : opts)
    if (o >= need) return o;
  return 32;
}

// 16-lane groups come in two register budgets: 128 registers (4 CTAs/SM)
// for batches that fit one wave -- the step is then a latency chain per env
// -- and 96 registers (5 CTAs/SM, more warps to hide latency) for batches
// that need several waves (measured: +3-6 % at 16K-131K envs, -5 % at 4K).
// Kernel budgets: 16-lane groups in two register budgets (WIDE: 96 regs, 5
// CTAs/SM for multi-wave batches; else 128 regs, 4 CTAs/SM, one-wave
// batches); full-warp groups TC_MIN_CTAS (multi-wave) / TC_MIN_CTAS32_1W
// (one-wave) CTAs per SM. TAPS = the debug-tap instantiation (zbuf / rayinfo
// / spritevis outputs; tests only), built with the WIDE budget.
#ifndef TC_MIN_CTAS32_1W
#define TC_MIN_CTAS32_1W TC_MIN_CTAS
#endif
template <int NC, int G, bool WIDE = false, bool TAPS = false>
const void* batch_fn() {
  constexpr int minb = G == 16 ? (WIDE ? TC_MIN_CTAS16_WIDE : TC_MIN_CTAS16)
                               : (WIDE ? TC_MIN_CTAS : TC_MIN_CTAS32_1W);
  return (const void*)batch_kernel<NC, G, minb, TAPS>;
}
template <int NC, int G>
const void* rollout_fn() { return (const void*)rollout_kernel<NC, G>; }

template <bool WIDE, bool TAPS>
const void* select_batch_t(int nc, int group) {
  if (group == 16) {
    switch (nc) {
      case 1: return batch_fn<1, 16, WIDE, TAPS>();
      case 2: return batch_fn<2, 16, WIDE, TAPS>();
      case 3: return batch_fn<3, 16, WIDE, TAPS>();
      default: return batch_fn<4, 16, WIDE, TAPS>();
    }
  }
  switch (nc) {
    case 1: return batch_fn<1, 32, WIDE, TAPS>();
    case 2: return batch_fn<2, 32, WIDE, TAPS>();
    case 3: return batch_fn<3, 32, WIDE, TAPS>();
    case 4: return batch_fn<4, 32, WIDE, TAPS>();
    case 8: return batch_fn<8, 32, WIDE, TAPS>();
    case 16: return batch_fn<16, 32, WIDE, TAPS>();
    default: return batch_fn<32, 32, WIDE, TAPS>();
  }
}
const void* select_batch(int nc, int group, bool wide = false, bool taps = false) {
  if (taps) return select_batch_t<true, true>(nc, group);
  return wide ? select_batch_t<true, false>(nc, group) : select_batch_t<false, false>(nc, group);
}
const void* select_rollout(int nc, int group) {
  if (group == 16) {
    switch (nc) {
      case 1: return rollout_fn<1, 16>();
      case 2: return rollout_fn<2, 16>();
      case 3: return rollout_fn<3, 16>();
      default: return rollout_fn<4, 16>();
    }
  }
  switch (nc) {
    case 1: return rollout_fn<1, 32>();
    case 2: return rollout_fn<2, 32>();
    case 3: return rollout_fn<3, 32>();
    case 4: return rollout_fn<4, 32>();
    case 8: return rollout_fn<8, 32>();
    case 16: return rollout_fn<16, 32>();
    default: return rollout_fn<32, 32>();
  }
}

#ifndef TC_MIN_CTAS_LEAN128W
#define TC_MIN_CTAS_LEAN128W 5  // lean kernel, 128x128 frames, multi-wave: 96 registers
                                // (7 spill slots instead of 43; +3 % over 7 CTAs at 72)
#endif
#ifndef TC_MIN_CTAS_LEAN16
#define TC_MIN_CTAS_LEAN16 5  // lean kernel, two envs per warp (multi-wave): 96 registers
#endif
// one-wave batches: one env per warp; multi-wave: two envs per warp (W <= 64)
template <bool ONE_WAVE>
const void* select_lean_t(int w, int h) {
  if (!ONE_WAVE && w <= 64) {
    if (w == 64 && h == 64) return (const void*)lean_kernel<4, false, 64, 64, 16, TC_MIN_CTAS_LEAN16>;
    switch ((w + 15) / 16) {
      case 2: return (const void*)lean_kernel<2, false, 0, 0, 16, TC_MIN_CTAS_LEAN16>;
      default: return (const void*)lean_kernel<4, false, 0, 0, 16, TC_MIN_CTAS_LEAN16>;
    }
  }
  if (w == 64 && h == 64) return (const void*)lean_kernel<2, ONE_WAVE, 64, 64, 32, TC_MIN_CTAS_LEAN>;
  if (w == 128 && h == 128)
    return ONE_WAVE ? (const void*)lean_kernel<4, ONE_WAVE, 128, 128, 32, TC_MIN_CTAS_LEAN>
                    : (const void*)lean_kernel<4, ONE_WAVE, 128, 128, 32, TC_MIN_CTAS_LEAN128W>;
  switch (w / 32) {
    case 1: return (const void*)lean_kernel<1, ONE_WAVE, 0, 0, 32, TC_MIN_CTAS_LEAN>;
    case 2: return (const void*)lean_kernel<2, ONE_WAVE, 0, 0, 32, TC_MIN_CTAS_LEAN>;
    default: return (const void*)lean_kernel<4, ONE_WAVE, 0, 0, 32, TC_MIN_CTAS_LEAN>;
  }
}
const void* select_lean(int w, int h, bool one_wave) {
  return one_wave ? select_lean_t<true>(w, h) : select_lean_t<false>(w, h);
}
// envs per CTA pass of the lean kernel
int lean_per_cta(int w, bool one_wave) { return WARPS_PER_CTA * ((!one_wave && w <= 64) ? 2 : 1); }

// validates host tables and builds the packed cell words
int validate_tables(const tc_tables* t, std::vector<uint32_t>& cells,
                    std::vector<uint32_t>& solid, int& sealed) {
  if (!t) return fail(TC_E_INVALID, "tables is NULL");
  if (t->h < 1 || t->w < 1) return fail(TC_E_INVALID, "empty map");
  if (t->obs_w < 8 || t->obs_h < 8) return fail(TC_E_INVALID, "observation must be at least 8x8");
  // the lane-parallel collision scan covers a 2x2 tile box (radius 0.2 in
  // every shipped spec, tables.py:19-31)
  if (!(t->fc[FC_RADIUS] >= 0.0 && t->fc[FC_RADIUS] < 0.5))
    return fail(TC_E_INVALID, "agent radius must be in [0, 0.5)");
  if (t->obs_w > TC_MAX_OBS_W || t->obs_h > TC_MAX_OBS_H)
    return fail(TC_E_CAPACITY, "observation larger than TC_MAX_OBS_W/H");
  if (t->n_entities < 0 || t->n_entities > TC_MAX_ENTITIES)
    return fail(TC_E_CAPACITY, "too many entities");
  if (t->n_doors < 0 || t->n_doors > TC_MAX_DOORS) return fail(TC_E_CAPACITY, "too many doors");
  if (t->n_spawns < 1) return fail(TC_E_INVALID, "map has no spawn candidates");
  if (t->n_pal < 1 || t->n_pal > 256) return fail(TC_E_INVALID, "palette size must be 1..256");
  const int cells_n = t->h * t->w;
  cells.assign(cells_n, 0);
  solid.assign(cells_n, 0);
  for (int k = 0; k < cells_n; k++) {
    const uint32_t tag = t->kind[k];
    uint32_t idx = 0;
    if (tag == C_WALL) {
      if (t->wcol[k] >= t->n_pal) return fail(TC_E_INVALID, "wall colour outside the palette");
      idx = t->wcol[k];
    } else if (tag == C_DOOR) {
      const int di = t->didx[k];
      if (di < 0 || di >= t->n_doors) return fail(TC_E_INVALID, "door cell without a door record");
      idx = (uint32_t)di;
    } else if (tag != C_FLOOR) {
      return fail(TC_E_INVALID, "cell tag must be 0 (floor), 1 (wall) or 2 (door)");
    }
    uint32_t eat = 0;
    const int ei = t->eat ? t->eat[k] : -1;
    if (ei >= 0) {
      if (ei >= t->n_entities) return fail(TC_E_INVALID, "eat[] entity index out of range");
      eat = (uint32_t)ei + 1;
    }
    cells[k] = idx | (tag << CELL_TAG_SHIFT) | (eat << CELL_EAT_SHIFT);
    solid[k] = tag == C_WALL ? 0xffffffffu : tag == C_DOOR ? (1u << idx) : 0u;
  }
  sealed = 1;
  for (int y = 0; y < t->h; y++)
    for (int x = 0; x < t->w; x++)
      if ((y == 0 || y == t->h - 1 || x == 0 || x == t->w - 1) && t->kind[y * t->w + x] != C_WALL)
        sealed = 0;
  for (int d = 0; d < t->n_doors; d++)
    if (t->dcol[d] > 2) return fail(TC_E_INVALID, "door colour must be 0..2");
  for (int e = 0; e < t->n_entities; e++) {
    if (t->ekind[e] > 2) return fail(TC_E_INVALID, "entity kind must be 0..2");
    if (t->ekind[e] == K_KEY && t->ecol[e] > 2) return fail(TC_E_INVALID, "key colour must be 0..2");
  }
  for (int g = 0; g < t->n_goals; g++)
    if (t->goal_ent[g] < 0 || t->goal_ent[g] >= t->n_entities)
      return fail(TC_E_INVALID, "goal_ent index out of range");
  return TC_OK;
}

struct BlobBuilder {
  std::vector<uint8_t> bytes;
  size_t add(const void* p, size_t n) {
    const size_t off = (bytes.size() + 15) & ~(size_t)15;
    bytes.resize(off + (n ? n : 16), 0);
    if (n) memcpy(bytes.data() + off, p, n);
    return off;
  }
};

int device_sm_count() {
  static int sms = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  });
  return sms;
}

// dynamic shared memory limit of a kernel = the opt-in maximum minus its
// static shared memory (the staging mbarrier)
int raise_smem(const void* fn, int optin) {
  cudaFuncAttributes fa;
  TC_CUDA(cudaFuncGetAttributes(&fa, fn));
  TC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               optin - (int)fa.sharedSizeBytes));
  return TC_OK;
}
#define TC_TRY_RC(x)              \
  do {                            \
    const int _rc = (x);          \
    if (_rc != TC_OK) return _rc; \
  } while (0)

int launch_geometry(tc_spec* s) {
  SpecDev& d = s->dev;
  const int row_bytes = d.obs_w * 3;
  d.quads = (d.obs_w % 4) == 0;
  d.bulk = (row_bytes % 16) == 0;
  d.mirror = (d.obs_h % 2 == 0 && d.obs_h <= 254 && d.obs_w % 16 == 0 && d.bulk) ? 1 : 0;
  d.mir_rpi = (d.obs_w / 16) >= 32 ? 1 : 32 / (d.obs_w / 16 > 0 ? d.obs_w / 16 : 1);
  d.mir_rpi16 = (d.obs_w / 16) >= 16 ? 1 : 16 / (d.obs_w / 16 > 0 ? d.obs_w / 16 : 1);
  const char* bb = getenv("TILECAST_BAND_BYTES");
  const int band_target = bb ? atoi(bb) : (d.mirror ? BAND_BYTES_TARGET / 2 : BAND_BYTES_TARGET);
  int rows = band_target / row_bytes;
  if (rows < 1) rows = 1;
  if (rows > d.obs_h) rows = d.obs_h;
  d.band_rows = rows;
  d.band_stride = align16(rows * row_bytes);
  // lanes per env: two envs per warp (16 lanes each) for obs_w <= 64, where
  // 16 lanes x 4 columns still cover a row (fits every env of a 4096-env
  // batch on the GPU at once); TILECAST_GROUP overrides (experiments)
  const char* gr = getenv("TILECAST_GROUP");
  d.group = gr ? atoi(gr) : (d.obs_w <= 64 ? 16 : 32);
  if (d.group != 16 || d.obs_w > 64) d.group = 32;
  // frame store path: 0 = staged bands + TMA bulk stores, 1 = 16-byte stores
  // straight from registers (no staging smem -> more resident envs), 2 =
  // staged bands + coalesced LDS/STG, 3 = 1 with the per-column lane layout.
  // Measured best: 1 whenever the lane-contiguous layout applies ((W/16) | G)
  // or with 16-lane groups, else 0; TILECAST_DIRECT overrides.
  const bool contig_ok = d.mirror && d.group % (d.obs_w / 16) == 0;
  const char* dr = getenv("TILECAST_DIRECT");
  d.direct = d.mirror ? (dr ? atoi(dr) : ((d.group == 16 || contig_ok) ? 1 : 0)) : 0;
  d.contig = d.direct == 1 && contig_ok;
  if (d.direct == 3) d.direct = 1;
  const char* np = getenv("TILECAST_NPAIRS");
  d.npairs = np ? atoi(np) : 2;
  if (d.npairs < 2) d.npairs = 2;
  if (d.npairs > 4) d.npairs = 4;
  d.warp_smem = warp_smem_layout(d, d.direct == 1 ? 0 : (d.mirror ? 2 * d.npairs : 2));
  d.smem_map = (d.h * d.w <= SMEM_MAP_MAX_CELLS) ? 1 : 0;
  d.smem_u8 = (!d.smem_map && s->code8_bytes <= SMEM_U8_MAX_BYTES) ? 1 : 0;
  d.stage_bytes = d.smem_map ? s->map_bytes : (d.smem_u8 ? s->code8_bytes : s->tab_bytes);
  const size_t map_bytes = (size_t)map_smem_bytes(d);
  // + the per-CTA scratch of the step kernel (actions / rewards / dones)
  s->smem_bytes = map_bytes + (size_t)WARPS_PER_CTA * (32 / d.group) * d.warp_smem + CTA_SCRATCH;
  s->nc = pick_nc(d.obs_w, d.group);
  const void* fns[4] = {select_batch(s->nc, d.group), select_rollout(s->nc, d.group),
                        select_batch(s->nc, d.group, true),
                        select_batch(s->nc, d.group, true, true)};
  // the attribute is per function, shared by every spec: raise it to the
  // device's opt-in maximum once instead of per spec (occupancy follows the
  // smem each launch actually asks for)
  int dev = 0, optin = 0;
  TC_CUDA(cudaGetDevice(&dev));
  TC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (s->smem_bytes + 64 > (size_t)optin)
    return fail(TC_E_CAPACITY, "per-CTA shared memory exceeds the device limit");
  for (const void* fn : fns)
    TC_TRY_RC(raise_smem(fn, optin));
  int per_sm = 0;
  TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[0], WARPS_PER_CTA * 32,
                                                        s->smem_bytes));
  if (per_sm < 1) return fail(TC_E_CAPACITY, "kernel does not fit on an SM");
  s->max_ctas = per_sm * device_sm_count();
  TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[2], WARPS_PER_CTA * 32,
                                                        s->smem_bytes));
  s->max_ctas_w = per_sm < 1 ? s->max_ctas : per_sm * device_sm_count();
  // lean kernel: a sealed map in shared memory, < 32 doors, the mirrored
  // lane-contiguous compose for full-warp groups (W / 16 divides 32, W <= 128)
  const char* ln = getenv("TILECAST_LEAN");
  d.lean = (ln ? atoi(ln) != 0 : true) && d.sealed && d.w >= 2 &&
           ((d.smem_map && d.n_doors < 32) || (d.smem_u8 && d.n_doors <= 30)) &&
           d.mirror && d.contig && d.direct == 1 && d.obs_w >= 32 && d.obs_w <= 128 &&
           32 % (d.obs_w / 16) == 0;
  if (d.lean) {
    const void* lf = select_lean(d.obs_w, d.obs_h, true);
    TC_TRY_RC(raise_smem(lf, optin));
    TC_TRY_RC(raise_smem(select_lean(d.obs_w, d.obs_h, false), optin));
    s->lean_smem = map_bytes + (size_t)WARPS_PER_CTA * d.warp_smem + CTA_SCRATCH;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lf, WARPS_PER_CTA * 32,
                                                          s->lean_smem));
    if (per_sm < 1) d.lean = 0;
    s->lean_ctas = per_sm * device_sm_count();
    s->lean16_ctas = 0;
    const char* l16 = getenv("TILECAST_LEAN16");
    if (d.lean && (l16 ? atoi(l16) != 0 : true)) {
      // multi-wave lean kernel: two envs per warp for W <= 64, one per warp
      // (with tickets) for W = 128
      const void* mf = select_lean(d.obs_w, d.obs_h, false);
      s->lean16_smem = map_bytes +
                       (size_t)lean_per_cta(d.obs_w, false) * d.warp_smem + CTA_SCRATCH;
      TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mf, WARPS_PER_CTA * 32,
                                                            s->lean16_smem));
      s->lean16_ctas = per_sm * device_sm_count();
    }
  }
  return TC_OK;
}

StateDev to_dev(const tc_state* s) {
  StateDev d;
  d.px = s->px; d.py = s->py; d.dx = s->dx; d.dy = s->dy; d.health = s->health;
  d.inv = s->inv;
  d.t = reinterpret_cast<long long*>(s->t);
  d.rkey = reinterpret_cast<unsigned long long*>(s->rkey);
  d.rctr = reinterpret_cast<unsigned long long*>(s->rctr);
  d.done = s->done; d.agoal = s->agoal; d.dopen = s->dopen; d.ealive = s->ealive;
  return d;
}

OutDev to_dev(const tc_out* o) {
  OutDev d;
  d.frames = o->frames; d.zbuf = o->zbuf; d.rewards = o->rewards; d.dones = o->dones;
  d.truncs = o->truncs; d.events = o->events; d.statuses = o->statuses;
  d.rayinfo = o->rayinfo;
  d.spritevis = reinterpret_cast<unsigned long long*>(o->spritevis);
  d.res_host = nullptr;
  d.flag_host = nullptr;
  return d;
}

// the step kernel for n envs: the wide variant when one wave of the
// latency variant cannot hold them all
bool use_wide(const tc_spec* s, int64_t n) {
  const int per_cta = WARPS_PER_CTA * (32 / s->dev.group);
  return n > (int64_t)s->max_ctas * per_cta;
}

// which kernel steps n envs: 1 = lean, one env per warp, one wave; 2 = lean
// multi-wave (env tickets); 0 = batch_kernel. (A batch past one wave of the
// lean kernel that still fits one wave of the 128-register batch_kernel runs
// there: measured +7 % on the 160x128-tile map; TILECAST_LEAN2_ANY=1 sends it
// to the multi-wave lean kernel instead, for experiments.)
int lean_kind(const tc_spec* s, int64_t n) {
  const SpecDev& d = s->dev;
  if (!d.lean) return 0;
  static const int force = [] {
    const char* e = getenv("TILECAST_LEAN_KIND");
    return e ? atoi(e) : -1;
  }();
  if (force == 2 && s->lean16_ctas > 0) return 2;
  if (n <= (int64_t)s->lean_ctas * WARPS_PER_CTA) return 1;
  static const bool any_n = [] {
    const char* e = getenv("TILECAST_LEAN2_ANY");
    return e && atoi(e) != 0;
  }();
  return (s->lean16_ctas > 0 && (use_wide(s, n) || any_n)) ? 2 : 0;
}

int grid_for(const tc_spec* s, int64_t n, bool wide = false) {
  const int per_cta = WARPS_PER_CTA * (32 / s->dev.group);  // envs per CTA pass
  const int64_t want = (n + per_cta - 1) / per_cta;
  const int max_ctas = wide ? s->max_ctas_w : s->max_ctas;
  if (want >= max_ctas) return max_ctas;
  // a partial wave: round the grid up to whole rounds of SMs (envs are
  // interleaved over CTAs, so every SM gets the same number of envs +-1)
  const int sms = device_sm_count();
  const int64_t g = (want + sms - 1) / sms * sms;
  return (int)(g < max_ctas ? g : max_ctas);
}

}  // namespace

extern "C" {

int tc_abi_version(void) { return TC_ABI_VERSION; }

// perf-experiment hook: per-env phase timestamps (TC_TRACE builds only)
int tc_debug_trace_cta(void* dev_buf) {
#if TC_TRACE
  TC_CUDA(cudaMemcpyToSymbol(g_trace_cta, &dev_buf, sizeof(void*)));
  static unsigned int zeros[16384] = {0};
  TC_CUDA(cudaMemcpyToSymbol(g_cta_gen, zeros, sizeof zeros));
  return TC_OK;
#else
  (void)dev_buf;
  return fail(TC_E_INVALID, "library built without TC_TRACE");
#endif
}
int tc_debug_trace(void* dev_buf) {
#if TC_TRACE
  TC_CUDA(cudaMemcpyToSymbol(g_trace, &dev_buf, sizeof(void*)));
  return TC_OK;
#else
  (void)dev_buf;
  return fail(TC_E_INVALID, "library built without TC_TRACE");
#endif
}
const char* tc_last_error(void) { return g_err.c_str(); }
const char* tc_build_info(void) {
  return "tilecast_b200 sm_100a; fp64 --fmad=false; 4 warps/CTA; spec tables + map staged "
         "per CTA by one TMA bulk copy (cp.async.bulk + mbarrier); one-wave steps: lean "
         "one-env-per-warp kernel; multi-wave: two envs per warp, ticket scheduler; frames "
         "by lane-contiguous 16-byte streaming stores (mirrored SWAR compose)";
}

const char* tc_step_kernel(const tc_spec* s, int64_t n) {
  if (!s) return "none";
  const SpecDev& d = s->dev;
  const int lk = lean_kind(s, n);
  if (lk == 1) return "lean_kernel (one env per warp, one wave, 72 registers)";
  if (lk == 2)
    return d.obs_w <= 64 ? "lean_kernel (two envs per warp, multi-wave env tickets, 96 registers)"
                         : "lean_kernel (one env per warp, multi-wave env tickets, 72 registers)";
  if (use_wide(s, n))
    return d.group == 16 ? "batch_kernel (two envs per warp, multi-wave, 96 registers)"
                         : "batch_kernel (one env per warp, multi-wave)";
  return d.group == 16 ? "batch_kernel (two envs per warp, one wave, 128 registers)"
                       : "batch_kernel (one env per warp, one wave)";
}

int tc_spec_create(const tc_tables* t, tc_spec** out) {
  if (!out) return fail(TC_E_INVALID, "out is NULL");
  *out = nullptr;
  std::vector<uint32_t> cells, solid;
  int sealed = 0;
  int rc = validate_tables(t, cells, solid, sealed);
  if (rc != TC_OK) return rc;

  std::vector<uint32_t> pal(t->n_pal), doorrgb(t->n_doors);
  for (int p = 0; p < t->n_pal; p++) pal[p] = pack_rgb(t->pal + 3 * p);
  for (int d = 0; d < t->n_doors; d++) doorrgb[d] = pack_rgb(t->door_rgb + 3 * t->dcol[d]);

  // blob: the small read-only tables first (always staged into shared
  // memory), then the packed cells and the guarded stop codes (staged when
  // the map fits, SpecDev::stage_bytes)
  BlobBuilder b;
  const size_t o_coef = b.add(t->coef, t->obs_w * 8);
  const size_t o_pal = b.add(pal.data(), pal.size() * 4);
  const size_t o_door = b.add(doorrgb.data(), doorrgb.size() * 4);
  const size_t o_epx = b.add(t->epx, t->n_entities * 8);
  const size_t o_epy = b.add(t->epy, t->n_entities * 8);
  const size_t o_spx = b.add(t->spx, t->n_spawns * 8);
  const size_t o_spy = b.add(t->spy, t->n_spawns * 8);
  const size_t o_goal = b.add(t->goal_ent, t->n_goals * 4);
  const size_t o_dcol = b.add(t->dcol, t->n_doors);
  const size_t o_dlock = b.add(t->dlock, t->n_doors);
  const size_t o_ekind = b.add(t->ekind, t->n_entities);
  const size_t o_ecol = b.add(t->ecol, t->n_entities);
  const size_t tab_end = (b.bytes.size() + 15) & ~(size_t)15;
  // u8 stop codes for large maps (0 floor, d + 1 door d, 31 wall), with the
  // same w+1-cell wall guards as the u32 codes
  std::vector<uint8_t> code8(cells.size() + 2 * (size_t)(t->w + 1), 31);
  for (size_t k = 0; k < cells.size(); k++) {
    const uint32_t tag = (cells[k] >> CELL_TAG_SHIFT) & 3u;
    code8[(size_t)(t->w + 1) + k] =
        tag == C_WALL ? 31 : tag == C_DOOR ? (uint8_t)((cells[k] & 31u) + 1) : 0;
  }
  const size_t o_code8 = b.add(code8.data(), code8.size()) + (size_t)(t->w + 1);
  const size_t code8_end = (b.bytes.size() + 15) & ~(size_t)15;
  const size_t o_cell = b.add(cells.data(), cells.size() * 4);
  // stop codes with a wall guard of w+1 cells on each side (speculative DDA)
  std::vector<uint32_t> gsolid(solid.size() + 2 * (size_t)(t->w + 1), 0xffffffffu);
  std::copy(solid.begin(), solid.end(), gsolid.begin() + (t->w + 1));
  const size_t o_solid = b.add(gsolid.data(), gsolid.size() * 4) + (size_t)(t->w + 1) * 4;
  const size_t map_end = (b.bytes.size() + 15) & ~(size_t)15;
  b.bytes.resize(map_end, 0);

  tc_spec* s = new tc_spec();
  cudaError_t e = cudaMalloc(&s->blob, b.bytes.size());
  if (e != cudaSuccess) { delete s; return cuda_fail(e, "cudaMalloc(spec)"); }
  e = cudaMemcpy(s->blob, b.bytes.data(), b.bytes.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(s->blob); delete s; return cuda_fail(e, "cudaMemcpy(spec)"); }
  uint8_t* base = static_cast<uint8_t*>(s->blob);
  SpecDev& d = s->dev;
  d.cell = (const uint32_t*)(base + o_cell);
  d.solid = (const uint32_t*)(base + o_solid);
  d.sealed = sealed;
  d.pal = (const uint32_t*)(base + o_pal);
  d.doorrgb = (const uint32_t*)(base + o_door);
  d.dcol = base + o_dcol;
  d.dlock = base + o_dlock;
  d.epx = (const double*)(base + o_epx);
  d.epy = (const double*)(base + o_epy);
  d.ekind = base + o_ekind;
  d.ecol = base + o_ecol;
  d.spx = (const double*)(base + o_spx);
  d.spy = (const double*)(base + o_spy);
  d.goal_ent = (const int32_t*)(base + o_goal);
  d.coef = (const double*)(base + o_coef);
  d.blob = base;
  d.b_coef = (int)o_coef; d.b_pal = (int)o_pal; d.b_door = (int)o_door;
  d.b_epx = (int)o_epx; d.b_epy = (int)o_epy; d.b_spx = (int)o_spx; d.b_spy = (int)o_spy;
  d.b_goal = (int)o_goal; d.b_dcol = (int)o_dcol; d.b_dlock = (int)o_dlock;
  d.b_ekind = (int)o_ekind; d.b_ecol = (int)o_ecol; d.b_cell = (int)o_cell;
  d.b_solid = (int)o_solid;
  d.b_code8 = (int)o_code8;
  s->tab_bytes = (int)tab_end;
  s->code8_bytes = (int)code8_end;
  s->map_bytes = (int)map_end;
  for (int k = 0; k < FC_COUNT; k++) d.fc[k] = t->fc[k];
  for (int k = 0; k < 8; k++) d.dirs[k] = t->dirs[k];
  d.max_steps = t->ic[0];
  d.goal_mode = (int)t->ic[1];
  d.use_health = (int)t->ic[2];
  d.ceil_rgb = pack_rgb(t->ceil_rgb);
  d.floor_rgb = pack_rgb(t->floor_rgb);
  d.goal_rgb = pack_rgb(t->goal_rgb);
  d.med_box = pack_rgb(t->med_box);
  d.med_cross = pack_rgb(t->med_cross);
  for (int k = 0; k < 3; k++) d.key_rgb[k] = pack_rgb(t->key_rgb + 3 * k);
  d.legal_mask = 0;
  for (int a = 0; a < A_COUNT; a++)
    if (t->legal == nullptr || t->legal[a]) d.legal_mask |= 1u << a;
  d.h = t->h; d.w = t->w; d.n_doors = t->n_doors; d.n_ent = t->n_entities;
  d.n_spawns = t->n_spawns; d.n_goals = t->n_goals; d.n_pal = t->n_pal;
  d.obs_h = t->obs_h; d.obs_w = t->obs_w;
  rc = launch_geometry(s);
  if (rc != TC_OK) {
    cudaFree(s->blob);
    delete s;
    return rc;
  }
  *out = s;
  return TC_OK;
}

int tc_spec_destroy(tc_spec* s) {
  if (!s) return TC_OK;
  cudaError_t e = cudaFree(s->blob);
  delete s;
  return e == cudaSuccess ? TC_OK : cuda_fail(e, "cudaFree(spec)");
}

// ---------------------------------------------- pipelined host step state
// tc_batch_step_pipelined launches step s+1 right after releasing step s,
// before the host knows step s+1's actions: the launch stages its tables,
// waits for step s's grid, then waits at a gate (LeanSched::gate_*). The
// next call with the matching arguments releases it with one host store
// instead of launching, so the launch call, the launch latency and the
// previous step's frame rendering are off the host's critical path. At most
// one such launch is pending per process; any other library launch cancels
// it first, and a watchdog thread cancels it if no call releases it within
// the timeout (TILECAST_PIPE_TIMEOUT_US, default 1000), so other work on the
// stream or the GPU is never held longer than that. After a timeout the
// pipeline backs off (exponentially, up to 4096 steps without speculation).
namespace {
struct PipeKey {
  const tc_spec* spec;
  tc_state in, out;  // pointer-only structs: compared bytewise
  tc_out ob;
  int64_t n;
  int32_t auto_reset, validate;
  tc_counters* counters;
  const int64_t* acts;
  uint8_t* res;
  int32_t* flag;
  void* stream;
};
PipeKey pipe_key(const tc_mapped_call& m, const tc_state* in, const tc_state* out,
                 const tc_out* ob) {
  PipeKey k;
  memset(&k, 0, sizeof(k));
  k.spec = m.spec; k.in = *in; k.out = *out; k.ob = *ob; k.n = m.n;
  k.auto_reset = m.auto_reset; k.validate = m.validate; k.counters = m.counters_dev;
  k.acts = m.actions_host; k.res = m.results_host; k.flag = m.flag_host; k.stream = m.stream;
  return k;
}
bool same_key(const PipeKey& a, const PipeKey& b) { return memcmp(&a, &b, sizeof(PipeKey)) == 0; }

struct Pipe {
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<bool> pending{false};
  PipeKey key;
  unsigned int q = 0;  // last gate number issued (host words hold the last go / cancel)
  double t_launch = 0.0, timeout_us = 1000.0;
  int skip = 0, backoff = 0;
  bool watchdog = false, idle = false;
  bool resident = false;  // the pending gate belongs to a resident loop kernel
  unsigned long long released = 0, cancelled = 0, timeouts = 0;
};
Pipe& pipe() {  // never destroyed: the watchdog thread may outlive static destruction
  static Pipe* p = [] {
    Pipe* x = new Pipe();
    const char* e = getenv("TILECAST_PIPE_TIMEOUT_US");
    if (e && atof(e) > 0) x->timeout_us = atof(e);
    return x;
  }();
  return *p;
}
// the cancel store (mu held): the gated kernel exits without any effect
void pipe_cancel_locked(Pipe& P, bool timeout) {
  if (!P.pending.load(std::memory_order_relaxed)) return;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  *reinterpret_cast<volatile uint32_t*>(P.key.flag + 5) = P.q;
  P.pending.store(false, std::memory_order_release);
  P.resident = false;
  P.cancelled++;
  if (timeout) {
    P.timeouts++;
    P.backoff = P.backoff ? std::min(2 * P.backoff, 4096) : 8;
    P.skip = P.backoff;
  }
}
void pipe_watchdog() {
  Pipe& P = pipe();
  std::unique_lock<std::mutex> lk(P.mu);
  for (;;) {
    if (!P.pending.load(std::memory_order_relaxed)) {
      P.idle = true;
      P.cv.wait(lk);
      P.idle = false;
      continue;
    }
    const double left = P.t_launch + P.timeout_us - host_us();
    if (left <= 0.0) {
      pipe_cancel_locked(P, true);
      continue;
    }
    P.cv.wait_for(lk, std::chrono::microseconds((long long)left + 1));
  }
}
}  // namespace

// TILECAST_PIPE_TRACE=1: the resident loop records its timeline (rstamp)
unsigned long long* g_pipe_trace = nullptr;
int g_pipe_trace_grid = 0;
static unsigned long long* pipe_trace_buf(int grid, void* stream) {
  static const bool on = [] {
    const char* e = getenv("TILECAST_PIPE_TRACE");
    return e && atoi(e) != 0;
  }();
  if (!on) return nullptr;
  if (g_pipe_trace_grid < grid) {
    if (g_pipe_trace) cudaFree(g_pipe_trace);
    g_pipe_trace = nullptr;
    if (cudaMalloc(&g_pipe_trace, (size_t)64 * 3 * grid * 8) != cudaSuccess) return nullptr;
    g_pipe_trace_grid = grid;
  }
  cudaMemsetAsync(g_pipe_trace, 0, (size_t)64 * 3 * grid * 8, (cudaStream_t)stream);
  return g_pipe_trace;
}

// TILECAST_PIPE_RESIDENT=0: one gated launch per pipelined step always
const bool g_pipe_resident = [] {
  const char* e = getenv("TILECAST_PIPE_RESIDENT");
  return e ? atoi(e) != 0 : true;
}();

static void pipe_cancel_if_pending() {
  Pipe& P = pipe();
  if (!P.pending.load(std::memory_order_acquire)) return;
  std::lock_guard<std::mutex> lk(P.mu);
  pipe_cancel_locked(P, false);
}

struct ChainArgs {
  unsigned int* flags;
  unsigned int* tickets;  // multi-wave: this launch's zeroed ticket counter
  unsigned int epoch, need_ready, need_done;
  unsigned int done_off;  // one wave: this ring slot's row of done epochs
};

struct GateArgs {  // a pipelined (gated) launch, LeanSched::gate_*
  unsigned int* dev;
  const unsigned long long* host;
  unsigned int q;
  const tc_out* out2;  // non-NULL: the resident host-step loop (RES kernel)
};

// the resident host-step loop kernel for a one-wave batch of this spec, or
// NULL (then the pipeline launches one gated kernel per step)
static const void* select_resident(const tc_spec* s) {
  if (s->dev.obs_w == 64 && s->dev.obs_h == 64)
    return (const void*)lean_kernel<2, true, 64, 64, 32, TC_MIN_CTAS_LEAN, true>;
  return nullptr;
}

static int launch_batch_kernel(const tc_spec* s, const tc_state* state, const tc_state* state_out,
                               const int64_t* actions_dev, const tc_out* out, int64_t n,
                               int32_t mode, int32_t auto_reset, int32_t validate,
                               tc_counters* counters_dev, void* stream,
                               uint8_t* res_host = nullptr, int32_t* flag_host = nullptr,
                               const ChainArgs* chain = nullptr, const GateArgs* gate = nullptr) {
  if (!s || !state || !out) return fail(TC_E_INVALID, "NULL spec/state/out");
  // any other launch first cancels a pipelined step still waiting for its
  // actions (it would hold every SM until the watchdog cancelled it)
  if (!gate) pipe_cancel_if_pending();
  if (n < 0) return fail(TC_E_INVALID, "n must be >= 0");
  if (mode != TC_MODE_RESET && mode != TC_MODE_STEP && mode != MODE_RENDER)
    return fail(TC_E_INVALID, "mode must be 0 (reset) or 1 (step)");
  if (mode == TC_MODE_STEP && (!actions_dev || !out->rewards || !out->dones || !out->truncs ||
                               !out->events))
    return fail(TC_E_INVALID, "step mode needs actions, rewards, dones, truncs, events");
  if (!out->frames || !out->statuses) return fail(TC_E_INVALID, "frames and statuses are required");
  if (n == 0) return TC_OK;
  const SpecDev& d = s->dev;
  if (d.bulk && (reinterpret_cast<uintptr_t>(out->frames) & 15u))
    return fail(TC_E_INVALID, "frames must be 16-byte aligned");
  StateDev sd = to_dev(state);
  StateDev so = to_dev(state_out ? state_out : state);
  OutDev od = to_dev(out);
  od.res_host = res_host;
  od.flag_host = flag_host;
  const bool taps = out->zbuf || out->rayinfo || out->spritevis;
  // the lean kernels: one env per warp for batches that fit one wave of it
  // (latency-bound), two envs per warp over a full wave with env tickets for
  // larger batches (issue-bound: the pair shares its convergent code)
  const int lk = lean_kind(s, n);
  const bool lean1 = lk == 1, lean2 = lk == 2;
  if (mode == TC_MODE_STEP && !taps && (lean1 || lean2)) {
    const int per_cta = lean_per_cta(d.obs_w, lean1);
    const int64_t want = (n + per_cta - 1) / per_cta;
    int grid = lean1 ? s->lean_ctas : s->lean16_ctas;
    if (want < grid) {
      const int sms = device_sm_count();
      const int64_t g = (want + sms - 1) / sms * sms;
      grid = (int)(g < grid ? g : grid);
    }
    LeanSched ls;
    ls.n = n;
    ls.stride = (long long)grid * per_cta;
    const bool one_wave = lean1;
    ls.epc = one_wave ? (int)((n + grid - 1) / grid) : 0;
    ls.early = res_host != nullptr;
    ls.ctas = one_wave ? (int)((n + ls.epc - 1) / ls.epc) : 0;
    ls.flags = ls.tickets = nullptr;
    ls.epoch = ls.need_ready = ls.need_done = 0;
    ls.done_off = 0;
    ls.gate_dev = gate ? gate->dev : nullptr;
    ls.gate_host = gate ? gate->host : nullptr;
    ls.gate_q = gate ? gate->q : 0u;
    ls.out2 = (gate && gate->out2) ? to_dev(gate->out2) : od;
    ls.rtrace = (gate && gate->out2) ? pipe_trace_buf(grid, stream) : nullptr;
    if (gate && gate->out2) {
      ls.out2.res_host = res_host;
      ls.out2.flag_host = flag_host;
    }
    if (chain && !res_host) {
      ls.flags = chain->flags;
      ls.tickets = chain->tickets;
      ls.epoch = chain->epoch;
      ls.need_ready = chain->need_ready;
      ls.need_done = one_wave ? chain->need_done : 0u;
      ls.done_off = chain->done_off;
    }
    const long long* acts = reinterpret_cast<const long long*>(actions_dev);
    int ar = auto_reset, va = validate;
    SpecDev spec = d;
    void* args[] = {&spec, &sd, &so, &acts, &od, &ls, &ar, &va, &counters_dev};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(WARPS_PER_CTA * 32);
    cfg.dynamicSmemBytes = lean1 ? s->lean_smem : s->lean16_smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const void* fn = (gate && gate->out2) ? select_resident(s) : select_lean(d.obs_w, d.obs_h, one_wave);
    if (!fn) return fail(TC_E_INVALID, "no resident kernel for this frame shape");
    TC_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    return TC_OK;
  }
  const bool wide = taps || use_wide(s, n);
  const int grid = grid_for(s, n, wide);
  const long long nn = n;
  const long long* acts = reinterpret_cast<const long long*>(actions_dev);
  int m = mode, ar = auto_reset, va = validate;
  SpecDev spec = d;
  void* args[] = {&spec, &sd, &so, &acts, &od, (void*)&nn, &m, &ar, &va, &counters_dev};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(WARPS_PER_CTA * 32);
  cfg.dynamicSmemBytes = s->smem_bytes;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TC_CUDA(cudaLaunchKernelExC(&cfg, select_batch(s->nc, s->dev.group, wide, taps), args));
  return TC_OK;
}

int tc_batch_kernel(const tc_spec* s, const tc_state* state, const int64_t* actions_dev,
                    const tc_out* out, int64_t n, int32_t mode, int32_t auto_reset,
                    int32_t validate, tc_counters* counters_dev, void* stream) {
  return launch_batch_kernel(s, state, nullptr, actions_dev, out, n, mode, auto_reset, validate,
                             counters_dev, stream);
}

int tc_batch_steps(const tc_spec* s, const tc_state* state_a, const tc_state* state_b,
                   const int64_t* actions_dev, const tc_out* outs, int32_t ring, int64_t n,
                   int32_t k_steps, int32_t auto_reset, int32_t validate,
                   tc_counters* counters_dev, uint32_t* flags_dev, uint32_t epoch0,
                   void* stream) {
  if (!state_a || !state_b || !actions_dev || !outs || !flags_dev)
    return fail(TC_E_INVALID, "NULL state / actions / outs / flags");
  if (ring < 1 || k_steps < 0 || n < 0) return fail(TC_E_INVALID, "bad ring / k / n");
  if (k_steps == 0 || n == 0) return TC_OK;
  // chaining needs a lean kernel on every launch (one wave: its fixed CTA ->
  // env mapping; multi-wave: env tickets with per-env epochs); other
  // batches, and rings with debug taps (batch_kernel), get K ordinary launches
  bool taps = false;
  for (int r = 0; r < ring; r++)
    taps = taps || outs[r].zbuf || outs[r].rayinfo || outs[r].spritevis;
  const int lk = s ? lean_kind(s, n) : 0;
  const bool lean1 = lk == 1, lean2 = lk == 2;
  // (multi-wave: only while the batch is a few waves deep -- chaining hides
  // the tail of each launch, but costs every env a device-scope fence after
  // its frame; at 2^20 envs, ~180 waves, the tail is < 1 % and the fences
  // cost ~20 %)
  const int64_t slots = lean2 ? (int64_t)s->lean16_ctas * lean_per_cta(s->dev.obs_w, false) : 0;
  // (one wave: a row of CHAIN_DONE_ROW done epochs per ring slot)
  const bool chain_ok = !taps && ((lean1 && ring <= CHAIN_MAX_RING && s->lean_ctas <= CHAIN_DONE_ROW) ||
                                  (lean2 && n <= CHAIN_MAX_WAVES * slots));
  // multi-wave: launch k draws env tickets from flags[n + k % n], zeroed
  // (stream-ordered after every earlier kernel) before each run of n launches
  uint32_t* const tickets = flags_dev + n;
  for (int k = 0; k < k_steps; k++) {
    const tc_state* in = (k & 1) ? state_b : state_a;
    const tc_state* outst = (k & 1) ? state_a : state_b;
    ChainArgs ca;
    ca.flags = flags_dev;
    ca.epoch = epoch0 + (uint32_t)k;
    // the first launch waits for the whole previous grid (whatever it was);
    // each later one for its env's state from step k - 1 and, once the ring
    // wraps, for the step that last wrote the output block it overwrites
    ca.need_ready = k == 0 ? 0u : ca.epoch - 1u;
    ca.need_done = (k >= ring) ? ca.epoch - (uint32_t)ring : 0u;
    ca.done_off = (unsigned int)(n + (int64_t)(k % ring) * CHAIN_DONE_ROW);
    ca.tickets = tickets + (k % n);
    if (chain_ok && lean2 && k % n == 0) {
      const int64_t run = std::min<int64_t>(n, (int64_t)k_steps - k);
      TC_CUDA(cudaMemsetAsync(tickets, 0, (size_t)run * 4, (cudaStream_t)stream));
      ca.need_ready = 0u;  // the memset already ordered this launch after the last
    }
    const int rc = launch_batch_kernel(s, in, outst, actions_dev + (size_t)k * (size_t)n,
                                       &outs[k % ring], n, TC_MODE_STEP, auto_reset, validate,
                                       counters_dev, stream, nullptr, nullptr,
                                       chain_ok ? &ca : nullptr);
    if (rc != TC_OK) return rc;
  }
  return TC_OK;
}

int tc_batch_step_into(const tc_spec* s, const tc_state* state_in, const tc_state* state_out,
                       const int64_t* actions_dev, const tc_out* out, int64_t n,
                       int32_t auto_reset, int32_t validate, tc_counters* counters_dev,
                       void* stream) {
  if (!state_out) return fail(TC_E_INVALID, "state_out is NULL");
  return launch_batch_kernel(s, state_in, state_out, actions_dev, out, n, TC_MODE_STEP,
                             auto_reset, validate, counters_dev, stream);
}

}  // extern "C"

namespace {
const void* select_multi(int nc, int group) {
  if (group == 16) {
    switch (nc) {
      case 1: return (const void*)multi_kernel<1, 16, TC_MIN_CTAS16_WIDE>;
      case 2: return (const void*)multi_kernel<2, 16, TC_MIN_CTAS16_WIDE>;
      case 3: return (const void*)multi_kernel<3, 16, TC_MIN_CTAS16_WIDE>;
      default: return (const void*)multi_kernel<4, 16, TC_MIN_CTAS16_WIDE>;
    }
  }
  switch (nc) {
    case 2: return (const void*)multi_kernel<2, 32, TC_MIN_CTAS>;
    case 4: return (const void*)multi_kernel<4, 32, TC_MIN_CTAS>;
    default: return nullptr;
  }
}

// one multi_kernel launch: each group gets a contiguous CTA range sized by
// its share of the envs (at least one CTA, at most one CTA per 8 / 4 envs),
// out of one wave at the largest group's shared-memory footprint
int launch_multi(const void* fn, const tc_spec* const* specs, const tc_state* states_in,
                 const tc_state* states_out, const int64_t* actions_dev, const tc_out* outs,
                 const int64_t* counts, int n_groups, int32_t auto_reset, int32_t validate,
                 tc_counters* const* counters, void* stream) {
  static thread_local MultiArgs A;
  size_t smem = 0;
  int64_t total = 0;
  for (int g = 0; g < n_groups; g++) {
    smem = std::max(smem, specs[g]->smem_bytes);
    total += counts[g];
  }
  int dev = 0, optin = 0, per_sm = 0;
  TC_CUDA(cudaGetDevice(&dev));
  TC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  static thread_local const void* raised = nullptr;
  if (raised != fn) {
    TC_TRY_RC(raise_smem(fn, optin));
    raised = fn;
  }
  TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, WARPS_PER_CTA * 32, smem));
  if (per_sm < 1) return fail(TC_E_CAPACITY, "multi-map step does not fit on an SM");
  const int wave = per_sm * device_sm_count();
  const int per_cta = WARPS_PER_CTA * (32 / specs[0]->dev.group);
  A.n_groups = n_groups;
  A.block_begin[0] = 0;
  A.ticket = counters[0];
  int64_t off = 0;
  for (int g = 0; g < n_groups; g++) {
    A.block_begin[g + 1] = A.block_begin[g] + (counts[g] + per_cta - 1) / per_cta;
    MultiGroup& m = A.g[g];
    m.spec = specs[g]->dev;
    m.st = to_dev(&states_in[g]);
    m.so = to_dev(&states_out[g]);
    m.out = to_dev(&outs[g]);
    m.out.res_host = nullptr;
    m.out.flag_host = nullptr;
    m.n = counts[g];
    m.off = off;
    m.counters = counters[g];
    off += counts[g];
    if (specs[g]->dev.bulk && (reinterpret_cast<uintptr_t>(outs[g].frames) & 15u))
      return fail(TC_E_INVALID, "frames must be 16-byte aligned");
  }
  A.total_blocks = A.block_begin[n_groups];
  // block tickets start after the grid's first blocks (block = blockIdx.x)
  const int grid = (int)std::min<int64_t>(wave, A.total_blocks);
  const long long* acts = reinterpret_cast<const long long*>(actions_dev);
  int ar = auto_reset, va = validate;
  void* args[] = {&A, &acts, &ar, &va};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(WARPS_PER_CTA * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TC_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  return TC_OK;
}
}  // namespace

extern "C" {

int tc_multi_step(const tc_spec* const* specs, const tc_state* states_in,
                  const tc_state* states_out, const int64_t* actions_dev, const tc_out* outs,
                  const int64_t* counts, int32_t n_groups, int32_t auto_reset, int32_t validate,
                  tc_counters* const* counters, void* stream) {
  pipe_cancel_if_pending();
  if (!specs || !states_in || !states_out || !actions_dev || !outs || !counts || !counters)
    return fail(TC_E_INVALID, "NULL group array");
  if (n_groups < 1) return fail(TC_E_INVALID, "n_groups must be >= 1");
  for (int g = 0; g < n_groups; g++) {
    if (!specs[g] || !counters[g]) return fail(TC_E_INVALID, "NULL spec / counters in a group");
    if (counts[g] < 1) return fail(TC_E_INVALID, "every group needs >= 1 env");
  }
  // ONE launch over all groups (multi_kernel) when they fit its group table
  // and kernel set; TILECAST_MULTI_LAUNCH=0 selects the per-group launches
  {
    const char* ml = getenv("TILECAST_MULTI_LAUNCH");
    const bool one = (ml ? atoi(ml) != 0 : true) && n_groups <= TC_MULTI_MAX && n_groups > 1;
    const void* fn = one ? select_multi(specs[0]->nc, specs[0]->dev.group) : nullptr;
    bool same = fn != nullptr;
    for (int g = 1; g < n_groups && same; g++)
      same = specs[g]->nc == specs[0]->nc && specs[g]->dev.group == specs[0]->dev.group &&
             specs[g]->dev.obs_w == specs[0]->dev.obs_w &&
             specs[g]->dev.obs_h == specs[0]->dev.obs_h;
    if (same) {
      return launch_multi(fn, specs, states_in, states_out, actions_dev, outs, counts, n_groups,
                          auto_reset, validate, counters, stream);
    }
  }
  // Groups run concurrently on side streams forked from / joined back into
  // the caller's stream, so one group's tail overlaps the others' work (each
  // group has its own counters: its env tickets are private).
  constexpr int kSide = 4;
  struct Side {
    int dev = -1;
    cudaStream_t st[kSide] = {};
    cudaEvent_t fork = nullptr, join[kSide] = {};
  };
  static thread_local Side side;
  int dev = 0;
  TC_CUDA(cudaGetDevice(&dev));
  if (side.dev != dev) {
    // one lazily created set per thread and device in use (re-created on a
    // device switch; the previous set is released)
    if (side.dev >= 0) {
      for (int k = 0; k < kSide; k++) {
        cudaStreamDestroy(side.st[k]);
        cudaEventDestroy(side.join[k]);
      }
      cudaEventDestroy(side.fork);
    }
    side.dev = -1;
    TC_CUDA(cudaEventCreateWithFlags(&side.fork, cudaEventDisableTiming));
    for (int k = 0; k < kSide; k++) {
      TC_CUDA(cudaStreamCreateWithFlags(&side.st[k], cudaStreamNonBlocking));
      TC_CUDA(cudaEventCreateWithFlags(&side.join[k], cudaEventDisableTiming));
    }
    side.dev = dev;
  }
  cudaStream_t main_st = (cudaStream_t)stream;
  const int used = n_groups < kSide ? n_groups : kSide;
  if (n_groups == 1) {
    return launch_batch_kernel(specs[0], &states_in[0], &states_out[0], actions_dev, &outs[0],
                               counts[0], TC_MODE_STEP, auto_reset, validate, counters[0], stream);
  }
  TC_CUDA(cudaEventRecord(side.fork, main_st));
  for (int k = 0; k < used; k++) TC_CUDA(cudaStreamWaitEvent(side.st[k], side.fork, 0));
  int64_t off = 0;
  for (int g = 0; g < n_groups; g++) {
    const int rc = launch_batch_kernel(specs[g], &states_in[g], &states_out[g], actions_dev + off,
                                       &outs[g], counts[g], TC_MODE_STEP, auto_reset, validate,
                                       counters[g], side.st[g % kSide]);
    if (rc != TC_OK) return rc;
    off += counts[g];
  }
  for (int k = 0; k < used; k++) {
    TC_CUDA(cudaEventRecord(side.join[k], side.st[k]));
    TC_CUDA(cudaStreamWaitEvent(main_st, side.join[k], 0));
  }
  return TC_OK;
}

int tc_batch_step_host(const tc_spec* s, const tc_state* state_in, const tc_state* state_out,
                       const int64_t* actions_host, int64_t* actions_dev, const tc_out* out,
                       int64_t n, int32_t auto_reset, int32_t validate,
                       tc_counters* counters_dev, double* rewards_host, uint8_t* dones_host,
                       void* stream) {
  if (!actions_host || !actions_dev) return fail(TC_E_INVALID, "NULL actions buffer");
  if (n <= 0) return n == 0 ? TC_OK : fail(TC_E_INVALID, "n must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  TC_CUDA(cudaMemcpyAsync(actions_dev, actions_host, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  const int rc = launch_batch_kernel(s, state_in, state_out ? state_out : state_in, actions_dev,
                                     out, n, TC_MODE_STEP, auto_reset, validate, counters_dev,
                                     stream);
  if (rc != TC_OK) return rc;
  // one copy when the host and device result buffers are both laid out as
  // [rewards f64[n] | dones u8[n]] (the Python host layer allocates them so)
  if (rewards_host && dones_host &&
      reinterpret_cast<uint8_t*>(out->rewards) + (size_t)n * 8 == out->dones &&
      reinterpret_cast<uint8_t*>(rewards_host) + (size_t)n * 8 == dones_host) {
    TC_CUDA(cudaMemcpyAsync(rewards_host, out->rewards, (size_t)n * 9, cudaMemcpyDeviceToHost, st));
  } else {
    if (rewards_host)
      TC_CUDA(cudaMemcpyAsync(rewards_host, out->rewards, (size_t)n * 8, cudaMemcpyDeviceToHost,
                              st));
    if (dones_host)
      TC_CUDA(cudaMemcpyAsync(dones_host, out->dones, (size_t)n, cudaMemcpyDeviceToHost, st));
  }
  TC_CUDA(cudaStreamSynchronize(st));
  return TC_OK;
}

int tc_batch_step_mapped(const tc_spec* s, const tc_state* state_in, const tc_state* state_out,
                         const int64_t* actions_host, const tc_out* out, int64_t n,
                         int32_t auto_reset, int32_t validate, tc_counters* counters_dev,
                         uint8_t* results_host, int32_t* flag_host, void* stream) {
  if (!actions_host || !results_host || !flag_host || !counters_dev)
    return fail(TC_E_INVALID, "NULL actions / results / flag / counters");
  if (!state_out) return fail(TC_E_INVALID, "state_out is NULL");
  if (n <= 0) return n == 0 ? TC_OK : fail(TC_E_INVALID, "n must be >= 0");
  if (!out || reinterpret_cast<uint8_t*>(out->rewards) + (size_t)n * 8 != out->dones)
    return fail(TC_E_INVALID, "out->dones must follow out->rewards ([rewards | dones])");
  if ((reinterpret_cast<uintptr_t>(out->rewards) | reinterpret_cast<uintptr_t>(results_host)) & 15u)
    return fail(TC_E_INVALID, "rewards / results_host must be 16-byte aligned");
  // the device reads / writes these host buffers directly: they must be
  // page-locked and mapped into the device's address space (UVA)
  // (checked once per buffer triple: a step loop reuses the same buffers)
  static thread_local const void* checked[3] = {nullptr, nullptr, nullptr};
  if (checked[0] != actions_host || checked[1] != results_host || checked[2] != flag_host) {
    for (const void* p : {(const void*)actions_host, (const void*)results_host,
                          (const void*)flag_host}) {
      cudaPointerAttributes a;
      if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeHost ||
          a.devicePointer != p) {
        cudaGetLastError();
        return fail(TC_E_INVALID, "host buffers must be pinned and UVA-mapped");
      }
    }
    checked[0] = actions_host; checked[1] = results_host; checked[2] = flag_host;
  }
  volatile int32_t* done = flag_host + 1;
  *done = 0;
  const double t0 = host_us();
  const int rc = launch_batch_kernel(s, state_in, state_out, actions_host, out, n, TC_MODE_STEP,
                                     auto_reset, validate, counters_dev, stream, results_host,
                                     flag_host);
  if (rc != TC_OK) return rc;
  const double t1 = host_us();
  // the last CTA raises *done after the results reached host memory: spin
  // on it (the kernel's teardown and the stream's completion need not be
  // waited for); poll the stream now and then so a faulting kernel surfaces
  for (unsigned spin = 1; *done == 0; spin++) {
    if ((spin & 1023u) == 0) {
      const cudaError_t q = cudaStreamQuery((cudaStream_t)stream);
      if (q == cudaSuccess) {
        if (*done == 0) return fail(TC_E_CUDA, "step kernel finished without results");
        break;
      }
      if (q != cudaErrorNotReady) {
        cudaGetLastError();
        return fail(TC_E_CUDA, cudaGetErrorString(q));
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  const double t2 = host_us();
  g_mapped_time[0] += t1 - t0;
  g_mapped_time[1] += t2 - t1;
  g_mapped_time[2] += 1.0;
  return TC_OK;
}

int tc_batch_step_mapped_call(const tc_mapped_call* c) {
  if (!c) return fail(TC_E_INVALID, "NULL call");
  return tc_batch_step_mapped(c->spec, c->state_in, c->state_out, c->actions_host, c->out, c->n,
                              c->auto_reset, c->validate, c->counters_dev, c->results_host,
                              c->flag_host, c->stream);
}

int tc_batch_step_pipelined(const tc_pipe_call* c) {
  if (!c) return fail(TC_E_INVALID, "NULL call");
  const tc_mapped_call& m = c->step;
  if (!m.actions_host || !m.results_host || !m.flag_host || !m.counters_dev)
    return fail(TC_E_INVALID, "NULL actions / results / flag / counters");
  if (!m.spec || !m.state_in || !m.state_out || !m.out)
    return fail(TC_E_INVALID, "NULL spec / state / out");
  if (m.n <= 0) return m.n == 0 ? TC_OK : fail(TC_E_INVALID, "n must be >= 0");
  if (reinterpret_cast<uint8_t*>(m.out->rewards) + (size_t)m.n * 8 != m.out->dones)
    return fail(TC_E_INVALID, "out->dones must follow out->rewards ([rewards | dones])");
  if ((reinterpret_cast<uintptr_t>(m.out->rewards) | reinterpret_cast<uintptr_t>(m.results_host) |
       reinterpret_cast<uintptr_t>(m.flag_host)) & 15u)
    return fail(TC_E_INVALID, "rewards / results_host / flag_host must be 16-byte aligned");
  const double t0 = host_us();
  // the call's device (the struct carries it: the caller need not switch)
  struct DevGuard {
    int prev = -1;
    explicit DevGuard(int want) {
      if (cudaGetDevice(&prev) == cudaSuccess && prev != want) cudaSetDevice(want);
      else prev = -1;
    }
    ~DevGuard() { if (prev >= 0) cudaSetDevice(prev); }
  } dev_guard(c->device);
  Pipe& P = pipe();
  std::unique_lock<std::mutex> lk(P.mu);
  volatile int32_t* done = m.flag_host + 1;
  bool released = false;
  if (P.pending.load(std::memory_order_relaxed)) {
    if (same_key(P.key, pipe_key(m, m.state_in, m.state_out, m.out))) {
      // this step is already resident behind its gate: open it. The host's
      // earlier stores (actions, the flag words) are ordered before the go
      // word (x86 TSO; the fence keeps the compiler from reordering them)
      *done = 0;
      std::atomic_thread_fence(std::memory_order_seq_cst);
      *reinterpret_cast<volatile uint32_t*>(m.flag_host + 4) = P.q;
      P.pending.store(false, std::memory_order_release);
      P.released++;
      P.backoff = 0;
      released = true;
      if (P.resident) {
        // the resident loop goes on to the next step of the ping-pong: it
        // is pending again (gate q + 1) without a launch
        P.q++;
        P.key = pipe_key(m, m.state_out, m.state_in, c->next_out);
        P.t_launch = host_us();
        P.pending.store(true, std::memory_order_release);
      }
    } else {
      pipe_cancel_locked(P, false);
    }
  }
  if (!released) {
    // the first step of a run (or after a cancel): an ordinary mapped launch
    if (tc_batch_step_mapped(m.spec, m.state_in, m.state_out, m.actions_host, m.out, m.n,
                             m.auto_reset, m.validate, m.counters_dev, m.results_host,
                             m.flag_host, m.stream) != TC_OK)
      return TC_E_CUDA;
    // (tc_batch_step_mapped waited for the results: nothing left to wait for
    // but the successor's launch below)
  }
  // the successor (reuse=True ping-pong: this step's out state is its input,
  // this step's input block its output state, c->next_out its output block)
  const bool taps = c->next_out && (c->next_out->zbuf || c->next_out->rayinfo ||
                                    c->next_out->spritevis);
  const int lkind = lean_kind(m.spec, m.n);
  if (c->speculate && c->next_out && c->gate_dev && !taps && lkind != 0 &&
      !P.pending.load(std::memory_order_relaxed)) {
    if (P.skip > 0) {
      P.skip--;
    } else {
      if (++P.q == 0) ++P.q;
      // one-wave 64x64 batches: a resident loop kernel (stays on the GPU
      // across steps); otherwise one gated launch per step
      const bool res = g_pipe_resident && lkind == 1 && select_resident(m.spec) != nullptr;
      GateArgs g{c->gate_dev, reinterpret_cast<const unsigned long long*>(m.flag_host + 4), P.q,
                 res ? m.out : nullptr};
      const int rc = launch_batch_kernel(m.spec, m.state_out, m.state_in, m.actions_host,
                                         c->next_out, m.n, TC_MODE_STEP, m.auto_reset,
                                         m.validate, m.counters_dev, m.stream, m.results_host,
                                         m.flag_host, nullptr, &g);
      if (rc != TC_OK) return rc;
      P.key = pipe_key(m, m.state_out, m.state_in, c->next_out);
      P.t_launch = host_us();
      P.resident = res;
      P.pending.store(true, std::memory_order_release);
      if (!P.watchdog) {
        std::thread(pipe_watchdog).detach();
        P.watchdog = true;
      } else if (P.idle) {
        P.cv.notify_one();
      }
    }
  }
  lk.unlock();
  if (!released) return TC_OK;
  const double t1 = host_us();
  // wait for the released step's results (as tc_batch_step_mapped): the
  // stream now also holds the successor, so a step that ended without
  // results surfaces once the successor is released or cancelled
  for (unsigned spin = 1; *done == 0; spin++) {
    if ((spin & 1023u) == 0) {
      const cudaError_t q = cudaStreamQuery((cudaStream_t)m.stream);
      if (q == cudaSuccess) {
        if (*done == 0) return fail(TC_E_CUDA, "step kernel finished without results");
        break;
      }
      if (q != cudaErrorNotReady) {
        cudaGetLastError();
        return fail(TC_E_CUDA, cudaGetErrorString(q));
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  {
    // the watchdog's clock for the launch waiting behind this step starts
    // now, when the caller gets control back (a step longer than the
    // timeout must not cancel its successor)
    std::lock_guard<std::mutex> g2(P.mu);
    if (P.pending.load(std::memory_order_relaxed) && P.key.flag == m.flag_host)
      P.t_launch = host_us();
  }
  // released steps: [3] release + bookkeeping, [4] wait for results, [5] count
  g_mapped_time[3] += t1 - t0;
  g_mapped_time[4] += host_us() - t1;
  g_mapped_time[5] += 1.0;
  return TC_OK;
}

int tc_debug_pipe_trace(uint64_t* host, int64_t cap, int32_t* grid) {
  if (grid) *grid = g_pipe_trace_grid;
  if (!g_pipe_trace || !host) return TC_OK;
  const size_t nb = std::min<size_t>((size_t)cap, (size_t)64 * 3 * g_pipe_trace_grid) * 8;
  TC_CUDA(cudaMemcpy(host, g_pipe_trace, nb, cudaMemcpyDeviceToHost));
  return TC_OK;
}

int tc_pipe_cancel(void) {
  pipe_cancel_if_pending();
  return TC_OK;
}

int tc_pipe_reset(void) {
  Pipe& P = pipe();
  std::lock_guard<std::mutex> lk(P.mu);
  pipe_cancel_locked(P, false);
  P.skip = P.backoff = 0;
  return TC_OK;
}

int tc_pipe_stats(uint64_t* out4) {
  if (!out4) return fail(TC_E_INVALID, "NULL out");
  Pipe& P = pipe();
  std::lock_guard<std::mutex> lk(P.mu);
  out4[0] = P.released;
  out4[1] = P.cancelled;
  out4[2] = P.timeouts;
  out4[3] = P.pending.load() ? 1u : 0u;
  return TC_OK;
}

// perf diagnostics of the mapped host step: mean host microseconds in the
// launch call and in the wait for the completion word since the last reset
int tc_debug_mapped_timing(double* out3, int32_t reset) {
  if (out3) {
    const double k = g_mapped_time[2] > 0 ? g_mapped_time[2] : 1.0;
    out3[0] = g_mapped_time[0] / k;
    out3[1] = g_mapped_time[1] / k;
    out3[2] = g_mapped_time[2];
  }
  if (out3 && reset == 2) {  // the pipelined released steps' split instead
    const double k = g_mapped_time[5] > 0 ? g_mapped_time[5] : 1.0;
    out3[0] = g_mapped_time[3] / k;
    out3[1] = g_mapped_time[4] / k;
    out3[2] = g_mapped_time[5];
  }
  if (reset) for (double& v : g_mapped_time) v = 0.0;
  return TC_OK;
}

int tc_rollout(const tc_spec* s, const tc_state* state, const tc_out* out, int64_t n,
               int64_t base, int64_t n_total, uint64_t policy_key, int64_t step0,
               int32_t k_steps, int32_t frame_ring, tc_counters* counters_dev, void* stream) {
  pipe_cancel_if_pending();
  if (!s || !state || !out || !out->frames) return fail(TC_E_INVALID, "NULL spec/state/out");
  if (n < 0 || k_steps < 0 || frame_ring < 1) return fail(TC_E_INVALID, "bad n/k/ring");
  if (n == 0 || k_steps == 0) return TC_OK;
  if (s->dev.bulk && (reinterpret_cast<uintptr_t>(out->frames) & 15u))
    return fail(TC_E_INVALID, "frames must be 16-byte aligned");
  RolloutArgs ra;
  ra.policy_key = policy_key;
  ra.base = base;
  ra.n_total = n_total;
  ra.step0 = step0;
  ra.k_steps = k_steps;
  ra.frame_ring = frame_ring;
  ra.n_tags = 0;
  for (int a = 0; a < A_COUNT; a++)
    if ((s->dev.legal_mask >> a) & 1u) ra.tags[ra.n_tags++] = a;
  if (ra.n_tags == 0) return fail(TC_E_INVALID, "spec has no legal actions");
  StateDev sd = to_dev(state);
  OutDev od = to_dev(out);
  const long long nn = n;
  SpecDev spec = s->dev;
  void* args[] = {&spec, &sd, &od, (void*)&nn, &ra, &counters_dev};
  const int grid = grid_for(s, n);
  TC_CUDA(cudaLaunchKernel(select_rollout(s->nc, s->dev.group), dim3(grid), dim3(WARPS_PER_CTA * 32), args,
                           s->smem_bytes, (cudaStream_t)stream));
  return TC_OK;
}

int tc_seed_streams(uint64_t seed, int64_t base, int64_t n, uint64_t* rkey_dev,
                    uint64_t* rctr_dev, void* stream) {
  if (n < 0 || (n > 0 && (!rkey_dev || !rctr_dev))) return fail(TC_E_INVALID, "bad seed args");
  if (n == 0) return TC_OK;
  // from_seed: the root key is mix(seed) (rng.py:36-38)
  uint64_t x = seed;
  x ^= x >> 30; x *= MIX1; x ^= x >> 27; x *= MIX2; x ^= x >> 31;
  const int threads = 256;
  const int64_t want = (n + threads - 1) / threads;
  const int blocks = (int)(want < 4096 ? want : 4096);
  seed_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
      x, base, n, reinterpret_cast<unsigned long long*>(rkey_dev),
      reinterpret_cast<unsigned long long*>(rctr_dev));
  TC_CUDA(cudaGetLastError());
  return TC_OK;
}

int tc_policy_actions(uint64_t policy_key, int64_t step, int64_t n_total, int64_t base,
                      int64_t n, const int64_t* action_tags_host, int32_t n_tags,
                      int64_t* actions_dev, void* stream) {
  if (n_tags < 1 || n_tags > A_COUNT || !action_tags_host)
    return fail(TC_E_INVALID, "n_tags must be 1..7");
  if (n < 0 || (n > 0 && !actions_dev)) return fail(TC_E_INVALID, "bad actions buffer");
  if (n == 0) return TC_OK;
  Tags tags;
  for (int k = 0; k < A_COUNT; k++) tags.v[k] = k < n_tags ? action_tags_host[k] : 0;
  const int threads = 256;
  const int64_t want = (n + threads - 1) / threads;
  const int blocks = (int)(want < 4096 ? want : 4096);
  policy_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
      policy_key, step, n_total, base, n, tags, n_tags,
      reinterpret_cast<long long*>(actions_dev));
  TC_CUDA(cudaGetLastError());
  return TC_OK;
}

// ------------------------------------------------ host-pointer parity entry
int tc_host_cast_ray(const uint8_t* kind, const int16_t* didx, const uint8_t* dopen, int32_t h,
                     int32_t w, double ox, double oy, double rx, double ry, int32_t* status,
                     int32_t* mapx, int32_t* mapy, int32_t* side, double* perp, double* wall_u,
                     int32_t* steps) {
  if (!kind || !didx || h < 1 || w < 1) return fail(TC_E_INVALID, "bad map");
  std::vector<uint32_t> cells(h * w);
  uint32_t dmask = 0;
  for (int k = 0; k < h * w; k++) {
    const uint32_t tag = kind[k];
    if (tag > C_DOOR) return fail(TC_E_INVALID, "cell tag must be 0..2");
    uint32_t idx = 0;
    if (tag == C_DOOR) {
      if (didx[k] < 0 || didx[k] >= TC_MAX_DOORS) return fail(TC_E_INVALID, "bad door index");
      idx = (uint32_t)didx[k];
      if (dopen && dopen[didx[k]]) dmask |= 1u << idx;
    }
    cells[k] = idx | (tag << CELL_TAG_SHIFT);
  }
  uint32_t* dcell = nullptr;
  int32_t* dio = nullptr;
  double* dd = nullptr;
  TC_CUDA(cudaMalloc(&dcell, cells.size() * 4));
  TC_CUDA(cudaMalloc(&dio, 5 * 4));
  TC_CUDA(cudaMalloc(&dd, 2 * 8));
  TC_CUDA(cudaMemcpy(dcell, cells.data(), cells.size() * 4, cudaMemcpyHostToDevice));
  cast_ray_kernel<<<1, 1>>>(dcell, h, w, dmask, ox, oy, rx, ry, dio, dd);
  int32_t io[5];
  double dv[2];
  cudaError_t e = cudaMemcpy(io, dio, sizeof io, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(dv, dd, sizeof dv, cudaMemcpyDeviceToHost);
  cudaFree(dcell);
  cudaFree(dio);
  cudaFree(dd);
  if (e != cudaSuccess) return cuda_fail(e, "cast_ray");
  *status = io[0]; *mapx = io[1]; *mapy = io[2]; *side = io[3]; *steps = io[4];
  *perp = dv[0]; *wall_u = dv[1];
  return TC_OK;
}

}  // extern "C"

namespace {
// device mirror of a host state/out block for the host-pointer entry points
struct DevBlock {
  std::vector<void*> ptrs;
  ~DevBlock() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  int up(T*& dst, const T* src, size_t count, bool copy) {
    dst = nullptr;
    if (!src) return TC_OK;
    void* p = nullptr;
    const size_t bytes = count ? count * sizeof(T) : 16;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(block)");
    ptrs.push_back(p);
    if (copy && count) {
      e = cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(H2D)");
    }
    dst = static_cast<T*>(p);
    return TC_OK;
  }
};
template <class T>
int down(T* host, const T* dev, size_t count) {
  if (!host || !dev || !count) return TC_OK;
  cudaError_t e = cudaMemcpy(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? TC_OK : cuda_fail(e, "cudaMemcpy(D2H)");
}
}  // namespace

#define TC_TRY(x)                 \
  do {                            \
    int _rc = (x);                \
    if (_rc != TC_OK) return _rc; \
  } while (0)

static int host_run(const tc_tables* t, const tc_state* sh, const int64_t* acts_h,
                    const tc_out* oh, int64_t n, int32_t mode, int32_t auto_reset,
                    int32_t validate, int64_t* violations) {
  tc_spec* s = nullptr;
  TC_TRY(tc_spec_create(t, &s));
  struct Guard {
    tc_spec* s;
    ~Guard() { tc_spec_destroy(s); }
  } guard{s};
  const size_t D = t->n_doors, E = t->n_entities, W = t->obs_w, H = t->obs_h;
  DevBlock blk;
  tc_state sd;
  tc_out od;
  TC_TRY(blk.up(sd.px, sh->px, n, true));
  TC_TRY(blk.up(sd.py, sh->py, n, true));
  TC_TRY(blk.up(sd.dx, sh->dx, n, true));
  TC_TRY(blk.up(sd.dy, sh->dy, n, true));
  TC_TRY(blk.up(sd.health, sh->health, n, true));
  TC_TRY(blk.up(sd.inv, sh->inv, n, true));
  TC_TRY(blk.up(sd.t, sh->t, n, true));
  TC_TRY(blk.up(sd.rkey, sh->rkey, n, true));
  TC_TRY(blk.up(sd.rctr, sh->rctr, n, true));
  TC_TRY(blk.up(sd.done, sh->done, n, true));
  TC_TRY(blk.up(sd.agoal, sh->agoal, n, true));
  TC_TRY(blk.up(sd.dopen, sh->dopen, n * D, true));
  TC_TRY(blk.up(sd.ealive, sh->ealive, n * E, true));
  const int64_t* da = nullptr;
  int64_t* dam = nullptr;
  if (mode == TC_MODE_STEP) {
    TC_TRY(blk.up(dam, acts_h, n, true));
    da = dam;
  }
  TC_TRY(blk.up(od.frames, oh->frames, n * H * W * 3, false));
  TC_TRY(blk.up(od.zbuf, oh->zbuf, n * W, false));
  TC_TRY(blk.up(od.rewards, oh->rewards, n, false));
  TC_TRY(blk.up(od.dones, oh->dones, n, false));
  TC_TRY(blk.up(od.truncs, oh->truncs, n, false));
  TC_TRY(blk.up(od.events, oh->events, n, false));
  TC_TRY(blk.up(od.statuses, oh->statuses, n, false));
  TC_TRY(blk.up(od.rayinfo, oh->rayinfo, n * W * 4, false));
  TC_TRY(blk.up(od.spritevis, oh->spritevis, n, false));
  tc_counters* dc = nullptr;
  TC_CUDA(cudaMalloc(&dc, sizeof(tc_counters)));
  blk.ptrs.push_back(dc);
  TC_CUDA(cudaMemset(dc, 0, sizeof(tc_counters)));
  if (od.zbuf) TC_CUDA(cudaMemset(od.zbuf, 0, n * W * 8));
  TC_TRY(tc_batch_kernel(s, &sd, da, &od, n, mode, auto_reset, validate, dc, nullptr));
  TC_CUDA(cudaDeviceSynchronize());
  TC_TRY(down(sh->px, sd.px, n));
  TC_TRY(down(sh->py, sd.py, n));
  TC_TRY(down(sh->dx, sd.dx, n));
  TC_TRY(down(sh->dy, sd.dy, n));
  TC_TRY(down(sh->health, sd.health, n));
  TC_TRY(down(sh->inv, sd.inv, n));
  TC_TRY(down(sh->t, sd.t, n));
  TC_TRY(down(sh->rkey, sd.rkey, n));
  TC_TRY(down(sh->rctr, sd.rctr, n));
  TC_TRY(down(sh->done, sd.done, n));
  TC_TRY(down(sh->agoal, sd.agoal, n));
  TC_TRY(down(sh->dopen, sd.dopen, n * D));
  TC_TRY(down(sh->ealive, sd.ealive, n * E));
  TC_TRY(down(oh->frames, od.frames, n * H * W * 3));
  TC_TRY(down(oh->zbuf, od.zbuf, n * W));
  TC_TRY(down(oh->rewards, od.rewards, n));
  TC_TRY(down(oh->dones, od.dones, n));
  TC_TRY(down(oh->truncs, od.truncs, n));
  TC_TRY(down(oh->events, od.events, n));
  TC_TRY(down(oh->statuses, od.statuses, n));
  TC_TRY(down(oh->rayinfo, od.rayinfo, n * W * 4));
  TC_TRY(down(oh->spritevis, od.spritevis, n));
  if (violations) {
    tc_counters hc;
    TC_CUDA(cudaMemcpy(&hc, dc, sizeof hc, cudaMemcpyDeviceToHost));
    *violations = (int64_t)hc.violations;
  }
  return TC_OK;
}

extern "C" {

int tc_host_render_into(const tc_tables* t, double px, double py, double dx, double dy,
                        const uint8_t* dopen_row, const uint8_t* ealive_row, int32_t agoal,
                        uint8_t* frame, double* zbuf, int32_t* status) {
  if (!t || !frame || !status) return fail(TC_E_INVALID, "NULL argument");
  double x = px, y = py, ddx = dx, ddy = dy, health = 100.0;
  uint8_t inv = 0, done = 0;
  int64_t tt = 0;
  uint64_t rkey = 0, rctr = 0;
  int32_t ag = agoal;
  uint8_t dop[TC_MAX_DOORS] = {0}, eal[TC_MAX_ENTITIES] = {0};
  if (t->n_doors > TC_MAX_DOORS || t->n_entities > TC_MAX_ENTITIES)
    return fail(TC_E_CAPACITY, "too many doors/entities");
  for (int d = 0; d < t->n_doors; d++) dop[d] = dopen_row ? dopen_row[d] : 0;
  for (int e = 0; e < t->n_entities; e++) eal[e] = ealive_row ? ealive_row[e] : 1;
  tc_state s = {&x, &y, &ddx, &ddy, &health, &inv, &tt, &rkey, &rctr, &done, &ag, dop, eal};
  std::vector<double> zb(t->obs_w, 0.0);
  tc_out o;
  memset(&o, 0, sizeof o);
  o.frames = frame;
  o.zbuf = zbuf ? zbuf : zb.data();
  o.statuses = status;
  return host_run(t, &s, nullptr, &o, 1, MODE_RENDER, 0, 0, nullptr);
}

int tc_host_batch_kernel(const tc_tables* t, const tc_state* state_host,
                         const int64_t* actions_host, const tc_out* out_host, int64_t n,
                         int32_t mode, int32_t auto_reset, int32_t validate,
                         int64_t* violations) {
  if (!t || !state_host || !out_host) return fail(TC_E_INVALID, "NULL argument");
  if (mode != TC_MODE_RESET && mode != TC_MODE_STEP) return fail(TC_E_INVALID, "bad mode");
  if (n < 0) return fail(TC_E_INVALID, "n must be >= 0");
  if (violations) *violations = 0;
  if (n == 0) return TC_OK;
  return host_run(t, state_host, actions_host, out_host, n, mode, auto_reset, validate,
                  violations);
}

}  // extern "C"
