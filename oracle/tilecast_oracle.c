/*
 * tilecast_oracle.c -- CPU restatement of the reference's batched env step.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker and the CPU baseline
 * port; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product path (the CUDA library under
 * paper_2605_19926_b200/csrc) never links or calls it.
 *
 * Semantics follow the reference's pure-Python kernels, which define the
 * engine bit for bit (/root/reference/pkg/src/tilecast/backend/_pycore.py:1-9),
 * statement by statement; citations are to that file unless noted. Compiled
 * with -O2 -ffp-contract=off like the reference's Cython build
 * (pkg/setup.py:20-27) so every a*b+c stays two IEEE roundings.
 *
 * Parity of this file is pinned against the reference itself: the Cython
 * module built by oracle/build_ref.sh into oracle/_ref and the golden
 * fixtures in tests/golden/ generated from the reference
 * (tests/golden/make_golden.py). See tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/tilecast_b200.h"

/* layout.py:8-19 / :22-25 / :28-66 */
enum { FC_MOVE_SPEED = 0, FC_RADIUS, FC_TURN_COS, FC_TURN_SIN, FC_ATTEN,
       FC_GOAL_REWARD, FC_LIVING_REWARD, FC_HEALTH_DECAY, FC_HEALTH_RESTORE,
       FC_SPRITE_K, FC_MIN_SPRITE_DEPTH };
enum { IC_MAX_STEPS = 0, IC_GOAL_MODE, IC_USE_HEALTH };
enum { A_FORWARD = 0, A_BACKWARD, A_TURN_LEFT, A_TURN_RIGHT, A_STRAFE_LEFT,
       A_STRAFE_RIGHT, A_NOOP };
enum { C_FLOOR = 0, C_WALL = 1, C_DOOR = 2 };
enum { K_KEY = 0, K_GOAL = 1, K_MEDKIT = 2 };
enum { EV_KEY_BASE_BIT = 0, EV_DOOR_BASE_BIT = 3, EV_MEDKIT_BIT = 6,
       EV_GOAL_BIT = 7, EV_DIED_BIT = 8, EV_TRUNCATED_BIT = 9 };

static const double PLANE_HALF_WIDTH = 0.66; /* geometry.py:18 */
static const uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;
static const uint64_t MIX1 = 0xBF58476D1CE4E5B9ULL;
static const uint64_t MIX2 = 0x94D049BB133111EBULL;
static const uint64_t SPLIT_SALT = 0x3C6EF372FE94F82AULL; /* rng.py:18 */

/* rng.py:26-33 */
static uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= MIX1;
  x ^= x >> 27;
  x *= MIX2;
  x ^= x >> 31;
  return x;
}

/* _pycore.py:27-35: draw in [0, n) by 128-bit multiply-high, bump counter */
static uint64_t draw_below(uint64_t key, uint64_t *ctr, uint64_t n) {
  uint64_t x = mix64(key + *ctr * GOLDEN);
  *ctr += 1;
  return (uint64_t)(((unsigned __int128)x * (unsigned __int128)n) >> 64);
}

/* _pycore.py:38-96 -- DDA along tile boundaries. */
static int cast_ray(const uint8_t *kind, const int16_t *didx,
                    const uint8_t *dopen, int h, int w, double ox, double oy,
                    double rx, double ry, int *mapx_o, int *mapy_o,
                    int *side_o, double *perp_o, double *wu_o, int *steps_o) {
  int mapx = (int)floor(ox);
  int mapy = (int)floor(oy);
  double ddx, ddy, sdx, sdy;
  int stepx, stepy;
  if (rx != 0.0) {
    ddx = fabs(1.0 / rx);
    stepx = rx > 0.0 ? 1 : -1;
    sdx = rx > 0.0 ? ((mapx + 1.0) - ox) * ddx : (ox - mapx) * ddx;
  } else {
    ddx = INFINITY;
    stepx = 0;
    sdx = INFINITY;
  }
  if (ry != 0.0) {
    ddy = fabs(1.0 / ry);
    stepy = ry > 0.0 ? 1 : -1;
    sdy = ry > 0.0 ? ((mapy + 1.0) - oy) * ddy : (oy - mapy) * ddy;
  } else {
    ddy = INFINITY;
    stepy = 0;
    sdy = INFINITY;
  }
  const int limit = 2 * (w + h);
  int side = 0, steps = 0;
  for (;;) {
    if (sdx < sdy) { /* ties step Y (_pycore.py:70) */
      sdx += ddx;
      mapx += stepx;
      side = 0;
    } else {
      sdy += ddy;
      mapy += stepy;
      side = 1;
    }
    steps += 1;
    if (steps > limit || mapx < 0 || mapx >= w || mapy < 0 || mapy >= h) {
      *mapx_o = mapx; *mapy_o = mapy; *side_o = side;
      *perp_o = 0.0; *wu_o = 0.0; *steps_o = steps;
      return steps > limit ? TC_ST_STEP_BUDGET : TC_ST_ESCAPED;
    }
    const int tag = kind[mapy * w + mapx];
    if (tag == C_WALL) break;
    if (tag == C_DOOR && dopen[didx[mapy * w + mapx]] == 0) break;
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
  *mapx_o = mapx; *mapy_o = mapy; *side_o = side;
  *perp_o = perp; *wu_o = wu; *steps_o = steps;
  return TC_ST_OK;
}

/* _pycore.py:99-129 */
static int sprite_mask(int kd, double aa, double v) {
  if (kd == K_GOAL) {
    double dv = v - 0.5;
    if (dv < 0.0) dv = -dv;
    return (aa + dv * 2.0 <= 0.8) ? 1 : 0;
  }
  if (kd == K_KEY) {
    const double ea = aa / 0.30;
    const double ev = (v - 0.30) / 0.18;
    const double e = ea * ea + ev * ev;
    if (0.30 <= e && e <= 1.0) return 1;
    if (aa <= 0.07 && 0.30 <= v && v <= 0.85) return 1;
    if (aa <= 0.24 && 0.62 <= v && v <= 0.70) return 1;
    if (aa <= 0.24 && 0.76 <= v && v <= 0.84) return 1;
    return 0;
  }
  if (aa <= 0.10 && 0.32 <= v && v <= 0.73) return 1;
  if (aa <= 0.38 && 0.47 <= v && v <= 0.60) return 1;
  if (aa <= 0.60 && 0.25 <= v && v <= 0.80) return 2;
  return 0;
}

static inline void put(uint8_t *frame, int obs_w, int row, int c, int r, int g,
                       int b) {
  uint8_t *p = frame + ((size_t)row * obs_w + c) * 3;
  p[0] = (uint8_t)r;
  p[1] = (uint8_t)g;
  p[2] = (uint8_t)b;
}

/* _pycore.py:132-271 -- walls per column, then sprites far to near.
 * rayinfo (i32[obs_w,4]) and spritevis are optional debug taps. */
static int render_into(const tc_tables *T, double px, double py, double dx,
                       double dy, const uint8_t *dopen_row,
                       const uint8_t *ealive_row, int agoal, uint8_t *frame,
                       double *zbuf, int32_t *rayinfo, uint64_t *spritevis) {
  const int obs_h = T->obs_h, obs_w = T->obs_w;
  const int h2 = obs_h / 2;
  const double atten = T->fc[FC_ATTEN];
  const double planex = -dy * PLANE_HALF_WIDTH;
  const double planey = dx * PLANE_HALF_WIDTH;
  const uint8_t *cc = T->ceil_rgb, *ff = T->floor_rgb;

  for (int c = 0; c < obs_w; c++) {
    const double k = T->coef[c];
    const double rx = dx + planex * k;
    const double ry = dy + planey * k;
    int mapx, mapy, side, steps;
    double perp, wu;
    const int status = cast_ray(T->kind, T->didx, dopen_row, T->h, T->w, px,
                                py, rx, ry, &mapx, &mapy, &side, &perp, &wu,
                                &steps);
    if (rayinfo) {
      rayinfo[c * 4 + 0] = mapx; rayinfo[c * 4 + 1] = mapy;
      rayinfo[c * 4 + 2] = side; rayinfo[c * 4 + 3] = steps;
    }
    if (status != TC_ST_OK) return status;
    zbuf[c] = perp;
    const double shade = 1.0 / (1.0 + atten * perp);
    const int cell = mapy * T->w + mapx;
    const uint8_t *base = (T->kind[cell] == C_DOOR)
                              ? T->door_rgb + 3 * T->dcol[T->didx[cell]]
                              : T->pal + 3 * T->wcol[cell];
    const int wr = (int)(base[0] * shade);
    const int wg = (int)(base[1] * shade);
    const int wb = (int)(base[2] * shade);
    double lh_f = obs_h / perp;
    if (lh_f > 1e9) lh_f = 1e9;
    const int half = (int)lh_f / 2;
    const int top = h2 - half, bot = h2 + half;
    const int t0 = top > 0 ? top : 0;
    const int b0 = bot < obs_h ? bot : obs_h;
    for (int row = 0; row < t0; row++) put(frame, obs_w, row, c, cc[0], cc[1], cc[2]);
    for (int row = t0; row < b0; row++) put(frame, obs_w, row, c, wr, wg, wb);
    for (int row = b0; row < obs_h; row++) put(frame, obs_w, row, c, ff[0], ff[1], ff[2]);
  }

  /* sprite gather in entity order, _pycore.py:192-209 */
  double deps[TC_MAX_ENTITIES], lats[TC_MAX_ENTITIES];
  int ents[TC_MAX_ENTITIES];
  int m = 0;
  const double det = planex * dy - dx * planey;
  if (det != 0.0) {
    const double invdet = 1.0 / det;
    for (int e = 0; e < T->n_entities; e++) {
      if (ealive_row[e] == 0) continue;
      if (T->ekind[e] == K_GOAL && e != agoal) continue;
      const double relx = T->epx[e] - px;
      const double rely = T->epy[e] - py;
      const double lat = invdet * (dy * relx - dx * rely);
      const double dep = invdet * (-planey * relx + planex * rely);
      if (dep < T->fc[FC_MIN_SPRITE_DEPTH]) continue;
      deps[m] = dep; lats[m] = lat; ents[m] = e; m++;
    }
  }
  /* stable insertion sort far -> near, _pycore.py:210-217 */
  for (int i = 1; i < m; i++) {
    const double d = deps[i], l = lats[i];
    const int e = ents[i];
    int j = i;
    while (j > 0 && deps[j - 1] < d) {
      deps[j] = deps[j - 1]; lats[j] = lats[j - 1]; ents[j] = ents[j - 1];
      j--;
    }
    deps[j] = d; lats[j] = l; ents[j] = e;
  }
  uint64_t vis = 0;
  /* draw, _pycore.py:219-270 */
  for (int oi = 0; oi < m; oi++) {
    const double dep = deps[oi], lat = lats[oi];
    const int e = ents[oi];
    const double ks = lat / dep;
    const double halfk = T->fc[FC_SPRITE_K] / dep;
    const double shade = 1.0 / (1.0 + atten * dep);
    double sh_f = obs_h / dep;
    if (sh_f > 1e9) sh_f = 1e9;
    const int vhalf = (int)sh_f / 2;
    const int vtop = h2 - vhalf, vbot = h2 + vhalf;
    const int denom = vbot - vtop;
    if (denom <= 0) continue;
    const int r0 = vtop > 0 ? vtop : 0;
    const int r1 = vbot < obs_h ? vbot : obs_h;
    const int kd = T->ekind[e];
    const uint8_t *m1 = kd == K_KEY ? T->key_rgb + 3 * T->ecol[e]
                        : kd == K_GOAL ? T->goal_rgb : T->med_cross;
    const int s1r = (int)(m1[0] * shade), s1g = (int)(m1[1] * shade),
              s1b = (int)(m1[2] * shade);
    const int s2r = (int)(T->med_box[0] * shade),
              s2g = (int)(T->med_box[1] * shade),
              s2b = (int)(T->med_box[2] * shade);
    for (int c = 0; c < obs_w; c++) {
      if (zbuf[c] <= dep) continue;
      const double a = (T->coef[c] - ks) / halfk;
      if (a <= -1.0 || a >= 1.0) continue;
      const double aa = a >= 0.0 ? a : -a;
      if (r0 < r1) vis |= 1ULL << e;
      for (int row = r0; row < r1; row++) {
        const double v = ((row - vtop) + 0.5) / denom;
        const int mk = sprite_mask(kd, aa, v);
        if (mk == 1) put(frame, obs_w, row, c, s1r, s1g, s1b);
        else if (mk == 2) put(frame, obs_w, row, c, s2r, s2g, s2b);
      }
    }
  }
  if (spritevis) *spritevis = vis;
  return TC_ST_OK;
}

/* _pycore.py:274-304 */
static int blocked(const tc_tables *T, const uint8_t *dopen_row, double cx,
                   double cy, double radius) {
  const int tx0 = (int)floor(cx - radius), tx1 = (int)floor(cx + radius);
  const int ty0 = (int)floor(cy - radius), ty1 = (int)floor(cy + radius);
  const double r2 = radius * radius;
  for (int ty = ty0; ty <= ty1; ty++) {
    for (int tx = tx0; tx <= tx1; tx++) {
      if (tx < 0 || tx >= T->w || ty < 0 || ty >= T->h) return 1;
      const int tag = T->kind[ty * T->w + tx];
      if (tag == C_FLOOR) continue;
      if (tag == C_DOOR && dopen_row[T->didx[ty * T->w + tx]] != 0) continue;
      double nx = cx;
      if (nx < tx) nx = tx;
      else if (nx > tx + 1.0) nx = tx + 1.0;
      double ny = cy;
      if (ny < ty) ny = ty;
      else if (ny > ty + 1.0) ny = ty + 1.0;
      const double ddx = cx - nx, ddy = cy - ny;
      if (ddx * ddx + ddy * ddy < r2) return 1;
    }
  }
  return 0;
}

/* _pycore.py:307-343 */
static uint32_t touch_doors(const tc_tables *T, uint8_t *dopen_row, double cx,
                            double cy, double radius, uint8_t inv) {
  uint32_t events = 0;
  const int tx0 = (int)floor(cx - radius), tx1 = (int)floor(cx + radius);
  const int ty0 = (int)floor(cy - radius), ty1 = (int)floor(cy + radius);
  const double r2 = radius * radius;
  for (int ty = ty0; ty <= ty1; ty++) {
    for (int tx = tx0; tx <= tx1; tx++) {
      if (tx < 0 || tx >= T->w || ty < 0 || ty >= T->h) continue;
      if (T->kind[ty * T->w + tx] != C_DOOR) continue;
      const int di = T->didx[ty * T->w + tx];
      if (dopen_row[di] != 0) continue;
      double nx = cx;
      if (nx < tx) nx = tx;
      else if (nx > tx + 1.0) nx = tx + 1.0;
      double ny = cy;
      if (ny < ty) ny = ty;
      else if (ny > ty + 1.0) ny = ty + 1.0;
      const double ddx = cx - nx, ddy = cy - ny;
      if (ddx * ddx + ddy * ddy >= r2) continue;
      if (T->dlock[di] != 0 && ((inv >> T->dcol[di]) & 1) == 0) continue;
      dopen_row[di] = 1;
      events |= 1u << (EV_DOOR_BASE_BIT + T->dcol[di]);
    }
  }
  return events;
}

static int render_env(const tc_tables *T, const tc_state *S, const tc_out *O,
                      int64_t i, double *zscratch) {
  const int D = T->n_doors, E = T->n_entities;
  double *zb = O->zbuf ? O->zbuf + i * T->obs_w : zscratch;
  return render_into(
      T, S->px[i], S->py[i], S->dx[i], S->dy[i], S->dopen + i * D,
      S->ealive + i * E, S->agoal[i],
      O->frames + (size_t)i * T->obs_h * T->obs_w * 3, zb,
      O->rayinfo ? O->rayinfo + (size_t)i * T->obs_w * 4 : 0,
      O->spritevis ? O->spritevis + i : 0);
}

/* _pycore.py:390-428 */
static void reset_env(const tc_tables *T, const tc_state *S, const tc_out *O,
                      int64_t i, double *zscratch) {
  const uint64_t key = S->rkey[i];
  uint64_t ctr = S->rctr[i];
  uint64_t v = draw_below(key, &ctr, (uint64_t)T->n_spawns);
  S->px[i] = T->spx[v];
  S->py[i] = T->spy[v];
  v = draw_below(key, &ctr, 4);
  S->dx[i] = T->dirs[v * 2 + 0];
  S->dy[i] = T->dirs[v * 2 + 1];
  if (T->ic[IC_GOAL_MODE] == 1 && T->n_goals > 0) {
    v = draw_below(key, &ctr, (uint64_t)T->n_goals);
    S->agoal[i] = T->goal_ent[v];
  } else if (T->n_goals > 0) {
    S->agoal[i] = T->goal_ent[0];
  } else {
    S->agoal[i] = -1;
  }
  S->rctr[i] = ctr;
  S->health[i] = 100.0;
  S->inv[i] = 0;
  S->t[i] = 0;
  S->done[i] = 0;
  for (int d = 0; d < T->n_doors; d++) S->dopen[i * T->n_doors + d] = 0;
  for (int e = 0; e < T->n_entities; e++) S->ealive[i * T->n_entities + e] = 1;
  O->statuses[i] = render_env(T, S, O, i, zscratch);
}

/* _pycore.py:431-547 */
static int step_env(const tc_tables *T, const tc_state *S, const int64_t *acts,
                    const tc_out *O, int64_t i, int auto_reset, int validate,
                    double *zscratch) {
  const int D = T->n_doors, E = T->n_entities;
  uint8_t *dopen = S->dopen + i * D;
  uint8_t *ealive = S->ealive + i * E;
  double x = S->px[i], y = S->py[i], dxx = S->dx[i], dyy = S->dy[i];
  const int64_t act = acts[i];
  uint32_t ev = 0;
  double reward = 0.0;
  int terminated = 0, truncated = 0, violations = 0;
  const double ms = T->fc[FC_MOVE_SPEED], radius = T->fc[FC_RADIUS];

  if (act == A_TURN_LEFT || act == A_TURN_RIGHT) {
    const double s = act == A_TURN_RIGHT ? T->fc[FC_TURN_SIN] : -T->fc[FC_TURN_SIN];
    const double cs = T->fc[FC_TURN_COS];
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
    const double nx = x + mvx;
    ev |= touch_doors(T, dopen, nx, y, radius, S->inv[i]);
    if (blocked(T, dopen, nx, y, radius) == 0) x = nx;
    const double ny = y + mvy;
    ev |= touch_doors(T, dopen, x, ny, radius, S->inv[i]);
    if (blocked(T, dopen, x, ny, radius) == 0) y = ny;
    if (validate && blocked(T, dopen, x, y, radius)) violations = 1;
  }

  const int ctx = (int)floor(x), cty = (int)floor(y);
  const int e = T->eat[cty * T->w + ctx];
  if (e >= 0 && ealive[e] != 0) {
    const int kd = T->ekind[e];
    if (kd == K_KEY) {
      S->inv[i] |= (uint8_t)(1 << T->ecol[e]);
      ealive[e] = 0;
      ev |= 1u << (EV_KEY_BASE_BIT + T->ecol[e]);
    } else if (kd == K_MEDKIT) {
      ealive[e] = 0;
      const double hv = S->health[i] + T->fc[FC_HEALTH_RESTORE];
      S->health[i] = hv > 100.0 ? 100.0 : hv;
      ev |= 1u << EV_MEDKIT_BIT;
    } else if (kd == K_GOAL && e == S->agoal[i]) {
      reward = reward + T->fc[FC_GOAL_REWARD];
      terminated = 1;
      ev |= 1u << EV_GOAL_BIT;
    }
  }
  if (T->ic[IC_USE_HEALTH] != 0 && terminated == 0) {
    reward = reward + T->fc[FC_LIVING_REWARD];
    S->health[i] = S->health[i] - T->fc[FC_HEALTH_DECAY];
    if (S->health[i] <= 0.0) {
      S->health[i] = 0.0;
      terminated = 1;
      reward = 0.0;
      ev |= 1u << EV_DIED_BIT;
    }
  }
  S->t[i] = S->t[i] + 1;
  if (terminated == 0 && S->t[i] >= T->ic[IC_MAX_STEPS]) {
    truncated = 1;
    ev |= 1u << EV_TRUNCATED_BIT;
  }
  S->px[i] = x; S->py[i] = y; S->dx[i] = dxx; S->dy[i] = dyy;
  S->done[i] = (terminated != 0 || truncated != 0) ? 1 : 0;
  O->rewards[i] = reward;
  O->dones[i] = S->done[i];
  O->truncs[i] = (uint8_t)truncated;
  O->events[i] = ev;
  if (S->done[i] != 0 && auto_reset != 0) reset_env(T, S, O, i, zscratch);
  else O->statuses[i] = render_env(T, S, O, i, zscratch);
  return violations;
}

/* ---------------------------------------------------------------- exports */

int orc_cast_ray(const uint8_t *kind, const int16_t *didx,
                 const uint8_t *dopen, int32_t h, int32_t w, double ox,
                 double oy, double rx, double ry, int32_t *out4, double *out2) {
  int mapx, mapy, side, steps;
  double perp, wu;
  int st = cast_ray(kind, didx, dopen, h, w, ox, oy, rx, ry, &mapx, &mapy,
                    &side, &perp, &wu, &steps);
  out4[0] = mapx; out4[1] = mapy; out4[2] = side; out4[3] = steps;
  out2[0] = perp; out2[1] = wu;
  return st;
}

int orc_render_into(const tc_tables *T, double px, double py, double dx,
                    double dy, const uint8_t *dopen_row,
                    const uint8_t *ealive_row, int32_t agoal, uint8_t *frame,
                    double *zbuf, int32_t *rayinfo, uint64_t *spritevis) {
  return render_into(T, px, py, dx, dy, dopen_row, ealive_row, agoal, frame,
                     zbuf, rayinfo, spritevis);
}

/* _pycore.py:346-387; OpenMP static schedule over envs like _core.pyx:745-762.
 * Results never depend on n_threads. */
int64_t orc_batch_kernel(const tc_tables *T, const tc_state *S,
                         const int64_t *actions, const tc_out *O, int64_t n,
                         int32_t mode, int32_t auto_reset, int32_t validate,
                         int32_t n_threads) {
  int64_t violations = 0;
  const int nt = n_threads > 0 ? n_threads : 1;
  (void)nt;
#pragma omp parallel num_threads(nt) reduction(+ : violations)
  {
    double zscratch[TC_MAX_OBS_W];
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; i++) {
      if (mode == TC_MODE_RESET) reset_env(T, S, O, i, zscratch);
      else violations += step_env(T, S, actions, O, i, auto_reset, validate, zscratch);
    }
  }
  return violations;
}

/* batch.py:81-85 with rng.py:36-38 / :56-59 */
void orc_seed_streams(uint64_t seed, int64_t base, int64_t n, uint64_t *rkey,
                      uint64_t *rctr) {
  const uint64_t root = mix64(seed);
  for (int64_t i = 0; i < n; i++) {
    rkey[i] = mix64(root + SPLIT_SALT + (uint64_t)(base + i) * GOLDEN);
    rctr[i] = 0;
  }
}

/* batch.py:141-153 with rng.py:62-93 (one step row of the action table) */
void orc_policy_actions(uint64_t policy_key, int64_t step, int64_t n_total,
                        int64_t base, int64_t n, const int64_t *tags,
                        int32_t n_tags, int64_t *actions) {
  for (int64_t i = 0; i < n; i++) {
    uint64_t ctr = (uint64_t)(step * n_total + base + i);
    actions[i] = tags[draw_below(policy_key, &ctr, (uint64_t)n_tags)];
  }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
