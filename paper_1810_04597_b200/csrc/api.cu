// api.cu — the C-ABI of include/echo.h: context, device allocations, stage
// orchestration on one CUDA stream, CFL readback, counters, profiling.
// Every step of the path runs in the kernels of march.cu / update.cu; this file
// only allocates, validates, launches and copies.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/echo.h"
#include "echo_dev.cuh"
#include "echo_kernels.h"
#include "metric_tables.h"

using namespace echo;

namespace {

enum KernelClass {
  kSweepX = 0, kSweepY, kSweepZ, kUpdateStage, kUpdateRhs, kC2P, kMaxSpeed, kPrim2Cons, kGetPrims, kLayout,
  kCflDt, kUctEmf, kUctInduct, kUctCell, kNanScan, kUpdateSweepX, kNumClasses
};
const char* kNames[kNumClasses] = {"sweep_x",   "sweep_y",   "sweep_z",   "update_stage", "update_rhs",
                                   "con2prim",  "max_speed", "prim2cons", "get_prims",    "layout",
                                   "cfl_dt",    "uct_emf",   "uct_induct", "uct_cell", "nan_scan", "update_sweep_x"};

std::string g_create_error;

}  // namespace

struct echo_ctx {
  GridP g;
  EosP e;
  bool ks = false;
  MetTables mt{};
  double* tables = nullptr;
  // cell-interleaved device state (echo_kernels.h): 8 doubles per cell each
  double* alloc_base[4] = {nullptr, nullptr, nullptr, nullptr};  // allocations (slab mode: incl. ghost planes)
  echo_ctx* link[2] = {nullptr, nullptr};  // slab mode: neighbours whose ghost planes K3 writes (echo_halo_link)
  std::vector<echo_ctx*> linked_by;         // contexts whose link[] points here (cleared by echo_destroy)
  // ... or a neighbour in another process: its P, Un, Us (plane 0) mapped by CUDA IPC
  struct Remote {
    double* base[3] = {nullptr, nullptr, nullptr};  // opened allocation bases (P, Un, Us)
    double* P = nullptr;
    double* Un = nullptr;
    double* Us = nullptr;
    int nz = 0;
  } rlink[2];
  int swept = 0;                           // stage whose sweeps ran (echo_stage_sweeps), 0 = none
  int swept_int = 0;                       // stage whose interior sweeps ran (echo_stage_sweeps_interior)
  int inducted = 0;                        // UCT slabs: stage whose induction ran (echo_stage_update_field)
  size_t plane = 0;       // doubles per z plane of a record array (pitch n2)
  double* Un = nullptr;   // U^n
  double* Us = nullptr;   // U^s
  double* P = nullptr;    // rho, u~, p, B
  double* R = nullptr;    // rhs + EMF accumulator
  // fused update + x sweep (fused.cu): the update of a stage writes the x sweep of the state it
  // produces into the OTHER accumulator (its own curl still reads this stage's EMF)
  double* R2 = nullptr;   // second accumulator (fuse only)
  double* uct_base[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // allocations of Bst, FS[3], Ed
  // guard bands (ECHO_GUARD_BANDS=1, contexts without halo boundaries): `guard` doubles of 0xA5
  // bytes before and after every state array, checked by echo_check_guards
  size_t guard = 0;
  std::vector<std::pair<double*, size_t>> guarded;  // (allocation base, doubles between the bands)
  int rsel = 0;           // accumulator of the current stage input: 0 R, 1 R2
  bool xahead = false;    // racc() already holds the x sweep of the current stage input
  bool fuse = false;      // fused update + x sweep (Minkowski, no slabs, no UCT; opt-in ECHO_FUSED_UPDATE=1)
  cudaGraphExec_t step_exec_p[2] = {nullptr, nullptr};  // echo_advance step graphs by entry rsel (fuse)
  // UCT (divb = 2, uct.cu): staggered field (slots 0..2 b^n, 3..5 b^s), face data per axis, edge EMFs
  double* Bst = nullptr;
  double* FS[3] = {nullptr, nullptr, nullptr};
  double* Ed = nullptr;
  bool have_faces = false;
  double* scratch = nullptr;  // 8N, lazily for layout conversions / host-buffer transfers
  unsigned long long* dcnt = nullptr;  // [0] floors [1] failures [2] max speed bits
  long long* dbad = nullptr;
  long long* dnan = nullptr;  // first non-finite value (cell id * 16 + slot) of the debug scan
  int debug = 0;              // ECHO_DEBUG_* flags
  unsigned long long* hpin = nullptr;  // pinned readback
  cudaStream_t st = nullptr;
  bool have_state = false;
  bool cfl_valid = false;  // dcnt[2] holds the CFL max of the current state (fused into the last update)
  int next_stage = 1;
  unsigned long long steps = 0, stages = 0;
  long long launches = 0;
  // device-driven time loop (echo_advance): adv = [dt, halt, steps done], then the dt log
  double* dadv = nullptr;
  long long dlog_cap = 0;
  cudaStream_t cap_st = nullptr;       // private stream the step graph is captured on
  cudaGraphExec_t step_exec = nullptr;  // one step: k_cfl_dt + 3 x (3 sweeps + update)
  double step_cfl = 0.0;               // the cfl baked into step_exec
  long long step_kernels = 0;          // kernels per replay
  std::string err;
  // profiling
  bool prof = false;
  struct Rec { int cls; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  double prof_ms[kNumClasses] = {0};
  long long prof_n[kNumClasses] = {0};
};

static int fail(echo_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  else g_create_error = msg;
  return code;
}
static int cuda_fail(echo_ctx* c, cudaError_t e, const char* where) {
  return fail(c, ECHO_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(call, where)                          \
  do {                                           \
    cudaError_t _e = (call);                     \
    if (_e != cudaSuccess) return cuda_fail(c, _e, where); \
  } while (0)

// launch bracket: profiling events + launch count
template <class F>
static cudaError_t launch(echo_ctx* c, int cls, F&& f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->prof) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, c->st);
  }
  cudaError_t e = f();
  c->launches++;
  if (c->prof) {
    cudaEventRecord(b, c->st);
    c->recs.push_back({cls, a, b});
  }
  return e;
}

static double* racc(echo_ctx* c) { return c->rsel ? c->R2 : c->R; }
static const double* ucur(echo_ctx* c) { return c->next_stage == 1 ? c->Un : c->Us; }
static double* ucur_mut(echo_ctx* c) { return c->next_stage == 1 ? c->Un : c->Us; }

static int ensure_scratch(echo_ctx* c) {
  if (c->scratch) return ECHO_OK;
  cudaError_t e = cudaMalloc(&c->scratch, sizeof(double) * 8 * c->g.N);
  if (e != cudaSuccess) return fail(c, ECHO_E_OOM, "echo: scratch allocation failed");
  return ECHO_OK;
}

static bool is_uct(const echo_ctx* c) { return c->g.divb == 2; }
// the stage-input staggered field (UCT)
static double* bcur(echo_ctx* c) { return c->Bst + (c->next_stage == 1 ? 0 : 3) * c->g.vs; }

// sweeps x, y, z of the current stage input P (B included) into R; UCT: then the edge EMFs.
// part (slab mode, the halo exchange overlapped): 1 = x/y over the owned planes only (they read
// no ghost plane), 2 = x/y over the first ghost plane of each side, then z; 0 = everything.
static int run_sweeps(echo_ctx* c, int part = 0) {
  const bool uct = is_uct(c);
  auto sweep = [&](int ax, PlaneRange zr) {
    cudaError_t e = launch(c, kSweepX + ax, [&] {
      return launch_march(ax, c->ks, c->g, c->e, c->mt, c->P, c->ks ? c->P : ucur(c), racc(c), c->st,
                          uct ? bcur(c) : nullptr, uct ? c->FS[ax] : nullptr, zr);
    });
    return e == cudaSuccess ? ECHO_OK : cuda_fail(c, e, "sweep launch");
  };
  if (part == 1 || part == 2) {
    for (int ax = 0; ax < 2; ax++) {
      if (part == 1) {
        int rc = sweep(ax, PlaneRange{0, c->g.n[2]});
        if (rc) return rc;
      } else {
        for (int zb : {-1, c->g.n[2]}) {
          int rc = sweep(ax, PlaneRange{zb, 1});
          if (rc) return rc;
        }
      }
    }
    return part == 2 ? sweep(2, PlaneRange{}) : ECHO_OK;
  }
  for (int ax = c->xahead ? 1 : 0; ax < 3; ax++) {  // (the fused update already swept x)
    int rc = sweep(ax, PlaneRange{});
    if (rc) return rc;
  }
  c->xahead = false;
  if (uct) {
    const double* fs[3] = {c->FS[0], c->FS[1], c->FS[2]};
    cudaError_t e = launch(c, kUctEmf, [&] { return launch_uct_emf(c->g, fs, bcur(c), c->Ed, c->st); });
    if (e != cudaSuccess) return cuda_fail(c, e, "uct emf launch");
  }
  return ECHO_OK;
}

static void ipc_close(echo_ctx::Remote& rm) {
  for (double*& b : rm.base)
    if (b) {
      cudaIpcCloseMemHandle(b);
      b = nullptr;
    }
  rm.P = rm.Un = rm.Us = nullptr;
}

// the fused ghost exchange of slab mode for stage s (targets: the linked neighbours' P and
// same-role U arrays, shifted so that my record offset lands in their ghost planes)
static GhostLinks ghost_links(echo_ctx* c, int s) {
  GhostLinks gl{};
  if (!c->g.zhalo) return gl;
  const long long plane = (long long)c->g.n[1] * c->g.pitch;
  for (int side = 0; side < 2; side++) {
    echo_ctx* nb = c->link[side];
    const echo_ctx::Remote& rm = c->rlink[side];
    double *nP = nullptr, *nUn = nullptr, *nUs = nullptr;
    int nnz = 0;
    if (nb) {
      nP = nb->P, nUn = nb->Un, nUs = nb->Us, nnz = nb->g.n[2];
    } else if (rm.P) {
      nP = rm.P, nUn = rm.Un, nUs = rm.Us, nnz = rm.nz;
    }
    if (nP) {
      // side 0: my plane k (< 6) -> the lower neighbour's plane nz_nb + k;
      // side 1: my plane k (>= nz - 6) -> the upper neighbour's plane k - nz
      const long long shift = side == 0 ? (long long)nnz * plane : -(long long)c->g.n[2] * plane;
      gl.dstP[side] = nP + shift;
      gl.dstU[side] = (s == 3 ? nUn : nUs) + shift;
      gl.on = 1;
    }
    if (c->g.bc[2][side] == ECHO_BC_OUTFLOW) {
      gl.replicate[side] = 1;
      gl.on = 1;
    }
  }
  return gl;
}

// part (UCT slabs, whose cell update centres the new b^z of 3 ghost faces that the neighbour's
// induction writes): 1 = the induction only, 2 = the cell update only, 0 = both
static int run_update(echo_ctx* c, int s, double dt, const double* dtp = nullptr, int part = 0) {
  const double* Uin = (s == 1) ? c->Un : c->Us;
  double* Uout = (s == 3) ? c->Un : c->Us;
  // the last stage also reduces the CFL rate of the new state (a9 fused into K3)
  unsigned long long* cfl = (s == 3) ? c->dcnt + 2 : nullptr;
  if (cfl) CK(cudaMemsetAsync(cfl, 0, sizeof(unsigned long long), c->st), "stage");
  if (is_uct(c)) {  // staggered field first (A41), then the cells read its centring (A37)
    cudaError_t e = cudaSuccess;
    if (part != 2)
      e = launch(c, kUctInduct, [&] {
        return launch_uct_induct(c->g, 0, s, dt, dtp, c->Ed, c->Bst, nullptr, c->st);
      });
    if (part == 1) {
      if (e != cudaSuccess) return cuda_fail(c, e, "uct induction launch");
      c->inducted = s;
      return ECHO_OK;
    }
    c->inducted = 0;
    if (e == cudaSuccess)
      e = launch(c, kUctCell, [&] {
        return launch_uct_cell(c->ks, c->g, c->e, c->mt, s, dt, dtp, racc(c), c->Un, Uin, Uout, c->P, c->Bst, c->dcnt,
                               cfl, c->st);
      });
    if (e != cudaSuccess) return cuda_fail(c, e, "uct update launch");
    if (c->debug & ECHO_DEBUG_NANSCAN) {
      e = launch(c, kNanScan, [&] { return launch_nanscan(c->g, Uout, c->P, c->ks ? 8 : 5, c->dnan, dtp ? c->dadv : nullptr, c->st); });
      if (e != cudaSuccess) return cuda_fail(c, e, "nan scan launch");
    }
    c->cfl_valid = (s == 3);
    c->stages++;
    c->next_stage = (s == 3) ? 1 : s + 1;
    c->swept = 0;
  c->swept_int = 0;
  c->inducted = 0;
    return ECHO_OK;
  }
  const GhostLinks gl = ghost_links(c, s);
  cudaError_t e;
  if (c->fuse) {  // the update of stage s + the x sweep of the state it produces (fused.cu)
    double* Rnew = c->rsel ? c->R : c->R2;
    e = launch(c, kUpdateSweepX, [&] {
      return launch_update_march(c->ks, c->g, c->e, c->mt, s, dt, dtp, racc(c), c->Un, Uin, Uout, c->P, c->dcnt, cfl,
                                 Rnew, c->st);
    });
    c->rsel ^= 1;
    c->xahead = true;
  } else {
    e = launch(c, kUpdateStage, [&] {
      return launch_update(kModeStage, c->ks, c->g, c->e, c->mt, s, dt, racc(c), c->Un, Uin, Uout, c->P, nullptr,
                           c->dcnt, cfl, c->st, &gl, dtp);
    });
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "update launch");
  if (c->debug & ECHO_DEBUG_NANSCAN) {
    e = launch(c, kNanScan, [&] { return launch_nanscan(c->g, Uout, c->P, c->ks ? 8 : 5, c->dnan, dtp ? c->dadv : nullptr, c->st); });
    if (e != cudaSuccess) return cuda_fail(c, e, "nan scan launch");
  }
  c->cfl_valid = (s == 3);
  c->stages++;
  c->next_stage = (s == 3) ? 1 : s + 1;
  c->swept = 0;
  c->swept_int = 0;
  c->inducted = 0;
  return ECHO_OK;
}

// the debug scan's verdict (synchronises): ECHO_E_NONFINITE naming the first bad value
static int nan_report(echo_ctx* c, const char* where) {
  long long code = LLONG_MAX;
  CK(cudaMemcpyAsync(&code, c->dnan, sizeof code, cudaMemcpyDeviceToHost, c->st), where);
  CK(cudaStreamSynchronize(c->st), where);
  if (code == LLONG_MAX) return ECHO_OK;
  const long long id = code / 16;
  const int q = (int)(code % 16);
  double v = 0.0;
  const long long r = id / c->g.n[0];
  const long long off = r * c->g.pitch + (id - r * c->g.n[0]) + (long long)(q % 8) * c->g.vs;
  cudaMemcpy(&v, (q < 8 ? (const double*)ucur(c) : c->P) + off, sizeof v, cudaMemcpyDeviceToHost);
  const long long i = id % c->g.n[0], j = (id / c->g.n[0]) % c->g.n[1], k = id / ((long long)c->g.n[0] * c->g.n[1]);
  char buf[300];
  std::snprintf(buf, sizeof buf, "%s: non-finite state value %s[%d] = %g at cell (%lld,%lld,%lld)", where,
                q < 8 ? "U" : "P", q % 8, v, i, j, k);
  const long long init = LLONG_MAX;
  cudaMemcpy(c->dnan, &init, sizeof init, cudaMemcpyHostToDevice);
  return fail(c, ECHO_E_NONFINITE, buf);
}

static int run_stage(echo_ctx* c, int s, double dt) {
  int rc = run_sweeps(c);
  if (rc) return rc;
  rc = run_update(c, s, dt);
  if (rc) return rc;
  if (c->debug & ECHO_DEBUG_NANSCAN) return nan_report(c, s == 1 ? "stage 1" : (s == 2 ? "stage 2" : "stage 3"));
  return ECHO_OK;
}

extern "C" {

int echo_create(const echo_grid* grid, const echo_metric* metric, const echo_eos* eos, echo_ctx** out) {
  echo_ctx* c = nullptr;
  if (out) *out = nullptr;
  if (!grid || !metric || !eos || !out) return fail(nullptr, ECHO_E_ARG, "echo_create: NULL argument");
  for (int a = 0; a < 3; a++) {
    if (grid->n[a] < 1) return fail(nullptr, ECHO_E_ARG, "echo_create: n[a] >= 1 violated");
    if (!(grid->hi[a] > grid->lo[a])) return fail(nullptr, ECHO_E_ARG, "echo_create: lo < hi violated");
    for (int s = 0; s < 2; s++)
      if (grid->bc[a][s] != ECHO_BC_PERIODIC && grid->bc[a][s] != ECHO_BC_OUTFLOW &&
          !(grid->bc[a][s] == ECHO_BC_HALO && a == 2))
        return fail(nullptr, ECHO_E_ARG, "echo_create: unknown boundary condition (ECHO_BC_HALO only on axis 2)");
    if ((grid->bc[a][0] == ECHO_BC_PERIODIC) != (grid->bc[a][1] == ECHO_BC_PERIODIC))
      return fail(nullptr, ECHO_E_ARG, "echo_create: periodic must be set on both sides of an axis");
  }
  {
    const bool zh = grid->bc[2][0] == ECHO_BC_HALO || grid->bc[2][1] == ECHO_BC_HALO;
    if (zh && grid->n[2] < (grid->divb == 2 ? ECHO_HALO_PLANES_UCT : ECHO_HALO_PLANES))
      return fail(nullptr, ECHO_E_ARG,
                  "echo_create: a slab with halo boundaries needs n[2] >= ECHO_HALO_PLANES (UCT: ECHO_HALO_PLANES_UCT)");
  }
  if (grid->rec < 0 || grid->rec > 6) return fail(nullptr, ECHO_E_ARG, "echo_create: rec must be 0..6");
  if (grid->rec == 6 && (metric->kind != ECHO_METRIC_MINKOWSKI || grid->divb == 2))
    return fail(nullptr, ECHO_E_ARG, "echo_create: rec = 6 (characteristic-wise, A44) needs the Minkowski metric and divb != 2");
  if (grid->der != 2 && grid->der != 4 && grid->der != 6) return fail(nullptr, ECHO_E_ARG, "echo_create: der must be 2, 4 or 6");
  if (grid->divb < 0 || grid->divb > 2) return fail(nullptr, ECHO_E_ARG, "echo_create: divb must be 0, 1 or 2");
  // UCT (A37, A42, A43): periodic, outflow or (z) slab axes, any metric; slabs with the copy exchange
  if (!(eos->gamma > 1.0)) return fail(nullptr, ECHO_E_ARG, "echo_create: gamma > 1 violated");
  if (!(eos->rho_floor > 0.0) || !(eos->p_floor > 0.0)) return fail(nullptr, ECHO_E_ARG, "echo_create: floors > 0 violated");
  if (!(eos->w_max > 1.0)) return fail(nullptr, ECHO_E_ARG, "echo_create: w_max > 1 violated");
  if (eos->c2p_max_iter < 1 || !(eos->c2p_tol > 0.0)) return fail(nullptr, ECHO_E_ARG, "echo_create: c2p controls invalid");
  if (metric->kind != ECHO_METRIC_MINKOWSKI && metric->kind != ECHO_METRIC_KERR_SCHILD)
    return fail(nullptr, ECHO_E_ARG, "echo_create: unknown metric kind");
  const bool ks = metric->kind == ECHO_METRIC_KERR_SCHILD;
  if (ks) {
    if (!(metric->M >= 0.0)) return fail(nullptr, ECHO_E_ARG, "echo_create: Kerr-Schild needs M >= 0");
    // every centre and face of the ghost-extended theta range must avoid the polar axis (sin theta = 0)
    double d2 = (grid->hi[1] - grid->lo[1]) / grid->n[1];
    for (int h = -2 * kG; h <= 2 * grid->n[1] + 2 * kG; h++) {
      double th = grid->lo[1] + 0.5 * h * d2;
      if (!(std::fabs(std::sin(th)) > 1e-12))
        return fail(nullptr, ECHO_E_ARG, "echo_create: Kerr-Schild theta grid (with 5 ghost cells) touches sin(theta) = 0");
    }
  }
  int dev;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return fail(nullptr, ECHO_E_CUDA, std::string("echo_create: no CUDA device: ") + cudaGetErrorString(ce));

  c = new echo_ctx();
  GridP& g = c->g;
  g.N = 1;
  for (int a = 0; a < 3; a++) {
    g.n[a] = grid->n[a];
    g.N *= grid->n[a];
    g.lo[a] = grid->lo[a];
    g.dx[a] = (grid->hi[a] - grid->lo[a]) / grid->n[a];
    g.idx[a] = 1.0 / g.dx[a];
    g.bc[a][0] = grid->bc[a][0];
    g.bc[a][1] = grid->bc[a][1];
  }
  if (grid->dz > 0.0) {  // a slab: the global grid's Delta_z bit for bit (echo.h)
    if (!(std::fabs(grid->dz * grid->n[2] - (grid->hi[2] - grid->lo[2])) <= 1e-12 * std::fabs(grid->hi[2] - grid->lo[2]))) {
      delete c;
      return fail(nullptr, ECHO_E_ARG, "echo_create: dz * n[2] must equal hi[2] - lo[2]");
    }
    g.dx[2] = grid->dz;
    g.idx[2] = 1.0 / grid->dz;
  }
  g.rec = grid->rec;
  g.der = grid->der;
  g.divb = grid->divb;
  g.der_jump = grid->der_jump > 0.0 ? grid->der_jump : INFINITY;  // A31 off: a test that never fires
  EosP& e = c->e;
  e.gamma = eos->gamma;
  e.gfac = eos->gamma / (eos->gamma - 1.0);
  e.gm = (eos->gamma - 1.0) / eos->gamma;
  e.rho_floor = eos->rho_floor;
  e.p_floor = eos->p_floor;
  e.w_max = eos->w_max;
  e.v2max = 1.0 - 1.0 / (eos->w_max * eos->w_max);
  e.maxit = eos->c2p_max_iter;
  e.tol = eos->c2p_tol;
  c->ks = ks;

  // record rows: 8 n1 doubles + 8 (64 B) padding, so that row and plane strides
  // are not powers of two (DRAM channel spread of the y/z pencils)
  g.vs = g.n[0] + (g.n[0] & 1);
  g.pitch = 8LL * g.vs + 8;
  // slab mode (z boundaries of kind ECHO_BC_HALO): kZH stored ghost planes below and above
  // the owned ones in every record array; the array pointers point at plane 0
  g.zhalo = (g.bc[2][0] == ECHO_BC_HALO || g.bc[2][1] == ECHO_BC_HALO) ? (g.divb == 2 ? kZHU : kZH) : 0;
  c->plane = (size_t)g.pitch * g.n[1];
  const size_t ghost = (size_t)g.zhalo * c->plane;
  const size_t rec = c->plane * g.n[2] + 2 * ghost;  // doubles per record array
  {
    const char* gb = std::getenv("ECHO_GUARD_BANDS");
    c->guard = (gb && gb[0] == '1' && !g.zhalo) ? 4096 : 0;  // 32 KB per side
  }
  // a state array of n doubles between two guard bands; *base = the allocation (for cudaFree / IPC)
  auto galloc = [&](size_t n, double** base) -> double* {
    *base = nullptr;
    if (cudaMalloc(base, sizeof(double) * (n + 2 * c->guard)) != cudaSuccess) {
      *base = nullptr;
      return nullptr;
    }
    if (c->guard) {
      cudaMemset(*base, 0xA5, sizeof(double) * c->guard);
      cudaMemset(*base + c->guard + n, 0xA5, sizeof(double) * c->guard);
      c->guarded.push_back({*base, n});
    }
    return *base + c->guard;
  };
  auto alloc = [&](int slot, double** p) {
    double* q = galloc(rec, &c->alloc_base[slot]);
    *p = q ? q + ghost : nullptr;
    return q ? cudaSuccess : cudaErrorMemoryAllocation;
  };
  if (alloc(0, &c->Un) != cudaSuccess || alloc(1, &c->Us) != cudaSuccess || alloc(2, &c->P) != cudaSuccess ||
      alloc(3, &c->R) != cudaSuccess ||
      cudaMalloc(&c->dcnt, 4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&c->dbad, sizeof(long long)) != cudaSuccess || cudaMalloc(&c->dnan, sizeof(long long)) != cudaSuccess ||
      cudaMallocHost(&c->hpin, 4 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    echo_destroy(c);
    return fail(nullptr, ECHO_E_OOM, "echo_create: device allocation failed");
  }
  {  // fused update + x sweep (opt-in, ECHO_FUSED_UPDATE=1: measured slower): a second
     // accumulator (without memory for it the kernels stay separate)
    const char* fu = std::getenv("ECHO_FUSED_UPDATE");
    c->fuse = !ks && !g.zhalo && g.divb != 2 && fu && fu[0] == '1';
    double* base = nullptr;
    if (c->fuse && !(c->R2 = galloc(rec, &base))) {
      cudaGetLastError();
      c->fuse = false;
    }
  }
  if (g.divb == 2) {
    // (slab mode: like the record arrays, the pointers point at plane 0, ghost planes before)
    double** uct_arrays[5] = {&c->Bst, &c->FS[0], &c->FS[1], &c->FS[2], &c->Ed};
    for (int q = 0; q < 5; q++) {
      double* a = galloc(rec, &c->uct_base[q]);
      if (!a) {
        cudaGetLastError();
        echo_destroy(c);
        return fail(nullptr, ECHO_E_OOM, "echo_create: UCT field allocation failed");
      }
      cudaMemset(a, 0, sizeof(double) * rec);
      *uct_arrays[q] = a + ghost;
    }
  }
  cudaMemset(c->dcnt, 0, 4 * sizeof(unsigned long long));
  for (double* b : c->alloc_base)
    if (b) cudaMemset(b + c->guard, 0, sizeof(double) * rec);
  if (ks) {
    KsTables t;
    build_ks_tables(metric->M, metric->a, g.n, g.lo, g.dx, &t);
    size_t total = t.cen.size() + t.der.size() + t.f0.size() + t.f1.size();
    if (cudaMalloc(&c->tables, sizeof(double) * total) != cudaSuccess) {
      echo_destroy(c);
      return fail(nullptr, ECHO_E_OOM, "echo_create: metric table allocation failed");
    }
    double* p = c->tables;
    cudaMemcpy(p, t.cen.data(), sizeof(double) * t.cen.size(), cudaMemcpyHostToDevice);
    c->mt.cen = p;
    p += t.cen.size();
    cudaMemcpy(p, t.der.data(), sizeof(double) * t.der.size(), cudaMemcpyHostToDevice);
    c->mt.der = p;
    p += t.der.size();
    cudaMemcpy(p, t.f0.data(), sizeof(double) * t.f0.size(), cudaMemcpyHostToDevice);
    c->mt.f0 = p;
    p += t.f0.size();
    cudaMemcpy(p, t.f1.data(), sizeof(double) * t.f1.size(), cudaMemcpyHostToDevice);
    c->mt.f1 = p;
    c->mt.w0 = t.w0;
  }
  {
    const long long init = LLONG_MAX;
    cudaMemcpy(c->dnan, &init, sizeof init, cudaMemcpyHostToDevice);
    const char* dbg = std::getenv("ECHO_DEBUG_NANSCAN");
    if (dbg && dbg[0] == '1') c->debug = ECHO_DEBUG_NANSCAN;
  }
  ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) {
    echo_destroy(c);
    return fail(nullptr, ECHO_E_CUDA, std::string("echo_create: ") + cudaGetErrorString(ce));
  }
  *out = c;
  return ECHO_OK;
}

static void drop_backref(echo_ctx* peer, echo_ctx* c) {
  auto& v = peer->linked_by;
  for (size_t i = 0; i < v.size(); i++)
    if (v[i] == c) {
      v.erase(v.begin() + i);
      return;
    }
}

void echo_destroy(echo_ctx* c) {
  if (!c) return;
  // unlink both ways: no surviving context may keep storing into this one's ghost planes
  for (echo_ctx* x : c->linked_by)
    for (auto& l : x->link)
      if (l == c) l = nullptr;
  for (auto& l : c->link)
    if (l && l != c) drop_backref(l, c);
  for (auto& rm : c->rlink) ipc_close(rm);
  for (double* b : c->alloc_base) cudaFree(b);
  cudaFree(c->scratch);
  cudaFree(c->dcnt);
  cudaFree(c->dbad);
  cudaFree(c->dnan);
  cudaFree(c->R2 ? c->R2 - c->guard : nullptr);
  for (auto& x : c->step_exec_p)
    if (x) cudaGraphExecDestroy(x);
  cudaFree(c->tables);
  cudaFree(c->dadv);
  for (double* b : c->uct_base) cudaFree(b);
  if (c->step_exec) cudaGraphExecDestroy(c->step_exec);
  if (c->cap_st) cudaStreamDestroy(c->cap_st);
  if (c->hpin) cudaFreeHost(c->hpin);
  for (auto& r : c->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  delete c;
}

int echo_set_stream(echo_ctx* c, void* stream) {
  if (!c) return ECHO_E_ARG;
  c->st = (cudaStream_t)stream;
  return ECHO_OK;
}

int echo_set_prims(echo_ctx* c, const double* p8, int on_device) {
  if (!c || !p8) return c ? fail(c, ECHO_E_ARG, "echo_set_prims: NULL buffer") : ECHO_E_ARG;
  const size_t bytes = sizeof(double) * 8 * c->g.N;
  const double* src = p8;
  if (!on_device) {
    int rc = ensure_scratch(c);
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->scratch, p8, bytes, cudaMemcpyHostToDevice, c->st), "echo_set_prims copy");
    src = c->scratch;
  }
  const long long init = LLONG_MAX;
  CK(cudaMemcpyAsync(c->dbad, &init, sizeof(long long), cudaMemcpyHostToDevice, c->st), "echo_set_prims");
  cudaError_t e = launch(c, kPrim2Cons, [&] {
    return launch_prim2cons(c->ks, c->g, c->e, c->mt, src, c->P, c->Un, c->dbad, c->st);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "prim2cons launch");
  long long bad = 0;
  CK(cudaMemcpyAsync(&bad, c->dbad, sizeof(long long), cudaMemcpyDeviceToHost, c->st), "echo_set_prims");
  CK(cudaStreamSynchronize(c->st), "echo_set_prims");
  if (bad != LLONG_MAX) {
    double v[8];
    const double* base = on_device ? p8 : nullptr;
    for (int q = 0; q < 8; q++) {
      if (base) cudaMemcpy(&v[q], base + q * c->g.N + bad, sizeof(double), cudaMemcpyDeviceToHost);
      else v[q] = p8[q * c->g.N + bad];
    }
    long long i = bad % c->g.n[0], j = (bad / c->g.n[0]) % c->g.n[1], k = bad / ((long long)c->g.n[0] * c->g.n[1]);
    char buf[400];
    snprintf(buf, sizeof buf,
             "echo_set_prims: unphysical state (rho > 0, p > 0, v^2 < 1 violated) at cell (%lld,%lld,%lld): "
             "rho=%.17g v=(%.17g,%.17g,%.17g) p=%.17g B=(%.17g,%.17g,%.17g)",
             i, j, k, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
    c->have_state = false;
    return fail(c, ECHO_E_UNPHYSICAL, buf);
  }
  c->have_state = true;
  c->have_faces = false;
  c->cfl_valid = false;
  c->next_stage = 1;
  c->xahead = false;
  c->swept = 0;
  c->swept_int = 0;
  c->inducted = 0;
  return ECHO_OK;
}

int echo_get_prims(echo_ctx* c, double* p8, int on_device) {
  if (!c || !p8) return c ? fail(c, ECHO_E_ARG, "echo_get_prims: NULL buffer") : ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_get_prims: no state (call echo_set_prims first)");
  double* dst = p8;
  if (!on_device) {
    int rc = ensure_scratch(c);
    if (rc) return rc;
    dst = c->scratch;
  }
  cudaError_t e = launch(c, kGetPrims, [&] { return launch_get_prims(c->ks, c->g, c->mt, c->P, ucur(c), dst, c->st); });
  if (e != cudaSuccess) return cuda_fail(c, e, "get_prims launch");
  if (!on_device) {
    CK(cudaMemcpyAsync(p8, c->scratch, sizeof(double) * 8 * c->g.N, cudaMemcpyDeviceToHost, c->st), "echo_get_prims");
    CK(cudaStreamSynchronize(c->st), "echo_get_prims");
  }
  return ECHO_OK;
}

// device record array [cell][8] -> caller array [q][cell] (first nq slots)
static int export_field(echo_ctx* c, double* dst, const double* src, int nq, int on_device, const char* where) {
  double* d = dst;
  if (!on_device) {
    int rc = ensure_scratch(c);
    if (rc) return rc;
    d = c->scratch;
  }
  CK(launch(c, kLayout, [&] { return launch_layout(c->g, src, d, nq, true, c->st); }), where);
  if (!on_device) {
    CK(cudaMemcpyAsync(dst, c->scratch, sizeof(double) * nq * c->g.N, cudaMemcpyDeviceToHost, c->st), where);
    CK(cudaStreamSynchronize(c->st), where);
  }
  return ECHO_OK;
}

int echo_get_cons(echo_ctx* c, double* u8, int on_device) {
  if (!c || !u8) return c ? fail(c, ECHO_E_ARG, "echo_get_cons: NULL buffer") : ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_get_cons: no state");
  return export_field(c, u8, ucur(c), 8, on_device, "echo_get_cons");
}

int echo_get_state(echo_ctx* c, double* un8, double* us8, double* p5, int on_device) {
  if (!c) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_get_state: no state");
  int rc = ECHO_OK;
  if (un8 && !rc) rc = export_field(c, un8, c->Un, 8, on_device, "echo_get_state");
  if (us8 && !rc) rc = export_field(c, us8, c->Us, 8, on_device, "echo_get_state");
  if (p5 && !rc) rc = export_field(c, p5, c->P, 5, on_device, "echo_get_state");
  return rc;
}

int echo_set_face_field(echo_ctx* c, const double* b3, int on_device) {
  if (!c || !b3) return c ? fail(c, ECHO_E_ARG, "echo_set_face_field: NULL buffer") : ECHO_E_ARG;
  if (!is_uct(c)) return fail(c, ECHO_E_ORDER, "echo_set_face_field: the context is not divb = 2 (UCT)");
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_set_face_field: needs a prior echo_set_prims (hydro state)");
  const double* src = b3;
  if (!on_device) {
    int rc = ensure_scratch(c);
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->scratch, b3, sizeof(double) * 3 * c->g.N, cudaMemcpyHostToDevice, c->st),
       "echo_set_face_field");
    src = c->scratch;
  }
  CK(launch(c, kLayout, [&] { return launch_layout(c->g, src, c->Bst, 3, false, c->st); }), "echo_set_face_field");
  CK(launch(c, kPrim2Cons, [&] { return launch_uct_centre_p2c(c->ks, c->g, c->e, c->mt, c->P, c->Un, c->Bst, c->st); }),
     "echo_set_face_field");
  if (!on_device) CK(cudaStreamSynchronize(c->st), "echo_set_face_field");
  c->have_faces = true;
  c->cfl_valid = false;
  c->next_stage = 1;
  c->xahead = false;
  c->swept = 0;
  c->swept_int = 0;
  c->inducted = 0;
  return ECHO_OK;
}

int echo_get_face_field(echo_ctx* c, double* b3, int on_device) {
  if (!c || !b3) return c ? fail(c, ECHO_E_ARG, "echo_get_face_field: NULL buffer") : ECHO_E_ARG;
  if (!is_uct(c) || !c->have_faces) return fail(c, ECHO_E_ORDER, "echo_get_face_field: no staggered field (divb = 2)");
  return export_field(c, b3, bcur(c), 3, on_device, "echo_get_face_field");
}

// ---- checkpoint / restart (SURVEY §5 "Checkpoint/resume"): the raw device state the next step
// reads — U^n, the P record (hydro primitives, the per-cell Newton guess / the curved-metric B)
// and, with divb = 2, the staggered field record — owned planes only, record layout
static int ckpt_arrays(echo_ctx* c, double* arr[3]) {
  arr[0] = c->Un;
  arr[1] = c->P;
  arr[2] = is_uct(c) ? c->Bst : nullptr;
  return is_uct(c) ? 3 : 2;
}

long long echo_checkpoint_doubles(const echo_ctx* c) {
  if (!c || c->g.zhalo) return 0;
  const long long per = (long long)c->plane * c->g.n[2];
  return (c->g.divb == 2 ? 3 : 2) * per;
}

static int ckpt_copy(echo_ctx* c, double* buf, bool save, int on_device, const char* where) {
  double* arr[3];
  const int na = ckpt_arrays(c, arr);
  const size_t per = c->plane * (size_t)c->g.n[2];
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice
                                        : (save ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
  for (int a = 0; a < na; a++) {
    double* dev = arr[a];
    double* usr = buf + a * per;
    CK(cudaMemcpyAsync(save ? usr : dev, save ? dev : usr, sizeof(double) * per, kind, c->st), where);
  }
  if (!on_device) CK(cudaStreamSynchronize(c->st), where);
  return ECHO_OK;
}

int echo_checkpoint_save(echo_ctx* c, double* buf, int on_device) {
  if (!c || !buf) return c ? fail(c, ECHO_E_ARG, "echo_checkpoint_save: NULL buffer") : ECHO_E_ARG;
  if (c->g.zhalo) return fail(c, ECHO_E_ORDER, "echo_checkpoint_save: not for slab contexts (halo boundaries)");
  if (!c->have_state || (is_uct(c) && !c->have_faces))
    return fail(c, ECHO_E_ORDER, "echo_checkpoint_save: no state (echo_set_prims / echo_set_face_field first)");
  if (c->next_stage != 1 || c->swept)
    return fail(c, ECHO_E_ORDER, "echo_checkpoint_save: inside a step (stage 1 or 2 done): finish it with echo_stage");
  return ckpt_copy(c, buf, true, on_device, "echo_checkpoint_save");
}

int echo_checkpoint_load(echo_ctx* c, const double* buf, int on_device) {
  if (!c || !buf) return c ? fail(c, ECHO_E_ARG, "echo_checkpoint_load: NULL buffer") : ECHO_E_ARG;
  if (c->g.zhalo) return fail(c, ECHO_E_ORDER, "echo_checkpoint_load: not for slab contexts (halo boundaries)");
  int rc = ckpt_copy(c, const_cast<double*>(buf), false, on_device, "echo_checkpoint_load");
  if (rc) return rc;
  c->have_state = true;
  c->have_faces = is_uct(c);
  c->cfl_valid = false;
  c->next_stage = 1;
  c->xahead = false;
  c->swept = 0;
  c->swept_int = 0;
  c->inducted = 0;
  return ECHO_OK;
}

int echo_set_cons(echo_ctx* c, const double* u8, int on_device) {
  if (!c || !u8) return c ? fail(c, ECHO_E_ARG, "echo_set_cons: NULL buffer") : ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_set_cons: needs a prior echo_set_prims (con2prim guess)");
  if (is_uct(c))
    return fail(c, ECHO_E_ORDER, "echo_set_cons: with divb = 2 the field is staggered: use echo_set_prims + echo_set_face_field");
  const double* src = u8;
  if (!on_device) {
    int rc = ensure_scratch(c);
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->scratch, u8, sizeof(double) * 8 * c->g.N, cudaMemcpyHostToDevice, c->st), "echo_set_cons");
    src = c->scratch;
  }
  CK(launch(c, kLayout, [&] { return launch_layout(c->g, src, c->Un, 8, false, c->st); }), "echo_set_cons");
  c->next_stage = 1;
  c->xahead = false;
  c->swept = 0;  // a half-done stage (echo_stage_sweeps) of the old state is void
  c->swept_int = 0;
  return echo_con2prim(c, nullptr);
}

int echo_rhs(echo_ctx* c, double* l8, int on_device) {
  if (!c || !l8) return c ? fail(c, ECHO_E_ARG, "echo_rhs: NULL buffer") : ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_rhs: no state");
  if (is_uct(c) && !c->have_faces) return fail(c, ECHO_E_ORDER, "echo_rhs: divb = 2 needs echo_set_face_field first");
  double* dst = l8;
  if (!on_device) {
    int rc = ensure_scratch(c);
    if (rc) return rc;
    dst = c->scratch;
  }
  const double* U = ucur(c);
  int rc = run_sweeps(c);
  if (rc) return rc;
  cudaError_t e = launch(c, kUpdateRhs, [&] {
    return launch_update(kModeRhs, c->ks, c->g, c->e, c->mt, 0, 0.0, racc(c), U, U, nullptr, c->P, dst, c->dcnt,
                         nullptr, c->st);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "update(rhs) launch");
  if (is_uct(c)) {
    e = launch(c, kUctInduct, [&] { return launch_uct_induct(c->g, 1, 0, 0.0, nullptr, c->Ed, c->Bst, dst, c->st); });
    if (e != cudaSuccess) return cuda_fail(c, e, "uct induct(rhs) launch");
  }
  if (!on_device) {
    CK(cudaMemcpyAsync(l8, c->scratch, sizeof(double) * 8 * c->g.N, cudaMemcpyDeviceToHost, c->st), "echo_rhs");
    CK(cudaStreamSynchronize(c->st), "echo_rhs");
  }
  return ECHO_OK;
}

int echo_con2prim(echo_ctx* c, echo_stats_t* delta) {
  if (!c) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_con2prim: no state");
  unsigned long long before[2] = {0, 0}, after[2] = {0, 0};
  if (delta) {
    CK(cudaMemcpyAsync(c->hpin, c->dcnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->st), "echo_con2prim");
    CK(cudaStreamSynchronize(c->st), "echo_con2prim");
    before[0] = c->hpin[0];
    before[1] = c->hpin[1];
  }
  double* U = ucur_mut(c);
  c->xahead = false;  // the state changes
  CK(cudaMemsetAsync(c->dcnt + 2, 0, sizeof(unsigned long long), c->st), "echo_con2prim");
  cudaError_t e = launch(c, kC2P, [&] {
    return launch_update(kModeC2P, c->ks, c->g, c->e, c->mt, 0, 0.0, c->R, U, U, U, c->P, nullptr, c->dcnt,
                         c->dcnt + 2, c->st);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "con2prim launch");
  c->cfl_valid = true;
  if (delta) {
    CK(cudaMemcpyAsync(c->hpin, c->dcnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->st), "echo_con2prim");
    CK(cudaStreamSynchronize(c->st), "echo_con2prim");
    after[0] = c->hpin[0];
    after[1] = c->hpin[1];
    delta->floor_events = after[0] - before[0];
    delta->c2p_failures = after[1] - before[1];
    delta->steps = 0;
    delta->stages = 0;
  }
  return ECHO_OK;
}

int echo_stage(echo_ctx* c, int s, double dt) {
  if (!c) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_stage: no state (call echo_set_prims first)");
  if (is_uct(c) && !c->have_faces) return fail(c, ECHO_E_ORDER, "echo_stage: divb = 2 needs echo_set_face_field first");
  if (s < 1 || s > 3) return fail(c, ECHO_E_ARG, "echo_stage: s must be 1, 2 or 3");
  if (s != c->next_stage || c->swept || c->swept_int) return fail(c, ECHO_E_ORDER, "echo_stage: stages must run in order 1, 2, 3");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(c, ECHO_E_ARG, "echo_stage: dt > 0 violated");
  if (is_uct(c) && c->g.zhalo)
    return fail(c, ECHO_E_ORDER,
                "echo_stage: UCT slabs: echo_stage_sweeps, echo_stage_update_field, the new-field halo exchange, "
                "echo_stage_update_cells");
  return run_stage(c, s, dt);
}

int echo_step(echo_ctx* c, double dt) {
  if (!c) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_step: no state (call echo_set_prims first)");
  if (is_uct(c) && !c->have_faces) return fail(c, ECHO_E_ORDER, "echo_step: divb = 2 needs echo_set_face_field first");
  if (c->next_stage != 1) return fail(c, ECHO_E_ORDER, "echo_step: a step is in progress (finish its stages)");
  if (c->g.zhalo)
    return fail(c, ECHO_E_ORDER,
                "echo_step: halo (slab) boundaries need a halo exchange before every stage: use echo_stage");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(c, ECHO_E_ARG, "echo_step: dt > 0 violated");
  for (int s = 1; s <= 3; s++) {
    int rc = run_stage(c, s, dt);
    if (rc) return rc;
  }
  c->steps++;
  return ECHO_OK;
}

int echo_max_dt(echo_ctx* c, double cfl, double* dt_out) {
  if (!c || !dt_out) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_max_dt: no state");
  if (!(cfl > 0.0)) return fail(c, ECHO_E_ARG, "echo_max_dt: cfl > 0 violated");
  if (!c->cfl_valid) {  // otherwise the last update already reduced it for this state
    CK(cudaMemsetAsync(c->dcnt + 2, 0, sizeof(unsigned long long), c->st), "echo_max_dt");
    cudaError_t e = launch(c, kMaxSpeed, [&] {
      return launch_max_speed(c->ks, c->g, c->e, c->mt, c->P, ucur(c), c->dcnt + 2, c->st);
    });
    if (e != cudaSuccess) return cuda_fail(c, e, "max_speed launch");
    c->cfl_valid = true;
  }
  CK(cudaMemcpyAsync(c->hpin + 2, c->dcnt + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->st), "echo_max_dt");
  CK(cudaStreamSynchronize(c->st), "echo_max_dt");
  double m;
  std::memcpy(&m, c->hpin + 2, sizeof m);
  if (!(m > 0.0) || !std::isfinite(m))
    return fail(c, ECHO_E_NONFINITE, "echo_max_dt: max signal speed is zero or not finite (static field, dt unbounded)");
  *dt_out = cfl / m;
  return ECHO_OK;
}

// ------------------------------------------------- device-driven time loop
// one step with dt computed on the device (k_cfl_dt) from the previous reduction
static int issue_step_dev(echo_ctx* c, double cfl) {
  CK(launch(c, kCflDt, [&] { return launch_cfl_dt(cfl, c->dcnt + 2, c->dadv, c->dadv + 4, c->dlog_cap, c->st); }),
     "echo_advance");
  for (int s = 1; s <= 3; s++) {
    int rc = run_sweeps(c);
    if (!rc) rc = run_update(c, s, 0.0, c->dadv);
    if (rc) return rc;
  }
  return ECHO_OK;
}

static void drop_graphs(echo_ctx* c) {
  if (c->step_exec) cudaGraphExecDestroy(c->step_exec);
  c->step_exec = nullptr;
  for (auto& x : c->step_exec_p) {
    if (x) cudaGraphExecDestroy(x);
    x = nullptr;
  }
}

// capture issue_step_dev into *target (on a private stream: the caller's may be the legacy
// default stream, which cannot be captured); host bookkeeping is restored after.  With the
// fused update the accumulator parity alternates step by step (3 updates per step), so there
// are two step graphs, one per entry parity (c->rsel at capture).
static int capture_step(echo_ctx* c, double cfl, cudaGraphExec_t* target) {
  if (*target) {
    cudaGraphExecDestroy(*target);
    *target = nullptr;
  }
  if (!c->cap_st) CK(cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking), "echo_advance");
  const cudaStream_t user = c->st;
  const long long launches0 = c->launches;
  const unsigned long long stages0 = c->stages;
  const int rsel0 = c->rsel;
  const bool xahead0 = c->xahead;
  c->st = c->cap_st;
  CK(cudaStreamBeginCapture(c->cap_st, cudaStreamCaptureModeThreadLocal), "echo_advance capture");
  int rc = issue_step_dev(c, cfl);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->cap_st, &graph);
  c->st = user;
  c->step_kernels = c->launches - launches0;
  c->launches = launches0;
  c->stages = stages0;
  c->rsel = rsel0;
  c->xahead = xahead0;
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "echo_advance capture");
  e = cudaGraphInstantiate(target, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(c, e, "echo_advance instantiate");
  c->step_cfl = cfl;
  return ECHO_OK;
}

int echo_advance(echo_ctx* c, int nsteps, double cfl, double* dt_log, int* steps_done) {
  if (steps_done) *steps_done = 0;
  if (!c) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_advance: no state (call echo_set_prims first)");
  if (is_uct(c) && !c->have_faces) return fail(c, ECHO_E_ORDER, "echo_advance: divb = 2 needs echo_set_face_field first");
  if (c->next_stage != 1 || c->swept) return fail(c, ECHO_E_ORDER, "echo_advance: a step is in progress (finish its stages)");
  if (c->g.zhalo)
    return fail(c, ECHO_E_ORDER, "echo_advance: halo (slab) boundaries need a halo exchange before every stage");
  if (nsteps < 0) return fail(c, ECHO_E_ARG, "echo_advance: nsteps >= 0 violated");
  if (!(cfl > 0.0) || !std::isfinite(cfl)) return fail(c, ECHO_E_ARG, "echo_advance: cfl > 0 violated");
  if (nsteps == 0) return ECHO_OK;
  const unsigned long long stages0 = c->stages;
  const long long cap = dt_log ? nsteps : 0;
  if (!c->dadv || cap > c->dlog_cap) {  // adv block + log; a new buffer invalidates the captured step
    cudaFree(c->dadv);
    c->dadv = nullptr;
    // at least 4096 entries: a later call with a longer log (e.g. warm-up without a log, then a
    // timed loop with one) does not reallocate and re-capture the step
    long long ncap = cap > c->dlog_cap ? cap : c->dlog_cap;
    if (ncap < 4096) ncap = 4096;
    if (cudaMalloc(&c->dadv, sizeof(double) * (4 + ncap)) != cudaSuccess)
      return fail(c, ECHO_E_OOM, "echo_advance: dt log allocation failed");
    c->dlog_cap = ncap;
    drop_graphs(c);
  }
  if (!c->cfl_valid) {  // the first dt needs the reduction of the current state
    CK(cudaMemsetAsync(c->dcnt + 2, 0, sizeof(unsigned long long), c->st), "echo_advance");
    cudaError_t e = launch(c, kMaxSpeed, [&] {
      return launch_max_speed(c->ks, c->g, c->e, c->mt, c->P, ucur(c), c->dcnt + 2, c->st);
    });
    if (e != cudaSuccess) return cuda_fail(c, e, "max_speed launch");
  }
  CK(cudaMemsetAsync(c->dadv, 0, 4 * sizeof(double), c->st), "echo_advance");
  if (c->prof) {  // per-kernel events cannot live inside a graph: issue the launches directly
    for (int n = 0; n < nsteps; n++) {
      int rc = issue_step_dev(c, cfl);
      if (rc) return rc;
    }
  } else {
    if (c->fuse && !c->xahead) {  // the step graph starts from a swept x (its last update sweeps the next)
      cudaError_t e = launch(c, kSweepX, [&] {
        return launch_march(0, c->ks, c->g, c->e, c->mt, c->P, c->ks ? c->P : ucur(c), racc(c), c->st);
      });
      if (e != cudaSuccess) return cuda_fail(c, e, "sweep launch");
      c->xahead = true;
    }
    if (c->step_cfl != cfl) drop_graphs(c);
    for (int n = 0; n < nsteps; n++) {
      cudaGraphExec_t& ex = c->fuse ? c->step_exec_p[c->rsel] : c->step_exec;
      if (!ex) {
        int rc = capture_step(c, cfl, &ex);
        if (rc) return rc;
      }
      CK(cudaGraphLaunch(ex, c->st), "echo_advance graph launch");
      c->launches += c->step_kernels;
      if (c->fuse) c->rsel ^= 1;  // three updates per step, each flips the accumulator
    }
  }
  // one readback for the whole loop: [dt, halt, steps done] and the dt log
  double adv[4];
  CK(cudaMemcpyAsync(adv, c->dadv, sizeof adv, cudaMemcpyDeviceToHost, c->st), "echo_advance");
  if (dt_log) CK(cudaMemcpyAsync(dt_log, c->dadv + 4, sizeof(double) * nsteps, cudaMemcpyDeviceToHost, c->st), "echo_advance");
  CK(cudaStreamSynchronize(c->st), "echo_advance");
  const int done = (int)adv[2];
  c->steps += done;
  c->stages = stages0 + 3ull * done;
  if (steps_done) *steps_done = done;
  if (adv[1] != 0.0) c->xahead = false;  // a halted loop skipped its later updates (and their x sweeps)
  if (adv[1] == 2.0) {  // the debug scan halted the loop
    c->cfl_valid = false;
    return nan_report(c, "echo_advance (debug scan)");
  }
  if (adv[1] != 0.0) {
    c->cfl_valid = false;
    return fail(c, ECHO_E_NONFINITE,
                "echo_advance: max signal speed is zero or not finite (static field, dt unbounded); "
                "the state is that after the steps done");
  }
  c->cfl_valid = true;
  return ECHO_OK;
}

int echo_set_debug(echo_ctx* c, int flags) {
  if (!c) return ECHO_E_ARG;
  if (flags & ~ECHO_DEBUG_NANSCAN) return fail(c, ECHO_E_ARG, "echo_set_debug: unknown flag");
  const long long init = LLONG_MAX;
  CK(cudaMemcpyAsync(c->dnan, &init, sizeof init, cudaMemcpyHostToDevice, c->st), "echo_set_debug");
  CK(cudaStreamSynchronize(c->st), "echo_set_debug");
  if (flags != c->debug) drop_graphs(c);  // the captured step holds (or lacks) the scans
  c->debug = flags;
  return ECHO_OK;
}

int echo_check_finite(echo_ctx* c) {
  if (!c) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_check_finite: no state");
  const long long init = LLONG_MAX;
  CK(cudaMemcpyAsync(c->dnan, &init, sizeof init, cudaMemcpyHostToDevice, c->st), "echo_check_finite");
  cudaError_t e = launch(c, kNanScan, [&] { return launch_nanscan(c->g, ucur(c), c->P, c->ks ? 8 : 5, c->dnan, nullptr, c->st); });
  if (e != cudaSuccess) return cuda_fail(c, e, "nan scan launch");
  return nan_report(c, "echo_check_finite");
}

int echo_check_guards(echo_ctx* c) {
  if (!c) return ECHO_E_ARG;
  if (!c->guard) return fail(c, ECHO_E_ORDER, "echo_check_guards: no guard bands (ECHO_GUARD_BANDS=1 at echo_create)");
  CK(cudaStreamSynchronize(c->st), "echo_check_guards");
  std::vector<unsigned long long> h(c->guard);
  const unsigned long long pat = 0xA5A5A5A5A5A5A5A5ull;
  for (size_t a = 0; a < c->guarded.size(); a++) {
    for (int side = 0; side < 2; side++) {
      const double* src = c->guarded[a].first + (side ? c->guard + c->guarded[a].second : 0);
      CK(cudaMemcpy(h.data(), src, sizeof(double) * c->guard, cudaMemcpyDeviceToHost), "echo_check_guards");
      for (size_t k = 0; k < c->guard; k++)
        if (h[side ? k : c->guard - 1 - k] != pat) {  // nearest to the array first
          char buf[200];
          std::snprintf(buf, sizeof buf, "echo_check_guards: state array %zu written out of bounds, %s its end by %zu doubles",
                        a, side ? "after" : "before", k + 1);
          return fail(c, ECHO_E_CUDA, buf);
        }
    }
  }
  return ECHO_OK;
}

int echo_stats(echo_ctx* c, echo_stats_t* out) {
  if (!c || !out) return ECHO_E_ARG;
  CK(cudaMemcpyAsync(c->hpin, c->dcnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->st), "echo_stats");
  CK(cudaStreamSynchronize(c->st), "echo_stats");
  out->floor_events = c->hpin[0];
  out->c2p_failures = c->hpin[1];
  out->steps = c->steps;
  out->stages = c->stages;
  return ECHO_OK;
}

// ------------------------------------------------------------ stage halves
int echo_stage_sweeps(echo_ctx* c, int s) {
  if (!c) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_stage_sweeps: no state");
  if (is_uct(c) && !c->have_faces) return fail(c, ECHO_E_ORDER, "echo_stage_sweeps: divb = 2 needs echo_set_face_field first");
  if (s < 1 || s > 3) return fail(c, ECHO_E_ARG, "echo_stage_sweeps: s must be 1, 2 or 3");
  if (s != c->next_stage || c->swept || c->swept_int) return fail(c, ECHO_E_ORDER, "echo_stage_sweeps: stages must run in order");
  int rc = run_sweeps(c);
  if (rc) return rc;
  c->swept = s;
  return ECHO_OK;
}

int echo_stage_sweeps_interior(echo_ctx* c, int s) {
  if (!c) return ECHO_E_ARG;
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_stage_sweeps_interior: no state");
  if (!c->g.zhalo || is_uct(c))
    return fail(c, ECHO_E_ORDER, "echo_stage_sweeps_interior: only for slab contexts (halo boundaries), not UCT");
  if (s < 1 || s > 3) return fail(c, ECHO_E_ARG, "echo_stage_sweeps_interior: s must be 1, 2 or 3");
  if (s != c->next_stage || c->swept || c->swept_int)
    return fail(c, ECHO_E_ORDER, "echo_stage_sweeps_interior: stages must run in order");
  int rc = run_sweeps(c, 1);
  if (rc) return rc;
  c->swept_int = s;
  return ECHO_OK;
}

int echo_stage_sweeps_boundary(echo_ctx* c, int s) {
  if (!c) return ECHO_E_ARG;
  if (c->swept_int != s || c->swept)
    return fail(c, ECHO_E_ORDER, "echo_stage_sweeps_boundary: echo_stage_sweeps_interior(s) must come first");
  int rc = run_sweeps(c, 2);
  if (rc) return rc;
  c->swept_int = 0;
  c->swept = s;
  return ECHO_OK;
}

int echo_stage_update(echo_ctx* c, int s, double dt) {
  if (!c) return ECHO_E_ARG;
  if (c->swept != s) return fail(c, ECHO_E_ORDER, "echo_stage_update: echo_stage_sweeps(s) must come first");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(c, ECHO_E_ARG, "echo_stage_update: dt > 0 violated");
  if (is_uct(c) && c->g.zhalo)
    return fail(c, ECHO_E_ORDER,
                "echo_stage_update: UCT slabs: echo_stage_update_field, the new-field halo exchange, echo_stage_update_cells");
  return run_update(c, s, dt);
}

int echo_stage_update_field(echo_ctx* c, int s, double dt) {
  if (!c) return ECHO_E_ARG;
  if (!is_uct(c) || !c->g.zhalo) return fail(c, ECHO_E_ORDER, "echo_stage_update_field: UCT slab contexts only");
  if (c->swept != s || c->inducted) return fail(c, ECHO_E_ORDER, "echo_stage_update_field: echo_stage_sweeps(s) must come first");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(c, ECHO_E_ARG, "echo_stage_update_field: dt > 0 violated");
  return run_update(c, s, dt, nullptr, 1);
}

int echo_stage_update_cells(echo_ctx* c, int s, double dt) {
  if (!c) return ECHO_E_ARG;
  if (c->inducted != s || c->swept != s)
    return fail(c, ECHO_E_ORDER, "echo_stage_update_cells: echo_stage_update_field(s) must come first");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(c, ECHO_E_ARG, "echo_stage_update_cells: dt > 0 violated");
  return run_update(c, s, dt, nullptr, 2);
}

// the new b^z of the 3 owned faces next to `side` (written by this stage's induction: slot 2 of the
// b^n half at stage 3, of the b^s half before), for the neighbour's centring of its edge cells
static int field_copy(echo_ctx* c, int side, double* buf, bool out, int on_device, const char* where) {
  if (!is_uct(c) || !c->g.zhalo) return fail(c, ECHO_E_ORDER, (std::string(where) + ": UCT slab contexts only").c_str());
  if (!c->inducted) return fail(c, ECHO_E_ORDER, (std::string(where) + ": after echo_stage_update_field").c_str());
  const int H = 3;
  const long long rows = (long long)H * c->g.n[1];
  const long long k0 = out ? (side == 0 ? 0 : c->g.n[2] - H) : (side == 0 ? -H : c->g.n[2]);
  const long long slot = (c->inducted == 3 ? 0 : 3) + 2;  // b^z of the new field
  double* dev = c->Bst + k0 * (long long)c->plane + slot * c->g.vs;
  const size_t w = sizeof(double) * c->g.vs, pitchB = sizeof(double) * c->g.pitch;
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : (out ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
  cudaError_t e = out ? cudaMemcpy2DAsync(buf, w, dev, pitchB, w, rows, kind, c->st)
                      : cudaMemcpy2DAsync(dev, pitchB, buf, w, w, rows, kind, c->st);
  if (e != cudaSuccess) return cuda_fail(c, e, where);
  if (!on_device) CK(cudaStreamSynchronize(c->st), where);
  return ECHO_OK;
}

long long echo_halo_field_doubles(const echo_ctx* c) {
  if (!c || !c->g.zhalo || c->g.divb != 2) return 0;
  return 3LL * c->g.vs * c->g.n[1];
}

int echo_halo_export_field(echo_ctx* c, int side, double* buf, int on_device) {
  if (!c || !buf || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_export_field: bad argument") : ECHO_E_ARG;
  return field_copy(c, side, buf, true, on_device, "echo_halo_export_field");
}

int echo_halo_import_field(echo_ctx* c, int side, const double* buf, int on_device) {
  if (!c || !buf || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_import_field: bad argument") : ECHO_E_ARG;
  return field_copy(c, side, const_cast<double*>(buf), false, on_device, "echo_halo_import_field");
}

// a physical outflow side: the new b^z of the edge face replicated into the 3 ghost faces (A42)
int echo_halo_fill_field(echo_ctx* c, int side) {
  if (!c || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_fill_field: bad argument") : ECHO_E_ARG;
  if (!is_uct(c) || !c->g.zhalo || !c->inducted)
    return fail(c, ECHO_E_ORDER, "echo_halo_fill_field: UCT slab contexts, after echo_stage_update_field");
  if (c->g.bc[2][side] != ECHO_BC_OUTFLOW) return fail(c, ECHO_E_ARG, "echo_halo_fill_field: only an outflow side");
  const long long slot = (c->inducted == 3 ? 0 : 3) + 2;
  const long long edge = side == 0 ? 0 : c->g.n[2] - 1;
  for (int h = 1; h <= 3; h++) {
    const long long k = side == 0 ? -h : c->g.n[2] - 1 + h;
    CK(cudaMemcpy2DAsync(c->Bst + k * (long long)c->plane + slot * c->g.vs, sizeof(double) * c->g.pitch,
                         c->Bst + edge * (long long)c->plane + slot * c->g.vs, sizeof(double) * c->g.pitch,
                         sizeof(double) * c->g.vs, c->g.n[1], cudaMemcpyDeviceToDevice, c->st),
       "echo_halo_fill_field");
  }
  return ECHO_OK;
}

// ------------------------------------------------------------ slab halos
// CUDA IPC: the allocation handles of P, Un, Us (3 x cudaIpcMemHandle_t) and n[2]
int echo_ipc_export(echo_ctx* c, void* handles, int* nz) {
  if (!c || !handles) return c ? fail(c, ECHO_E_ARG, "echo_ipc_export: NULL buffer") : ECHO_E_ARG;
  if (!c->g.zhalo) return fail(c, ECHO_E_ORDER, "echo_ipc_export: the context has no halo boundary");
  cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(handles);
  const int slot[3] = {2, 0, 1};  // P, Un, Us
  for (int q = 0; q < 3; q++) CK(cudaIpcGetMemHandle(&h[q], c->alloc_base[slot[q]]), "echo_ipc_export");
  if (nz) *nz = c->g.n[2];
  return ECHO_OK;
}

int echo_halo_link_ipc(echo_ctx* c, int side, const void* handles, int peer_nz) {
  if (!c || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_link_ipc: bad argument") : ECHO_E_ARG;
  ipc_close(c->rlink[side]);
  if (!handles) return ECHO_OK;
  if (is_uct(c)) return fail(c, ECHO_E_ARG, "echo_halo_link_ipc: UCT slabs use the copy exchange (export / import)");
  if (!c->g.zhalo || c->g.bc[2][side] != ECHO_BC_HALO || peer_nz < ECHO_HALO_PLANES)
    return fail(c, ECHO_E_ARG, "echo_halo_link_ipc: the side must be a halo boundary facing a slab of >= 6 planes");
  const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(handles);
  echo_ctx::Remote& rm = c->rlink[side];
  for (int q = 0; q < 3; q++) {
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      ipc_close(rm);
      return cuda_fail(c, e, "echo_halo_link_ipc");
    }
    rm.base[q] = static_cast<double*>(p);
  }
  // the peer's arrays start kZH ghost planes into their allocations (same n[0], n[1], pitch)
  const long long ghost = (long long)kZH * (long long)c->g.n[1] * c->g.pitch;
  rm.P = rm.base[0] + ghost;
  rm.Un = rm.base[1] + ghost;
  rm.Us = rm.base[2] + ghost;
  rm.nz = peer_nz;
  return ECHO_OK;
}

// fill the ghost planes of `side` from the linked neighbour's edge planes (peer / IPC reads)
int echo_halo_pull(echo_ctx* c, int side) {
  if (!c || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_pull: bad argument") : ECHO_E_ARG;
  echo_ctx* nb = c->link[side];
  const echo_ctx::Remote& rm = c->rlink[side];
  double *nP = nullptr, *nU = nullptr;
  int nnz = 0;
  const bool first = c->next_stage == 1;  // the stage-input role of U: U^n before stage 1, U^s after
  if (nb) {
    nP = nb->P, nU = first ? nb->Un : nb->Us, nnz = nb->g.n[2];
  } else if (rm.P) {
    nP = rm.P, nU = first ? rm.Un : rm.Us, nnz = rm.nz;
  } else {
    return fail(c, ECHO_E_ORDER, "echo_halo_pull: the side is not linked");
  }
  const long long plane = (long long)c->g.n[1] * c->g.pitch;
  const long long src_k = side == 0 ? nnz - ECHO_HALO_PLANES : 0;
  const long long dst_k = side == 0 ? -ECHO_HALO_PLANES : c->g.n[2];
  const size_t bytes = sizeof(double) * ECHO_HALO_PLANES * plane;
  CK(cudaMemcpyAsync(c->P + dst_k * plane, nP + src_k * plane, bytes, cudaMemcpyDefault, c->st), "echo_halo_pull");
  CK(cudaMemcpyAsync(ucur_mut(c) + dst_k * plane, nU + src_k * plane, bytes, cudaMemcpyDefault, c->st), "echo_halo_pull");
  return ECHO_OK;
}

int echo_halo_link(echo_ctx* c, int side, echo_ctx* peer) {
  if (!c || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_link: bad argument") : ECHO_E_ARG;
  if (!peer) {
    if (c->link[side]) drop_backref(c->link[side], c);
    c->link[side] = nullptr;
    return ECHO_OK;
  }
  if (is_uct(c)) return fail(c, ECHO_E_ARG, "echo_halo_link: UCT slabs use the copy exchange (export / import)");
  if (!c->g.zhalo || c->g.bc[2][side] != ECHO_BC_HALO || !peer->g.zhalo || peer->g.bc[2][1 - side] != ECHO_BC_HALO)
    return fail(c, ECHO_E_ARG, "echo_halo_link: both facing sides must be halo boundaries");
  if (peer->g.n[0] != c->g.n[0] || peer->g.n[1] != c->g.n[1] || peer->g.pitch != c->g.pitch || peer->ks != c->ks)
    return fail(c, ECHO_E_ARG, "echo_halo_link: the slabs must share n[0], n[1] and the metric");
  if (c->link[side]) drop_backref(c->link[side], c);
  c->link[side] = peer;
  peer->linked_by.push_back(c);
  return ECHO_OK;
}


long long echo_halo_doubles(const echo_ctx* c) {
  if (!c || !c->g.zhalo) return 0;
  // halo_copy: 8 slots x vs per row (+ 3 for UCT's staggered field), zhalo planes
  return (is_uct(c) ? 11LL : 8LL) * c->g.vs * c->g.zhalo * (long long)c->g.n[1];
}

// A halo message holds, for each of the zhalo x n2 rows next to a side, what the neighbour reads
// of a ghost cell: the primitives rho, u~, p (P slots 0..4) and B (Minkowski: U slots 5..7 of the
// stage-input U; Kerr-Schild: P slots 5..7) — 8 vs doubles per row — and with UCT the stage-input
// staggered field b^1..3 (3 vs more), rows packed part by part.  Z0 (P slot 5, Minkowski) and the
// hydro U of ghost cells are never read there.
static int halo_copy(echo_ctx* c, int side, double* buf, bool out, int on_device, const char* where) {
  const int H = c->g.zhalo;
  const long long rows = (long long)H * c->g.n[1];
  const long long k0 = out ? (side == 0 ? 0 : c->g.n[2] - H) : (side == 0 ? -H : c->g.n[2]);
  const size_t pitchB = sizeof(double) * c->g.pitch;
  const long long vs = c->g.vs;
  cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : (out ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
  struct Part {
    double* arr;
    long long slot0, nslot;
  };
  Part parts[3];
  int np = 0;
  if (c->ks) {
    parts[np++] = {c->P, 0, 8};
  } else {
    parts[np++] = {c->P, 0, 5};
    parts[np++] = {ucur_mut(c), 5, 3};
  }
  if (is_uct(c)) parts[np++] = {bcur(c), 0, 3};  // the stage-input staggered field b^1..3
  long long off = 0;
  for (int q = 0; q < np; q++) {
    const Part& pt = parts[q];
    double* dev = pt.arr + k0 * (long long)c->plane + pt.slot0 * vs;
    const size_t w = sizeof(double) * pt.nslot * vs;
    cudaError_t e = out ? cudaMemcpy2DAsync(buf + off, w, dev, pitchB, w, rows, kind, c->st)
                        : cudaMemcpy2DAsync(dev, pitchB, buf + off, w, w, rows, kind, c->st);
    if (e != cudaSuccess) return cuda_fail(c, e, where);
    off += pt.nslot * vs * rows;
  }
  if (!on_device) CK(cudaStreamSynchronize(c->st), where);
  return ECHO_OK;
}

int echo_halo_export(echo_ctx* c, int side, double* buf, int on_device) {
  if (!c || !buf || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_export: bad argument") : ECHO_E_ARG;
  if (!c->g.zhalo) return fail(c, ECHO_E_ORDER, "echo_halo_export: the context has no halo boundary");
  if (!c->have_state) return fail(c, ECHO_E_ORDER, "echo_halo_export: no state");
  return halo_copy(c, side, buf, true, on_device, "echo_halo_export");
}

int echo_halo_import(echo_ctx* c, int side, const double* buf, int on_device) {
  if (!c || !buf || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_import: bad argument") : ECHO_E_ARG;
  if (!c->g.zhalo) return fail(c, ECHO_E_ORDER, "echo_halo_import: the context has no halo boundary");
  return halo_copy(c, side, const_cast<double*>(buf), false, on_device, "echo_halo_import");
}

// a physical outflow side of a slab: every ghost plane = the owned edge plane (A13)
int echo_halo_fill(echo_ctx* c, int side) {
  if (!c || (side != 0 && side != 1)) return c ? fail(c, ECHO_E_ARG, "echo_halo_fill: bad argument") : ECHO_E_ARG;
  if (!c->g.zhalo) return fail(c, ECHO_E_ORDER, "echo_halo_fill: the context has no halo boundary");
  if (c->g.bc[2][side] != ECHO_BC_OUTFLOW)
    return fail(c, ECHO_E_ARG, "echo_halo_fill: only an outflow side is filled locally (halo sides are imported)");
  const long long edge = side == 0 ? 0 : c->g.n[2] - 1;
  for (int h = 1; h <= c->g.zhalo; h++) {
    const long long k = side == 0 ? -h : c->g.n[2] - 1 + h;
    // (UCT: also the staggered field, A42: a ghost face takes the nearest owned face)
    for (double* a : {c->P, ucur_mut(c), is_uct(c) ? c->Bst : nullptr}) {
      if (!a) continue;
      CK(cudaMemcpyAsync(a + k * (long long)c->plane, a + edge * (long long)c->plane, sizeof(double) * c->plane,
                         cudaMemcpyDeviceToDevice, c->st),
         "echo_halo_fill");
    }
  }
  return ECHO_OK;
}

const char* echo_last_error(const echo_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

int echo_profile(echo_ctx* c, int enable) {
  if (!c) return ECHO_E_ARG;
  if (enable) {
    for (int k = 0; k < kNumClasses; k++) {
      c->prof_ms[k] = 0.0;
      c->prof_n[k] = 0;
    }
  }
  c->prof = enable != 0;
  return ECHO_OK;
}

int echo_profile_read(echo_ctx* c, int id, double* ms, long long* n) {
  if (!c || id < 0 || id >= kNumClasses) return ECHO_E_ARG;
  CK(cudaStreamSynchronize(c->st), "echo_profile_read");
  for (auto& r : c->recs) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
      c->prof_ms[r.cls] += t;
      c->prof_n[r.cls] += 1;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  c->recs.clear();
  if (ms) *ms = c->prof_ms[id];
  if (n) *n = c->prof_n[id];
  return ECHO_OK;
}

int echo_kernel_classes(void) { return kNumClasses; }
const char* echo_kernel_name(int id) { return (id >= 0 && id < kNumClasses) ? kNames[id] : ""; }
long long echo_launch_count(const echo_ctx* c) { return c ? c->launches : 0; }

}  // extern "C"
