// STF tile-task DAG of the GPT-2 block ("nodes correspond to tasks and
// directed edges correspond to tiles", P:80-84 sequential task flow), with the
// access-mode dependency rules of S:46 and the lowering used by nnt_block_fwd /
// nnt_block_bwd.  Host-only integer code: the block plans' task counts / levels are
// tested bit-exactly (tests/test_abi.py), the graph builder itself by a serializability
// fuzz against a sequential Python executor through nnt_stf_build (tests/test_dag.py).
#include "dag.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "nnt_internal.h"

namespace nnt {

int StfGraph::new_tensor(int64_t n_tiles) {
  int id = (int)base_.size();
  int64_t b = hs_.size();
  base_.push_back(b);
  param_grad_.push_back(0);
  hs_.resize(b + n_tiles);
  return id;
}

void StfGraph::mark_param_grad(int tensor) { param_grad_[tensor] = 1; }

int StfGraph::tensor_of(int64_t handle) const {
  return (int)(std::upper_bound(base_.begin(), base_.end(), handle) - base_.begin()) - 1;
}

static void add_unique(std::vector<int>& v, int x) {
  if (std::find(v.begin(), v.end(), x) == v.end()) v.push_back(x);
}

// Dependency rules between two tasks sharing a handle, in submission order
// (S:46): R->R none; R->W/RW edge; W/RW->anything edge; Reduce->Reduce none;
// Reduce<->(R/W/RW) edge.
int StfGraph::submit(int op, const int64_t tile[3], const std::vector<std::pair<int64_t, int>>& hm) {
  Task t;
  t.op = op;
  t.tile[0] = tile[0];
  t.tile[1] = tile[1];
  t.tile[2] = tile[2];
  t.level = 0;
  t.group = -1;
  t.writes_only_grads = true;
  for (auto& [h, mode] : hm)
    if (mode != ACC_R && !param_grad_[tensor_of(h)]) t.writes_only_grads = false;
  const int id = (int)tasks.size();
  for (auto& [h, mode] : hm) {
    HState& s = hs_[h];
    if (mode == ACC_R) {
      for (int d : s.writers) add_unique(t.deps, d);
      for (int d : s.reducers) add_unique(t.deps, d);
    } else if (mode == ACC_REDUCE) {
      for (int d : s.writers) add_unique(t.deps, d);
      for (int d : s.readers) add_unique(t.deps, d);
    } else {  // W / RW
      for (int d : s.writers) add_unique(t.deps, d);
      for (int d : s.readers) add_unique(t.deps, d);
      for (int d : s.reducers) add_unique(t.deps, d);
    }
  }
  for (auto& [h, mode] : hm) {
    HState& s = hs_[h];
    if (mode == ACC_R) {
      if (!s.reducers.empty()) {  // a read closes the open reduction group
        s.writers = s.reducers;
        s.reducers.clear();
        s.readers.clear();
      }
      add_unique(s.readers, id);
    } else if (mode == ACC_REDUCE) {
      add_unique(s.reducers, id);
    } else {
      s.writers.assign(1, id);
      s.readers.clear();
      s.reducers.clear();
    }
  }
  for (int d : t.deps) t.level = std::max(t.level, tasks[d].level + 1);
  tasks.push_back(std::move(t));
  return id;
}

// Lowering: every op becomes ONE launch group (one kernel executes all of its
// tile tasks), launched at the highest level any of its tasks reached (a task
// may be ready earlier, e.g. the v-columns of dqkv; delaying it is legal).
// The lowering is valid iff every dependency edge goes from a strictly lower
// launch level to a higher one — checked here; groups are ordered by
// (launch level, first submission).  Ops sharing a launch level are mutually
// independent.  Returns false (and sets the error) if the check fails.
bool StfGraph::lower(BlockPlan* plan) {
  std::map<int, int> op_level, op_first;
  for (size_t i = 0; i < tasks.size(); ++i) {
    const Task& t = tasks[i];
    auto it = op_level.find(t.op);
    if (it == op_level.end()) {
      op_level[t.op] = t.level;
      op_first[t.op] = (int)i;
    } else {
      it->second = std::max(it->second, t.level);
    }
  }
  for (const Task& t : tasks)
    for (int d : t.deps)
      if (op_level[tasks[d].op] >= op_level[t.op]) {
        set_error("DAG lowering: edge %s -> %s does not cross launch levels", nnt_op_name(tasks[d].op),
                  nnt_op_name(t.op));
        return false;
      }
  std::vector<std::tuple<int, int, int>> order;  // (launch level, first task, op)
  for (auto& [op, lv] : op_level) order.emplace_back(lv, op_first[op], op);
  std::sort(order.begin(), order.end());
  std::map<int, int> group_of;
  plan->groups.clear();
  for (auto& [lv, first, op] : order) {
    group_of[op] = (int)plan->groups.size();
    plan->groups.push_back({op, lv, 0, true});
  }
  for (auto& t : tasks) {
    t.group = group_of[t.op];
    LaunchGroup& gr = plan->groups[t.group];
    gr.n_tasks++;
    if (!t.writes_only_grads) gr.side_ok = false;
  }
  for (const Task& t : tasks)  // an op with a dependent in another op stays on the critical chain
    for (int d : t.deps)
      if (tasks[d].op != t.op) plan->groups[group_of[tasks[d].op]].side_ok = false;
  plan->tasks = tasks;
  return true;
}

namespace {

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t clamp_tile(int64_t tile, int64_t dim) { return tile < dim ? tile : dim; }

// A row-major 2-D tensor tiled (tr x tc).
struct T2 {
  int id = -1;
  int64_t rows = 0, cols = 0, tr = 1, tc = 1, nr = 0, nc = 0;
  void make(StfGraph& g, int64_t r, int64_t c, int64_t tile_r, int64_t tile_c) {
    rows = r;
    cols = c;
    tr = clamp_tile(tile_r, r);
    tc = clamp_tile(tile_c, c);
    nr = ceil_div(r, tr);
    nc = ceil_div(c, tc);
    id = g.new_tensor(nr * nc);
  }
  // handles of every tile overlapping rows [r0,r1) x cols [c0,c1)
  void region(const StfGraph& g, int64_t r0, int64_t r1, int64_t c0, int64_t c1, int mode,
              std::vector<std::pair<int64_t, int>>& out) const {
    for (int64_t i = r0 / tr; i <= (r1 - 1) / tr; ++i)
      for (int64_t j = c0 / tc; j <= (c1 - 1) / tc; ++j) out.emplace_back(g.handle(id, i * nc + j), mode);
  }
  void tile(const StfGraph& g, int64_t i, int64_t j, int mode, std::vector<std::pair<int64_t, int>>& out) const {
    out.emplace_back(g.handle(id, i * nc + j), mode);
  }
  void row(const StfGraph& g, int64_t i, int mode, std::vector<std::pair<int64_t, int>>& out) const {
    for (int64_t j = 0; j < nc; ++j) out.emplace_back(g.handle(id, i * nc + j), mode);
  }
  int64_t r_begin(int64_t i) const { return i * tr; }
  int64_t r_end(int64_t i) const { return std::min(rows, (i + 1) * tr); }
  int64_t c_begin(int64_t j) const { return j * tc; }
  int64_t c_end(int64_t j) const { return std::min(cols, (j + 1) * tc); }
};

struct Shapes {
  int64_t E, H, S, B, T, F, Dh, te, tf, ts, tt;
  bool causal, bf16;
};

// Attention [B][H][S][S] tiled by (ts x ts) per (b, h).
struct TAtt {
  int id = -1;
  int64_t B, H, nq;
  void make(StfGraph& g, const Shapes& s) {
    B = s.B;
    H = s.H;
    nq = ceil_div(s.S, clamp_tile(s.ts, s.S));
    id = g.new_tensor(B * H * nq * nq);
  }
  int64_t h(const StfGraph& g, int64_t b, int64_t hh, int64_t qi, int64_t kj) const {
    return g.handle(id, ((b * H + hh) * nq + qi) * nq + kj);
  }
};

struct TStats {
  int id = -1;
  int64_t H, nq;
  void make(StfGraph& g, const Shapes& s) {
    H = s.H;
    nq = ceil_div(s.S, clamp_tile(s.ts, s.S));
    id = g.new_tensor(s.B * H * nq);
  }
  int64_t h(const StfGraph& g, int64_t b, int64_t hh, int64_t qi) const { return g.handle(id, (b * H + hh) * nq + qi); }
};

struct BlockTensors {
  // forward activations / parameters
  T2 x, h1, qkv, O, x1, h2, u, g, y, stats1, stats2;
  T2 ln1, ln2, wqkv, bqkv, wo, bo, wfc, bfc, wpr, bpr;
  TAtt scores, P;
  TStats stats;
  // backward
  T2 dy, dyA, du, dh, dx1, dx1A, dO, dqkv, dx;
  T2 gln1, gln2, gwqkv, gbqkv, gwo, gbo, gwfc, gbfc, gwpr, gbpr;
  TAtt dP, dA;
  TStats Dv;  // bf16 path: D = rowdot(dO, O) per query tile
};

using Acc = std::vector<std::pair<int64_t, int>>;

void make_tensors(StfGraph& g, const Shapes& s, BlockTensors& t) {
  const int64_t T = s.T, E = s.E, F = s.F;
  t.x.make(g, T, E, s.tt, s.te);
  t.h1.make(g, T, E, s.tt, s.te);
  t.qkv.make(g, T, 3 * E, s.tt, s.te);
  t.O.make(g, T, E, s.tt, s.te);
  t.x1.make(g, T, E, s.tt, s.te);
  t.h2.make(g, T, E, s.tt, s.te);
  t.u.make(g, T, F, s.tt, s.tf);
  t.g.make(g, T, F, s.tt, s.tf);
  t.y.make(g, T, E, s.tt, s.te);
  t.stats1.make(g, T, 1, s.tt, 1);
  t.stats2.make(g, T, 1, s.tt, 1);
  t.ln1.make(g, 1, E, 1, s.te);
  t.ln2.make(g, 1, E, 1, s.te);
  t.wqkv.make(g, 3 * E, E, s.te, s.te);
  t.bqkv.make(g, 1, 3 * E, 1, s.te);
  t.wo.make(g, E, E, s.te, s.te);
  t.bo.make(g, 1, E, 1, s.te);
  t.wfc.make(g, F, E, s.tf, s.te);
  t.bfc.make(g, 1, F, 1, s.tf);
  t.wpr.make(g, E, F, s.te, s.tf);
  t.bpr.make(g, 1, E, 1, s.te);
  t.scores.make(g, s);
  t.P.make(g, s);
  t.stats.make(g, s);
}

void make_bwd_tensors(StfGraph& g, const Shapes& s, BlockTensors& t) {
  const int64_t T = s.T, E = s.E, F = s.F;
  t.dy.make(g, T, E, s.tt, s.te);
  t.dyA = t.dy;
  if (s.bf16) t.dyA.make(g, T, E, s.tt, s.te);
  t.du.make(g, T, F, s.tt, s.tf);
  t.dh.make(g, T, E, s.tt, s.te);
  t.dx1.make(g, T, E, s.tt, s.te);
  t.dx1A = t.dx1;
  if (s.bf16) t.dx1A.make(g, T, E, s.tt, s.te);
  t.dO.make(g, T, E, s.tt, s.te);
  t.dqkv.make(g, T, 3 * E, s.tt, s.te);
  t.dx.make(g, T, E, s.tt, s.te);
  t.gln1.make(g, 1, E, 1, s.te);
  t.gln2.make(g, 1, E, 1, s.te);
  t.gwqkv.make(g, 3 * E, E, s.te, s.te);
  t.gbqkv.make(g, 1, 3 * E, 1, s.te);
  t.gwo.make(g, E, E, s.te, s.te);
  t.gbo.make(g, 1, E, 1, s.te);
  t.gwfc.make(g, F, E, s.tf, s.te);
  t.gbfc.make(g, 1, F, 1, s.tf);
  t.gwpr.make(g, E, F, s.te, s.tf);
  t.gbpr.make(g, 1, E, 1, s.te);
  for (const T2* pg : {&t.gln1, &t.gln2, &t.gwqkv, &t.gbqkv, &t.gwo, &t.gbo, &t.gwfc, &t.gbfc, &t.gwpr, &t.gbpr})
    g.mark_param_grad(pg->id);
  t.dP.make(g, s);
  t.dA.make(g, s);
  t.Dv.make(g, s);
}

// LayerNorm: one task per token tile (steps 1-3 of P:162 over every E-tile of the row block).
void submit_ln_fwd(StfGraph& g, int op, const T2& x, const T2& prm, const T2& y, const T2& st) {
  for (int64_t i = 0; i < x.nr; ++i) {
    Acc a;
    x.row(g, i, ACC_R, a);
    prm.row(g, 0, ACC_R, a);
    y.row(g, i, ACC_W, a);
    st.tile(g, i, 0, ACC_W, a);
    int64_t tl[3] = {i, 0, 0};
    g.submit(op, tl, a);
  }
}

// Linear C(i,j) (+)= sum_k A(i,k) W(j,k)^T: one task per (i, j, k), Reduce over k.
void submit_linear(StfGraph& g, int op, const T2& A, const T2& W, const T2* bias, const T2* resid, const T2& C,
                   const T2* C2) {
  for (int64_t i = 0; i < C.nr; ++i)
    for (int64_t j = 0; j < C.nc; ++j)
      for (int64_t k = 0; k < A.nc; ++k) {
        Acc a;
        A.tile(g, i, k, ACC_R, a);
        W.region(g, C.c_begin(j), C.c_end(j), A.c_begin(k), A.c_end(k), ACC_R, a);
        if (bias) bias->region(g, 0, 1, C.c_begin(j), C.c_end(j), ACC_R, a);
        if (resid) resid->tile(g, i, j, ACC_R, a);
        C.tile(g, i, j, ACC_REDUCE, a);
        if (C2) C2->tile(g, i, j, ACC_REDUCE, a);
        int64_t tl[3] = {i, j, k};
        g.submit(op, tl, a);
      }
}

// Backward of a linear: dW(j,k) (+)= sum_i dY(i,j)^T X(i,k) — task per (j, k, i).
void submit_dw(StfGraph& g, int op, const T2& dY, const T2& X, const T2& dW) {
  for (int64_t j = 0; j < dY.nc; ++j)
    for (int64_t k = 0; k < X.nc; ++k)
      for (int64_t i = 0; i < dY.nr; ++i) {
        Acc a;
        dY.tile(g, i, j, ACC_R, a);
        X.tile(g, i, k, ACC_R, a);
        dW.region(g, dY.c_begin(j), dY.c_end(j), X.c_begin(k), X.c_end(k), ACC_REDUCE, a);
        int64_t tl[3] = {j, k, i};
        g.submit(op, tl, a);
      }
}

// dX(i,k) (+)= sum_j dY(i,j) W(j,k), optionally gated by GELU'(aux(i,k)).
void submit_dx(StfGraph& g, int op, const T2& dY, const T2& W, const T2* aux, const T2& dX) {
  for (int64_t i = 0; i < dX.nr; ++i)
    for (int64_t k = 0; k < dX.nc; ++k)
      for (int64_t j = 0; j < dY.nc; ++j) {
        Acc a;
        dY.tile(g, i, j, ACC_R, a);
        W.region(g, dY.c_begin(j), dY.c_end(j), dX.c_begin(k), dX.c_end(k), ACC_R, a);
        if (aux) aux->tile(g, i, k, ACC_R, a);
        dX.tile(g, i, k, ACC_REDUCE, a);
        int64_t tl[3] = {i, k, j};
        g.submit(op, tl, a);
      }
}

void submit_db(StfGraph& g, int op, const T2& dY, const T2& db, const T2* copy) {
  for (int64_t i = 0; i < dY.nr; ++i)
    for (int64_t j = 0; j < dY.nc; ++j) {
      Acc a;
      dY.tile(g, i, j, ACC_R, a);
      if (copy) copy->tile(g, i, j, ACC_W, a);
      db.region(g, 0, 1, dY.c_begin(j), dY.c_end(j), ACC_REDUCE, a);
      int64_t tl[3] = {i, j, 0};
      g.submit(op, tl, a);
    }
}

// token-row range of (b, q-tile qi) and column range of head h in part `part` (0 q, 1 k, 2 v)
struct AttnGeom {
  const Shapes& s;
  int64_t ts;
  int64_t nq;
  int64_t row0(int64_t b, int64_t qi) const { return b * s.S + qi * ts; }
  int64_t row1(int64_t b, int64_t qi) const { return b * s.S + std::min(s.S, (qi + 1) * ts); }
  int64_t col0(int part, int64_t h) const { return part * s.E + h * s.Dh; }
  int64_t col1(int part, int64_t h) const { return part * s.E + (h + 1) * s.Dh; }
  bool needed(int64_t qi, int64_t kj) const { return !s.causal || kj <= qi; }
};

void build_fwd(StfGraph& g, const Shapes& s) {
  BlockTensors t;
  make_tensors(g, s, t);
  AttnGeom ag{s, clamp_tile(s.ts, s.S), ceil_div(s.S, clamp_tile(s.ts, s.S))};
  submit_ln_fwd(g, NNT_OP_LN1, t.x, t.ln1, t.h1, t.stats1);
  submit_linear(g, NNT_OP_QKV, t.h1, t.wqkv, &t.bqkv, nullptr, t.qkv, nullptr);
  for (int64_t b = 0; b < s.B; ++b)
    for (int64_t h = 0; h < s.H; ++h)
      for (int64_t qi = 0; qi < ag.nq; ++qi)
        for (int64_t kj = 0; kj < ag.nq; ++kj) {
          if (!ag.needed(qi, kj)) continue;
          Acc a;
          t.qkv.region(g, ag.row0(b, qi), ag.row1(b, qi), ag.col0(0, h), ag.col1(0, h), ACC_R, a);
          t.qkv.region(g, ag.row0(b, kj), ag.row1(b, kj), ag.col0(1, h), ag.col1(1, h), ACC_R, a);
          if (s.bf16)  // R26: score tile kept on chip, its subroutine-1 partial Reduced into the stats
            a.emplace_back(t.stats.h(g, b, h, qi), ACC_REDUCE);
          else
            a.emplace_back(t.scores.h(g, b, h, qi, kj), ACC_W);
          int64_t tl[3] = {b * s.H + h, qi, kj};
          g.submit(NNT_OP_SCORES, tl, a);
        }
  // softmax subroutine 1: per key tile partial, Reduce into the slice stats
  // (bf16 path: fused into NNT_OP_SCORES above)
  if (!s.bf16)
    for (int64_t b = 0; b < s.B; ++b)
      for (int64_t h = 0; h < s.H; ++h)
        for (int64_t qi = 0; qi < ag.nq; ++qi)
          for (int64_t kj = 0; kj < ag.nq; ++kj) {
            if (!ag.needed(qi, kj)) continue;
            Acc a;
            a.emplace_back(t.scores.h(g, b, h, qi, kj), ACC_R);
            a.emplace_back(t.stats.h(g, b, h, qi), ACC_REDUCE);
            int64_t tl[3] = {b * s.H + h, qi, kj};
            g.submit(NNT_OP_MAXSUMEXP, tl, a);
          }
  // subroutine 2: normalise every tile with the aggregated stats (bf16 path: on the recomputed
  // score tile, from q and k)
  for (int64_t b = 0; b < s.B; ++b)
    for (int64_t h = 0; h < s.H; ++h)
      for (int64_t qi = 0; qi < ag.nq; ++qi)
        for (int64_t kj = 0; kj < ag.nq; ++kj) {
          if (!ag.needed(qi, kj)) continue;
          Acc a;
          if (s.bf16) {
            t.qkv.region(g, ag.row0(b, qi), ag.row1(b, qi), ag.col0(0, h), ag.col1(0, h), ACC_R, a);
            t.qkv.region(g, ag.row0(b, kj), ag.row1(b, kj), ag.col0(1, h), ag.col1(1, h), ACC_R, a);
          } else {
            a.emplace_back(t.scores.h(g, b, h, qi, kj), ACC_R);
          }
          a.emplace_back(t.stats.h(g, b, h, qi), ACC_R);
          a.emplace_back(t.P.h(g, b, h, qi, kj), ACC_W);
          int64_t tl[3] = {b * s.H + h, qi, kj};
          g.submit(NNT_OP_SOFTMAX, tl, a);
        }
  for (int64_t b = 0; b < s.B; ++b)
    for (int64_t h = 0; h < s.H; ++h)
      for (int64_t qi = 0; qi < ag.nq; ++qi)
        for (int64_t kj = 0; kj < ag.nq; ++kj) {
          if (!ag.needed(qi, kj)) continue;
          Acc a;
          a.emplace_back(t.P.h(g, b, h, qi, kj), ACC_R);
          t.qkv.region(g, ag.row0(b, kj), ag.row1(b, kj), ag.col0(2, h), ag.col1(2, h), ACC_R, a);
          t.O.region(g, ag.row0(b, qi), ag.row1(b, qi), h * s.Dh, (h + 1) * s.Dh, ACC_REDUCE, a);
          int64_t tl[3] = {b * s.H + h, qi, kj};
          g.submit(NNT_OP_PV, tl, a);
        }
  submit_linear(g, NNT_OP_OUT, t.O, t.wo, &t.bo, &t.x, t.x1, nullptr);
  submit_ln_fwd(g, NNT_OP_LN2, t.x1, t.ln2, t.h2, t.stats2);
  submit_linear(g, NNT_OP_FC, t.h2, t.wfc, &t.bfc, nullptr, t.u, &t.g);
  submit_linear(g, NNT_OP_PROJ, t.g, t.wpr, &t.bpr, &t.x1, t.y, nullptr);
}

void build_bwd(StfGraph& g, const Shapes& s) {
  BlockTensors t;
  make_tensors(g, s, t);
  make_bwd_tensors(g, s, t);
  AttnGeom ag{s, clamp_tile(s.ts, s.S), ceil_div(s.S, clamp_tile(s.ts, s.S))};
  submit_db(g, NNT_OP_PROJ_DB, t.dy, t.gbpr, s.bf16 ? &t.dyA : nullptr);
  submit_dw(g, NNT_OP_PROJ_DW, t.dyA, t.g, t.gwpr);
  submit_dx(g, NNT_OP_PROJ_DX, t.dyA, t.wpr, &t.u, t.du);
  submit_db(g, NNT_OP_FC_DB, t.du, t.gbfc, nullptr);
  submit_dw(g, NNT_OP_FC_DW, t.du, t.h2, t.gwfc);
  submit_dx(g, NNT_OP_FC_DX, t.du, t.wfc, nullptr, t.dh);
  for (int64_t i = 0; i < t.dh.nr; ++i) {
    Acc a;
    t.dh.row(g, i, ACC_R, a);
    t.x1.row(g, i, ACC_R, a);
    t.stats2.tile(g, i, 0, ACC_R, a);
    t.ln2.row(g, 0, ACC_R, a);
    t.dy.row(g, i, ACC_R, a);
    t.dx1.row(g, i, ACC_W, a);
    if (s.bf16) t.dx1A.row(g, i, ACC_W, a);
    t.gln2.row(g, 0, ACC_REDUCE, a);
    int64_t tl[3] = {i, 0, 0};
    g.submit(NNT_OP_LN2_BWD, tl, a);
  }
  submit_db(g, NNT_OP_OUT_DB, t.dx1, t.gbo, nullptr);
  submit_dw(g, NNT_OP_OUT_DW, t.dx1A, t.O, t.gwo);
  submit_dx(g, NNT_OP_OUT_DX, t.dx1A, t.wo, nullptr, t.dO);
  auto each_pair = [&](auto fn) {
    for (int64_t b = 0; b < s.B; ++b)
      for (int64_t h = 0; h < s.H; ++h)
        for (int64_t qi = 0; qi < ag.nq; ++qi)
          for (int64_t kj = 0; kj < ag.nq; ++kj)
            if (ag.needed(qi, kj)) fn(b, h, qi, kj);
  };
  if (s.bf16) {
    // bf16 path: D = rowdot(dO, O) per query tile first (softmax-bwd reduction through the
    // dO.O identity), then dA = scale * P * (dO V^T - D) straight from the dP GEMM epilogue.
    for (int64_t b = 0; b < s.B; ++b)
      for (int64_t h = 0; h < s.H; ++h)
        for (int64_t qi = 0; qi < ag.nq; ++qi) {
          Acc a;
          t.dO.region(g, ag.row0(b, qi), ag.row1(b, qi), h * s.Dh, (h + 1) * s.Dh, ACC_R, a);
          t.O.region(g, ag.row0(b, qi), ag.row1(b, qi), h * s.Dh, (h + 1) * s.Dh, ACC_R, a);
          a.emplace_back(t.Dv.h(g, b, h, qi), ACC_W);
          int64_t tl[3] = {b * s.H + h, qi, 0};
          g.submit(NNT_OP_SOFTMAX_BWD, tl, a);
        }
    each_pair([&](int64_t b, int64_t h, int64_t qi, int64_t kj) {  // dA tile = f(dO V^T, P, D)
      Acc a;
      t.dO.region(g, ag.row0(b, qi), ag.row1(b, qi), h * s.Dh, (h + 1) * s.Dh, ACC_R, a);
      t.qkv.region(g, ag.row0(b, kj), ag.row1(b, kj), ag.col0(2, h), ag.col1(2, h), ACC_R, a);
      a.emplace_back(t.P.h(g, b, h, qi, kj), ACC_R);
      a.emplace_back(t.Dv.h(g, b, h, qi), ACC_R);
      a.emplace_back(t.dA.h(g, b, h, qi, kj), ACC_W);
      int64_t tl[3] = {b * s.H + h, qi, kj};
      g.submit(NNT_OP_ATT_DP, tl, a);
    });
  } else {
    each_pair([&](int64_t b, int64_t h, int64_t qi, int64_t kj) {  // dP = dO V^T
      Acc a;
      t.dO.region(g, ag.row0(b, qi), ag.row1(b, qi), h * s.Dh, (h + 1) * s.Dh, ACC_R, a);
      t.qkv.region(g, ag.row0(b, kj), ag.row1(b, kj), ag.col0(2, h), ag.col1(2, h), ACC_R, a);
      a.emplace_back(t.dP.h(g, b, h, qi, kj), ACC_W);
      int64_t tl[3] = {b * s.H + h, qi, kj};
      g.submit(NNT_OP_ATT_DP, tl, a);
    });
  }
  each_pair([&](int64_t b, int64_t h, int64_t qi, int64_t kj) {  // dV = P^T dO
    Acc a;
    a.emplace_back(t.P.h(g, b, h, qi, kj), ACC_R);
    t.dO.region(g, ag.row0(b, qi), ag.row1(b, qi), h * s.Dh, (h + 1) * s.Dh, ACC_R, a);
    t.dqkv.region(g, ag.row0(b, kj), ag.row1(b, kj), ag.col0(2, h), ag.col1(2, h), ACC_REDUCE, a);
    int64_t tl[3] = {b * s.H + h, kj, qi};
    g.submit(NNT_OP_ATT_DV, tl, a);
  });
  if (!s.bf16)
    for (int64_t b = 0; b < s.B; ++b)
      for (int64_t h = 0; h < s.H; ++h)
        for (int64_t qi = 0; qi < ag.nq; ++qi) {  // softmax bwd needs the whole slice for D
          Acc a;
          for (int64_t kj = 0; kj < ag.nq; ++kj) {
            if (!ag.needed(qi, kj)) continue;
            a.emplace_back(t.P.h(g, b, h, qi, kj), ACC_R);
            a.emplace_back(t.dP.h(g, b, h, qi, kj), ACC_R);
            a.emplace_back(t.dA.h(g, b, h, qi, kj), ACC_W);
          }
          int64_t tl[3] = {b * s.H + h, qi, 0};
          g.submit(NNT_OP_SOFTMAX_BWD, tl, a);
        }
  each_pair([&](int64_t b, int64_t h, int64_t qi, int64_t kj) {  // dQ = dA K
    Acc a;
    a.emplace_back(t.dA.h(g, b, h, qi, kj), ACC_R);
    t.qkv.region(g, ag.row0(b, kj), ag.row1(b, kj), ag.col0(1, h), ag.col1(1, h), ACC_R, a);
    t.dqkv.region(g, ag.row0(b, qi), ag.row1(b, qi), ag.col0(0, h), ag.col1(0, h), ACC_REDUCE, a);
    int64_t tl[3] = {b * s.H + h, qi, kj};
    g.submit(NNT_OP_ATT_DQ, tl, a);
  });
  each_pair([&](int64_t b, int64_t h, int64_t qi, int64_t kj) {  // dK = dA^T Q
    Acc a;
    a.emplace_back(t.dA.h(g, b, h, qi, kj), ACC_R);
    t.qkv.region(g, ag.row0(b, qi), ag.row1(b, qi), ag.col0(0, h), ag.col1(0, h), ACC_R, a);
    t.dqkv.region(g, ag.row0(b, kj), ag.row1(b, kj), ag.col0(1, h), ag.col1(1, h), ACC_REDUCE, a);
    int64_t tl[3] = {b * s.H + h, kj, qi};
    g.submit(NNT_OP_ATT_DK, tl, a);
  });
  submit_db(g, NNT_OP_QKV_DB, t.dqkv, t.gbqkv, nullptr);
  submit_dw(g, NNT_OP_QKV_DW, t.dqkv, t.h1, t.gwqkv);
  submit_dx(g, NNT_OP_QKV_DX, t.dqkv, t.wqkv, nullptr, t.dh);
  for (int64_t i = 0; i < t.dh.nr; ++i) {
    Acc a;
    t.dh.row(g, i, ACC_R, a);
    t.x.row(g, i, ACC_R, a);
    t.stats1.tile(g, i, 0, ACC_R, a);
    t.ln1.row(g, 0, ACC_R, a);
    t.dx1.row(g, i, ACC_R, a);
    t.dx.row(g, i, ACC_W, a);
    t.gln1.row(g, 0, ACC_REDUCE, a);
    int64_t tl[3] = {i, 0, 0};
    g.submit(NNT_OP_LN1_BWD, tl, a);
  }
}

struct CfgKey {
  int64_t v[10];
  bool operator<(const CfgKey& o) const { return std::lexicographical_compare(v, v + 10, o.v, o.v + 10); }
};

std::mutex g_plan_mu;
std::map<CfgKey, BlockPlan> g_plans;

}  // namespace

const BlockPlan* block_plan(const nnt_block_cfg& c, int pass) {
  if (c.E <= 0 || c.H <= 0 || c.S <= 0 || c.B <= 0 || c.E % c.H != 0) {
    set_error("block cfg: bad shape E=%lld H=%lld S=%lld B=%lld", (long long)c.E, (long long)c.H, (long long)c.S,
              (long long)c.B);
    return nullptr;
  }
  if (c.tile_e <= 0 || c.tile_f <= 0 || c.tile_s <= 0 || c.tile_t <= 0) {
    set_error("block cfg: tiles must be positive");
    return nullptr;
  }
  CfgKey key{{c.E, c.H, c.S, c.B, c.tile_e, c.tile_f, c.tile_s, c.tile_t, (int64_t)c.dtype * 2 + (c.causal ? 1 : 0),
              pass}};
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) return &it->second;
  Shapes s{c.E, c.H, c.S, c.B, c.B * c.S, 4 * c.E, c.E / c.H, c.tile_e, c.tile_f, c.tile_s, c.tile_t,
           c.causal != 0, c.dtype == NNT_BF16};
  StfGraph g;
  if (pass == 0)
    build_fwd(g, s);
  else
    build_bwd(g, s);
  BlockPlan plan;
  if (!g.lower(&plan)) return nullptr;
  return &(g_plans[key] = std::move(plan));
}

}  // namespace nnt

using namespace nnt;

extern "C" {

const char* nnt_op_name(int op) {
  static const char* names[NNT_OP_COUNT] = {
      "ln1",      "qkv",      "scores",   "maxsumexp", "softmax",     "pv",     "out",    "ln2",
      "fc",       "proj",     "proj_db",  "proj_dw",   "proj_dx",     "fc_db",  "fc_dw",  "fc_dx",
      "ln2_bwd",  "out_db",   "out_dw",   "out_dx",    "att_dp",      "att_dv", "softmax_bwd",
      "att_dq",   "att_dk",   "qkv_db",   "qkv_dw",    "qkv_dx",      "ln1_bwd"};
  if (op < 0 || op >= NNT_OP_COUNT) return "?";
  return names[op];
}

nnt_status nnt_stf_build(int64_t n_handles, int64_t n_tasks, const int32_t* n_acc, const int64_t* acc_handle,
                         const int32_t* acc_mode, int32_t* level, int64_t* dep_offsets, int32_t* dep_ids,
                         int64_t dep_cap) {
  NNT_REQUIRE(n_handles > 0 && n_tasks >= 0 && n_handles < (1ll << 31) && n_tasks < (1ll << 31), NNT_ERR_SHAPE,
              "nnt_stf_build: n_handles=%lld n_tasks=%lld", (long long)n_handles, (long long)n_tasks);
  NNT_REQUIRE(n_tasks == 0 || (n_acc && acc_handle && acc_mode && level && dep_offsets), NNT_ERR_NULL,
              "nnt_stf_build: NULL argument");
  StfGraph g;
  const int tensor = g.new_tensor(n_handles);
  int64_t a = 0;
  const int64_t zero[3] = {0, 0, 0};
  for (int64_t t = 0; t < n_tasks; ++t) {
    NNT_REQUIRE(n_acc[t] > 0, NNT_ERR_ARG, "nnt_stf_build: task %lld has no access", (long long)t);
    std::vector<std::pair<int64_t, int>> hm;
    for (int32_t i = 0; i < n_acc[t]; ++i, ++a) {
      const int64_t h = acc_handle[a];
      const int m = acc_mode[a];
      NNT_REQUIRE(h >= 0 && h < n_handles && m >= ACC_R && m <= ACC_REDUCE, NNT_ERR_ARG,
                  "nnt_stf_build: access (%lld, %d)", (long long)h, m);
      for (auto& e : hm)
        NNT_REQUIRE(e.first != g.handle(tensor, h), NNT_ERR_ARG, "nnt_stf_build: handle %lld twice in task %lld",
                    (long long)h, (long long)t);
      hm.emplace_back(g.handle(tensor, h), m);
    }
    g.submit((int)(t % NNT_OP_COUNT), zero, hm);
  }
  int64_t n = 0;
  dep_offsets[0] = 0;
  for (int64_t t = 0; t < n_tasks; ++t) {
    level[t] = g.tasks[t].level;
    n += (int64_t)g.tasks[t].deps.size();
    dep_offsets[t + 1] = n;
  }
  NNT_REQUIRE(n <= dep_cap && (n == 0 || dep_ids), NNT_ERR_WORKSPACE, "nnt_stf_build: %lld dependencies > cap %lld",
              (long long)n, (long long)dep_cap);
  for (int64_t t = 0; t < n_tasks; ++t) {
    std::vector<int> d = g.tasks[t].deps;
    std::sort(d.begin(), d.end());
    for (size_t i = 0; i < d.size(); ++i) dep_ids[dep_offsets[t] + (int64_t)i] = d[i];
  }
  return NNT_OK;
}

nnt_status nnt_block_dag_describe(const nnt_block_cfg* cfg, int pass, nnt_task* tasks, int64_t task_cap,
                                  int64_t* n_tasks, nnt_launch_group* groups, int64_t group_cap, int64_t* n_groups) {
  NNT_REQUIRE(cfg && n_tasks && n_groups, NNT_ERR_NULL, "nnt_block_dag_describe: NULL argument");
  NNT_REQUIRE(pass == 0 || pass == 1, NNT_ERR_ARG, "nnt_block_dag_describe: pass=%d", pass);
  const BlockPlan* p = block_plan(*cfg, pass);
  if (!p) return NNT_ERR_SHAPE;
  *n_tasks = (int64_t)p->tasks.size();
  *n_groups = (int64_t)p->groups.size();
  if (tasks)
    for (int64_t i = 0; i < task_cap && i < *n_tasks; ++i) {
      const Task& t = p->tasks[i];
      tasks[i].op = t.op;
      tasks[i].level = t.level;
      tasks[i].tile[0] = t.tile[0];
      tasks[i].tile[1] = t.tile[1];
      tasks[i].tile[2] = t.tile[2];
      tasks[i].n_deps = (int32_t)t.deps.size();
      tasks[i].group = t.group;
    }
  if (groups)
    for (int64_t i = 0; i < group_cap && i < *n_groups; ++i) {
      groups[i].op = p->groups[i].op;
      groups[i].level = p->groups[i].level;
      groups[i].n_tasks = p->groups[i].n_tasks;
      groups[i].side_stream_ok = p->groups[i].side_ok ? 1 : 0;
    }
  return NNT_OK;
}

}  // extern "C"
