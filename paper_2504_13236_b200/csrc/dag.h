// Per-GPU tile-task DAG of one GPT-2 block pass: tasks are
// submitted in program order (STF) with R / W / RW / Reduce accesses on tile
// handles; dependencies follow S:46; tasks are levelled (longest chain) and
// lowered to launch groups, one per op at the op's highest task level (every
// edge must cross launch levels, checked).  Replaces StarPU's dynamic
// scheduler with a deterministic, cached, stream-ordered plan.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/nnt.h"

namespace nnt {

enum Access { ACC_R = 0, ACC_W = 1, ACC_RW = 2, ACC_REDUCE = 3 };

struct Task {
  int op;
  int64_t tile[3];
  int level;
  int group;
  std::vector<int> deps;
  bool writes_only_grads;  // every handle it writes belongs to a parameter-gradient tensor
};

struct LaunchGroup {
  int op;
  int level;
  int64_t n_tasks;
  // no task of another op depends on this op's tasks and all it writes are parameter gradients:
  // it may run on a second stream beside the critical chain (nnt_block_bwd_streams)
  bool side_ok;
};

struct BlockPlan {
  std::vector<Task> tasks;
  std::vector<LaunchGroup> groups;  // execution order
};

// Generic STF graph builder.
class StfGraph {
 public:
  int new_tensor(int64_t n_tiles);
  void mark_param_grad(int tensor);  // the tensor's tiles are parameter gradients (pass outputs)
  // Submit a task; accesses are (tensor, tile index, mode).
  int submit(int op, const int64_t tile[3], const std::vector<std::pair<int64_t, int>>& handle_modes);
  int64_t handle(int tensor, int64_t tile) const { return base_[tensor] + tile; }
  bool lower(BlockPlan* plan);
  std::vector<Task> tasks;

 private:
  struct HState {
    std::vector<int> writers, readers, reducers;
  };
  std::vector<int64_t> base_;
  std::vector<HState> hs_;
  std::vector<char> param_grad_;  // per tensor
  int tensor_of(int64_t handle) const;
};

// Cached plan for (cfg, pass).  Returns nullptr and sets the error on failure.
const BlockPlan* block_plan(const nnt_block_cfg& cfg, int pass);

}  // namespace nnt
