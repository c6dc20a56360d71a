// Opaque handle definitions behind the C ABI.
#pragma once
#include "../planner/planner.hpp"
#include "../../../include/vdnn.h"

struct vdnn_graph {
  vdnnp::Net net;
};
struct vdnn_decision {
  vdnnp::Decision d;
};
struct vdnn_report {
  vdnnp::Report r;
};
struct vdnn_dyn {
  vdnnp::DynResult res;
};

namespace vdnncapi {
vdnnp::Cost cost_from(const vdnn_cost_model* cm);
}
