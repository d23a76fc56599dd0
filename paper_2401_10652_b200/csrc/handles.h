// Opaque handle types behind include/ac.h.
#pragma once
#include <memory>

#include "graph.h"

struct ac_graph {
  std::shared_ptr<const ac::Graph> g;
};

struct ac_chunk_plan {
  std::shared_ptr<const ac::Graph> g;
  ac::Plan plan;
};
