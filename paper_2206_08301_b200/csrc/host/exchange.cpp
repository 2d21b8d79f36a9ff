// Block redistribution plans between two placements of one tensor.
// Restates proj/src/redistribute.cpp: per-dimension segments (Eq. 25/27,
// 9-38), matching ranks (Eq. 28, 40-49) and the message plan with canonical
// source replicas, destination fan-out and self messages (51-148).  The
// execution side (copy_ranges / apply_plan, 152-206) lives on the GPU:
// executor.cpp drives eb_copy_box / NCCL send-recv per message.
#include <algorithm>

#include "einplan_host.hpp"

namespace einplan {

DimPartition dim_partition(std::int64_t block_y, std::int64_t p_y, std::int64_t block_x,
                           std::int64_t extent) {
  if (block_x < 1 || block_y < 1)
    fail(errc::invalid_argument, "dim_partition: block sizes must be positive");
  const std::int64_t start = p_y * block_y;
  if (start < 0 || start >= extent)
    fail(errc::invalid_argument, "dim_partition: source block outside the extent");
  const std::int64_t len = std::min(block_y, extent - start);
  DimPartition part;
  part.xi = start / block_x;
  part.lambda = start % block_x;
  // Walk the source block, cutting it at destination block boundaries.
  std::int64_t done = 0;
  std::int64_t dst = part.xi;
  std::int64_t dst_off = part.lambda;
  while (done < len) {
    const std::int64_t piece = std::min(block_x - dst_off, len - done);
    DimSegment seg;
    seg.p_x = dst;
    seg.oy_lo = done;
    seg.oy_hi = done + piece;
    seg.ox_lo = dst_off;
    seg.ox_hi = dst_off + piece;
    part.segments.push_back(seg);
    done += piece;
    ++dst;
    dst_off = 0;
  }
  return part;
}

std::pair<std::int64_t, std::int64_t> matching_ranks(std::int64_t p_x, std::int64_t block_x,
                                                     std::int64_t block_y) {
  if (block_x < 1 || block_y < 1)
    fail(errc::invalid_argument, "matching_ranks: block sizes must be positive");
  const auto up = [](std::int64_t a, std::int64_t b) { return (a + b - 1) / b; };
  return {up(p_x * block_x + 1, block_y) - 1, up((p_x + 1) * block_x, block_y)};
}

RedistributionPlan plan_redistribution(const std::string& tensor, const TensorPlacement& source,
                                       const TensorPlacement& destination) {
  if (source.dist.extents != destination.dist.extents)
    fail(errc::invalid_argument,
         "plan: source and destination cover different index spaces for \"" + tensor + "\"");
  RedistributionPlan plan;
  plan.tensor = tensor;
  plan.source = source;
  plan.destination = destination;

  // Both grids number their ranks from one shared pool (a smaller grid is a
  // prefix of it).
  const std::int64_t src_ranks = source.term_grid.total();
  const BlockDistribution& from = source.dist;
  const BlockDistribution& to = destination.dist;
  const std::size_t nd = from.extents.size();

  std::vector<std::int64_t> src_block(nd, 0);
  for (;;) {
    // Segments of this source block along every dimension.
    std::vector<DimPartition> cuts;
    cuts.reserve(nd);
    for (std::size_t d = 0; d < nd; ++d)
      cuts.push_back(dim_partition(from.blocks[d], src_block[d], to.blocks[d], from.extents[d]));
    const std::int64_t sender = source.canonical_rank(src_block);

    // Cartesian product of the per-dimension segments (last dim fastest).
    std::vector<std::size_t> sel(nd, 0);
    for (;;) {
      Message box;
      box.src_block = src_block;
      box.dst_block.resize(nd);
      box.elements = 1;
      for (std::size_t d = 0; d < nd; ++d) {
        const DimSegment& sg = cuts[d].segments[sel[d]];
        box.dst_block[d] = sg.p_x;
        box.oy_lo.push_back(sg.oy_lo);
        box.oy_hi.push_back(sg.oy_hi);
        box.ox_lo.push_back(sg.ox_lo);
        box.ox_hi.push_back(sg.ox_hi);
        box.elements *= sg.oy_hi - sg.oy_lo;
      }
      for (std::int64_t receiver : destination.replica_ranks(box.dst_block)) {
        Message m = box;
        m.dst_rank = receiver;
        // A receiver that already holds this source block copies locally.
        m.self = receiver < src_ranks && source.block_coords_of(receiver) == src_block;
        m.src_rank = m.self ? receiver : sender;
        if (m.self) {
          ++plan.self_messages;
        } else {
          plan.transmitted_volume += m.elements;
          if (destination.is_canonical(receiver)) plan.logical_volume += m.elements;
        }
        plan.messages.push_back(std::move(m));
      }
      int d = static_cast<int>(nd) - 1;
      while (d >= 0) {
        const std::size_t u = static_cast<std::size_t>(d);
        if (++sel[u] < cuts[u].segments.size()) break;
        sel[u] = 0;
        --d;
      }
      if (d < 0) break;
    }

    // Next source block (row-major over the source owner grid).
    int d = static_cast<int>(nd) - 1;
    while (d >= 0) {
      const std::size_t u = static_cast<std::size_t>(d);
      if (++src_block[u] < from.grid.dims[u]) break;
      src_block[u] = 0;
      --d;
    }
    if (d < 0) break;
  }
  return plan;
}

}  // namespace einplan
