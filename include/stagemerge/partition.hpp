// stagemerge/partition.hpp — multi-GPU placement of a plan.
//
// Root subtrees of a plan are independent after their shared init (no data flows between
// them), so ranks split the work by root: LPT (longest processing time first) over subtree step
// extents, ties by root id.  Every rank computes the identical map from its identical plan
// (insertion is deterministic), so no communication is needed; new roots (tuner insertions)
// are placed incrementally on the least-loaded rank.
#pragma once

#include <map>
#include <set>

#include "stagemerge/plan.hpp"

namespace stagemerge {

/// Step extent of every root subtree: sum over its nodes of (furthest request end or child
/// boundary) - start_step.  This is the unique training work the subtree still describes.
std::map<NodeId, StepCount> root_work(const SearchPlan& plan);

/// Extends `owner` (root -> rank) with every root of `plan` not yet placed, LPT by root_work.
void assign_roots(const SearchPlan& plan, int world, std::map<NodeId, int>& owner);

/// Root of the subtree containing `node`.
NodeId root_of(const SearchPlan& plan, NodeId node);

/// In-process placement of every plan node on one of `devices` GPUs: LPT over
/// placement units by step extent.  Units start as root subtrees; while the heaviest unit
/// exceeds total / devices it is split at its first branch point -- every child subtree but the
/// heaviest becomes its own unit -- so one dominant root no longer serialises on one GPU.  A
/// split-off subtree's first stage LOADs its branch checkpoint from the parent's GPU with one
/// peer copy (K7).  Deterministic (plan only); ties: heavier first, then smaller node id, then
/// the lowest device.
std::map<NodeId, int> place_nodes(const SearchPlan& plan, int devices);

}  // namespace stagemerge
