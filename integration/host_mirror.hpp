// Write tracking for host buffers the device mirrors (the drop-in's VoxelGrid
// payload / occupancy, RMSProp state and keyframes), so repeat calls skip the
// upload of anything the caller did not change.
//
// The reference API passes VoxelGrid by (const) reference with value semantics
// and no version counter (voxel_grid.hpp:112-175), and mapping_step mutates it in
// place (mapping.hpp:80-82). Once the device copy matches a host buffer, the
// buffer's whole pages are made read-only. A write by anyone faults once per
// 2 MB granule; the handler makes that granule writable again and the write
// proceeds. A buffer's dirty set is then every tracked granule that lies in a
// writable mapping (read from /proc/self/maps), which also catches a buffer that
// was freed and re-mapped at the same address. The partial pages at a buffer's
// two ends cannot be protected: they are compared against copies taken when the
// buffer was last made clean (small buffers entirely so). A kernel write on the
// caller's behalf (read(2) straight into a tracked buffer) fails with EFAULT
// instead of faulting: tracked buffers must be written from user space
// (VoxelGrid::load builds a fresh buffer, so the reference never does that).
#pragma once

#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

namespace voxrf_b200 {

class HostMirror {
 public:
  // Starts (or restarts) tracking [ptr, ptr + bytes), clean and read-only.
  static void track(const void* ptr, std::size_t bytes);
  // True when [ptr, ptr + bytes) is a tracked buffer of exactly that extent.
  static bool tracked(const void* ptr, std::size_t bytes);
  // Re-reads the process's writable mappings; dirty() answers from this snapshot
  // (one /proc/self/maps read per API call, however many buffers it checks).
  static void refresh();
  // Byte ranges [begin, end) of the buffer written since track() / clean()
  // (as of the last refresh()), sorted and merged (granule runs plus any changed
  // end page).
  static std::vector<std::pair<std::size_t, std::size_t>> dirty(const void* ptr);
  // Marks the buffer clean again (read-only).
  static void clean(const void* ptr);
  // Makes the whole buffer writable (our own write-back); clean() afterwards.
  static void unprotect(const void* ptr);
  static void untrack(const void* ptr);
  // Write faults taken so far (tests).
  static std::uint64_t faults();
};

}  // namespace voxrf_b200
