// HostMirror: page-protection write tracking (see host_mirror.hpp).
#include "host_mirror.hpp"

#include <signal.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>

#ifndef MADV_COLLAPSE
#define MADV_COLLAPSE 25
#endif

namespace voxrf_b200 {
namespace {

constexpr int kMaxRegions = 4096;
constexpr std::size_t kGranule = std::size_t(2) << 20;  // bounds the VMA splits per buffer
// Buffers at least this large are moved onto 2 MB pages (MADV_COLLAPSE, in the
// background): mprotect of a 3.8 GB buffer costs ~40 ms on 4 KB pages and ~0.3 ms
// on 2 MB pages, and every mapping_step re-protects the grid and RMSProp state.
constexpr std::size_t kCollapseBytes = std::size_t(256) << 20;

struct Region {
  std::uintptr_t begin = 0;                    // buffer start; 0 = free slot
  std::size_t bytes = 0;
  std::atomic<std::uintptr_t> pb{0}, pe{0};    // protected whole-page span
  // copies of the unprotectable partial pages at the two ends (compared, not trapped)
  std::vector<unsigned char> head, tail;
};

Region g_regions[kMaxRegions];
std::mutex g_mu;
struct sigaction g_prev;
bool g_installed = false;
std::atomic<std::uint64_t> g_faults{0};
std::size_t g_page = 4096;
std::vector<std::pair<std::uintptr_t, std::uintptr_t>> g_vmas;  // refresh() snapshot

void on_segv(int sig, siginfo_t* si, void* uc) {
  const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(si->si_addr);
  for (Region& r : g_regions) {
    const std::uintptr_t pb = r.pb.load(std::memory_order_acquire);
    const std::uintptr_t pe = r.pe.load(std::memory_order_acquire);
    if (pb != 0 && a >= pb && a < pe) {
      const std::uintptr_t g0 = pb + (a - pb) / kGranule * kGranule;
      const std::uintptr_t g1 = std::min(pe, g0 + kGranule);
      g_faults.fetch_add(1, std::memory_order_relaxed);
      if (mprotect(reinterpret_cast<void*>(g0), g1 - g0, PROT_READ | PROT_WRITE) == 0) return;
      break;  // cannot unprotect: fall through to the previous disposition
    }
  }
  if (g_prev.sa_flags & SA_SIGINFO) {
    if (g_prev.sa_sigaction) return g_prev.sa_sigaction(sig, si, uc);
  } else if (g_prev.sa_handler != SIG_DFL && g_prev.sa_handler != SIG_IGN) {
    return g_prev.sa_handler(sig);
  }
  signal(SIGSEGV, SIG_DFL);  // the store re-executes and takes the default action
}

void install() {
  if (g_installed) return;
  g_installed = true;
  g_page = (std::size_t)sysconf(_SC_PAGESIZE);
  struct sigaction sa;
  std::memset(&sa, 0, sizeof(sa));
  sa.sa_sigaction = on_segv;
  sa.sa_flags = SA_SIGINFO | SA_NODEFER;
  sigemptyset(&sa.sa_mask);
  sigaction(SIGSEGV, &sa, &g_prev);
}

Region* find(const void* ptr) {
  const std::uintptr_t b = reinterpret_cast<std::uintptr_t>(ptr);
  if (b == 0) return nullptr;
  for (Region& r : g_regions)
    if (r.begin == b) return &r;
  return nullptr;
}

void protect(Region& r) {
  const std::uintptr_t b = r.begin, pb = r.pb.load(), pe = r.pe.load();
  if (pe > pb) mprotect(reinterpret_cast<void*>(pb), pe - pb, PROT_READ);
  // snapshot the ends (the whole buffer when no page of it can be protected)
  const unsigned char* p = reinterpret_cast<const unsigned char*>(b);
  const std::size_t h = pb ? pb - b : r.bytes, t0 = pb ? pe - b : r.bytes;
  r.head.assign(p, p + h);
  r.tail.assign(p + t0, p + r.bytes);
}

void release(Region& r) {
  const std::uintptr_t pb = r.pb.load(), pe = r.pe.load();
  r.pb.store(0, std::memory_order_release);
  r.pe.store(0, std::memory_order_release);
  // (if the buffer was unmapped meanwhile this fails harmlessly)
  if (pe > pb) mprotect(reinterpret_cast<void*>(pb), pe - pb, PROT_READ | PROT_WRITE);
  r.begin = 0;
  r.bytes = 0;
  r.head.clear();
  r.tail.clear();
}

// Writable mappings of the process: [start, end) pairs from /proc/self/maps.
std::vector<std::pair<std::uintptr_t, std::uintptr_t>> writable_vmas() {
  std::vector<std::pair<std::uintptr_t, std::uintptr_t>> out;
  FILE* f = std::fopen("/proc/self/maps", "r");
  if (!f) return out;
  char line[512];
  while (std::fgets(line, sizeof(line), f)) {
    unsigned long s = 0, e = 0;
    char perms[8] = {0};
    if (std::sscanf(line, "%lx-%lx %7s", &s, &e, perms) == 3 && perms[1] == 'w')
      out.emplace_back((std::uintptr_t)s, (std::uintptr_t)e);
  }
  std::fclose(f);
  return out;
}

}  // namespace

void HostMirror::track(const void* ptr, std::size_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  install();
  if (Region* old = find(ptr)) release(*old);
  Region* r = nullptr;
  for (Region& x : g_regions)
    if (x.begin == 0) {
      r = &x;
      break;
    }
  if (!r) {  // full: drop the first (its buffer is simply re-uploaded next time)
    release(g_regions[0]);
    r = &g_regions[0];
  }
  const std::uintptr_t b = reinterpret_cast<std::uintptr_t>(ptr);
  const std::uintptr_t pb = (b + g_page - 1) / g_page * g_page;
  const std::uintptr_t pe = (b + bytes) / g_page * g_page;
  r->begin = b;
  r->bytes = bytes;
  r->pb.store(pe > pb ? pb : 0, std::memory_order_release);
  r->pe.store(pe > pb ? pe : 0, std::memory_order_release);
  protect(*r);
  if (bytes >= kCollapseBytes) {
    const std::uintptr_t hb = (b + kGranule - 1) / kGranule * kGranule;
    const std::uintptr_t he = (b + bytes) / kGranule * kGranule;
    if (he > hb)  // best effort (THP off or an older kernel: stays on 4 KB pages)
      std::thread([hb, he] {
        madvise(reinterpret_cast<void*>(hb), he - hb, MADV_HUGEPAGE);
        madvise(reinterpret_cast<void*>(hb), he - hb, MADV_COLLAPSE);
      }).detach();
  }
}

bool HostMirror::tracked(const void* ptr, std::size_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  const Region* r = find(ptr);
  return r && r->bytes == bytes;
}

std::vector<std::pair<std::size_t, std::size_t>> HostMirror::dirty(const void* ptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<std::pair<std::size_t, std::size_t>> out;
  const Region* r = find(ptr);
  if (!r) return out;
  const std::uintptr_t b = r->begin, pb = r->pb.load(), pe = r->pe.load();
  // (a remapped buffer shows up as a writable mapping over the protected span;
  // its end pages are compared against the snapshots)
  auto add = [&out](std::size_t s, std::size_t e) {
    if (e <= s) return;
    if (!out.empty() && out.back().second >= s)
      out.back().second = std::max(out.back().second, e);
    else
      out.emplace_back(s, e);
  };
  const unsigned char* p = reinterpret_cast<const unsigned char*>(b);
  auto changed = [p](std::size_t off, const std::vector<unsigned char>& snap) {
    return !snap.empty() && std::memcmp(p + off, snap.data(), snap.size()) != 0;
  };
  if (pb == 0) {  // nothing protectable: compare the whole snapshot
    if (changed(0, r->head)) add(0, r->bytes);
    return out;
  }
  if (changed(0, r->head)) add(0, pb - b);  // head partial page
  std::vector<std::pair<std::size_t, std::size_t>> mid;
  for (const auto& v : g_vmas) {
    const std::uintptr_t s = std::max(v.first, pb), e = std::min(v.second, pe);
    if (s < e) mid.emplace_back(s - b, e - b);
  }
  std::sort(mid.begin(), mid.end());
  for (const auto& m : mid) add(m.first, m.second);
  if (changed(pe - b, r->tail)) add(pe - b, r->bytes);  // tail partial page
  return out;
}

void HostMirror::refresh() {
  auto v = writable_vmas();
  std::lock_guard<std::mutex> lk(g_mu);
  g_vmas.swap(v);
}

void HostMirror::clean(const void* ptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (Region* r = find(ptr)) protect(*r);
}

void HostMirror::unprotect(const void* ptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  const Region* r = find(ptr);
  if (!r) return;
  const std::uintptr_t pb = r->pb.load(), pe = r->pe.load();
  if (pe > pb) mprotect(reinterpret_cast<void*>(pb), pe - pb, PROT_READ | PROT_WRITE);
}

void HostMirror::untrack(const void* ptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (Region* r = find(ptr)) release(*r);
}

std::uint64_t HostMirror::faults() { return g_faults.load(); }

}  // namespace voxrf_b200
