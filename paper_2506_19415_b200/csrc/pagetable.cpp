// Subsystem [3] host side: the page table / LRU residency cache with the
// exact semantics of runtime.PageTable + update_page_table
// (pkg/src/vmsplat/runtime.py:161-346), re-built on ordered sets so every
// allocation is O(log capacity) instead of the reference's O(capacity) scans
// (SURVEY Appendix A.4):
//
//   open[level]   entries of that level with a free slot, by index
//                 -> "first entry of the same level with a free slot"
//   empty_        empty entries by index -> "first empty entry"
//   lru_          (last_used, index) of every non-empty entry -> LRU victim,
//                 skipping the entries protected this frame
//
// The per-frame work list is sorted by (class, -encoded depth, page id),
// pass 2 breaks (never skips) on the staging budget and continues past a
// failed allocation, exactly as the reference.
#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <map>
#include <set>
#include <tuple>
#include <vector>

#include "../../include/vmsplat_b200.h"

namespace vms {
void set_error(const char* fmt, ...);
}

struct vms_pagetable {
  struct Entry {
    int level = -1;
    int64_t last = -1;
    int occupied = 0;
    std::vector<uint32_t> slots;
  };
  std::vector<Entry> e;
  std::map<uint32_t, std::pair<int32_t, int32_t>> resident;
  std::vector<std::set<int32_t>> open;
  std::set<int32_t> empty_;
  std::set<std::pair<int64_t, int32_t>> lru_;
  std::vector<uint8_t> prot;
  std::vector<int32_t> prot_list;

  explicit vms_pagetable(int64_t cap) : e(cap), open(32), prot(cap, 0) {
    for (int32_t i = 0; i < cap; ++i) empty_.insert(i);
  }

  void protect(int32_t ei) {
    if (!prot[ei]) {
      prot[ei] = 1;
      prot_list.push_back(ei);
    }
  }
  void touch(int32_t ei, int64_t frame) {
    Entry& x = e[ei];
    if (x.level >= 0) lru_.erase({x.last, ei});
    x.last = frame;
    if (x.level >= 0) lru_.insert({x.last, ei});
  }
  void activate(int32_t ei, int level) {
    Entry& x = e[ei];
    empty_.erase(ei);
    x.level = level;
    x.slots.assign(size_t(1) << level, 0u);
    x.occupied = 0;
    open[level].insert(ei);
    lru_.insert({x.last, ei});
  }
  void clear(int32_t ei) {
    Entry& x = e[ei];
    open[x.level].erase(ei);
    lru_.erase({x.last, ei});
    x.level = -1;
    x.slots.clear();
    x.occupied = 0;
    empty_.insert(ei);
  }
  // runtime.py:238-264
  bool alloc(int level, int32_t* ei_out, int32_t* si_out) {
    if (!open[level].empty()) {
      int32_t ei = *open[level].begin();
      const Entry& x = e[ei];
      for (size_t si = 0; si < x.slots.size(); ++si)
        if (x.slots[si] == 0) {
          *ei_out = ei;
          *si_out = (int32_t)si;
          return true;
        }
    }
    if (!empty_.empty()) {
      int32_t ei = *empty_.begin();
      activate(ei, level);
      *ei_out = ei;
      *si_out = 0;
      return true;
    }
    for (auto it = lru_.begin(); it != lru_.end(); ++it) {
      const int32_t ei = it->second;
      if (prot[ei]) continue;
      for (uint32_t pid : e[ei].slots)  // runtime.py:266-271
        if (pid) resident.erase(pid);
      clear(ei);
      activate(ei, level);
      *ei_out = ei;
      *si_out = 0;
      return true;
    }
    return false;
  }
  // runtime.py:273-283
  void place(uint32_t pid, int32_t ei, int32_t si, int64_t frame) {
    auto old = resident.find(pid);
    bool had = old != resident.end();
    std::pair<int32_t, int32_t> prev = had ? old->second : std::make_pair(-1, -1);
    Entry& x = e[ei];
    x.slots[si] = pid;
    if (++x.occupied == (int)x.slots.size()) open[x.level].erase(ei);
    touch(ei, frame);
    resident[pid] = {ei, si};
    if (had && prev != std::make_pair(ei, si)) {
      Entry& o = e[prev.first];
      o.slots[prev.second] = 0;
      --o.occupied;
      open[o.level].insert(prev.first);
      if (o.occupied == 0) clear(prev.first);
    }
  }
};

extern "C" {

vms_pagetable* vms_pt_create(int64_t capacity) {
  if (capacity < 1) {
    vms::set_error("page table needs at least one entry");
    return nullptr;
  }
  try {
    return new vms_pagetable(capacity);
  } catch (...) {
    vms::set_error("page table allocation failed");
    return nullptr;
  }
}

void vms_pt_destroy(vms_pagetable* pt) { delete pt; }

int32_t vms_pt_update(vms_pagetable* pt, const uint32_t* pid, const uint32_t* enc,
                      const uint8_t* direct, const uint8_t* level, int64_t n, int64_t frame,
                      double budget, uint32_t* plan_pid, uint8_t* plan_level,
                      int32_t* plan_entry, int32_t* plan_slot, int64_t plan_cap,
                      int64_t* n_plan, int64_t* missing) {
  if (!pt) {
    vms::set_error("null page table");
    return VMS_ERR_INVALID;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (level[i] > 30) {
      vms::set_error("LOD level %d out of range", (int)level[i]);
      return VMS_ERR_INVALID;
    }
  }
  // pass 1 (runtime.py:312-327)
  struct Work {
    int cls;
    int64_t neg_enc;
    uint32_t pid;
    int level;
    bool operator<(const Work& o) const {
      return std::tie(cls, neg_enc, pid) < std::tie(o.cls, o.neg_enc, o.pid);
    }
  };
  std::vector<Work> work;
  work.reserve(n);
  for (int64_t i = 0; i < n; ++i) {
    auto it = pt->resident.find(pid[i]);
    if (it != pt->resident.end()) {
      const int32_t ei = it->second.first;
      pt->touch(ei, frame);
      pt->protect(ei);
      if (pt->e[ei].level != (int)level[i])
        work.push_back({2, -(int64_t)enc[i], pid[i], (int)level[i]});
    } else {
      work.push_back({direct[i] ? 0 : 1, -(int64_t)enc[i], pid[i], (int)level[i]});
    }
  }
  std::sort(work.begin(), work.end());
  // pass 2 (runtime.py:330-343)
  int64_t np_ = 0;
  double spent = 0.0;
  for (const Work& w : work) {
    const double cost = 1.0 / (double)(int64_t(1) << w.level);
    if (spent + cost > budget) break;
    int32_t ei, si;
    if (!pt->alloc(w.level, &ei, &si)) continue;
    pt->place(w.pid, ei, si, frame);
    pt->protect(ei);
    if (np_ < plan_cap) {
      plan_pid[np_] = w.pid;
      plan_level[np_] = (uint8_t)w.level;
      plan_entry[np_] = ei;
      plan_slot[np_] = si;
    }
    ++np_;
    spent += cost;
  }
  int64_t miss = 0;
  for (int64_t i = 0; i < n; ++i) miss += pt->resident.count(pid[i]) ? 0 : 1;
  for (int32_t ei : pt->prot_list) pt->prot[ei] = 0;
  pt->prot_list.clear();
  *n_plan = np_;
  *missing = miss;
  if (np_ > plan_cap) {
    vms::set_error("plan capacity %lld < %lld", (long long)plan_cap, (long long)np_);
    return VMS_ERR_NOMEM;
  }
  return VMS_OK;
}

int64_t vms_pt_capacity(const vms_pagetable* pt) { return pt ? (int64_t)pt->e.size() : -1; }

int64_t vms_pt_occupied(const vms_pagetable* pt) {
  return pt ? (int64_t)(pt->e.size() - pt->empty_.size()) : -1;
}

int64_t vms_pt_resident_count(const vms_pagetable* pt) {
  return pt ? (int64_t)pt->resident.size() : -1;
}

int32_t vms_pt_resident(const vms_pagetable* pt, uint32_t* pid, int32_t* entry, int32_t* slot,
                        int64_t cap) {
  if (!pt || cap < (int64_t)pt->resident.size()) {
    vms::set_error("resident export: bad table or capacity");
    return VMS_ERR_INVALID;
  }
  int64_t i = 0;
  for (const auto& kv : pt->resident) {
    pid[i] = kv.first;
    entry[i] = kv.second.first;
    slot[i] = kv.second.second;
    ++i;
  }
  return VMS_OK;
}

int32_t vms_pt_entries(const vms_pagetable* pt, int32_t* level, int64_t* last_used,
                       uint32_t* slots, int32_t max_slots) {
  if (!pt) return VMS_ERR_INVALID;
  for (size_t i = 0; i < pt->e.size(); ++i) {
    const auto& x = pt->e[i];
    level[i] = x.level;
    last_used[i] = x.last;
    for (int32_t s = 0; s < max_slots; ++s)
      slots[i * max_slots + s] = s < (int32_t)x.slots.size() ? x.slots[s] : 0u;
    if ((int32_t)x.slots.size() > max_slots) {
      vms::set_error("entry %zu has %zu slots > %d", i, x.slots.size(), max_slots);
      return VMS_ERR_INVALID;
    }
  }
  return VMS_OK;
}

int32_t vms_pt_resident_counts(const vms_pagetable* pt, int64_t* counts, int32_t levels) {
  if (!pt) return VMS_ERR_INVALID;
  for (int32_t k = 0; k < levels; ++k) counts[k] = 0;
  for (const auto& kv : pt->resident) {
    const int lv = pt->e[kv.second.first].level;
    if (lv < 0 || lv >= levels) {
      vms::set_error("resident level %d outside [0, %d)", lv, levels);
      return VMS_ERR_INVARIANT;
    }
    counts[lv] += 1;
  }
  return VMS_OK;
}

// runtime.py:218-234 plus the index structures' own consistency.
int32_t vms_pt_check(const vms_pagetable* pt) {
  if (!pt) return VMS_ERR_INVALID;
  std::map<uint32_t, std::pair<int32_t, int32_t>> seen;
  for (size_t ei = 0; ei < pt->e.size(); ++ei) {
    const auto& x = pt->e[ei];
    if (x.level < 0) {
      if (!x.slots.empty()) {
        vms::set_error("empty entry %zu has slots", ei);
        return VMS_ERR_INVARIANT;
      }
      if (!pt->empty_.count((int32_t)ei)) {
        vms::set_error("empty entry %zu missing from the free set", ei);
        return VMS_ERR_INVARIANT;
      }
      continue;
    }
    if (x.slots.size() != (size_t(1) << x.level)) {
      vms::set_error("entry %zu slot count mismatch", ei);
      return VMS_ERR_INVARIANT;
    }
    int occ = 0;
    for (size_t si = 0; si < x.slots.size(); ++si) {
      const uint32_t pid = x.slots[si];
      if (!pid) continue;
      ++occ;
      if (seen.count(pid)) {
        vms::set_error("page %u resident twice", pid);
        return VMS_ERR_INVARIANT;
      }
      seen[pid] = {(int32_t)ei, (int32_t)si};
    }
    const bool is_open = pt->open[x.level].count((int32_t)ei) != 0;
    if (occ != x.occupied || is_open != (occ < (int)x.slots.size()) ||
        !pt->lru_.count({x.last, (int32_t)ei})) {
      vms::set_error("entry %zu index structures out of sync", ei);
      return VMS_ERR_INVARIANT;
    }
  }
  if (seen != pt->resident) {
    vms::set_error("residency map out of sync with entries");
    return VMS_ERR_INVARIANT;
  }
  return VMS_OK;
}

int64_t vms_pt_chunks(const vms_pagetable* pt, int64_t page_size, vms_chunk* out, int64_t cap,
                      int64_t* n_records) {
  if (!pt || page_size <= 0) return -1;
  const uint32_t kChunk = 128;
  int64_t n = 0;
  uint64_t gather = 0;
  for (const auto& kv : pt->resident) {
    const int32_t ei = kv.second.first, si = kv.second.second;
    const int lv = pt->e[ei].level;
    const uint64_t per = (uint64_t)page_size >> lv;
    uint64_t row = (uint64_t)ei * page_size + (uint64_t)si * per;
    for (uint64_t k = 0; k < per; k += kChunk) {
      const uint32_t c = (uint32_t)std::min<uint64_t>(kChunk, per - k);
      if (n < cap) out[n] = vms_chunk{(uint32_t)(row + k), (uint32_t)(gather + k), c, 0u};
      ++n;
    }
    gather += per;
  }
  if (n_records) *n_records = (int64_t)gather;
  return n;
}

}  // extern "C"
