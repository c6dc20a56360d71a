// Device-arena address map (placement rule of memory_pool.hpp:55-86; see
// planner.hpp for the representation). The map is a vector of segments in
// address order that tiles [0, capacity); allocating splits a free segment,
// freeing merges the freed segment with free neighbours, so the free
// segments are exactly the coalesced free extents the placement rule ranges
// over.
#include <algorithm>

#include "planner.hpp"

namespace vdnnp {

Arena::Arena(u64 capacity, bool trace) : cap_(capacity), trace_(trace) {
  if (capacity > 0) segs_.push_back(Seg{0, capacity, false, 0, -1});
}

// The byte*ns usage integral needs a clock that never runs backwards
// (memory_pool.hpp:174-180).
void Arena::clock_to(i64 t) {
  if (t < now_) throw PlanError(Err::Pool, "arena clock moved backwards (" + std::to_string(t) + " < " +
                                               std::to_string(now_) + ")");
  area_ += static_cast<u128>(live_) * static_cast<u128>(t - now_);
  now_ = t;
}

size_t Arena::seg_at(u64 off) const {
  auto it = std::lower_bound(segs_.begin(), segs_.end(), off, [](const Seg& s, u64 o) { return s.off < o; });
  if (it == segs_.end() || it->off != off || !it->used)
    throw PlanError(Err::Pool, "no live allocation starts at offset " + std::to_string(off));
  return static_cast<size_t>(it - segs_.begin());
}

std::optional<u64> Arena::place(u64 bytes, const std::string& tag, i64 t, bool pinned) {
  if (bytes == 0) throw PlanError(Err::Pool, "arena: a 0-byte request");
  clock_to(t);
  const u64 len = round_up(bytes, kAlign);
  const bool from_top = pinned || len <= cap_ / 8;
  size_t pick = segs_.size();
  for (size_t i = 0; i < segs_.size(); ++i) {
    const Seg& s = segs_[i];
    if (s.used || s.len < len) continue;
    // top: the last (highest) fitting gap; bottom: the first of the narrowest
    if (from_top || pick == segs_.size() || s.len < segs_[pick].len) pick = i;
  }
  if (pick == segs_.size()) return std::nullopt;
  Seg gap = segs_[pick];
  const u64 spare = gap.len - len;
  const u64 off = from_top ? gap.off + spare : gap.off;
  int32_t tag_id = -1;
  if (trace_) {
    tag_id = static_cast<int32_t>(tags_.size());
    tags_.push_back(tag);
  }
  Seg blk{off, len, true, bytes, tag_id};
  if (spare == 0) {
    segs_[pick] = blk;
  } else if (from_top) {
    segs_[pick].len = spare;
    segs_.insert(segs_.begin() + static_cast<std::ptrdiff_t>(pick) + 1, blk);
  } else {
    segs_[pick] = blk;
    segs_.insert(segs_.begin() + static_cast<std::ptrdiff_t>(pick) + 1, Seg{off + len, spare, false, 0, -1});
  }
  live_ += len;
  hw_ = std::max(hw_, live_);
  if (trace_) rows_.push_back(TraceRow{t, 'a', tag, off, len, live_, hw_});
  return off;
}

void Arena::free_at(u64 off, i64 t) {
  clock_to(t);
  size_t i = seg_at(off);
  const Seg gone = segs_[i];
  live_ -= gone.len;
  segs_[i] = Seg{gone.off, gone.len, false, 0, -1};
  // merge with a free right neighbour, then with a free left neighbour
  if (i + 1 < segs_.size() && !segs_[i + 1].used) {
    segs_[i].len += segs_[i + 1].len;
    segs_.erase(segs_.begin() + static_cast<std::ptrdiff_t>(i) + 1);
  }
  if (i > 0 && !segs_[i - 1].used) {
    segs_[i - 1].len += segs_[i].len;
    segs_.erase(segs_.begin() + static_cast<std::ptrdiff_t>(i));
  }
  if (trace_) rows_.push_back(TraceRow{t, 'f', tags_[static_cast<size_t>(gone.tag)], gone.off, gone.len, live_, hw_});
}

u64 Arena::requested_at(u64 off) const { return segs_[seg_at(off)].req; }

std::pair<u64, u64> Arena::widest_gap() const {
  std::pair<u64, u64> best{0, 0};
  for (const Seg& s : segs_)
    if (!s.used && s.len > best.second) best = {s.off, s.len};
  return best;
}

u64 Arena::free_total() const {
  u64 t = 0;
  for (const Seg& s : segs_)
    if (!s.used) t += s.len;
  return t;
}

bool Arena::would_fragment(u64 bytes) const {
  const u64 len = round_up(bytes, kAlign);
  return len <= free_total() && len > widest_gap().second;
}

u128 Arena::byte_ns_until(i64 t) {
  clock_to(t);
  return area_;
}

void Arena::audit() const {
  u64 at = 0, used = 0;
  for (size_t i = 0; i < segs_.size(); ++i) {
    const Seg& s = segs_[i];
    if (s.off != at) throw PlanError(Err::Pool, "arena audit: segments do not tile the address range");
    if (s.len == 0) throw PlanError(Err::Pool, "arena audit: empty segment");
    if (!s.used && i > 0 && !segs_[i - 1].used) throw PlanError(Err::Pool, "arena audit: neighbouring free segments");
    if (s.used) used += s.len;
    at += s.len;
  }
  if (at != cap_) throw PlanError(Err::Pool, "arena audit: segments do not cover the capacity");
  if (used != live_) throw PlanError(Err::Pool, "arena audit: live byte count drifted");
}

}  // namespace vdnnp
