// Memory model, LRU device plan and physical placement.
//
// simulate_model: §II-C: for c_i (i) load the leaf operands not in
//   memory, (ii) produce the output, (iii) release tensors no remaining contraction needs,
//   including a ROOT output; M_i after (iii), transient after (ii) (reading G-5).
// lru_plan: MemHC-style "pre-protected LRU" eviction to host, readings E-1..E-8,
// or (policy EVICT_NEXT_USE, reading E-9) Belady-style: the victim is the resident non-operand
// whose next use in the known schedule is farthest away, ties to the least recently used:
//   before c_i evict least-recently-used non-operand tensors until operands + output fit;
//   leaves are dropped (no D2H), an intermediate is copied to host on its first eviction
//   and the host copy is kept until release; fetches are touches; LRU ties cannot occur
//   (one clock tick per touch: operands left then right, then the output).
//   Peer-HBM tier (readings E-10, E-11): a victim with no copy off the device other than a
//   leaf's caller host copy goes to the peer tier (P2P_OUT) while peer_cap has room, and its
//   re-fetches are P2P_IN; the peer copy lives until release.  Peer-homed leaves are always
//   fetched P2P_IN and dropped on eviction.
// build_phys: offline placement of every residency in the device pool (best fit) and the
//   host pool, plus cross-stream event dependencies: RAW on data (ready op of each operand,
//   D2H before a re-fetch) and WAR/WAW on reused byte ranges.
#include "plan.hpp"

#include <algorithm>
#include <limits>

namespace cc {

void check_order(const Dag& g, const std::vector<int32_t>& order) {
  std::vector<int32_t> pos(g.nodes.size(), -1);
  for (size_t i = 0; i < order.size(); ++i) {
    const int32_t u = order[i];
    if (u < 0 || u >= int32_t(g.nodes.size())) throw Error(CC_E_INVAL, "schedule: bad node");
    if (g.nodes[u].leaf()) throw Error(CC_E_INVAL, "schedule: leaf " + std::to_string(g.nodes[u].id) + " scheduled");
    if (pos[u] >= 0) throw Error(CC_E_INVAL, "schedule: node " + std::to_string(g.nodes[u].id) + " twice");
    pos[u] = int32_t(i);
  }
  if (int64_t(order.size()) != g.n_contr) throw Error(CC_E_INVAL, "schedule: missing contractions");
  for (size_t i = 0; i < order.size(); ++i) {
    const Node& n = g.nodes[order[i]];
    for (int32_t c : {n.l, n.r})
      if (!g.nodes[c].leaf() && pos[c] > int32_t(i))
        throw Error(CC_E_INVAL, "schedule: node " + std::to_string(n.id) + " before its child " +
                                    std::to_string(g.nodes[c].id));
  }
}

ModelTrace simulate_model(const Dag& g, const std::vector<int32_t>& order) {
  ModelTrace tr;
  std::vector<int32_t> remaining(g.nodes.size());
  std::vector<uint8_t> resident(g.nodes.size(), 0);
  for (size_t u = 0; u < g.nodes.size(); ++u) remaining[u] = int32_t(g.nodes[u].parents.size());
  int64_t used = 0;
  tr.M.reserve(order.size() + 1);
  tr.transient.reserve(order.size());
  tr.M.push_back(0);
  for (int32_t u : order) {
    const Node& n = g.nodes[u];
    for (int32_t c : {n.l, n.r})                  // (i) lazy leaf loads
      if (g.nodes[c].leaf() && !resident[c]) {
        resident[c] = 1;
        used += g.nodes[c].size;
      }
    resident[u] = 1;                               // (ii)
    used += n.size;
    tr.transient.push_back(used);
    tr.transient_peak = std::max(tr.transient_peak, used);
    for (int32_t c : {n.l, n.r})                  // (iii)
      if (--remaining[c] == 0) {
        resident[c] = 0;
        used -= g.nodes[c].size;
      }
    if (remaining[u] == 0) {
      resident[u] = 0;
      used -= n.size;
    }
    tr.M.push_back(used);
    tr.peak = std::max(tr.peak, used);
  }
  return tr;
}

LruPlan lru_plan(const Dag& g, const std::vector<int32_t>& order, int64_t cap, EvictPolicy policy, int64_t peer_cap,
                 const std::vector<uint8_t>* peer_home) {
  const bool bounded = cap > 0;
  const bool next_use = policy == EVICT_NEXT_USE;
  const size_t n = g.nodes.size();
  LruPlan p;
  std::vector<int32_t> remaining(n);
  std::vector<uint8_t> resident(n, 0), host_copy(n, 0), peer_copy(n, 0);
  auto homed = [&](int32_t x) { return peer_home && (*peer_home)[size_t(x)] != 0; };
  int64_t peer_used = 0;
  std::vector<int64_t> stamp(n, 0);
  for (size_t u = 0; u < n; ++u) remaining[u] = int32_t(g.nodes[u].parents.size());
  // E-9: the steps reading each tensor, in order (CSR), and a cursor to its next use
  std::vector<int32_t> use_start(n + 1, 0), use_step, cursor(n, 0);
  if (next_use) {
    for (int32_t u : order) {
      ++use_start[size_t(g.nodes[u].l) + 1];
      ++use_start[size_t(g.nodes[u].r) + 1];
    }
    for (size_t x = 0; x < n; ++x) use_start[x + 1] += use_start[x];
    use_step.resize(size_t(use_start[n]));
    std::vector<int32_t> fill(use_start.begin(), use_start.end() - 1);
    for (size_t i = 0; i < order.size(); ++i) {
      const Node& nd = g.nodes[size_t(order[i])];
      use_step[size_t(fill[size_t(nd.l)]++)] = int32_t(i);
      use_step[size_t(fill[size_t(nd.r)]++)] = int32_t(i);
    }
  }
  auto nxt = [&](int32_t x) -> int64_t { return use_step[size_t(use_start[size_t(x)] + cursor[size_t(x)])]; };
  // resident tensors in eviction order: LRU (E-1): (stamp, node); next use (E-9):
  // (-next use, stamp) with the node in the second slot of a tuple-like key
  auto key = [&](int32_t x) -> std::pair<int64_t, int64_t> {
    return next_use ? std::make_pair(-nxt(x), stamp[x]) : std::make_pair(stamp[x], int64_t(0));
  };
  std::set<std::pair<std::pair<int64_t, int64_t>, int32_t>> lru;
  int64_t clock = 0, used = 0, host = 0;
  p.used.reserve(order.size() + 1);
  p.used.push_back(0);
  auto erase = [&](int32_t x) { lru.erase({key(x), x}); };
  auto insert = [&](int32_t x) { lru.insert({key(x), x}); };
  for (int32_t u : order) {
    const Node& nd = g.nodes[u];
    const int32_t ops[2] = {nd.l, nd.r};
    const int64_t work = g.nodes[nd.l].size + g.nodes[nd.r].size + nd.size;
    if (bounded && work > cap)
      throw Error(CC_E_INFEASIBLE, "contraction " + std::to_string(nd.id) + " needs " + std::to_string(work) +
                                       " bytes > cap " + std::to_string(cap));
    int64_t need = nd.size;
    for (int32_t x : ops)
      if (!resident[x]) need += g.nodes[x].size;
    while (bounded && used + need > cap) {          // E-1 (victim order: E-1 LRU or E-9 next use)
      auto it = lru.begin();
      while (it != lru.end() && (it->second == ops[0] || it->second == ops[1])) ++it;
      if (it == lru.end()) throw Error(CC_E_INFEASIBLE, "no evictable tensor");
      const int32_t v = it->second;
      lru.erase(it);
      ++p.evictions;
      const int64_t vs = g.nodes[v].size;
      const bool stash = !peer_copy[v] && !homed(v) && !host_copy[v];
      if (stash && peer_used + vs <= peer_cap) {      // E-10: copy to the peer tier
        ++p.p2p_out_count;
        p.p2p_out_bytes += vs;
        peer_copy[v] = 1;
        peer_used += vs;
        p.peer_peak = std::max(p.peer_peak, peer_used);
        p.ops.push_back({OP_P2P_OUT, v});
      } else if (!g.nodes[v].leaf() && stash) {       // E-4: first eviction copies to host
        ++p.d2h_count;
        p.d2h_bytes += g.nodes[v].size;
        host_copy[v] = 1;
        host += g.nodes[v].size;
        p.host_peak = std::max(p.host_peak, host);
        p.ops.push_back({OP_D2H, v});
      } else {                                       // E-3 / clean re-eviction
        p.ops.push_back({OP_DROP, v});
      }
      resident[v] = 0;
      used -= g.nodes[v].size;
    }
    for (int32_t x : ops)                            // this step's use is consumed (keys change)
      if (resident[x]) erase(x);
    for (int32_t x : ops) ++cursor[size_t(x)];
    for (int32_t x : ops) {                          // fetch + touch, left then right (E-2)
      if (!resident[x]) {
        if (peer_copy[x] || homed(x)) {              // E-10 / E-11: over NVLink
          ++p.p2p_in_count;
          p.p2p_in_bytes += g.nodes[x].size;
          p.ops.push_back({OP_P2P_IN, x});
        } else {
          ++p.h2d_count;
          p.h2d_bytes += g.nodes[x].size;
          p.ops.push_back({OP_H2D, x});
        }
        used += g.nodes[x].size;
        resident[x] = 1;
      }
      stamp[x] = ++clock;
    }
    // operands are (re-)inserted below only while they stay resident
    used += nd.size;                                  // output
    stamp[u] = ++clock;
    resident[u] = 1;
    p.ops.push_back({OP_CONTRACT, u});
    p.transient_peak = std::max(p.transient_peak, used);
    for (int32_t x : ops)                             // release at last use (E-8)
      if (--remaining[x] == 0) {
        resident[x] = 0;
        used -= g.nodes[x].size;
        if (host_copy[x]) {
          host_copy[x] = 0;
          host -= g.nodes[x].size;
        }
        if (peer_copy[x]) {
          peer_copy[x] = 0;
          peer_used -= g.nodes[x].size;
        }
        p.ops.push_back({OP_FREE, x});
      }
    for (int32_t x : ops)
      if (resident[x]) insert(x);
    if (remaining[u] == 0) {                          // ROOT output released at once
      resident[u] = 0;
      used -= nd.size;
      p.ops.push_back({OP_FREE, u});
    } else {
      insert(u);
    }
    p.peak = std::max(p.peak, used);
    p.used.push_back(used);
  }
  if (used != 0 || host != 0 || peer_used != 0) throw Error(CC_E_STATE, "plan: accounting did not return to zero");
  return p;
}

// ---------------------------------------------------------------------------------------
RangeAlloc::RangeAlloc(int64_t capacity, Policy policy) : policy_(policy) {
  if (capacity > 0) {
    by_off_[0] = capacity;
    by_size_.insert({capacity, 0});
  }
}

int64_t RangeAlloc::take(int64_t off, int64_t size, int64_t bytes) {
  by_size_.erase({size, off});
  by_off_.erase(off);
  if (size > bytes) {
    by_off_[off + bytes] = size - bytes;
    by_size_.insert({size - bytes, off + bytes});
  }
  high_ = std::max(high_, off + bytes);
  return off;
}

int64_t RangeAlloc::alloc(int64_t bytes) {
  if (policy_ == NEXT_FIT) {
    // first fit at or after the cursor (a block straddling the cursor is used from the
    // cursor on), then wrap around once
    for (int pass = 0; pass < 2; ++pass) {
      auto it = by_off_.upper_bound(pass == 0 ? cursor_ : -1);
      if (it != by_off_.begin()) {
        auto prev = std::prev(it);
        if (pass == 0 && prev->first + prev->second > cursor_) it = prev;
      }
      for (; it != by_off_.end(); ++it) {
        int64_t off = it->first, size = it->second;
        if (pass == 0 && off < cursor_) {
          // split the block at the cursor so allocation proceeds forward
          const int64_t lo = cursor_ - off;
          if (size - lo < bytes) continue;
          by_size_.erase({size, off});
          by_off_.erase(off);
          by_off_[off] = lo;
          by_size_.insert({lo, off});
          off = cursor_;
          size -= lo;
          by_off_[off] = size;
          by_size_.insert({size, off});
        }
        if (size >= bytes) {
          cursor_ = off + bytes;
          return take(off, size, bytes);
        }
      }
    }
    return -1;
  }
  auto it = by_size_.lower_bound({bytes, std::numeric_limits<int64_t>::min()});
  if (it == by_size_.end()) return -1;
  return take(it->second, it->first, bytes);
}

bool RangeAlloc::take_range(int64_t off, int64_t bytes) {
  auto it = by_off_.upper_bound(off);
  if (it == by_off_.begin()) return false;
  --it;
  if (it->first > off || it->first + it->second < off + bytes) return false;
  const int64_t b = it->first, size = it->second;
  by_size_.erase({size, b});
  by_off_.erase(it);
  if (off > b) {
    by_off_[b] = off - b;
    by_size_.insert({off - b, b});
  }
  if (b + size > off + bytes) {
    by_off_[off + bytes] = b + size - off - bytes;
    by_size_.insert({b + size - off - bytes, off + bytes});
  }
  high_ = std::max(high_, off + bytes);
  return true;
}

int64_t RangeAlloc::free_bytes() const {
  int64_t t = 0;
  for (const auto& kv : by_off_) t += kv.second;
  return t;
}

void RangeAlloc::free(int64_t off, int64_t bytes) {
  auto next = by_off_.lower_bound(off);
  if (next != by_off_.end() && next->first == off + bytes) {
    bytes += next->second;
    by_size_.erase({next->second, next->first});
    next = by_off_.erase(next);
  }
  if (next != by_off_.begin()) {
    auto prev = std::prev(next);
    if (prev->first + prev->second == off) {
      off = prev->first;
      bytes += prev->second;
      by_size_.erase({prev->second, prev->first});
      by_off_.erase(prev);
    }
  }
  by_off_[off] = bytes;
  by_size_.insert({bytes, off});
}

RangeTracker::RangeTracker(int64_t capacity) {
  pieces_[0] = Piece{capacity, {-1, -1, -1}};
}

void RangeTracker::split(int64_t at) {
  auto it = pieces_.upper_bound(at);
  if (it == pieces_.begin()) return;
  --it;
  if (it->first == at || it->second.end <= at) return;
  Piece hi = it->second;
  it->second.end = at;
  pieces_[at] = hi;
}

void RangeTracker::access(int64_t off, int64_t bytes, int stream, int32_t op, std::vector<int32_t>& deps,
                          std::vector<int32_t>* same) {
  split(off);
  split(off + bytes);
  for (auto it = pieces_.find(off); it != pieces_.end() && it->first < off + bytes; ++it) {
    for (int s = 0; s < 3; ++s)
      if (s != stream && it->second.last[s] >= 0) deps.push_back(it->second.last[s]);
    if (same && it->second.last[stream] >= 0) same->push_back(it->second.last[stream]);
    it->second.last[stream] = op;
  }
}

static int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

PhysPlan build_phys(const Dag& g, const LruPlan& lp, const std::vector<uint8_t>& leaf_on_device,
                    int64_t pool_bytes, int64_t align, RangeAlloc::Policy policy, int64_t peer_bytes, bool leaf_slots,
                    bool compact) {
  PhysPlan pp;
  const size_t n = g.nodes.size();
  // fixed leaf slots: assigned in first-load order from offset 0; the intermediates share
  // [leaf_region, pool) (the top of the pool stays free for the executor's metadata)
  std::vector<int64_t> slot(n, -1);
  int64_t leaf_region = 0;
  if (leaf_slots) {
    for (const auto& op : lp.ops)
      if ((op.kind == OP_H2D || op.kind == OP_P2P_IN) && g.nodes[size_t(op.node)].leaf() &&
          !leaf_on_device[size_t(op.node)] && slot[size_t(op.node)] < 0) {
        slot[size_t(op.node)] = leaf_region;
        leaf_region += round_up(g.nodes[size_t(op.node)].size, align);
      }
    if (leaf_region > pool_bytes) throw Error(CC_E_NOMEM, "leaf slots exceed the pool");
  }
  // host pool: sized for the worst case (sum of all D2H'd sizes), placed best-fit
  int64_t host_cap = 0;
  for (const auto& op : lp.ops)
    if (op.kind == OP_D2H) host_cap += round_up(g.nodes[op.node].size, align);
  RangeAlloc dev0(pool_bytes - leaf_region, policy), hostp(host_cap), peerp(peer_bytes);
  // the intermediates' allocator works on [leaf_region, pool)
  struct Shifted {
    RangeAlloc& a;
    int64_t base;
    int64_t alloc(int64_t b) {
      const int64_t o = a.alloc(b);
      return o < 0 ? o : o + base;
    }
    void free(int64_t o, int64_t b) { a.free(o - base, b); }
    bool take_range(int64_t o, int64_t b) { return a.take_range(o - base, b); }
  } dev{dev0, leaf_region};
  RangeTracker dtr(pool_bytes), htr(std::max<int64_t>(host_cap, 1)), ptr(std::max<int64_t>(peer_bytes, 1));
  std::vector<int64_t> dev_off(n, -1), host_off(n, -1), peer_off(n, -1);
  std::vector<int32_t> ready(n, -1), ready_stream(n, -1), d2h_op(n, -1), p2p_op(n, -1);
  auto need_ready = [&](int32_t x, int stream, std::vector<int32_t>& deps) {
    if (ready[x] >= 0 && ready_stream[x] != stream) deps.push_back(ready[x]);
  };
  // tensors placed in the shared region (not leaf slots): offset -> node, for compaction
  std::map<int64_t, int32_t> placed;
  // allocation for op `me` on `stream`: a free block, else (compact) a cleared window
  auto alloc_for = [&](int64_t rb, int stream, int32_t me, PhysOp& op, int32_t self) -> int64_t {
    int64_t off = dev.alloc(rb);
    if (off >= 0 || !compact) return off;
    // windows start at a free block's start or right after a placed tensor; the cheapest has
    // the fewest bytes of resident tensors, each at most half the request (so they fit
    // elsewhere) and none of them an operand the op is about to read
    std::vector<int64_t> starts;
    for (const auto& kv : dev0.free_blocks()) starts.push_back(kv.first + leaf_region);
    for (const auto& kv : placed) starts.push_back(kv.first + round_up(g.nodes[size_t(kv.second)].size, align));
    const Node& me_node = g.nodes[size_t(self)];
    int64_t best = -1, best_cost = INT64_MAX;
    for (int64_t w0 : starts) {
      if (w0 < leaf_region || w0 + rb > pool_bytes) continue;
      int64_t cost = 0;
      bool ok = true;
      auto it = placed.upper_bound(w0);
      if (it != placed.begin()) --it;
      for (; it != placed.end() && it->first < w0 + rb; ++it) {
        const int32_t y = it->second;
        const int64_t ys = round_up(g.nodes[size_t(y)].size, align);
        if (it->first + ys <= w0) continue;
        if (ys * 2 > rb || (op.kind == OP_CONTRACT && (y == me_node.l || y == me_node.r))) {
          ok = false;
          break;
        }
        cost += ys;
      }
      if (ok && cost < best_cost && dev0.free_bytes() - (rb - cost) >= cost) {
        best = w0;
        best_cost = cost;
      }
    }
    if (best < 0) return -1;
    // reserve the window's free pieces, move its tensors out, then allocate it whole
    std::vector<std::pair<int64_t, int64_t>> reserved;
    for (const auto& kv : std::map<int64_t, int64_t>(dev0.free_blocks())) {
      const int64_t a = std::max(kv.first + leaf_region, best), b = std::min(kv.first + leaf_region + kv.second, best + rb);
      if (b > a && dev.take_range(a, b - a)) reserved.push_back({a, b - a});
    }
    std::vector<int32_t> movers;
    for (auto it = placed.lower_bound(0); it != placed.end(); ++it) {
      const int64_t ys = round_up(g.nodes[size_t(it->second)].size, align);
      if (it->first < best + rb && it->first + ys > best) movers.push_back(it->second);
    }
    for (int32_t y : movers) {
      const int64_t ys = round_up(g.nodes[size_t(y)].size, align);
      const int64_t src = dev_off[size_t(y)];
      const int64_t dst = dev.alloc(ys);
      if (dst < 0) throw Error(CC_E_NOMEM, "compaction: no room to relocate node " + std::to_string(g.nodes[size_t(y)].id));
      need_ready(y, stream, op.deps);
      dtr.access(src, ys, stream, me, op.deps);         // read the old range (after its writer)
      dtr.access(dst, ys, stream, me, op.deps);         // write the new range (after its readers)
      op.pre_moves.push_back(Move{y, src, dst, g.nodes[size_t(y)].size});
      ++pp.n_moves;
      pp.move_bytes += g.nodes[size_t(y)].size;
      placed.erase(src);
      placed[dst] = y;
      dev_off[size_t(y)] = dst;
      ready[size_t(y)] = me;
      ready_stream[size_t(y)] = stream;
      reserved.push_back({src, ys});                    // its old range is inside the window
    }
    for (const auto& r : reserved) dev.free(r.first, r.second);
    if (!dev.take_range(best, rb)) throw Error(CC_E_STATE, "compaction: window not free");
    return best;
  };
  for (const auto& lop : lp.ops) {
    const int32_t x = lop.node;
    const Node& nd = g.nodes[x];
    const int32_t me = int32_t(pp.ops.size());
    PhysOp op{lop.kind, x, S_NONE};
    op.bytes = nd.size;
    const int64_t rb = round_up(nd.size, align);
    switch (lop.kind) {
      case OP_H2D: {
        if (nd.leaf() && leaf_on_device[x]) break;            // already in HBM: no copy
        const int64_t off = slot[x] >= 0 ? slot[x] : alloc_for(rb, S_H2D, me, op, x);
        if (off < 0) throw Error(CC_E_NOMEM, "device pool fragmented/too small for node " + std::to_string(nd.id));
        dev_off[x] = off;
        if (slot[x] < 0) placed[off] = x;
        op.stream = S_H2D;
        op.dev_off = off;
        dtr.access(off, rb, S_H2D, me, op.deps, &op.same_deps);
        if (!nd.leaf()) {                                       // re-fetch of an evicted intermediate
          op.host_off = host_off[x];
          if (d2h_op[x] >= 0) op.deps.push_back(d2h_op[x]);
          htr.access(host_off[x], rb, S_H2D, me, op.deps, &op.same_deps);
        }
        ready[x] = me;
        ready_stream[x] = S_H2D;
        pp.h2d_bytes += nd.size;
        break;
      }
      case OP_P2P_IN: {
        if (nd.leaf() && leaf_on_device[x]) break;            // already in HBM: no copy
        const int64_t off = slot[x] >= 0 ? slot[x] : alloc_for(rb, S_H2D, me, op, x);
        if (off < 0) throw Error(CC_E_NOMEM, "device pool fragmented/too small for node " + std::to_string(nd.id));
        dev_off[x] = off;
        if (slot[x] < 0) placed[off] = x;
        op.stream = S_H2D;                                      // inbound copies share the H2D stream
        op.dev_off = off;
        dtr.access(off, rb, S_H2D, me, op.deps, &op.same_deps);
        if (peer_off[x] >= 0) {                                 // stashed copy in the peer tier
          op.peer_off = peer_off[x];
          if (p2p_op[x] >= 0) op.deps.push_back(p2p_op[x]);
          ptr.access(peer_off[x], rb, S_H2D, me, op.deps, &op.same_deps);
        }
        ready[x] = me;
        ready_stream[x] = S_H2D;
        pp.p2p_in_bytes += nd.size;
        break;
      }
      case OP_P2P_OUT: {
        if (nd.leaf() && leaf_on_device[x]) break;            // caller device leaf: nothing to move
        const int64_t poff = peerp.alloc(rb);
        if (poff < 0) throw Error(CC_E_NOMEM, "peer tier fragmented/too small for node " + std::to_string(nd.id));
        peer_off[x] = poff;
        op.stream = S_D2H;                                      // outbound copies share the D2H stream
        op.dev_off = dev_off[x];
        op.peer_off = poff;
        need_ready(x, S_D2H, op.deps);
        dtr.access(dev_off[x], rb, S_D2H, me, op.deps);
        ptr.access(poff, rb, S_D2H, me, op.deps);
        p2p_op[x] = me;
        if (slot[x] < 0) {                            // a leaf slot stays reserved
          dev.free(dev_off[x], rb);
          placed.erase(dev_off[x]);
        }
        dev_off[x] = -1;
        pp.p2p_out_bytes += nd.size;
        break;
      }
      case OP_D2H: {
        const int64_t hoff = hostp.alloc(rb);
        if (hoff < 0) throw Error(CC_E_NOMEM, "host pool allocation failed");
        host_off[x] = hoff;
        op.stream = S_D2H;
        op.dev_off = dev_off[x];
        op.host_off = hoff;
        need_ready(x, S_D2H, op.deps);
        dtr.access(dev_off[x], rb, S_D2H, me, op.deps);
        htr.access(hoff, rb, S_D2H, me, op.deps);
        d2h_op[x] = me;
        if (slot[x] < 0) {                            // a leaf slot stays reserved
          dev.free(dev_off[x], rb);
          placed.erase(dev_off[x]);
        }
        dev_off[x] = -1;
        pp.d2h_bytes += nd.size;
        break;
      }
      case OP_DROP: {
        if (dev_off[x] >= 0) {
          if (slot[x] < 0) {                            // a leaf slot stays reserved
          dev.free(dev_off[x], rb);
          placed.erase(dev_off[x]);
        }
          dev_off[x] = -1;
        }
        break;
      }
      case OP_CONTRACT: {
        op.stream = S_COMPUTE;
        const int32_t ab[2] = {nd.l, nd.r};
        for (int k = 0; k < 2; ++k) {
          const int32_t c = ab[k];
          int32_t& loc = k ? op.loc_b : op.loc_a;
          int64_t& off = k ? op.off_b : op.off_a;
          if (g.nodes[c].leaf() && leaf_on_device[c]) {
            loc = LOC_DEVLEAF;
            off = -1;
          } else {
            if (dev_off[c] < 0) throw Error(CC_E_STATE, "plan: operand not resident");
            loc = LOC_POOL;
            off = dev_off[c];
            need_ready(c, S_COMPUTE, op.deps);
            dtr.access(off, round_up(g.nodes[c].size, align), S_COMPUTE, me, op.deps);
          }
        }
        if (nd.type == ROOT) {
          op.dev_off = -1;                                      // root values buffer
        } else {
          const int64_t off = alloc_for(rb, S_COMPUTE, me, op, x);
          if (off < 0) throw Error(CC_E_NOMEM, "device pool fragmented/too small for node " + std::to_string(nd.id));
          dev_off[x] = off;
          op.dev_off = off;
          placed[off] = x;
          dtr.access(off, rb, S_COMPUTE, me, op.deps);
        }
        ready[x] = me;
        ready_stream[x] = S_COMPUTE;
        break;
      }
      case OP_FREE: {
        if (dev_off[x] >= 0) {
          if (slot[x] < 0) {                            // a leaf slot stays reserved
          dev.free(dev_off[x], rb);
          placed.erase(dev_off[x]);
        }
          dev_off[x] = -1;
        }
        if (host_off[x] >= 0) {
          hostp.free(host_off[x], rb);
          host_off[x] = -1;
        }
        if (peer_off[x] >= 0) {
          peerp.free(peer_off[x], rb);
          peer_off[x] = -1;
        }
        break;
      }
    }
    std::sort(op.deps.begin(), op.deps.end());
    op.deps.erase(std::unique(op.deps.begin(), op.deps.end()), op.deps.end());
    std::sort(op.same_deps.begin(), op.same_deps.end());
    op.same_deps.erase(std::unique(op.same_deps.begin(), op.same_deps.end()), op.same_deps.end());
    pp.ops.push_back(std::move(op));
  }
  for (auto& op : pp.ops) {
    for (int32_t d : op.deps) pp.ops[size_t(d)].source = true;
    for (int32_t d : op.same_deps) pp.ops[size_t(d)].source = true;
  }
  pp.pool_high_water = leaf_region + dev0.high_water();
  pp.host_pool_bytes = host_cap;
  pp.peer_high_water = peerp.high_water();
  return pp;
}

}  // namespace cc
