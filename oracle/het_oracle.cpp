// HET cache-protocol ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded CPU implementation of the per-iteration
// sparse-embedding step of HET (Miao et al., arXiv 2112.07221, PVLDB), written
// from the paper, step by step, in the paper's order and notation.  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library; the product path never does.
// It shares no code with paper_2112_07221_b200/ (no headers, helpers,
// constants or generators).
//
// Citations: "P:n" = /root/reference/PAPER.md line n (canonical copy,
// lines 168-810); "S:n" = SPEC.md line n; "Rn" = the readings table in
// DESIGN.md (= SURVEY.md §8(c)).
//
// Protocol, for iteration t over N workers in lock-step BSP phases (R1):
//   L1  U_i = sorted(unique(K_i)), inverse, stable perm, seg_off   (Alg.1 l.5; R2)
//   L2  hit iff u in cache_i                                       (Cache.Find, Alg.2 l.3)
//   L3  c1 = cc - cs <= s; if c1 and s != inf: cg_obs = cg[u] now,
//       c2 = cg_obs <= cc + s; valid = c1 && c2                    (CheckValid; R3, R4)
//   L4  server applies sync pushes of expired dirty hits,
//       rank asc then key asc: W += p, cg = max(cg, cc)            (Cache.Evict(key); R5)
//   L5  install expired hits and misses: v = W[u], p = 0,
//       cs = cc = cg[u]                                            (Cache.Fetch; R6)
//   L6  count_i[u] += 1, tick[u] = t                               (LFU/LRU; R7, R8)
//       light-LFU (R27): a pinned entry skips the count update;
//       an unpinned one reaching count >= theta is pinned, ascending key,
//       while fewer than floor(C/2) entries are pinned
//   L7  out[pos] = v[K_i[pos]]                                     (Cache.Get)
//   U1  acc = +0.0f; acc += G[pos] for pos ascending among u's
//       occurrences                                                (Cache.Update, Alg.3 l.2; R11)
//   U2  d = (-lr)*acc; v += d; p += d; cc += 1                     (Cache.Update + Cache.Clock)
//   U3  while |cache_i| > C: evict min (count,key) [LFU] or
//       (tick,key) [LRU]; dirty (cc > cs) victims push (k,p,cc)    (Cache.Evict(); R9, R13)
//       light-LFU: pinned entries are exempt                        (R27)
//   U4  server applies eviction pushes rank asc, key asc
//   flush (het_sync): every worker pushes all dirty entries
//       (rank asc, key asc) and empties its cache                  (R16)
//
// Floating point: IEEE fp32, round-to-nearest-even, built with
// -ffp-contract=off so no FMA contraction (R17).  The paper counts the
// embedding table in "floats", which fixes fp32.
//
// Row values are kept only for "tracked" keys (all keys when track_div <= 1);
// cache decisions never depend on row values (SURVEY.md §8(c) value
// independence), so large configs run clocks-only (D = 0) or tracked.
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>
#include <algorithm>

namespace {

const uint32_t S_INF = 0xFFFFFFFFu;  // s = infinity (R4)
enum Status : uint8_t { HIT = 0, EXP1 = 1, EXP2 = 2, MISS = 3 };

// splitmix64 finalizer (the oracle's own copy of the counter hash, R14)
uint64_t fmix(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31; return x;
}

// R14: W0[k][d] = (int32)((mix64(seed0,k,d) >> 40) - 2^23) * 2^-30, exact in fp32,
// in [-2^-7, 2^-7), never -0.  mix64(seed0,k,d) = fmix(fmix(fmix(seed0) ^ k) ^ d).
float w0(uint64_t seed0, int64_t k, uint32_t d) {
  uint64_t h = fmix(fmix(fmix(seed0) ^ (uint64_t)k) ^ (uint64_t)d);
  int32_t q = (int32_t)(h >> 40) - (1 << 23);
  return (float)q * (1.0f / 1073741824.0f);  // 2^-30, exact scaling
}

struct Entry {
  std::vector<float> v;  // cached row incl. own updates (read-my-updates)
  std::vector<float> p;  // pending accumulated deltas owed to the server
  uint32_t cs = 0;       // start clock c_s
  uint32_t cc = 0;       // current clock c_c
  uint32_t tick = 0;     // LRU recency (R8)
  uint32_t own_count = 0;  // LFU count when lfu_persist == 0 (reset on install)
  bool pinned = false;     // light-LFU direct-access entry (R27)
};

struct Push { int64_t key; std::vector<float> p; uint32_t cc; };

struct Worker {
  std::map<int64_t, Entry> cache;                 // the cache embedding table
  std::unordered_map<int64_t, uint32_t> count;    // persistent LFU count per key (R7)
  std::set<std::pair<uint64_t, int64_t>> order;   // (policy primary, key) of unpinned residents
  int64_t npinned = 0;                            // light-LFU pinned residents
  // last lookup (L1-L3) — kept for the matching update (het_update contract)
  std::vector<int64_t> keys, uniq;
  std::vector<int32_t> inverse, perm, seg_off;
  std::vector<uint8_t> status;
  bool have_lookup = false;
  std::vector<int64_t> victims;                   // last U3, in eviction order
  std::vector<uint8_t> victim_dirty;
  uint64_t st[9] = {0};  // lookups, keys, unique, hits, exp1, exp2, misses, evictions, dirty_pushes
};

struct Oracle {
  int64_t R; uint32_t D; int64_t C; uint32_t s; int policy; int N; int lfu_persist;
  uint32_t pin_thr = 0;    // light-LFU threshold theta (policy 2), R27
  uint64_t seed0; int64_t track_div;
  // server: global embedding table W (lazy rows) and global clocks c_g
  std::unordered_map<int64_t, std::vector<float>> W;
  std::unordered_map<int64_t, uint32_t> cg;
  std::vector<Worker> w;

  bool tracked(int64_t k) const {
    if (D == 0) return false;
    if (track_div <= 1) return true;
    return (int64_t)(fmix((uint64_t)k ^ 0x7472616Bull) % (uint64_t)track_div) == 0;
  }
  std::vector<float>& Wrow(int64_t k) {
    auto it = W.find(k);
    if (it != W.end()) return it->second;
    std::vector<float> r(D);
    for (uint32_t d = 0; d < D; ++d) r[d] = w0(seed0, k, d);
    return W.emplace(k, std::move(r)).first->second;
  }
  uint32_t get_cg(int64_t k) const { auto it = cg.find(k); return it == cg.end() ? 0u : it->second; }

  uint32_t lfu_count(Worker& wk, int64_t k, const Entry& e) {
    if (lfu_persist) { auto it = wk.count.find(k); return it == wk.count.end() ? 0u : it->second; }
    return e.own_count;
  }
  uint64_t primary(Worker& wk, int64_t k, const Entry& e) {
    return policy == 1 ? (uint64_t)e.tick : (uint64_t)lfu_count(wk, k, e);   // 0 LFU, 2 light-LFU
  }
  // light-LFU pin cap (R27): at most floor(C/2) pinned entries, so an
  // overflow can always be evicted among the unpinned ones
  int64_t pin_max() const { return C / 2; }

  // Server side of Cache.Evict(key): W += p, c_g = max(c_g, c_c)
  void server_apply(int64_t k, const std::vector<float>& p, uint32_t cc) {
    if (tracked(k)) {
      std::vector<float>& row = Wrow(k);
      for (uint32_t d = 0; d < D; ++d) row[d] = row[d] + p[d];
    }
    uint32_t g = get_cg(k);
    cg[k] = g > cc ? g : cc;
  }

  // ---------------------------------------------------------------- Read
  int lookup(uint64_t t, const int64_t* keys, const int64_t* n_per, float* out) {
    std::vector<int64_t> base(N + 1, 0);
    for (int i = 0; i < N; ++i) base[i + 1] = base[i] + n_per[i];
    for (int i = 0; i < N; ++i)
      for (int64_t j = base[i]; j < base[i + 1]; ++j)
        if (keys[j] < 0 || keys[j] >= R) return 2;  // HET_ERR_KEY_RANGE
    // L1-L3 for every worker
    for (int i = 0; i < N; ++i) {
      Worker& wk = w[i];
      int64_t n = n_per[i];
      wk.keys.assign(keys + base[i], keys + base[i + 1]);
      // L1: unique keys ascending (R2); perm groups positions by key, ascending pos
      std::vector<std::pair<int64_t, int32_t>> kp(n);
      for (int64_t j = 0; j < n; ++j) kp[j] = {wk.keys[j], (int32_t)j};
      std::sort(kp.begin(), kp.end());
      wk.uniq.clear(); wk.seg_off.clear(); wk.perm.assign(n, 0); wk.inverse.assign(n, 0);
      for (int64_t j = 0; j < n; ++j) {
        if (j == 0 || kp[j].first != kp[j - 1].first) {
          wk.uniq.push_back(kp[j].first);
          wk.seg_off.push_back((int32_t)j);
        }
        wk.perm[j] = kp[j].second;
        wk.inverse[kp[j].second] = (int32_t)wk.uniq.size() - 1;
      }
      wk.seg_off.push_back((int32_t)n);
      // L2 + L3
      wk.status.assign(wk.uniq.size(), MISS);
      for (size_t u = 0; u < wk.uniq.size(); ++u) {
        auto it = wk.cache.find(wk.uniq[u]);
        if (it == wk.cache.end()) { wk.status[u] = MISS; continue; }
        const Entry& e = it->second;
        if (s == S_INF) { wk.status[u] = HIT; continue; }  // R4: no clock query
        bool c1 = (e.cc - e.cs) <= s;                       // condition (1)
        if (!c1) { wk.status[u] = EXP1; continue; }         // R3: no query for EXP1
        uint32_t g = get_cg(wk.uniq[u]);                    // clock check
        bool c2 = (g <= e.cc) || (g - e.cc <= s);           // condition (2)
        wk.status[u] = c2 ? HIT : EXP2;
      }
      wk.have_lookup = true;
      wk.st[0] += 1; wk.st[1] += (uint64_t)n; wk.st[2] += wk.uniq.size();
      for (uint8_t sv : wk.status) wk.st[3 + sv] += 1;
    }
    // L4: sync pushes of expired dirty hits, rank asc then key asc (R1, R5)
    for (int i = 0; i < N; ++i) {
      Worker& wk = w[i];
      for (size_t u = 0; u < wk.uniq.size(); ++u) {
        if (wk.status[u] != EXP1 && wk.status[u] != EXP2) continue;
        Entry& e = wk.cache.at(wk.uniq[u]);
        if (e.cc > e.cs) server_apply(wk.uniq[u], e.p, e.cc);  // dirty <=> cc > cs (R13)
      }
    }
    // L5: Fetch for expired hits and misses: v = W, p = 0, cs = cc = cg
    for (int i = 0; i < N; ++i) {
      Worker& wk = w[i];
      for (size_t u = 0; u < wk.uniq.size(); ++u) {
        if (wk.status[u] == HIT) continue;
        int64_t k = wk.uniq[u];
        auto it = wk.cache.find(k);
        if (it != wk.cache.end() && !it->second.pinned) wk.order.erase({primary(wk, k, it->second), k});
        Entry& e = wk.cache[k];
        if (tracked(k)) { e.v = Wrow(k); e.p.assign(D, 0.0f); }
        e.cs = e.cc = get_cg(k);
        if (wk.status[u] == MISS) e.own_count = 0;  // reset-LFU reading only
        if (!e.pinned) wk.order.insert({primary(wk, k, e), k});
      }
    }
    // L6: LFU count +1 per unique key per lookup, LRU tick = t (R7, R8)
    for (int i = 0; i < N; ++i) {
      Worker& wk = w[i];
      for (int64_t k : wk.uniq) {                  // ascending key
        Entry& e = wk.cache.at(k);
        if (e.pinned) continue;                    // light-LFU: no frequency maintenance
        wk.order.erase({primary(wk, k, e), k});
        wk.count[k] += 1;
        e.own_count += 1;
        e.tick = (uint32_t)t;
        if (policy == 2 && lfu_count(wk, k, e) >= pin_thr && wk.npinned < pin_max()) {
          e.pinned = true;                         // direct access index
          wk.npinned += 1;
          continue;
        }
        wk.order.insert({primary(wk, k, e), k});
      }
    }
    // L7: Get — out[pos] = v[K_i[pos]]
    if (out) {
      for (int i = 0; i < N; ++i) {
        Worker& wk = w[i];
        for (size_t j = 0; j < wk.keys.size(); ++j) {
          float* o = out + (size_t)(base[i] + j) * D;
          const Entry& e = wk.cache.at(wk.keys[j]);
          if (tracked(wk.keys[j])) std::memcpy(o, e.v.data(), sizeof(float) * D);
        }
      }
    }
    return 0;
  }

  // ---------------------------------------------------------------- Write
  int update(const float* grads, float lr) {
    int64_t base = 0;
    for (int i = 0; i < N; ++i) if (!w[i].have_lookup) return 3;  // write without read
    for (int i = 0; i < N; ++i) {
      Worker& wk = w[i];
      for (size_t u = 0; u < wk.uniq.size(); ++u) {
        int64_t k = wk.uniq[u];
        Entry& e = wk.cache.at(k);
        if (tracked(k) && grads) {
          for (uint32_t d = 0; d < D; ++d) {
            float acc = 0.0f;                               // U1, R11
            for (int32_t j = wk.seg_off[u]; j < wk.seg_off[u + 1]; ++j)
              acc = acc + grads[(size_t)(base + wk.perm[j]) * D + d];
            float delta = (-lr) * acc;                       // U2
            e.v[d] = e.v[d] + delta;
            e.p[d] = e.p[d] + delta;
          }
        }
        e.cc += 1;                                           // Cache.Clock
      }
      base += (int64_t)wk.keys.size();
      wk.have_lookup = false;
    }
    // U3: Evict() overflow (R9)
    std::vector<std::vector<Push>> pushes(N);
    for (int i = 0; i < N; ++i) evict_overflow(i, pushes[i]);
    // U4: apply eviction pushes rank asc, key asc
    apply_pushes(pushes);
    return 0;
  }

  void evict_one(int i, int64_t k, std::vector<Push>& out) {
    Worker& wk = w[i];
    Entry& e = wk.cache.at(k);
    bool dirty = e.cc > e.cs;
    if (dirty) out.push_back({k, e.p, e.cc});
    wk.victims.push_back(k);
    wk.victim_dirty.push_back(dirty ? 1 : 0);
    if (e.pinned) wk.npinned -= 1;
    else wk.order.erase({primary(wk, k, e), k});
    wk.cache.erase(k);
    wk.st[7] += 1; if (dirty) wk.st[8] += 1;
  }

  void evict_overflow(int i, std::vector<Push>& out) {
    Worker& wk = w[i];
    wk.victims.clear(); wk.victim_dirty.clear();
    while ((int64_t)wk.cache.size() > C) {
      // the minimum over all residents by (primary, key)
      int64_t k = wk.order.begin()->second;
      evict_one(i, k, out);
    }
  }

  void apply_pushes(std::vector<std::vector<Push>>& pushes) {
    for (int i = 0; i < N; ++i) {
      std::sort(pushes[i].begin(), pushes[i].end(),
                [](const Push& a, const Push& b) { return a.key < b.key; });
      for (const Push& ps : pushes[i]) server_apply(ps.key, ps.p, ps.cc);
    }
  }

  int evict_keys(const int64_t* keys, const int64_t* n_per) {
    std::vector<std::vector<Push>> pushes(N);
    int64_t b = 0;
    for (int i = 0; i < N; ++i) {
      w[i].victims.clear(); w[i].victim_dirty.clear();
      std::vector<int64_t> ks(keys + b, keys + b + n_per[i]);
      b += n_per[i];
      std::sort(ks.begin(), ks.end());
      ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
      for (int64_t k : ks) if (w[i].cache.count(k)) evict_one(i, k, pushes[i]);
    }
    apply_pushes(pushes);
    return 0;
  }

  int evict_overflow_all() {
    std::vector<std::vector<Push>> pushes(N);
    for (int i = 0; i < N; ++i) evict_overflow(i, pushes[i]);
    apply_pushes(pushes);
    return 0;
  }

  // het_sync: push all dirty entries (rank asc, key asc), empty the caches (R16)
  int flush() {
    std::vector<std::vector<Push>> pushes(N);
    for (int i = 0; i < N; ++i) {
      Worker& wk = w[i];
      for (auto& kv : wk.cache)  // std::map iterates in ascending key
        if (kv.second.cc > kv.second.cs) pushes[i].push_back({kv.first, kv.second.p, kv.second.cc});
      wk.cache.clear();
      wk.order.clear();
      wk.npinned = 0;
      wk.have_lookup = false;
    }
    apply_pushes(pushes);
    return 0;
  }
};

}  // namespace

extern "C" {

void* orc_create(int64_t R, uint32_t D, int64_t C, uint32_t s, int policy, int N,
                 int lfu_persist, uint64_t seed0, int64_t track_div, uint32_t pin_thr) {
  Oracle* o = new Oracle();
  o->R = R; o->D = D; o->C = C; o->s = s; o->policy = policy; o->N = N;
  o->pin_thr = pin_thr;
  o->lfu_persist = lfu_persist; o->seed0 = seed0; o->track_div = track_div;
  o->w.resize(N);
  return o;
}
void orc_destroy(void* h) { delete (Oracle*)h; }
// Bench infrastructure only (bench.py cpu_baseline / --impl reference; no
// parity test calls it): change which keys carry row values.  A clocks-only
// fill (track_div huge) brings the cache to steady state fast; switching to
// full rows then gives every resident entry that had none the server row as
// at a Fetch (v = W[k], p = 0).  Decisions never depend on row values,
// so the protocol phase is unchanged; row VALUES after the switch are not the
// protocol's and must not be compared.
void orc_set_track_div(void* h, int64_t track_div) {
  Oracle* o = (Oracle*)h;
  o->track_div = track_div;
  for (Worker& wk : o->w)
    for (auto& kv : wk.cache)
      if (o->tracked(kv.first) && kv.second.v.size() != o->D) {
        kv.second.v = o->Wrow(kv.first);
        kv.second.p.assign(o->D, 0.0f);
      }
}
int orc_lookup(void* h, uint64_t t, const int64_t* keys, const int64_t* n_per, float* out) {
  return ((Oracle*)h)->lookup(t, keys, n_per, out);
}
int orc_update(void* h, const float* grads, float lr) { return ((Oracle*)h)->update(grads, lr); }
int orc_flush(void* h) { return ((Oracle*)h)->flush(); }
int orc_evict_keys(void* h, const int64_t* keys, const int64_t* n_per) {
  return ((Oracle*)h)->evict_keys(keys, n_per);
}
int orc_evict_overflow(void* h) { return ((Oracle*)h)->evict_overflow_all(); }

int64_t orc_num_unique(void* h, int i) { return (int64_t)((Oracle*)h)->w[i].uniq.size(); }
void orc_get_lookup_log(void* h, int i, int64_t* uniq, int32_t* inverse, int32_t* perm,
                        int32_t* seg_off, uint8_t* status) {
  Worker& wk = ((Oracle*)h)->w[i];
  size_t U = wk.uniq.size(), n = wk.keys.size();
  if (uniq) std::memcpy(uniq, wk.uniq.data(), U * 8);
  if (inverse) std::memcpy(inverse, wk.inverse.data(), n * 4);
  if (perm) std::memcpy(perm, wk.perm.data(), n * 4);
  if (seg_off) std::memcpy(seg_off, wk.seg_off.data(), (U + 1) * 4);
  if (status) std::memcpy(status, wk.status.data(), U);
}
int64_t orc_num_victims(void* h, int i) { return (int64_t)((Oracle*)h)->w[i].victims.size(); }
void orc_get_victims(void* h, int i, int64_t* keys, uint8_t* dirty) {
  Worker& wk = ((Oracle*)h)->w[i];
  std::memcpy(keys, wk.victims.data(), wk.victims.size() * 8);
  if (dirty) std::memcpy(dirty, wk.victim_dirty.data(), wk.victims.size());
}
void orc_get_stats(void* h, int i, uint64_t* out9) { std::memcpy(out9, ((Oracle*)h)->w[i].st, 9 * 8); }
int64_t orc_cache_size(void* h, int i) { return (int64_t)((Oracle*)h)->w[i].cache.size(); }
// resident entries in ascending key; v/p only meaningful for tracked keys
void orc_dump_cache(void* h, int i, int64_t* keys, float* v, float* p, uint32_t* cs,
                    uint32_t* cc, uint32_t* count, uint32_t* tick) {
  Oracle* o = (Oracle*)h;
  Worker& wk = o->w[i];
  size_t j = 0;
  for (auto& kv : wk.cache) {
    const Entry& e = kv.second;
    keys[j] = kv.first;
    if (v && o->tracked(kv.first)) std::memcpy(v + j * o->D, e.v.data(), o->D * 4);
    if (p && o->tracked(kv.first)) std::memcpy(p + j * o->D, e.p.data(), o->D * 4);
    if (cs) cs[j] = e.cs;
    if (cc) cc[j] = e.cc;
    if (count) count[j] = o->lfu_count(wk, kv.first, e);
    if (tick) tick[j] = e.pinned ? 0xFFFFFFFEu : e.tick;   // light-LFU: pinned marker
    ++j;
  }
}
void orc_read_global(void* h, const int64_t* keys, int64_t n, float* rows, uint32_t* cgs) {
  Oracle* o = (Oracle*)h;
  for (int64_t j = 0; j < n; ++j) {
    if (rows && o->D) {
      if (o->tracked(keys[j])) {
        auto it = o->W.find(keys[j]);
        for (uint32_t d = 0; d < o->D; ++d)
          rows[j * o->D + d] = it == o->W.end() ? w0(o->seed0, keys[j], d) : it->second[d];
      }
    }
    if (cgs) cgs[j] = o->get_cg(keys[j]);
  }
}
float orc_w0(uint64_t seed0, int64_t k, uint32_t d) { return w0(seed0, k, d); }

}  // extern "C"
