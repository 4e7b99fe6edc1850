// LoopProgram JSON -> batched sm_100a CUDA kernel.  See lp_program.h for the
// execution model; the reference semantics followed here are those of
// emit_c (reference scheduling.py:617-738):
//   ZeroFill  -> buffer[z] = 0.0                       (:707-709)
//   Assign    -> target[addr] = expr                   (:710-713)
//   Accumulate-> target[addr] += expr                  (:714-717)
//   Delta     -> ((i == j) ? 1.0 : 0.0)                (:666-667)
//   Comparison-> ((a op b) ? 1.0 : 0.0)                (:685-686)
//   MathFunction via _C_FUNCTIONS (ln -> log, abs -> fabs)  (:601-602)
// with row-major strides for Indexed tables / variables (:654-661) and the
// explicit (offset, terms) address of FlexiblyIndexed (:662-663).
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <set>
#include <sstream>
#include <stdexcept>

#include "lp_program.h"
#include "sfk_options.h"

namespace sfk {
namespace lp {

// ---------------------------------------------------------------------------
// parsing (mirror of parse_program, reference scheduling.py:535-596)

namespace {

struct Reader {
  Program& P;
  std::map<std::string, int> table_ids;

  Entry entry(const json::Value& v) {
    Entry e;
    if (v.is_arr()) {
      e.idx = idx(v);
    } else {
      e.val = v.i();
    }
    return e;
  }
  int idx(const json::Value& v) {
    if (!v.is_arr() || v.size() != 3 || v.at(0).s() != "idx")
      throw std::runtime_error("LoopProgram: bad index spec");
    const int id = (int)v.at(1).i();
    const int ext = (int)v.at(2).i();
    auto it = P.extents.find(id);
    if (it != P.extents.end() && it->second != ext)
      throw std::runtime_error("LoopProgram: index extent mismatch");
    P.extents[id] = ext;
    return id;
  }
  static std::vector<long long> row_major(const std::vector<long long>& shape) {
    std::vector<long long> s(shape.size());
    long long acc = 1;
    for (size_t k = shape.size(); k-- > 0;) {
      s[k] = acc;
      acc *= shape[k];
    }
    return s;
  }
  int table(const json::Value& t) {
    Table tb;
    for (const auto& d : t.at(1).arr) tb.shape.push_back(d.i());
    for (const auto& x : t.at(2).arr) tb.values.push_back(x.d());
    long long n = 1;
    for (auto d : tb.shape) n *= d;
    if ((long long)tb.values.size() != n) throw std::runtime_error("LoopProgram: table size");
    std::string key((const char*)tb.shape.data(), tb.shape.size() * sizeof(long long));
    key.append((const char*)tb.values.data(), tb.values.size() * sizeof(double));
    auto it = table_ids.find(key);
    if (it != table_ids.end()) return it->second;
    const int id = (int)P.tables.size();
    P.tables.push_back(std::move(tb));
    table_ids.emplace(std::move(key), id);
    return id;
  }
  ExprP expr(const json::Value& v) {
    const std::string& tag = v.at(0).s();
    auto e = std::make_shared<Expr>();
    if (tag == "lit") {
      e->k = Expr::LIT;
      e->lit = v.at(1).d();
    } else if (tag == "indexed") {
      const json::Value& base = v.at(1);
      const json::Value& mi = v.at(2);
      std::vector<long long> shape;
      const std::string& btag = base.at(0).s();
      if (btag == "table") {
        e->k = Expr::TABLE;
        e->table = table(base);
        shape = P.tables[e->table].shape;
      } else if (btag == "var") {
        e->k = Expr::LOAD;
        e->name = base.at(1).s();
        for (const auto& d : base.at(2).arr) shape.push_back(d.i());
      } else {
        throw std::runtime_error("LoopProgram: indexed base '" + btag + "'");
      }
      if (shape.size() != mi.size()) throw std::runtime_error("LoopProgram: rank mismatch");
      const auto strides = row_major(shape);
      for (size_t k = 0; k < mi.size(); ++k) e->terms.push_back({entry(mi.at(k)), strides[k]});
    } else if (tag == "flex") {
      const json::Value& base = v.at(1);
      if (base.at(0).s() != "var") throw std::runtime_error("LoopProgram: flex base");
      e->k = Expr::LOAD;
      e->name = base.at(1).s();
      e->offset = v.at(2).i();
      for (const auto& t : v.at(3).arr) e->terms.push_back({entry(t.at(0)), t.at(1).i()});
    } else if (tag == "delta") {
      e->k = Expr::DELTA;
      e->d0 = entry(v.at(1));
      e->d1 = entry(v.at(2));
    } else if (tag == "+" || tag == "*" || tag == "/" || tag == "pow" || tag == "min" ||
               tag == "max") {
      e->k = tag == "+" ? Expr::ADD : tag == "*" ? Expr::MUL : tag == "/" ? Expr::DIV
           : tag == "pow" ? Expr::POW : tag == "min" ? Expr::MIN : Expr::MAX;
      e->a = expr(v.at(1));
      e->b = expr(v.at(2));
    } else if (tag == "call") {
      e->k = Expr::CALL;
      e->name = v.at(1).s();
      e->a = expr(v.at(2));
    } else if (tag == "cmp") {
      e->k = Expr::CMP;
      e->name = v.at(1).s();
      e->a = expr(v.at(2));
      e->b = expr(v.at(3));
    } else if (tag == "var" || tag == "table") {
      throw std::runtime_error("LoopProgram: bare " + tag);
    } else {
      throw std::runtime_error("LoopProgram: cannot parse '" + tag + "'");
    }
    return e;
  }
  void ref(const json::Value& r, Stmt& s) {
    s.name = r.at(0).s();
    s.offset = r.at(1).i();
    for (const auto& t : r.at(2).arr) s.terms.push_back({entry(t.at(0)), t.at(1).i()});
  }
  Stmt stmt(const json::Value& v) {
    const std::string& tag = v.at(0).s();
    Stmt s;
    if (tag == "loop") {
      s.k = Stmt::LOOP;
      s.idx = idx(v.at(1));
      s.extent = P.extents[s.idx];
      for (const auto& b : v.at(2).arr) s.body.push_back(stmt(b));
    } else if (tag == "assign" || tag == "accumulate") {
      s.k = tag == "assign" ? Stmt::ASSIGN : Stmt::ACCUM;
      ref(v.at(1), s);
      s.e = expr(v.at(2));
    } else if (tag == "zero") {
      s.k = Stmt::ZERO;
      s.name = v.at(1).s();
      s.size = v.at(2).i();
    } else {
      throw std::runtime_error("LoopProgram: unknown statement '" + tag + "'");
    }
    return s;
  }
};

}  // namespace

Program parse_program(const char* text, size_t n) {
  const json::Value doc = json::parse(text, n);
  Program P;
  Reader r{P, {}};
  P.name = doc.at("name").s();
  P.ret_name = doc.at("return").at(0).s();
  P.ret_size = doc.at("return").at(1).i();
  for (const auto& a : doc.at("arguments").arr) P.args.emplace_back(a.at(0).s(), a.at(1).i());
  for (const auto& t : doc.at("temporaries").arr) P.temps.emplace_back(t.at(0).s(), t.at(1).i());
  for (const auto& s : doc.at("body").arr) P.body.push_back(r.stmt(s));
  return P;
}

// ---------------------------------------------------------------------------
// analysis

namespace {

struct Phase {
  enum K { ZERO, NEST, SERIAL } k = ZERO;
  const Stmt* top = nullptr;
  const Stmt* leaf = nullptr;
  std::vector<std::pair<int, int>> par, red;   // (index id, extent), nest order
  long long npar = 1;
  // output blocking: the parallel index `blk` (extent blk_ext) is handled
  // inside one thread, so loads that do not depend on it are shared by the
  // blk_ext outputs (accumulators in registers); opar = par without blk
  int blk = -1, blk_ext = 1;
  std::vector<std::pair<int, int>> opar;
  long long nitem = 1;                          // items per cell = npar / blk_ext
  bool zero_init = false;                      // folded ZeroFill (ACCUM starts at 0)
  std::string zname;
  long long zsize = 0;
  std::set<std::string> reads, writes;
};

void expr_reads(const Expr& e, std::set<std::string>& out) {
  if (e.k == Expr::LOAD) out.insert(e.name);
  if (e.a) expr_reads(*e.a, out);
  if (e.b) expr_reads(*e.b, out);
}

void stmt_rw(const Stmt& s, std::set<std::string>& r, std::set<std::string>& w) {
  switch (s.k) {
    case Stmt::LOOP:
      for (const auto& b : s.body) stmt_rw(b, r, w);
      break;
    case Stmt::ZERO:
      w.insert(s.name);
      break;
    case Stmt::ASSIGN:
      w.insert(s.name);
      expr_reads(*s.e, r);
      break;
    case Stmt::ACCUM:
      w.insert(s.name);
      r.insert(s.name);
      expr_reads(*s.e, r);
      break;
  }
}

// Target addresses of a perfect nest over its parallel box: injective?  Does
// the set equal {0..size-1}?
void target_map(const Stmt& leaf, const std::vector<std::pair<int, int>>& par,
                long long cover_size, bool& injective, bool& covers) {
  long long base = leaf.offset;
  std::map<int, long long> stride;
  for (const auto& t : leaf.terms) {
    if (t.e.idx < 0) base += t.e.val * t.stride;
    else stride[t.e.idx] += t.stride;
  }
  long long total = 1;
  for (const auto& pr : par) total *= pr.second;
  injective = false;
  covers = false;
  if (total > (1LL << 24)) return;
  long long lo = base, hi = base;
  for (const auto& pr : par) {
    const long long s = stride[pr.first] * (pr.second - 1);
    if (s < 0) lo += s; else hi += s;
  }
  if (lo < 0) return;
  std::vector<char> seen((size_t)(hi - lo + 1), 0);
  std::vector<int> it(par.size(), 0);
  for (long long n = 0; n < total; ++n) {
    long long a = base;
    for (size_t k = 0; k < par.size(); ++k) a += stride[par[k].first] * it[k];
    if (seen[a - lo]) return;
    seen[a - lo] = 1;
    for (size_t k = par.size(); k-- > 0;) {
      if (++it[k] < par[k].second) break;
      it[k] = 0;
    }
  }
  injective = true;
  covers = (lo == 0 && hi == cover_size - 1 && total == cover_size);
}

Phase classify(const Stmt& s) {
  Phase ph;
  ph.top = &s;
  stmt_rw(s, ph.reads, ph.writes);
  // descend the perfect nest
  std::vector<std::pair<int, int>> loops;
  const Stmt* cur = &s;
  while (cur->k == Stmt::LOOP && cur->body.size() == 1) {
    loops.emplace_back(cur->idx, cur->extent);
    cur = &cur->body[0];
  }
  if (cur->k == Stmt::LOOP || cur->k == Stmt::ZERO) {  // imperfect nest
    ph.k = Phase::SERIAL;
    return ph;
  }
  ph.leaf = cur;
  std::set<int> tgt;
  for (const auto& t : cur->terms)
    if (t.e.idx >= 0 && t.stride != 0) tgt.insert(t.e.idx);
  std::set<int> loop_ids;
  for (const auto& l : loops) loop_ids.insert(l.first);
  for (int id : tgt)
    if (!loop_ids.count(id)) { ph.k = Phase::SERIAL; return ph; }
  for (const auto& l : loops) (tgt.count(l.first) ? ph.par : ph.red).push_back(l);
  std::set<std::string> er;
  expr_reads(*cur->e, er);
  bool inj = false, cov = false;
  target_map(*cur, ph.par, -1, inj, cov);
  if (!inj || er.count(cur->name)) {
    ph.k = Phase::SERIAL;
    ph.par.clear();
    ph.red.clear();
    return ph;
  }
  ph.k = Phase::NEST;
  for (const auto& pr : ph.par) ph.npar *= pr.second;
  // output blocking: pick the parallel index most loads do not depend on
  {
    std::vector<const Expr*> lds;
    std::function<void(const Expr&)> col = [&](const Expr& e) {
      if (e.k == Expr::LOAD || e.k == Expr::TABLE) lds.push_back(&e);
      if (e.a) col(*e.a);
      if (e.b) col(*e.b);
    };
    col(*cur->e);
    // (a variant restricted to reductions reusing a temporary lost most of the
    // gain: profiles/r01av_lp_block.jsonl)
    int best = 0;
    for (const auto& pr : ph.par) {
      if (pr.second < 2 || pr.second > 16) continue;
      int score = 0;
      for (const Expr* ld : lds) {
        bool dep = false;
        for (const auto& t : ld->terms) dep = dep || (t.e.idx == pr.first && t.stride != 0);
        score += dep ? 0 : 1;
      }
      if (score > best || (score == best && score > 0 && pr.second > ph.blk_ext)) {
        best = score;
        ph.blk = pr.first;
        ph.blk_ext = pr.second;
      }
    }
    if (best == 0) ph.blk = -1, ph.blk_ext = 1;
    for (const auto& pr : ph.par)
      if (pr.first != ph.blk) ph.opar.push_back(pr);
    ph.nitem = ph.npar / ph.blk_ext;
  }
  return ph;
}

bool nest_covers(const Phase& ph, long long size) {
  bool inj = false, cov = false;
  target_map(*ph.leaf, ph.par, size, inj, cov);
  return inj && cov;
}

std::string fmt_double(double x) {
  if (std::isnan(x) || std::isinf(x)) {
    long long bits;
    std::memcpy(&bits, &x, 8);
    char buf[64];
    std::snprintf(buf, sizeof buf, "__longlong_as_double(0x%016llxLL)", (unsigned long long)bits);
    return buf;
  }
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", x);  // exact (hex float literal)
  return buf;
}


// Exact barrier placement.  Phase k needs a __syncthreads() before it iff
// some shared-memory element it touches was touched since the last barrier
// by a DIFFERENT thread, with at least one of the two accesses a write
// (thread of item w = w % T, as the generated loops deal items).  Same-thread
// chains (pointwise statements reading what the same item wrote) need none.
// Phases too large to enumerate fall back to "barrier before and after".
struct Access {
  long long elem;
  int thread;
  bool write;
  int item = -1;   // loop item (w) of a NEST phase; -1 elsewhere (never fusable)
};

void collect_loads(const Expr& e, std::vector<const Expr*>& out) {
  if (e.k == Expr::LOAD) out.push_back(&e);
  if (e.a) collect_loads(*e.a, out);
  if (e.b) collect_loads(*e.b, out);
}

long long eval_addr(long long off, const std::vector<Term>& terms, const std::vector<long long>& val) {
  long long a = off;
  for (const auto& t : terms) a += t.stride * (t.e.idx >= 0 ? val[t.e.idx] : t.e.val);
  return a;
}

// Returns false if the phase is too large to enumerate.
bool phase_accesses(const Phase& ph, const std::map<std::string, long long>& base,
                    const std::map<std::string, long long>& bufsize, int NC, int T, int max_idx,
                    std::vector<Access>& out) {
  const long long kBudget = 1LL << 23;
  out.clear();
  auto elem = [&](long long slot, int c) { return slot * NC + c; };
  if (ph.k == Phase::ZERO) {
    const long long b = base.at(ph.zname);
    for (long long e = 0; e < NC * ph.zsize; ++e)
      out.push_back({elem(b + e / NC, (int)(e % NC)), (int)(e % T), true});
    return true;
  }
  if (ph.k == Phase::SERIAL) {
    long long n = 0;
    for (const auto& nm : ph.reads) n += bufsize.at(nm);
    for (const auto& nm : ph.writes) n += bufsize.at(nm);
    if (n * NC > kBudget) return false;
    for (int c = 0; c < NC; ++c) {
      for (const auto& nm : ph.reads)
        for (long long z = 0; z < bufsize.at(nm); ++z)
          out.push_back({elem(base.at(nm) + z, c), c % T, false});
      for (const auto& nm : ph.writes)
        for (long long z = 0; z < bufsize.at(nm); ++z)
          out.push_back({elem(base.at(nm) + z, c), c % T, true});
    }
    return true;
  }
  const Stmt& L = *ph.leaf;
  std::vector<const Expr*> loads;
  collect_loads(*L.e, loads);
  long long nred = 1;
  for (const auto& r : ph.red) nred *= r.second;
  if ((long long)NC * ph.npar * (1 + nred * (long long)loads.size()) > kBudget) return false;
  std::vector<long long> val(max_idx + 1, 0);
  const long long tb = base.at(L.name);
  for (long long w = 0; w < NC * ph.nitem; ++w) {
    const int c = (int)(w % NC);
    long long q = w / NC;
    for (size_t j = ph.opar.size(); j-- > 0;) {
      if (j == 0) { val[ph.opar[j].first] = q; break; }
      val[ph.opar[j].first] = q % ph.opar[j].second;
      q /= ph.opar[j].second;
    }
    const int t = (int)(w % T);
    for (int bv = 0; bv < ph.blk_ext; ++bv) {
      if (ph.blk >= 0) val[ph.blk] = bv;
      out.push_back({elem(tb + eval_addr(L.offset, L.terms, val), c), t, true, (int)w});
      if (loads.empty()) continue;
      std::vector<int> it(ph.red.size(), 0);
      for (long long r = 0; r < nred; ++r) {
        for (size_t j = 0; j < ph.red.size(); ++j) val[ph.red[j].first] = it[j];
        for (const Expr* ld : loads)
          out.push_back({elem(base.at(ld->name) + eval_addr(ld->offset, ld->terms, val), c), t,
                         false, (int)w});
        for (size_t j = ph.red.size(); j-- > 0;) {
          if (++it[j] < ph.red[j].second) break;
          it[j] = 0;
        }
      }
    }
  }
  return true;
}

struct Window {
  std::vector<int> writer, reader;
  std::vector<char> multi;
  std::vector<long long> touched;
  bool poisoned = false;
  explicit Window(long long n) : writer(n, -1), reader(n, -1), multi(n, 0) {}
  bool conflicts(const std::vector<Access>& acc) const {
    if (poisoned) return true;
    for (const auto& a : acc) {
      const int w = writer[a.elem];
      if (w >= 0 && w != a.thread) return true;
      if (a.write) {
        const int r = reader[a.elem];
        if (r >= 0 && (r != a.thread || multi[a.elem])) return true;
      }
    }
    return false;
  }
  void add(const std::vector<Access>& acc) {
    for (const auto& a : acc) {
      if (writer[a.elem] < 0 && reader[a.elem] < 0) touched.push_back(a.elem);
      if (a.write) {
        writer[a.elem] = a.thread;
      } else if (reader[a.elem] < 0) {
        reader[a.elem] = a.thread;
      } else if (reader[a.elem] != a.thread) {
        multi[a.elem] = 1;
      }
    }
  }
  void clear() {
    for (long long e : touched) { writer[e] = -1; reader[e] = -1; multi[e] = 0; }
    touched.clear();
    poisoned = false;
  }
};

// Item-level dependence inside a fused loop group: every element touched by
// two phases of the group (at least one write) must be touched by the SAME
// item w, so running the phases' bodies back to back per item preserves
// every dependence.
struct ItemWindow {
  std::vector<int> writer, reader;   // -1 none, -2 several items
  std::vector<long long> touched;
  explicit ItemWindow(long long n) : writer(n, -1), reader(n, -1) {}
  bool compatible(const std::vector<Access>& acc) const {
    for (const auto& a : acc) {
      if (a.item < 0) return false;
      const int w = writer[a.elem], r = reader[a.elem];
      if (w != -1 && w != a.item) return false;
      if (a.write && r != -1 && r != a.item) return false;
    }
    return true;
  }
  void add(const std::vector<Access>& acc) {
    for (const auto& a : acc) {
      if (writer[a.elem] == -1 && reader[a.elem] == -1) touched.push_back(a.elem);
      if (a.write) {
        writer[a.elem] = (writer[a.elem] == -1 || writer[a.elem] == a.item) ? a.item : -2;
      } else {
        reader[a.elem] = (reader[a.elem] == -1 || reader[a.elem] == a.item) ? a.item : -2;
      }
    }
  }
  void clear() {
    for (long long e : touched) { writer[e] = -1; reader[e] = -1; }
    touched.clear();
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// generation

Generated generate(const Program& P, int64_t smem_limit, bool allow_fma) {
  (void)allow_fma;
  std::map<std::string, long long> bufsize;
  bufsize[P.ret_name] = P.ret_size;
  for (const auto& a : P.args) bufsize[a.first] = a.second;
  for (const auto& t : P.temps) bufsize[t.first] = t.second;

  // 1. phases with ZeroFill folding
  std::vector<Phase> phases;
  std::map<std::string, long long> pending;  // name -> zero size
  auto flush_zero = [&](const std::string& nm) {
    Phase z;
    z.k = Phase::ZERO;
    z.zname = nm;
    z.zsize = pending[nm];
    z.writes.insert(nm);
    phases.push_back(z);
    pending.erase(nm);
  };
  for (const auto& s : P.body) {
    if (s.k == Stmt::ZERO) {
      if (!bufsize.count(s.name)) throw std::runtime_error("LoopProgram: unknown buffer " + s.name);
      if (pending.count(s.name)) flush_zero(s.name);
      pending[s.name] = s.size;
      continue;
    }
    Phase ph = classify(s);
    std::set<std::string> touched = ph.reads;
    touched.insert(ph.writes.begin(), ph.writes.end());
    for (const auto& nm : touched) {
      if (!bufsize.count(nm)) throw std::runtime_error("LoopProgram: unknown buffer " + nm);
      if (!pending.count(nm)) continue;
      std::set<std::string> er;
      if (ph.k == Phase::NEST) expr_reads(*ph.leaf->e, er);
      const bool fold = ph.k == Phase::NEST && ph.leaf->name == nm && !er.count(nm) &&
                        pending[nm] == bufsize[nm] && nest_covers(ph, pending[nm]);
      if (fold) {
        if (ph.leaf->k == Stmt::ACCUM) ph.zero_init = true;
        pending.erase(nm);
      } else {
        flush_zero(nm);
      }
    }
    phases.push_back(std::move(ph));
  }
  if (pending.count(P.ret_name)) flush_zero(P.ret_name);

  // 2. storage: args, A fixed; temporaries packed by liveness
  std::map<std::string, long long> base;
  long long fixed = 0;
  for (const auto& a : P.args) { base[a.first] = fixed; fixed += a.second; }
  base[P.ret_name] = fixed;
  fixed += P.ret_size;
  std::map<std::string, int> first, last;
  for (int k = 0; k < (int)phases.size(); ++k) {
    std::set<std::string> t = phases[k].reads;
    t.insert(phases[k].writes.begin(), phases[k].writes.end());
    for (const auto& nm : t) {
      if (!first.count(nm)) first[nm] = k;
      last[nm] = k;
    }
  }
  long long peak = fixed;
  {
    std::vector<std::pair<long long, long long>> used;  // [start, end) of live temps
    std::vector<std::pair<int, std::string>> live;      // (last, name)
    for (int k = 0; k < (int)phases.size(); ++k) {
      for (size_t j = 0; j < live.size();) {
        if (live[j].first < k) {
          const long long s = base[live[j].second];
          used.erase(std::find_if(used.begin(), used.end(),
                                  [&](const std::pair<long long, long long>& u) { return u.first == s; }));
          live.erase(live.begin() + j);
        } else {
          ++j;
        }
      }
      for (const auto& t : P.temps) {
        if (!first.count(t.first) || first[t.first] != k) continue;
        std::sort(used.begin(), used.end());
        long long at = fixed;
        for (const auto& u : used) {
          if (at + t.second <= u.first) break;
          at = std::max(at, u.second);
        }
        base[t.first] = at;
        used.emplace_back(at, at + t.second);
        live.emplace_back(last[t.first], t.first);
        peak = std::max(peak, at + t.second);
      }
    }
  }
  for (const auto& t : P.temps)
    if (!base.count(t.first)) base[t.first] = 0;  // never touched

  // 3. launch geometry
  Generated G;
  Config& C = G.cfg;
  C.slots = peak;
  long long tbl_doubles = 0;
  std::vector<long long> toff;
  for (const auto& t : P.tables) { toff.push_back(tbl_doubles); tbl_doubles += (long long)t.values.size(); }
  const long long tbl_bytes_smem = ((tbl_doubles * 8 + 15) / 16) * 16;
  C.tables_in_smem = tbl_bytes_smem <= 64 * 1024;
  const long long tb = C.tables_in_smem ? tbl_bytes_smem : 0;
  // cell stride of a slot: NC (cell-fastest, so a warp touching consecutive
  // items of one phase reads consecutive doubles: conflict-free)
  auto ncp_of = [](int nc) { return nc; };
  auto bytes_of = [&](int nc) { return tb + peak * ncp_of(nc) * 8; };
  int nc = 0;
  long long cta_budget = 56 * 1024;  // ~4 CTAs per SM (measured best, tools/lp_sweep.sh)
  if (option(OPT_LP_SMEM_KB) > 0) cta_budget = option(OPT_LP_SMEM_KB) * 1024;
  for (int cand = 32; cand >= 1; cand /= 2)
    if (bytes_of(cand) <= cta_budget) { nc = cand; break; }
  if (!nc && bytes_of(1) <= smem_limit) nc = 1;
  if (nc) {
    C.cells_per_block = nc;
    C.ncp = ncp_of(nc);
    C.smem_bytes = bytes_of(nc);
  } else {
    C.global_scratch = true;
    C.cells_per_block = 1;
    C.ncp = 1;
    C.smem_bytes = tb;
    C.arena_doubles_per_block = ((peak + 31) / 32) * 32;
  }
  // CTA size (tools/lp_sweep.sh): 256 threads, one item each in the widest
  // phase if fewer suffice -- unless the work-weighted median phase needs two
  // rounds of 256 but fits one round of <= 512 (then one round).  The launch
  // bound keeps <= 128 registers so the ~4 CTAs the 56 KB smem budget allows
  // are not register-limited.
  long long maxitems = 1;
  std::vector<std::pair<long long, double>> items;  // (items, work)
  double work_total = 0;
  for (const auto& ph : phases) {
    if (ph.k != Phase::NEST) continue;
    long long nred = 1;
    for (const auto& r : ph.red) nred *= r.second;
    const long long it = ph.nitem * C.cells_per_block;
    maxitems = std::max(maxitems, it);
    items.emplace_back(it, (double)it * nred);
    work_total += (double)it * nred;
  }
  std::sort(items.begin(), items.end());
  long long median = 0;
  double acc_w = 0;
  for (const auto& it : items) {
    acc_w += it.second;
    if (acc_w >= 0.5 * work_total) { median = it.first; break; }
  }
  long long tmax = 256;
  if (median > 256 && median <= 512) maxitems = median, tmax = 512;
  if (option(OPT_LP_MAX_THREADS) > 0) tmax = option(OPT_LP_MAX_THREADS);
  C.threads = (int)std::min<long long>(tmax, std::max<long long>(64, ((maxitems + 31) / 32) * 32));

  // warp mode: with at least one cell per warp, every warp owns whole cells
  // through all phases, so all dependencies stay inside a warp and the
  // barriers become __syncwarp (the CTA-wide version spent 18% of its stalls
  // at barriers, profiles/r01av_lp_p3.md).  option lp_warp = -1 disables it.
  {
    // measured (profiles/r01bc_lp_warp.jsonl): a win for matrix-shaped
    // programs (laplace hex p=2 1.04 -> 0.72 ms, curl_curl, prism matrices),
    // a loss for the actions, whose large phases want many threads per cell
    bool wm = C.cells_per_block >= 2 && !C.global_scratch && P.ret_size >= 128;
    if (option(OPT_LP_WARP) < 0) wm = false;
    if (wm) {
      // largest power of two <= min(threads / 32, NC) (NC is a power of two)
      const int cap = std::max(1, std::min(C.threads / 32, C.cells_per_block));
      int warps = 1;
      while (warps * 2 <= cap) warps *= 2;
      C.threads = 32 * warps;
      C.warp_mode = 1;
      C.cells_per_warp = C.cells_per_block / warps;
    }
  }

  // 4. emission
  const int NC = C.cells_per_block, NCP = C.ncp, T = C.threads;
  const bool WM = C.warp_mode != 0;
  const int LN = WM ? C.cells_per_warp : NC;   // cells of one loop group (warp or CTA)
  const int LT = WM ? 32 : T;                  // threads of one loop group
  const std::string TID = WM ? "lane" : "threadIdx.x";
  // warp mode: each warp has its own [slot][LN] region (Sw), c is the
  // warp-local cell and wbase + c the CTA cell (global addressing, nvalid)
  const std::string CB = WM ? "wbase + " : "";
  const std::string SYNC = WM ? "__syncwarp()" : "__syncthreads()";
  std::ostringstream o;
  auto slot = [&](const std::string& nm, const std::string& addr) {
    std::ostringstream s;
    const long long b = base.at(nm);
    const int stride = WM ? LN : NCP;
    const char* arr = WM ? "Sw" : "S";
    if (stride == 1) s << arr << "[" << b << " + (" << addr << ")]";
    else s << arr << "[(" << b << " + (" << addr << ")) * " << stride << " + c]";
    return s.str();
  };
  auto ent = [](const Entry& e) { return e.idx >= 0 ? "i" + std::to_string(e.idx) : std::to_string(e.val); };
  auto addr = [&](long long off, const std::vector<Term>& terms) {
    std::ostringstream s;
    long long c0 = off;
    bool any = false;
    for (const auto& t : terms) {
      if (t.e.idx < 0) { c0 += t.e.val * t.stride; continue; }
      if (t.stride == 0) continue;
      if (any) s << " + ";
      if (t.stride == 1) s << "i" << t.e.idx;
      else s << t.stride << " * i" << t.e.idx;
      any = true;
    }
    if (c0 || !any) { if (any) s << " + "; s << c0; }
    return s.str();
  };
  std::function<std::string(const Expr&)> ex = [&](const Expr& e) -> std::string {
    switch (e.k) {
      case Expr::LIT: return fmt_double(e.lit);
      case Expr::LOAD: return slot(e.name, addr(e.offset, e.terms));
      case Expr::TABLE: {
        std::ostringstream s;
        s << (C.tables_in_smem ? "Tb[" : "sfk_tables[") << toff[e.table] << " + ("
          << addr(0, e.terms) << ")]";
        return s.str();
      }
      case Expr::DELTA: return "((" + ent(e.d0) + " == " + ent(e.d1) + ") ? 1.0 : 0.0)";
      case Expr::ADD: return "(" + ex(*e.a) + " + " + ex(*e.b) + ")";
      case Expr::MUL: return "(" + ex(*e.a) + " * " + ex(*e.b) + ")";
      case Expr::DIV: return "(" + ex(*e.a) + " / " + ex(*e.b) + ")";
      case Expr::POW: return "pow(" + ex(*e.a) + ", " + ex(*e.b) + ")";
      case Expr::MIN: return "fmin(" + ex(*e.a) + ", " + ex(*e.b) + ")";
      case Expr::MAX: return "fmax(" + ex(*e.a) + ", " + ex(*e.b) + ")";
      case Expr::CALL: {
        static const std::map<std::string, std::string> fn = {
            {"sqrt", "sqrt"}, {"sin", "sin"}, {"cos", "cos"}, {"tan", "tan"},
            {"exp", "exp"},   {"ln", "log"},  {"abs", "fabs"}};
        auto it = fn.find(e.name);
        if (it == fn.end()) throw std::runtime_error("LoopProgram: unsupported function " + e.name);
        return it->second + "(" + ex(*e.a) + ")";
      }
      case Expr::CMP: {
        static const std::set<std::string> ops = {"<", ">", "<=", ">=", "==", "!="};
        if (!ops.count(e.name)) throw std::runtime_error("LoopProgram: comparison " + e.name);
        return "((" + ex(*e.a) + " " + e.name + " " + ex(*e.b) + ") ? 1.0 : 0.0)";
      }
    }
    return "0.0";
  };
  std::function<void(const Stmt&, int)> serial = [&](const Stmt& s, int ind) {
    const std::string pad(ind * 2, ' ');
    switch (s.k) {
      case Stmt::LOOP:
        o << pad << "for (int i" << s.idx << " = 0; i" << s.idx << " < " << s.extent << "; ++i"
          << s.idx << ") {\n";
        for (const auto& b : s.body) serial(b, ind + 1);
        o << pad << "}\n";
        break;
      case Stmt::ZERO:
        o << pad << "for (int z = 0; z < " << s.size << "; ++z) " << slot(s.name, "z") << " = 0.0;\n";
        break;
      case Stmt::ASSIGN:
        o << pad << slot(s.name, addr(s.offset, s.terms)) << " = " << ex(*s.e) << ";\n";
        break;
      case Stmt::ACCUM: {
        const std::string t = slot(s.name, addr(s.offset, s.terms));
        o << pad << t << " = " << t << " + " << ex(*s.e) << ";\n";
        break;
      }
    }
  };

  G.entry = "sfk_lp_" + P.name;
  for (auto& ch : G.entry)
    if (!std::isalnum((unsigned char)ch) && ch != '_') ch = '_';
  o << "// generated by libsfk from the LoopProgram '" << P.name << "'\n"
    << "// NC=" << NC << " cells/CTA, " << T << " threads, " << C.slots << " slots/cell, "
    << (C.global_scratch ? "global arena" : "shared memory") << "\n";
  if (tbl_doubles) {
    o << "__device__ const double sfk_tables[" << tbl_doubles << "] = {";
    long long n = 0;
    for (const auto& t : P.tables)
      for (double v : t.values) o << (n++ ? ", " : "") << fmt_double(v);
    o << "};\n";
  }
  // registers: enough CTAs for the smem budget, at most 1024 threads per SM
  const long long smem_ctas = std::max<long long>(1, (228 * 1024) / (C.smem_bytes + 1024));
  long long minb = std::max<long long>(1, std::min<long long>(smem_ctas, 1024 / T));
  if (option(OPT_LP_MINB) > 0) minb = option(OPT_LP_MINB);
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ", " << minb << ") "
    << G.entry
    << "(double* __restrict__ gA";
  for (size_t a = 0; a < P.args.size(); ++a) o << ", const double* __restrict__ g" << a;
  o << ", long long ncells, double* __restrict__ arena) {\n"
    << "  extern __shared__ __align__(16) double smem[];\n";
  if (C.tables_in_smem && tbl_doubles) {
    o << "  double* Tb = smem;\n"
      << "  for (int k = threadIdx.x; k < " << tbl_doubles << "; k += " << T
      << ") Tb[k] = sfk_tables[k];\n"
      << "  __syncthreads();\n";
  }
  if (C.global_scratch)
    o << "  double* __restrict__ S = arena + (long long)blockIdx.x * " << C.arena_doubles_per_block
      << ";\n";
  else
    o << "  double* S = smem + " << tb / 8 << ";\n";
  o << "  const long long nchunks = (ncells + " << NC - 1 << ") / " << NC << ";\n"
    << "  for (long long chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {\n"
    << "    const long long c0 = chunk * " << NC << ";\n"
    << "    const int nvalid = (int)((ncells - c0) < " << NC << " ? (ncells - c0) : " << NC << ");\n";
  if (NC == 1) o << "    const int c = 0; (void)c;\n";
  if (WM)
    o << "    const int lane = threadIdx.x & 31, wbase = (threadIdx.x >> 5) * " << LN << ";\n"
      << "    double* Sw = S + (threadIdx.x >> 5) * " << C.slots * LN << ";\n";
  // global <-> shared transfers: each warp moves G consecutive elements of
  // 32/G cells (G*NC = 32 when NC <= 32): G-double runs per cell in HBM,
  // 32 consecutive doubles in shared memory (element k of cell c at k*NC + c)
  std::vector<Access> acc;
  auto xfer_g = [&](long long sz) { return std::min<long long>(sz, std::max(1, 32 / LN)); };
  auto xfer_items = [&](long long sz) {
    const long long g = xfer_g(sz);
    return LN * g * ((sz + g - 1) / g);
  };
  auto xfer_open = [&](long long sz) {
    const long long g = xfer_g(sz);
    o << "    for (int e = " << TID << "; e < " << xfer_items(sz) << "; e += " << LT << ") {\n";
    if (NC > 1)
      o << "      const int c = (e / " << g << ") % " << LN << ", k = (e / " << g * LN
        << ") * " << g << " + e % " << g << ";\n";
    else
      o << "      const int k = e;\n";
  };
  // accesses of one loop group (element = slot * LN + group-local cell)
  auto xfer_access = [&](long long sz, long long b, bool write) {
    const long long g = xfer_g(sz);
    acc.clear();
    for (long long e = 0; e < xfer_items(sz); ++e) {
      const long long c = NC > 1 ? (e / g) % LN : 0;
      const long long k = NC > 1 ? (e / (g * LN)) * g + e % g : e;
      if (k < sz) acc.push_back({(b + k) * LN + c, (int)(e % LT), write});
    }
  };
  for (size_t a = 0; a < P.args.size(); ++a) {
    const long long sz = P.args[a].second;
    xfer_open(sz);
    o << "      if (k < " << sz << ") " << slot(P.args[a].first, "k") << " = (" << CB
      << "c < nvalid) ? g" << a << "[(c0 + " << CB << "c) * " << sz << " + k] : 0.0;\n    }\n";
  }
  // barrier plan (see Window): the argument loads open the window
  int max_idx = 0;
  for (const auto& kv : P.extents) max_idx = std::max(max_idx, kv.first);
  Window win(C.slots * LN);
  for (size_t a = 0; a < P.args.size(); ++a) {
    xfer_access(P.args[a].second, base.at(P.args[a].first), true);
    win.add(acc);
  }
  // fused loop groups: consecutive NEST phases with the same trip count, no
  // barrier between them and only same-item dependences share one loop over w
  bool fusion = true;
  if (option(OPT_LP_FUSE) < 0) fusion = false;
  ItemWindow iwin(C.slots * LN);
  long long group_trips = -1;   // trip count of the open loop group (-1: none open)
  auto close_group = [&]() {
    if (group_trips >= 0) o << "    }\n";
    group_trips = -1;
    iwin.clear();
  };
  auto barrier_for = [&](bool known) {
    const bool need = !known || win.conflicts(acc);
    if (need) {
      close_group();
      o << "    " << SYNC << ";\n";
      ++C.barriers;
      win.clear();
    }
    if (known) win.add(acc);
    else win.poisoned = true;
    return need;
  };
  C.phases = (int)phases.size();
  for (size_t k = 0; k < phases.size(); ++k) {
    const Phase& ph = phases[k];
    const bool known = phase_accesses(ph, base, bufsize, LN, LT, max_idx, acc);
    barrier_for(known);
    if (ph.k != Phase::NEST) close_group();
    if (ph.k == Phase::ZERO) {
      o << "    // phase " << k << ": zero " << ph.zname << "\n"
        << "    for (int e = " << TID << "; e < " << LN * ph.zsize << "; e += " << LT << ") {\n";
      if (NC > 1) o << "      const int c = e % " << LN << ", z = e / " << LN << ";\n";
      else o << "      const int z = e;\n";
      o << "      " << slot(ph.zname, "z") << " = 0.0;\n    }\n";
    } else if (ph.k == Phase::SERIAL) {
      ++C.serial_phases;
      o << "    // phase " << k << ": serial nest (thread per cell)\n";
      if (NC > 1)
        o << "    for (int c = " << TID << "; c < " << LN << "; c += " << LT << ") {\n";
      else o << "    if (threadIdx.x == 0) {\n";
      serial(*ph.top, 3);
      o << "    }\n";
    } else {
      const Stmt& L = *ph.leaf;
      const int E = ph.blk_ext;
      const std::string bv = ph.blk >= 0 ? "i" + std::to_string(ph.blk) : std::string();
      o << "    // phase " << k << ": " << (L.k == Stmt::ACCUM ? "accumulate " : "assign ") << L.name
        << " (" << ph.npar << " parallel";
      if (E > 1) o << ", " << E << " per thread along " << bv;
      o << " x " << ph.red.size() << " reduction loops)\n";
      const long long trips = LN * ph.nitem;
      const bool join = fusion && known && group_trips == trips && iwin.compatible(acc);
      if (!join) {
        close_group();
        o << "    for (int w = " << TID << "; w < " << trips << "; w += " << LT << ") {\n";
        if (NC > 1) o << "      const int c = w % " << LN << ";\n";
        group_trips = trips;
      } else {
        ++C.fused_phases;
      }
      iwin.add(acc);
      o << "     {\n";
      if (NC > 1) o << "      int q = w / " << LN << ";\n";
      else o << "      int q = w;\n";
      for (size_t j = ph.opar.size(); j-- > 0;) {
        const auto& pr = ph.opar[j];
        if (j == 0) o << "      const int i" << pr.first << " = q;\n";
        else o << "      const int i" << pr.first << " = q % " << pr.second << "; q /= " << pr.second << ";\n";
      }
      if (ph.opar.empty()) o << "      (void)q;\n";
      const std::string tgt = slot(L.name, addr(L.offset, L.terms));
      const std::string av = E > 1 ? "acc[" + bv + "]" : std::string("acc");
      // the E outputs of the block accumulate in registers and are stored at
      // the end, so loads independent of the block index are loaded once
      auto bopen = [&](const std::string& pad) {
        if (E > 1)
          o << pad << "#pragma unroll\n" << pad << "for (int " << bv << " = 0; " << bv << " < " << E
            << "; ++" << bv << ") ";
      };
      o << "      double acc" << (E > 1 ? "[" + std::to_string(E) + "]" : std::string()) << ";\n";
      if (L.k == Stmt::ACCUM) {
        bopen("      ");
        o << (E > 1 ? "" : "      ") << av << " = " << (ph.zero_init ? "0.0" : tgt) << ";\n";
      }
      std::string pad = "      ";
      for (size_t j = 0; j < ph.red.size(); ++j) {
        const auto& r = ph.red[j];
        if (j + 1 == ph.red.size() && r.second <= 32 && r.second * E <= 64)
          o << pad << "#pragma unroll\n";
        o << pad << "for (int i" << r.first << " = 0; i" << r.first << " < " << r.second << "; ++i"
          << r.first << ") {\n";
        pad += "  ";
      }
      if (E > 1) {
        o << pad << "#pragma unroll\n"
          << pad << "for (int " << bv << " = 0; " << bv << " < " << E << "; ++" << bv << ")\n  ";
      }
      o << pad << av << " = " << (L.k == Stmt::ACCUM ? av + " + " : std::string()) << ex(*L.e)
        << ";\n";
      for (size_t r = 0; r < ph.red.size(); ++r) {
        pad.resize(pad.size() - 2);
        o << pad << "}\n";
      }
      bopen("      ");
      o << (E > 1 ? "" : "      ") << tgt << " = " << av << ";\n";
      o << "     }\n";
    }
  }
  close_group();
  // store A
  xfer_access(P.ret_size, base.at(P.ret_name), false);
  barrier_for(true);
  xfer_open(P.ret_size);
  o << "      if (k < " << P.ret_size << " && " << CB << "c < nvalid) gA[(c0 + " << CB << "c) * "
    << P.ret_size << " + k] = " << slot(P.ret_name, "k") << ";\n    }\n";
  o << "    " << SYNC << ";\n  }\n}\n";
  G.source = o.str();
  return G;
}

}  // namespace lp
}  // namespace sfk
