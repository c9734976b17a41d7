// xir.cpp -- native reader of the stencil-level textual IR (the reference's `.xir` syntax,
// as printed by proj/core/src/ir/printer.cpp and parsed by parser.cpp) into hg_program.
//
// Covers what the device path executes: one all-field func.func with stencil.load,
// dmp.swap {grid, exchanges}, one stencil.apply (access / arith.constant / addf / subf / mulf /
// divf / stencil.return, any number of results), stencil.store, func.return; module
// attributes stencil.time_slots and dmp.topology (dmp.reference is read on request).
// Float literals are converted exactly like the reference (std::from_chars of the token in
// the literal's own type, parser.cpp:392-404), so constants carry identical bits.
#include "hg_internal.hpp"

#include <cctype>
#include <charconv>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace hg {
namespace {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Reader {
  const std::string &s;
  size_t i = 0;
  explicit Reader(const std::string &t) : s(t) {}

  [[noreturn]] void fail(const std::string &m) const {
    int line = 1, col = 1;
    for (size_t k = 0; k < i && k < s.size(); ++k) {
      if (s[k] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
    throw ParseError(std::to_string(line) + ":" + std::to_string(col) + ": " + m);
  }
  void ws() {
    for (;;) {
      while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i])))
        ++i;
      if (i + 1 < s.size() && s[i] == '/' && s[i + 1] == '/') {
        while (i < s.size() && s[i] != '\n')
          ++i;
        continue;
      }
      break;
    }
  }
  bool peek(const char *t) {
    ws();
    return s.compare(i, std::strlen(t), t) == 0;
  }
  bool accept(const char *t) {
    if (!peek(t))
      return false;
    i += std::strlen(t);
    return true;
  }
  void expect(const char *t) {
    if (!accept(t))
      fail(std::string("expected '") + t + "'");
  }
  static bool identChar(char c) {
    return std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '.' || c == '$';
  }
  std::string ident() {
    ws();
    size_t b = i;
    while (i < s.size() && identChar(s[i]))
      ++i;
    if (b == i)
      fail("expected an identifier");
    return s.substr(b, i - b);
  }
  std::string value() { // %name
    ws();
    if (i >= s.size() || s[i] != '%')
      fail("expected an SSA value");
    ++i;
    size_t b = i;
    while (i < s.size() && (std::isalnum(static_cast<unsigned char>(s[i])) || s[i] == '_'))
      ++i;
    if (b == i)
      fail("empty SSA value name");
    return s.substr(b, i - b);
  }
  int64_t integer() {
    ws();
    size_t b = i;
    if (i < s.size() && (s[i] == '-' || s[i] == '+'))
      ++i;
    while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i])))
      ++i;
    if (b == i || (i == b + 1 && !std::isdigit(static_cast<unsigned char>(s[b]))))
      fail("expected an integer");
    return std::stoll(s.substr(b, i - b));
  }
  std::string number() { // float or integer literal token
    ws();
    size_t b = i;
    if (i < s.size() && (s[i] == '-' || s[i] == '+'))
      ++i;
    while (i < s.size() &&
           (std::isalnum(static_cast<unsigned char>(s[i])) || s[i] == '.' ||
            ((s[i] == '-' || s[i] == '+') && (s[i - 1] == 'e' || s[i - 1] == 'E'))))
      ++i;
    if (b == i)
      fail("expected a number");
    return s.substr(b, i - b);
  }
  std::string balanced(char open, char close) { // from an `open` to its matching `close`
    ws();
    if (i >= s.size() || s[i] != open)
      fail(std::string("expected '") + open + "'");
    size_t b = i;
    int depth = 0;
    bool str = false;
    for (; i < s.size(); ++i) {
      char c = s[i];
      if (str) {
        if (c == '\\')
          ++i;
        else if (c == '"')
          str = false;
        continue;
      }
      if (c == '"')
        str = true;
      else if (c == open)
        ++depth;
      else if (c == close && --depth == 0) {
        ++i;
        return s.substr(b, i - b);
      }
    }
    fail("unbalanced bracket");
  }
  std::string str() {
    ws();
    if (i >= s.size() || s[i] != '"')
      fail("expected a string");
    std::string out;
    for (++i; i < s.size() && s[i] != '"'; ++i) {
      if (s[i] == '\\' && i + 1 < s.size()) {
        char n = s[++i];
        out += n == 'n' ? '\n' : n == 't' ? '\t' : n;
      } else {
        out += s[i];
      }
    }
    if (i >= s.size())
      fail("unterminated string");
    ++i;
    return out;
  }
};

struct TypeInfo {
  bool field = false, temp = false, known = false;
  int rank = 0;
  int dtype = 0; // HG_F32 / HG_F64, 0 for non-float
  int64_t lb[3] = {0, 0, 0}, ub[3] = {0, 0, 0};
};

int elemOf(const std::string &e) {
  if (e == "f32")
    return HG_F32;
  if (e == "f64")
    return HG_F64;
  return 0;
}

// "[a,b]x[c,d]" into bounds; returns rank
int parseBoundsText(Reader &R, const std::string &t, int64_t *lb, int64_t *ub) {
  int r = 0;
  size_t k = 0;
  while (k < t.size()) {
    if (t[k] != '[')
      R.fail("malformed bounds '" + t + "'");
    size_t c = t.find(',', k), e = t.find(']', k);
    if (c == std::string::npos || e == std::string::npos || r >= 3)
      R.fail("malformed bounds '" + t + "'");
    lb[r] = std::stoll(t.substr(k + 1, c - k - 1));
    ub[r] = std::stoll(t.substr(c + 1, e - c - 1));
    ++r;
    k = e + 1;
    if (k < t.size() && t[k] == 'x')
      ++k;
  }
  return r;
}

TypeInfo parseType(Reader &R) {
  TypeInfo ti;
  R.ws();
  if (R.peek("!field<") || R.peek("!temp<")) {
    const bool field = R.peek("!field<");
    R.i += field ? 6 : 5;
    std::string inner = R.balanced('<', '>');
    inner = inner.substr(1, inner.size() - 2);
    // split "<bounds>x<elem>" at the last 'x' at bracket depth 0
    size_t cut = inner.rfind('x');
    if (cut == std::string::npos)
      R.fail("malformed type");
    std::string b = inner.substr(0, cut), e = inner.substr(cut + 1);
    ti.field = field;
    ti.temp = !field;
    ti.dtype = elemOf(e);
    if (b != "?") {
      ti.rank = parseBoundsText(R, b, ti.lb, ti.ub);
      ti.known = true;
    }
    return ti;
  }
  if (R.accept("(")) { // tuple type (T, T, ...)
    R.i -= 1;
    R.balanced('(', ')');
    return ti;
  }
  std::string n = R.ident();
  ti.dtype = elemOf(n);
  return ti;
}

std::vector<int64_t> intList(Reader &R) { // [a, b, ...]
  std::vector<int64_t> v;
  R.expect("[");
  if (R.accept("]"))
    return v;
  do
    v.push_back(R.integer());
  while (R.accept(","));
  R.expect("]");
  return v;
}

hg_exchange parseExchange(Reader &R) {
  // #dmp.exchange<at [..] size [..] source offset [..] to [..]>
  R.expect("#dmp.exchange<");
  hg_exchange e;
  std::memset(&e, 0, sizeof e);
  auto copy = [&](int64_t *dst, const std::vector<int64_t> &v) {
    if (v.size() > 3)
      R.fail("exchange rank > 3");
    for (size_t k = 0; k < v.size(); ++k)
      dst[k] = v[k];
  };
  R.expect("at");
  copy(e.at, intList(R));
  R.expect("size");
  copy(e.size, intList(R));
  R.expect("source");
  R.expect("offset");
  copy(e.offset, intList(R));
  R.expect("to");
  copy(e.to, intList(R));
  R.expect(">");
  return e;
}

std::vector<int64_t> parseGrid(Reader &R) { // #dmp.grid<AxBxC>
  R.expect("#dmp.grid<");
  std::vector<int64_t> g;
  do
    g.push_back(R.integer());
  while (R.accept("x"));
  R.expect(">");
  return g;
}

// skip any attribute value
void skipAttr(Reader &R) {
  R.ws();
  if (R.peek("\"")) {
    R.str();
  } else if (R.peek("[")) {
    R.balanced('[', ']');
  } else if (R.peek("{")) {
    R.balanced('{', '}');
  } else if (R.peek("#")) {
    while (R.i < R.s.size() && R.s[R.i] != '<')
      ++R.i;
    R.balanced('<', '>');
  } else {
    R.number();
  }
  if (R.accept(":"))
    parseType(R);
}

struct PApply {
  std::vector<int> operands;  // >= 0 field, < 0 temp (-t-1)
  int op_begin = 0, nops = 0;
  std::vector<int> result_op; // slice-relative
  std::vector<int> result_temp;
  bool domainKnown = false;
  hg_bounds domain{};
};

struct PStore {
  int temp, field;
  hg_bounds region;
};

struct Parsed {
  hg_program prog{};
  std::vector<hg_op> ops;
  std::vector<hg_apply> applies;
  std::vector<PApply> papplies;
  std::vector<PStore> pstores;
  std::vector<int> loads; // stencil.load fields in step order
  int ntemps = 0;
  hg_decomp dc{};
  bool decomposed = false;
  std::string reference; // dmp.reference text, if any
  std::vector<std::vector<int>> groups;
};

void parseModule(const std::string &text, Parsed &P) {
  Reader R(text);
  std::memset(&P.prog, 0, sizeof P.prog);
  std::memset(&P.dc, 0, sizeof P.dc);
  R.expect("builtin.module");
  std::vector<int64_t> topology;
  if (R.accept("attributes")) {
    R.expect("{");
    if (!R.accept("}")) {
      do {
        std::string key = R.ident();
        R.expect("=");
        if (key == "stencil.time_slots") {
          R.expect("[");
          if (!R.accept("]")) {
            do {
              auto v = intList(R);
              P.groups.emplace_back(v.begin(), v.end());
            } while (R.accept(","));
            R.expect("]");
          }
        } else if (key == "dmp.topology") {
          topology = parseGrid(R);
        } else if (key == "dmp.reference") {
          P.reference = R.str();
        } else {
          skipAttr(R);
        }
      } while (R.accept(","));
      R.expect("}");
    }
  }
  R.expect("{");
  bool haveEntry = false;
  while (!R.accept("}")) {
    R.expect("func.func");
    R.expect("@");
    std::string fname = R.ident();
    // arguments
    R.expect("(");
    std::vector<std::string> argNames;
    std::vector<TypeInfo> argTypes;
    if (!R.accept(")")) {
      do {
        argNames.push_back(R.value());
        R.expect(":");
        argTypes.push_back(parseType(R));
      } while (R.accept(","));
      R.expect(")");
    }
    if (R.accept("->"))
      parseType(R);
    bool allFields = !argTypes.empty();
    for (auto &t : argTypes)
      allFields = allFields && t.field;
    if (!allFields || haveEntry) {
      R.balanced('{', '}'); // not the stencil entry: skip its body
      if (allFields && haveEntry)
        R.fail("module has more than one all-field function");
      continue;
    }
    haveEntry = true;
    hg_program &p = P.prog;
    p.nfields = static_cast<int>(argTypes.size());
    if (p.nfields > HG_MAX_FIELDS)
      R.fail("too many fields");
    std::map<std::string, int> argIdx, loadOf;
    for (int f = 0; f < p.nfields; ++f) {
      const TypeInfo &t = argTypes[static_cast<size_t>(f)];
      if (f == 0) {
        p.rank = t.rank;
        p.dtype = t.dtype;
      }
      if (t.rank != p.rank || t.dtype != p.dtype || !t.dtype)
        R.fail("fields must share rank and f32/f64 element type");
      for (int d = 0; d < t.rank; ++d) {
        p.fields[f].lb[d] = t.lb[d];
        p.fields[f].ub[d] = t.ub[d];
      }
      argIdx[argNames[static_cast<size_t>(f)]] = f;
    }
    std::map<std::string, int> tempOf; // apply result value -> temp id
    int &ntemps = P.ntemps;
    std::vector<PApply> &applies = P.papplies;
    std::vector<PStore> &stores = P.pstores;
    R.expect("{");
    while (!R.accept("}")) {
      if (R.peek("func.return")) {
        R.expect("func.return");
        continue;
      }
      if (R.peek("dmp.swap")) {
        R.expect("dmp.swap");
        R.expect("(");
        std::string v = R.value();
        R.expect(")");
        auto it = argIdx.find(v);
        if (it == argIdx.end())
          R.fail("dmp.swap of a non-argument");
        if (P.dc.nswaps >= HG_MAX_FIELDS)
          R.fail("too many swaps");
        hg_swap &sw = P.dc.swaps[P.dc.nswaps++];
        sw.field = it->second;
        R.expect("{");
        do {
          std::string key = R.ident();
          R.expect("=");
          if (key == "grid") {
            auto g = parseGrid(R);
            P.dc.ndim = static_cast<int>(g.size());
            for (size_t d = 0; d < g.size() && d < 3; ++d)
              P.dc.grid[d] = g[d];
          } else if (key == "exchanges") {
            R.expect("[");
            if (!R.accept("]")) {
              do {
                if (sw.nexchanges >= 2 * HG_MAX_RANK)
                  R.fail("too many exchanges");
                sw.ex[sw.nexchanges++] = parseExchange(R);
              } while (R.accept(","));
              R.expect("]");
            }
          } else {
            skipAttr(R);
          }
        } while (R.accept(","));
        R.expect("}");
        if (R.accept(":")) {
          parseType(R);
          R.expect("->");
          parseType(R);
        }
        P.decomposed = true;
        continue;
      }
      if (R.peek("stencil.store")) {
        R.expect("stencil.store");
        std::string src = R.value();
        R.expect("to");
        std::string dst = R.value();
        std::string b = R.balanced('(', ')');
        auto rit = tempOf.find(src);
        auto fit = argIdx.find(dst);
        if (rit == tempOf.end() || fit == argIdx.end())
          R.fail("stencil.store of a non-apply value or into a non-argument");
        PStore st{rit->second, fit->second, {}};
        int r = parseBoundsText(R, b.substr(1, b.size() - 2), st.region.lb, st.region.ub);
        if (r != p.rank)
          R.fail("store bounds rank mismatch");
        stores.push_back(st);
        R.expect(":");
        parseType(R);
        R.expect("to");
        parseType(R);
        continue;
      }
      // "%a[, %b ...] = <op>"
      std::vector<std::string> defs;
      do
        defs.push_back(R.value());
      while (R.accept(","));
      R.expect("=");
      std::string opn = R.ident();
      if (opn == "stencil.load") {
        std::string v = R.value();
        auto it = argIdx.find(v);
        if (it == argIdx.end())
          R.fail("stencil.load of a non-argument");
        loadOf[defs[0]] = it->second;
        P.loads.push_back(it->second);
        R.expect(":");
        parseType(R);
        R.expect("->");
        parseType(R);
        continue;
      }
      if (opn != "stencil.apply")
        R.fail("unsupported op in the step function: " + opn);
      if (applies.size() >= HG_MAX_APPLIES)
        R.fail("too many stencil.apply ops");
      applies.emplace_back();
      PApply &A = applies.back();
      A.op_begin = static_cast<int>(P.ops.size());
      R.expect("(");
      std::map<std::string, int> regionArg;
      if (!R.accept(")")) {
        do {
          std::string a = R.value();
          R.expect("=");
          std::string t = R.value();
          R.expect(":");
          parseType(R);
          auto it = loadOf.find(t);
          auto tt = tempOf.find(t);
          if (it != loadOf.end())
            A.operands.push_back(it->second);
          else if (tt != tempOf.end())
            A.operands.push_back(-tt->second - 1);
          else
            R.fail("apply operand is neither a stencil.load nor an apply result");
          regionArg[a] = static_cast<int>(A.operands.size()) - 1;
        } while (R.accept(","));
        R.expect(")");
        if (A.operands.size() > HG_MAX_FIELDS)
          R.fail("too many apply operands");
      }
      R.expect("->");
      {
        // result type(s): a single !temp or a (tuple); bounds give the evaluation domain
        R.ws();
        std::string rt;
        if (R.peek("(")) {
          rt = R.balanced('(', ')');
          Reader R2(rt);
          R2.expect("(");
          TypeInfo t0 = parseType(R2);
          A.domainKnown = t0.known;
          for (int d = 0; d < t0.rank; ++d) {
            A.domain.lb[d] = t0.lb[d];
            A.domain.ub[d] = t0.ub[d];
          }
        } else {
          TypeInfo t0 = parseType(R);
          A.domainKnown = t0.known;
          for (int d = 0; d < t0.rank; ++d) {
            A.domain.lb[d] = t0.lb[d];
            A.domain.ub[d] = t0.ub[d];
          }
        }
      }
      if (defs.size() > HG_MAX_RESULTS)
        R.fail("too many apply results");
      for (size_t k = 0; k < defs.size(); ++k) {
        A.result_temp.push_back(ntemps);
        tempOf[defs[k]] = ntemps++;
      }
      std::map<std::string, int> vid;
      R.expect("{");
      while (!R.accept("}")) {
        if (R.peek("stencil.return")) {
          R.expect("stencil.return");
          do {
            std::string v = R.value();
            auto it = vid.find(v);
            if (it == vid.end())
              R.fail("stencil.return of an undefined value %" + v);
            A.result_op.push_back(it->second - A.op_begin);
          } while (R.accept(","));
          if (A.result_op.size() != A.result_temp.size())
            R.fail("stencil.return arity mismatch");
          R.expect(":");
          do
            parseType(R);
          while (R.accept(","));
          continue;
        }
        std::string d = R.value();
        R.expect("=");
        std::string in = R.ident();
        hg_op h;
        std::memset(&h, 0, sizeof h);
        if (in == "stencil.access") {
          std::string a = R.value();
          auto it = regionArg.find(a);
          if (it == regionArg.end())
            R.fail("stencil.access of a non-region value %" + a);
          h.code = HG_OP_ACCESS;
          h.operand = it->second;
          auto off = intList(R);
          if (static_cast<int>(off.size()) != p.rank)
            R.fail("access offset rank mismatch");
          for (size_t k = 0; k < off.size(); ++k)
            h.off[k] = off[k];
          R.expect(":");
          parseType(R);
        } else if (in == "arith.constant") {
          std::string tok = R.number();
          R.expect(":");
          TypeInfo t = parseType(R);
          h.code = HG_OP_CONST;
          if (t.dtype == HG_F32) {
            float f = 0.0f;
            auto r = std::from_chars(tok.data(), tok.data() + tok.size(), f);
            if (r.ec != std::errc())
              R.fail("malformed float literal '" + tok + "'");
            uint32_t u;
            std::memcpy(&u, &f, 4);
            h.bits = u;
          } else if (t.dtype == HG_F64) {
            double v = 0.0;
            auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
            if (r.ec != std::errc())
              R.fail("malformed float literal '" + tok + "'");
            std::memcpy(&h.bits, &v, 8);
          } else {
            R.fail("only f32/f64 constants are supported");
          }
        } else if (in == "arith.addf" || in == "arith.subf" || in == "arith.mulf" ||
                   in == "arith.divf") {
          h.code = in == "arith.addf"   ? HG_OP_ADD
                   : in == "arith.subf" ? HG_OP_SUB
                   : in == "arith.mulf" ? HG_OP_MUL
                                        : HG_OP_DIV;
          std::string a = R.value();
          R.expect(",");
          std::string b = R.value();
          auto ia = vid.find(a), ib = vid.find(b);
          if (ia == vid.end() || ib == vid.end())
            R.fail("use before def in the apply region");
          h.a = ia->second - A.op_begin;
          h.b = ib->second - A.op_begin;
          R.expect(":");
          parseType(R);
        } else {
          R.fail("unsupported op in the apply region: " + in);
        }
        if (P.ops.size() >= HG_MAX_OPS)
          R.fail("too many ops");
        vid[d] = static_cast<int>(P.ops.size());
        P.ops.push_back(h);
      }
      A.nops = static_cast<int>(P.ops.size()) - A.op_begin;
    }
  }
  if (!haveEntry)
    R.fail("module has no single all-field step function");
  hg_program &p = P.prog;
  p.nops = static_cast<int>(P.ops.size());
  if (P.papplies.empty())
    R.fail("step function has no stencil.apply");
  bool chained = false;
  for (auto &A : P.papplies)
    for (int x : A.operands)
      chained = chained || x < 0;
  if (P.papplies.size() == 1 && !chained) {
    // the single-apply form: operands are loads, results are stored directly
    const PApply &A = P.papplies[0];
    p.noperands = static_cast<int>(A.operands.size());
    for (int o = 0; o < p.noperands; ++o)
      p.operand_field[o] = A.operands[static_cast<size_t>(o)];
    p.nresults = static_cast<int>(A.result_op.size());
    for (int k = 0; k < p.nresults; ++k)
      p.result_op[k] = A.result_op[static_cast<size_t>(k)];
    std::vector<char> stored(static_cast<size_t>(p.nresults), 0);
    for (const PStore &st : P.pstores) {
      if (st.temp >= p.nresults || stored[static_cast<size_t>(st.temp)])
        R.fail("each apply result must be stored exactly once");
      stored[static_cast<size_t>(st.temp)] = 1;
      p.store_field[st.temp] = st.field;
      p.store[st.temp] = st.region;
    }
    for (char c : stored)
      if (!c)
        R.fail("an apply result is never stored");
  } else {
    for (const PApply &A : P.papplies) {
      if (!A.domainKnown)
        R.fail("unresolved stencil.apply bounds (run propagate-bounds)");
      hg_apply h;
      std::memset(&h, 0, sizeof h);
      h.noperands = static_cast<int>(A.operands.size());
      for (int o = 0; o < h.noperands; ++o)
        h.operand[o] = A.operands[static_cast<size_t>(o)];
      h.op_begin = A.op_begin;
      h.nops = A.nops;
      h.nresults = static_cast<int>(A.result_op.size());
      for (int k = 0; k < h.nresults; ++k) {
        h.result_op[k] = A.result_op[static_cast<size_t>(k)];
        h.result_temp[k] = A.result_temp[static_cast<size_t>(k)];
      }
      h.domain = A.domain;
      P.applies.push_back(h);
    }
    p.napplies = static_cast<int>(P.applies.size());
    p.ntemps = P.ntemps;
    if (P.loads.size() > HG_MAX_FIELDS)
      R.fail("too many loads");
    p.noperands = static_cast<int>(P.loads.size());
    for (int o = 0; o < p.noperands; ++o)
      p.operand_field[o] = P.loads[static_cast<size_t>(o)];
    if (P.pstores.size() > HG_MAX_STORES)
      R.fail("too many stores");
    p.nstores = static_cast<int>(P.pstores.size());
    for (int k = 0; k < p.nstores; ++k) {
      p.mstore_temp[k] = P.pstores[static_cast<size_t>(k)].temp;
      p.mstore_field[k] = P.pstores[static_cast<size_t>(k)].field;
      p.mstore[k] = P.pstores[static_cast<size_t>(k)].region;
    }
  }
  int at = 0;
  for (auto &g : P.groups) {
    if (p.ngroups >= HG_MAX_FIELDS || at + static_cast<int>(g.size()) > HG_MAX_FIELDS)
      R.fail("too many time-slot entries");
    p.group_len[p.ngroups++] = static_cast<int>(g.size());
    for (int v : g)
      p.groups[at++] = v;
  }
  if (P.decomposed) {
    if (!topology.empty() && P.dc.ndim == 0) {
      P.dc.ndim = static_cast<int>(topology.size());
      for (size_t d = 0; d < topology.size() && d < 3; ++d)
        P.dc.grid[d] = topology[d];
    }
    for (int d = 0; d < p.rank; ++d)
      P.dc.core[d] = storedRegion(p, 0).ub[d] - storedRegion(p, 0).lb[d];
  }
}

} // namespace
} // namespace hg

using namespace hg;

extern "C" int hg_parse_program(const char *text, hg_program *prog, hg_op *ops, int cap_ops,
                                hg_apply *applies, int cap_applies, hg_decomp *decomp,
                                int *decomposed, char *reference, size_t ref_cap) {
  if (!text || !prog || !ops)
    return setError(HG_EINVAL, "null argument");
  Parsed P;
  try {
    parseModule(text, P);
  } catch (const ParseError &e) {
    return setError(HG_EINVAL, std::string("<xir>:") + e.what());
  } catch (const std::exception &e) {
    return setError(HG_EINVAL, std::string("<xir>: ") + e.what());
  }
  if (static_cast<int>(P.ops.size()) > cap_ops)
    return setError(HG_EINVAL, "op buffer too small");
  std::memcpy(ops, P.ops.data(), P.ops.size() * sizeof(hg_op));
  if (!P.applies.empty()) {
    if (!applies || static_cast<int>(P.applies.size()) > cap_applies)
      return setError(HG_EINVAL, "apply buffer too small");
    std::memcpy(applies, P.applies.data(), P.applies.size() * sizeof(hg_apply));
  }
  *prog = P.prog;
  prog->ops = ops;
  prog->applies = P.applies.empty() ? nullptr : applies;
  if (decomp)
    *decomp = P.dc;
  if (decomposed)
    *decomposed = P.decomposed ? 1 : 0;
  if (reference && ref_cap) {
    if (P.reference.size() + 1 > ref_cap)
      return setError(HG_EINVAL, "reference buffer too small");
    std::memcpy(reference, P.reference.c_str(), P.reference.size() + 1);
  }
  return validateProgram(*prog);
}
