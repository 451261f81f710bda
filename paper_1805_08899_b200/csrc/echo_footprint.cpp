// echo_footprint.cpp — host-side, graph-wide footprint estimator (row a8).
//
// Implements the adjusted NNVM pass pipeline of Fig. 14:
//   InferShape&Type -> Gradient dependencies -> EdgeUseRef -> Echo (Algorithm 1,
//   PAPER.md:488-541) -> DeadNodeElimination -> liveness planning,
// in exact integer bytes (int64).  Readings are listed in DESIGN.md (R11-R13, R22-R25):
//  * gradient dependencies per op: an FC keeps its inputs, not its output (Eq. 2,
//    PAPER.md:389-396); tanh / sigmoid keep their outputs; mul keeps both inputs;
//    add / slice / broadcast-add / stack keep nothing;
//  * partition: backward expansion from the graph outputs, stopped by placeholders, already
//    claimed nodes and compute-heavy ops, which become new seeds (Alg. 1 lines 1-10);
//  * the recomputation paths of all subgraphs are created first; forward trimming then visits
//    every subgraph's members in topological order; the co-removal group is the closure over
//    mirrored nodes sharing a currently stashed input edge (use references);
//    Rel / Alloc are the exact bytes that would leave / enter the stash set if the group were
//    removed from the mirror path, and the group is removed iff Rel >= Alloc;
//    both are evaluated incrementally over the group's input and output edges only;
//  * compute-heavy ops whose gradient needs no output become dead mirrors that forward the
//    recomputed inputs (Alg. 1 lines 13-17); binarizable ops keep a 1-bit mask
//    (line 18);
//  * `stack` is a view: a stashed stack output covers its inputs.
// The same semantics are written independently, slowly and by brute force, in
// oracle/footprint.py; tests/test_footprint.py checks the two agree byte for byte.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/echo.h"

namespace echo {
echo_status fail(echo_status s, const char* fmt, ...);
}

namespace {

// ============================================================================ minimal JSON
// Compact read-only DOM: values live in a JsonDoc's pool (stable addresses), containers point at
// arena arrays of child pointers (and, for objects, keys), strings are views into the source text
// (or into the doc when they contain escapes).  The source text must outlive the doc.
struct Json {
  enum Kind : uint8_t { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  bool b = false;
  double num = 0;
  std::string_view str;
  struct Range {                               // ARR elements / OBJ values
    const Json* const* p = nullptr;
    uint32_t n = 0;
    size_t size() const { return n; }
    const Json& operator[](size_t i) const { return *p[i]; }
    struct It {
      const Json* const* q;
      const Json& operator*() const { return **q; }
      It& operator++() { ++q; return *this; }
      bool operator!=(const It& o) const { return q != o.q; }
    };
    It begin() const { return {p}; }
    It end() const { return {p + n}; }
  } arr;
  const std::string_view* keys = nullptr;      // OBJ keys, parallel to arr
  const Json* get(std::string_view k) const {
    if (kind != OBJ) return nullptr;
    for (uint32_t i = 0; i < arr.n; ++i)
      if (keys[i] == k) return arr.p[i];
    return nullptr;
  }
  long long i64() const { return (long long)llround(num); }
};

struct ParseError : std::runtime_error {
  explicit ParseError(const std::string& s) : std::runtime_error(s) {}
};

struct JsonDoc {
  std::deque<Json> pool;
  std::deque<std::string> escaped;             // strings that contained escapes
  std::vector<std::unique_ptr<char[]>> blocks; // arena for child-pointer and key arrays
  char* cur = nullptr;
  size_t left = 0;
  const Json* root = nullptr;
  template <typename T> T* alloc(size_t n) {
    const size_t bytes = (n * sizeof(T) + 15) & ~(size_t)15;
    if (bytes > left) {
      const size_t sz = bytes > (1u << 20) ? bytes : (1u << 20);
      blocks.emplace_back(new char[sz]);
      cur = blocks.back().get();
      left = sz;
    }
    T* r = reinterpret_cast<T*>(cur);
    cur += bytes;
    left -= bytes;
    return r;
  }
};

// Recursive-descent parser.  Children of open containers are collected on one shared scratch stack
// and copied to the arena when the container closes; integers are parsed without strtod.
struct Parser {
  const char* p;
  const char* end;
  JsonDoc& doc;
  std::vector<const Json*> kid_stack;
  std::vector<std::string_view> key_stack;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r' || *p == '\f' || *p == '\v')) ++p;
  }
  [[noreturn]] void err(const char* what) { throw ParseError(std::string("json: ") + what); }
  std::string_view string_view_at() {          // at the opening quote
    const char* s0 = ++p;
    const char* q = p;
    while (q < end && *q != '"' && *q != '\\') ++q;
    if (q < end && *q == '"') {                // no escapes: a view into the source
      p = q + 1;
      return std::string_view(s0, (size_t)(q - s0));
    }
    doc.escaped.emplace_back(s0, q);
    std::string& out = doc.escaped.back();
    p = q;
    for (;;) {
      if (p >= end) err("unterminated string");
      if (*p == '"') { ++p; return std::string_view(out); }
      if (*p == '\\') {
        ++p;
        if (p >= end) err("bad escape");
        const char c = *p++;
        out.push_back(c == 'n' ? '\n' : c == 't' ? '\t' : c);
        continue;
      }
      q = p;
      while (q < end && *q != '"' && *q != '\\') ++q;
      out.append(p, q);
      p = q;
    }
  }
  void number_into(Json& j) {
    j.kind = Json::NUM;
    const char* q = p;
    bool neg = false;
    if (q < end && *q == '-') { neg = true; ++q; }
    const char* d0 = q;
    long long v = 0;
    while (q < end && *q >= '0' && *q <= '9' && q - d0 < 18) v = v * 10 + (*q++ - '0');
    if (q > d0 && (q >= end || (*q != '.' && *q != 'e' && *q != 'E' && !(*q >= '0' && *q <= '9')))) {
      j.num = (double)(neg ? -v : v);      // plain integer (exact below 10^18)
      p = q;
      return;
    }
    char* r = nullptr;
    j.num = strtod(p, &r);
    if (r == p) err("bad value");
    p = r;
  }
  void close(Json& j, size_t mark, bool obj) {
    const size_t n = kid_stack.size() - mark;
    j.arr.n = (uint32_t)n;
    if (!n) return;
    const Json** kids = doc.alloc<const Json*>(n);
    std::copy(kid_stack.begin() + mark, kid_stack.end(), kids);
    j.arr.p = kids;
    kid_stack.resize(mark);
    if (obj) {
      std::string_view* ks = doc.alloc<std::string_view>(n);
      std::copy(key_stack.end() - n, key_stack.end(), ks);
      j.keys = ks;
      key_stack.resize(key_stack.size() - n);
    }
  }
  const Json* value() {
    ws();
    if (p >= end) err("unexpected end");
    doc.pool.emplace_back();
    Json& j = doc.pool.back();
    if (*p == '{') {
      j.kind = Json::OBJ;
      ++p;
      ws();
      const size_t mark = kid_stack.size();
      if (p < end && *p == '}') { ++p; return &j; }
      for (;;) {
        ws();
        if (p >= end || *p != '"') {
          if (p < end) value();                // a non-string key: parse it for the error position
          err("object key must be a string");
        }
        key_stack.push_back(string_view_at());
        ws();
        if (p >= end || *p != ':') err("expected ':'");
        ++p;
        kid_stack.push_back(value());
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == '}') { ++p; break; }
        err("expected ',' or '}'");
      }
      close(j, mark, true);
    } else if (*p == '[') {
      j.kind = Json::ARR;
      ++p;
      ws();
      const size_t mark = kid_stack.size();
      if (p < end && *p == ']') { ++p; return &j; }
      for (;;) {
        kid_stack.push_back(value());
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == ']') { ++p; break; }
        err("expected ',' or ']'");
      }
      close(j, mark, false);
    } else if (*p == '"') {
      j.kind = Json::STR;
      j.str = string_view_at();
    } else if (end - p >= 4 && !strncmp(p, "true", 4)) {
      j.kind = Json::BOOL; j.b = true; p += 4;
    } else if (end - p >= 5 && !strncmp(p, "false", 5)) {
      j.kind = Json::BOOL; j.b = false; p += 5;
    } else if (end - p >= 4 && !strncmp(p, "null", 4)) {
      j.kind = Json::NUL; p += 4;
    } else {
      number_into(j);
    }
    return &j;
  }
};

// The returned doc views `s`: keep the text alive while the doc (or anything pointing into it) is used.
std::unique_ptr<JsonDoc> parse_json(const char* s) {
  auto doc = std::make_unique<JsonDoc>();
  Parser ps{s, s + strlen(s), *doc, {}, {}};
  doc->root = ps.value();
  ps.ws();
  if (ps.p != ps.end) throw ParseError("json: trailing characters");
  return doc;
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o.push_back('\\');
    o.push_back(c);
  }
  return o + "\"";
}

// ============================================================================ graph model
enum Op {
  FC, MATMUL, BDOT, EMBED, SLICE, ADD, BADD, STACK, CONCAT, SUM, MUL, SIGMOID, TANH, RELU, DROPOUT, DOTLAST,
  MSOFTMAX, WSUM, CE, SOFTMAX, TO_HEADS, FROM_HEADS, CONV2D, GELU, SILU, SCALE, LAYERNORM, N_OPS
};
struct OpInfo {
  const char* name;
  int min_in, max_in, n_out;
  unsigned needs_in;   // bit k: gradient reads input k
  unsigned needs_out;  // bit k: gradient reads output k
};
const OpInfo OPS[N_OPS] = {
    {"fully_connected", 2, 3, 1, 0b11, 0}, {"matmul", 2, 2, 1, 0b11, 0},   {"batched_dot", 2, 2, 1, 0b11, 0},
    {"embedding", 2, 2, 1, 0b01, 0},       {"slice", 1, 1, 1, 0, 0},       {"add", 2, 2, 1, 0, 0},
    {"broadcast_add", 2, 2, 1, 0, 0},      {"stack", 1, 1 << 20, 1, 0, 0}, {"concat", 1, 1 << 20, 1, 0, 0},
    {"sum_reduce", 1, 1, 1, 0, 0},         {"mul", 2, 2, 1, 0b11, 0},      {"sigmoid", 1, 1, 1, 0, 0b1},
    {"tanh", 1, 1, 1, 0, 0b1},             {"relu", 1, 1, 1, 0, 0b1},      {"dropout", 1, 1, 2, 0, 0b10},
    {"dot_last", 2, 2, 1, 0b11, 0},        {"masked_softmax", 2, 2, 1, 0b10, 0b1},
    {"weighted_sum", 2, 2, 1, 0b11, 0},    {"softmax_ce_loss", 2, 2, 2, 0, 0b10},
    {"softmax", 1, 1, 1, 0, 0b1},          {"to_heads", 1, 1, 1, 0, 0},    {"from_heads", 1, 1, 1, 0, 0},
    {"conv2d", 2, 3, 1, 0b11, 0},          // like an FC: its gradient reads its input and weight (Eq. 2)
    {"gelu", 1, 1, 1, 0b1, 0},             // gelu'(x), silu'(x) are functions of x: the input is read
    {"silu", 1, 1, 1, 0b1, 0},
    {"scale", 1, 1, 1, 0, 0},              // y = c x (constant c): dx = c dy reads nothing
    {"layer_norm", 1, 3, 3, 0b1, 0b110},   // (y, mean, rstd): the gradient reads x and the row statistics
};

double dtype_width(const std::string& d) {
  if (d == "f32" || d == "i32") return 4;
  if (d == "bf16") return 2;
  if (d == "f64" || d == "i64") return 8;
  if (d == "u8") return 1;
  if (d == "bit") return 0.125;
  throw ParseError("unknown dtype " + d);
}
bool is_float(const std::string& d) { return d == "f32" || d == "bf16" || d == "f64"; }

struct Edge {
  int node, out;
  std::vector<int64_t> shape;
  std::string dtype;
  int64_t numel() const {
    int64_t n = 1;
    for (auto s : shape) n *= s;
    return n;
  }
  int64_t bytes(bool bit = false) const {
    if (bit) return (numel() + 7) / 8;
    return (int64_t)std::ceil((double)numel() * dtype_width(dtype));
  }
};

struct Node {
  int id;
  bool placeholder = false;
  bool trainable = false;
  int op = -1;
  std::string tag;
  std::vector<int> in;    // edge indices
  std::vector<int> out;   // edge indices
  const Json* attrs = nullptr;
};

struct Graph {
  std::vector<Node> nodes;           // by id (dense)
  std::vector<Edge> edges;
  std::vector<int> first_out;        // per node id: index of its output 0 (outputs are contiguous), -1 if none yet
  int edge_of(long long node, long long k) const {   // -1 if (node, k) is not an edge
    if (node < 0 || node >= (long long)first_out.size() || first_out[node] < 0 || k < 0) return -1;
    const Node& n = nodes[node];
    return k < (long long)n.out.size() ? n.out[k] : -1;
  }
  std::vector<int> order;            // non-placeholder node ids, ascending (topological)
  std::vector<int> outputs;          // edge indices
  std::vector<std::vector<int>> consumers;     // per edge: consumer node ids (with multiplicity per use)
  std::vector<std::vector<int>> grad_readers;  // per edge: nodes whose gradient reads it
  std::vector<int> stacked_into;     // per edge: stack output edge if this edge is a stack input, else -1
};

int64_t attr_int(const Node& n, const char* k, int64_t def) {
  if (!n.attrs) return def;
  const Json* v = n.attrs->get(k);
  return v && v->kind == Json::NUM ? v->i64() : def;
}
std::string attr_str(const Node& n, const char* k) {
  if (!n.attrs) return "";
  const Json* v = n.attrs->get(k);
  return v && v->kind == Json::STR ? std::string(v->str) : std::string();
}

void infer(Graph& g, Node& n) {
  const OpInfo& oi = OPS[n.op];
  std::vector<const Edge*> I;
  I.reserve(n.in.size());
  for (int e : n.in) I.push_back(&g.edges[e]);
  std::vector<std::vector<int64_t>> out;
  auto need = [&](bool ok, const char* what) {
    if (!ok) throw ParseError(std::string("shape error in node ") + std::to_string(n.id) + " (" + oi.name + "): " + what);
  };
  switch (n.op) {
    case FC: {
      need(!I[0]->shape.empty() && I[1]->shape.size() == 2 && I[0]->shape.back() == I[1]->shape[1], "X[...,in] W[out,in]");
      auto s = I[0]->shape;
      s.back() = I[1]->shape[0];
      out.push_back(s);
      break;
    }
    case MATMUL:
      need(I[0]->shape.size() == 2 && I[1]->shape.size() == 2 && I[0]->shape[1] == I[1]->shape[0], "[m,k]x[k,n]");
      out.push_back({I[0]->shape[0], I[1]->shape[1]});
      break;
    case BDOT: {
      const bool tb = attr_int(n, "trans_b", 0) != 0;
      need(I[0]->shape.size() == 3 && I[1]->shape.size() == 3 && I[0]->shape[2] == I[1]->shape[tb ? 2 : 1],
           "[b,m,k]x[b,k,n] (or [b,n,k] with trans_b)");
      out.push_back({I[0]->shape[0], I[0]->shape[1], I[1]->shape[tb ? 1 : 2]});
      break;
    }
    case SOFTMAX: out.push_back(I[0]->shape); break;
    case TO_HEADS: {
      const int64_t Bt = attr_int(n, "batch", 1), Hh = attr_int(n, "heads", 1);
      need(I[0]->shape.size() == 2 && Bt > 0 && Hh > 0 && I[0]->shape[0] % Bt == 0 && I[0]->shape[1] % Hh == 0, "[B*L, d]");
      out.push_back({Bt * Hh, I[0]->shape[0] / Bt, I[0]->shape[1] / Hh});
      break;
    }
    case FROM_HEADS: {
      const int64_t Hh = attr_int(n, "heads", 1);
      need(I[0]->shape.size() == 3 && Hh > 0 && I[0]->shape[0] % Hh == 0, "[B*H, L, dh]");
      out.push_back({I[0]->shape[0] / Hh * I[0]->shape[1], Hh * I[0]->shape[2]});
      break;
    }
    case CONV2D: {   // x [N,C,H,W], W [O,C,kh,kw] (+ bias [O]); attrs stride, padding (dilation 1, groups 1)
      need(I[0]->shape.size() == 4 && I[1]->shape.size() == 4 && I[0]->shape[1] == I[1]->shape[1], "x[N,C,H,W] W[O,C,kh,kw]");
      const int64_t st = attr_int(n, "stride", 1), pd = attr_int(n, "padding", 0);
      need(st > 0 && pd >= 0, "stride > 0, padding >= 0");
      const int64_t oh = (I[0]->shape[2] + 2 * pd - I[1]->shape[2]) / st + 1;
      const int64_t ow = (I[0]->shape[3] + 2 * pd - I[1]->shape[3]) / st + 1;
      need(oh > 0 && ow > 0, "output size");
      out.push_back({I[0]->shape[0], I[1]->shape[0], oh, ow});
      break;
    }
    case EMBED: {
      need(I[1]->shape.size() == 2, "table [V,E]");
      auto s = I[0]->shape;
      s.push_back(I[1]->shape[1]);
      out.push_back(s);
      break;
    }
    case SLICE: {
      auto s = I[0]->shape;
      int64_t ax = attr_int(n, "axis", 0);
      need(ax >= 0 && ax < (int64_t)s.size(), "axis");
      if (attr_int(n, "squeeze", 0)) s.erase(s.begin() + ax);
      else s[ax] = attr_int(n, "end", 0) - attr_int(n, "begin", 0);
      out.push_back(s);
      break;
    }
    case ADD: case MUL:
      need(I[0]->shape == I[1]->shape, "equal shapes");
      out.push_back(I[0]->shape);
      break;
    case SIGMOID: case TANH: case RELU: case GELU: case SILU: case SCALE: out.push_back(I[0]->shape); break;
    case LAYERNORM: {   // statistics over the last norm_ndim dims, one per row
      const int64_t k = attr_int(n, "norm_ndim", 1);
      need(k >= 1 && k <= (int64_t)I[0]->shape.size(), "norm_ndim");
      std::vector<int64_t> st(I[0]->shape.begin(), I[0]->shape.end() - k);
      st.insert(st.end(), (size_t)k, 1);
      out.push_back(I[0]->shape);
      out.push_back(st);
      out.push_back(st);
      break;
    }
    case DROPOUT: out.push_back(I[0]->shape); out.push_back(I[0]->shape); break;
    case BADD:
      need(I[1]->shape.size() == I[0]->shape.size() + 1 &&
               std::equal(I[0]->shape.begin(), I[0]->shape.end(), I[1]->shape.begin() + 1), "a[S] b[T,S]");
      out.push_back(I[1]->shape);
      break;
    case STACK: {
      for (auto* e : I) need(e->shape == I[0]->shape, "equal shapes");
      std::vector<int64_t> s{(int64_t)I.size()};
      s.insert(s.end(), I[0]->shape.begin(), I[0]->shape.end());
      out.push_back(s);
      break;
    }
    case CONCAT: {
      auto s = I[0]->shape;
      int64_t ax = attr_int(n, "axis", 0);
      need(ax >= 0 && ax < (int64_t)s.size(), "axis");
      s[ax] = 0;
      for (auto* e : I) s[ax] += e->shape[ax];
      out.push_back(s);
      break;
    }
    case SUM: out.push_back({}); break;
    case DOTLAST: {
      need(!I[0]->shape.empty() && I[1]->shape.size() == 1 && I[0]->shape.back() == I[1]->shape[0], "E[...,A] v[A]");
      auto s = I[0]->shape;
      s.pop_back();
      out.push_back(s);
      break;
    }
    case MSOFTMAX: out.push_back(I[0]->shape); break;
    case WSUM: {
      need(I[1]->shape.size() >= 2, "H[Ts,...]");
      out.push_back(std::vector<int64_t>(I[1]->shape.begin() + 1, I[1]->shape.end()));
      break;
    }
    case CE: out.push_back({}); out.push_back(I[0]->shape); break;
  }
  std::string dt = attr_str(n, "dtype");
  if (dt.empty()) dt = n.op == EMBED ? I[1]->dtype : I[0]->dtype;
  dtype_width(dt);
  for (size_t k = 0; k < out.size(); ++k) {
    std::string dk = n.op == CE ? std::string("f32") : (n.op == DROPOUT && k == 1 ? std::string("u8") : dt);
    if (n.op == LAYERNORM && k > 0 && I[0]->dtype == "bf16") dk = "f32";   // fp32 statistics for bf16 inputs
    Edge e{n.id, (int)k, out[k], dk};
    for (auto s : e.shape) need(s >= 1, "non-positive dim");
    if (k == 0) g.first_out[n.id] = (int)g.edges.size();
    n.out.push_back((int)g.edges.size());
    g.edges.push_back(std::move(e));
  }
}

Graph build_graph(const Json& doc) {
  Graph g;
  if (doc.kind != Json::OBJ) throw ParseError("graph: document must be an object");
  const Json* ver = doc.get("version");
  if (!ver || ver->i64() != 1) throw ParseError("graph: version must be 1");
  const Json* phs = doc.get("placeholders");
  const Json* nds = doc.get("nodes");
  const Json* outs = doc.get("outputs");
  if (!phs || !nds || !outs || phs->kind != Json::ARR || nds->kind != Json::ARR || outs->kind != Json::ARR)
    throw ParseError("graph: needs arrays 'placeholders', 'nodes', 'outputs'");
  const size_t N = phs->arr.size() + nds->arr.size();
  g.nodes.resize(N);
  g.first_out.assign(N, -1);
  std::vector<const Json*> def(N, nullptr);
  std::vector<char> isph(N, 0);
  for (auto& p : phs->arr) {
    const Json* id = p.get("id");
    if (!id || id->i64() < 0 || id->i64() >= (long long)N) throw ParseError("graph: placeholder id out of range");
    if (def[id->i64()]) throw ParseError("graph: duplicate id");
    def[id->i64()] = &p;
    isph[id->i64()] = 1;
  }
  for (auto& p : nds->arr) {
    const Json* id = p.get("id");
    if (!id || id->i64() < 0 || id->i64() >= (long long)N) throw ParseError("graph: node id out of range");
    if (def[id->i64()]) throw ParseError("graph: duplicate id");
    def[id->i64()] = &p;
  }
  for (size_t i = 0; i < N; ++i) {
    Node& n = g.nodes[i];
    n.id = (int)i;
    const Json& d = *def[i];
    const Json* tag = d.get("tag");
    n.tag = tag && tag->kind == Json::STR ? std::string(tag->str) : std::string();
    if (isph[i]) {
      n.placeholder = true;
      const Json* tr = d.get("trainable");
      n.trainable = tr && tr->kind == Json::BOOL && tr->b;
      const Json* sh = d.get("shape");
      const Json* dt = d.get("dtype");
      if (!sh || sh->kind != Json::ARR || !dt || dt->kind != Json::STR) throw ParseError("graph: placeholder needs shape, dtype");
      Edge e{(int)i, 0, {}, std::string(dt->str)};
      for (auto& s : sh->arr) {
        if (s.i64() < 1) throw ParseError("graph: non-positive dim");
        e.shape.push_back(s.i64());
      }
      dtype_width(e.dtype);
      g.first_out[i] = (int)g.edges.size();
      n.out.push_back((int)g.edges.size());
      g.edges.push_back(std::move(e));
      continue;
    }
    const Json* op = d.get("op");
    if (!op || op->kind != Json::STR) throw ParseError("graph: node needs 'op'");
    n.op = -1;
    static const std::vector<std::string_view> op_names = [] {
      std::vector<std::string_view> v;
      for (int k = 0; k < N_OPS; ++k) v.emplace_back(OPS[k].name);
      return v;
    }();
    for (int k = 0; k < N_OPS && n.op < 0; ++k)
      if (op->str == op_names[k]) n.op = k;
    if (n.op < 0) throw ParseError("graph: unknown op '" + std::string(op->str) + "'");
    const Json* ins = d.get("inputs");
    if (!ins || ins->kind != Json::ARR) throw ParseError("graph: node needs 'inputs'");
    if ((int)ins->arr.size() < OPS[n.op].min_in || (int)ins->arr.size() > OPS[n.op].max_in)
      throw ParseError("graph: arity mismatch for node " + std::to_string(i) + " (" + std::string(op->str) + ")");
    for (auto& r : ins->arr) {
      if (r.kind != Json::ARR || r.arr.size() != 2) throw ParseError("graph: input must be [node, out]");
      long long src = r.arr[0].i64(), k = r.arr[1].i64();
      if (src < 0 || src >= (long long)i) throw ParseError("graph: input must reference an earlier id (cycle or forward ref)");
      const int e = g.edge_of(src, k);
      if (e < 0) throw ParseError("graph: dangling edge reference");
      n.in.push_back(e);
    }
    const Json* at = d.get("attrs");
    n.attrs = at && at->kind == Json::OBJ ? at : nullptr;
    infer(g, n);
    g.order.push_back((int)i);
  }
  for (auto& o : outs->arr) {
    if (o.kind != Json::ARR || o.arr.size() != 2) throw ParseError("graph: output must be [node, out]");
    const int e = g.edge_of(o.arr[0].i64(), o.arr[1].i64());
    if (e < 0) throw ParseError("graph: dangling output");
    g.outputs.push_back(e);
  }
  g.consumers.assign(g.edges.size(), {});
  g.grad_readers.assign(g.edges.size(), {});
  g.stacked_into.assign(g.edges.size(), -1);
  for (int i : g.order) {
    const Node& n = g.nodes[i];
    for (int e : n.in) g.consumers[e].push_back(i);
    for (size_t k = 0; k < n.in.size(); ++k)
      if (k < 32 && (OPS[n.op].needs_in >> k) & 1u) g.grad_readers[n.in[k]].push_back(i);
    for (size_t k = 0; k < n.out.size(); ++k)
      if ((OPS[n.op].needs_out >> k) & 1u) g.grad_readers[n.out[k]].push_back(i);
    if (n.op == STACK)
      for (int e : n.in) g.stacked_into[e] = n.out[0];
  }
  return g;
}

// ============================================================================ strategy
struct Config {
  std::string kind = "echo";
  std::set<std::string> heavy{"fully_connected", "matmul", "batched_dot", "conv2d"};
  std::set<std::string> binarizable{"relu", "dropout"};
  bool dead = true, binarize = true;
  bool regen = false;          // counter-based dropout masks may be regenerated (reading R30)
  bool has_threshold = false;
  double threshold = 0;
  double weight_multiplier = 1;
  bool self_verify = false;    // check the plan is sufficient for the backward (ECHO_ERR_MISMATCH if not)
  int unstash_node = -1, unstash_out = 0;   // test hook: drop this edge from the plan before verifying
};

Config parse_config(const char* s) {
  Config c;
  if (!s) return c;
  auto doc = parse_json(s);
  const Json& j = *doc->root;
  if (j.kind != Json::OBJ) throw ParseError("config: must be an object");
  // strict schema: an unknown key or a value of the wrong kind is an error, not silently ignored
  static const char* const kKeys[] = {"strategy", "compute_heavy_ops", "binarizable_ops", "enable_dead_node",
                                      "enable_binarization", "regenerate_masks", "flop_threshold",
                                      "weight_multiplier", "self_verify", "debug_unstash_edge"};
  for (uint32_t i = 0; i < j.arr.n; ++i) {
    bool known = false;
    for (const char* k : kKeys) known = known || j.keys[i] == k;
    if (!known) throw ParseError("config: unknown key '" + std::string(j.keys[i]) + "'");
  }
  auto kind_of = [&](const char* k, Json::Kind want, const char* what) {
    const Json* v = j.get(k);
    if (v && v->kind != want) throw ParseError(std::string("config: ") + k + " must be " + what);
    return v;
  };
  for (const char* k : {"enable_dead_node", "enable_binarization", "regenerate_masks", "self_verify"})
    kind_of(k, Json::BOOL, "a boolean");
  for (const char* k : {"compute_heavy_ops", "binarizable_ops"}) {
    if (const Json* v = kind_of(k, Json::ARR, "an array of op names"))
      for (auto& x : v->arr)
        if (x.kind != Json::STR) throw ParseError(std::string("config: ") + k + " must be an array of op names");
  }
  kind_of("strategy", Json::STR, "a string");
  kind_of("flop_threshold", Json::NUM, "a number");
  kind_of("weight_multiplier", Json::NUM, "a number");
  kind_of("debug_unstash_edge", Json::ARR, "[node, out]");
  if (auto* v = j.get("strategy")) c.kind = std::string(v->str);
  if (c.kind != "echo" && c.kind != "mirror" && c.kind != "baseline") throw ParseError("config: bad strategy");
  if (auto* v = j.get("compute_heavy_ops")) {
    c.heavy.clear();
    for (auto& x : v->arr) c.heavy.insert(std::string(x.str));
  }
  if (auto* v = j.get("binarizable_ops")) {
    c.binarizable.clear();
    for (auto& x : v->arr) c.binarizable.insert(std::string(x.str));
  }
  if (auto* v = j.get("enable_dead_node")) c.dead = v->b;
  if (auto* v = j.get("enable_binarization")) c.binarize = v->b;
  if (auto* v = j.get("regenerate_masks")) c.regen = v->b;
  if (auto* v = j.get("self_verify")) c.self_verify = v->b;
  if (auto* v = j.get("debug_unstash_edge"))                 // [node, out]: a corrupted plan (negative control)
    if (v->kind == Json::ARR && v->arr.size() == 2) {
      c.unstash_node = (int)v->arr[0].i64();
      c.unstash_out = (int)v->arr[1].i64();
      c.self_verify = true;
    }
  if (auto* v = j.get("flop_threshold"))
    if (v->kind == Json::NUM) { c.has_threshold = true; c.threshold = v->num; }
  if (auto* v = j.get("weight_multiplier"))
    if (v->kind == Json::NUM) c.weight_multiplier = v->num;
  if (c.kind != "echo") {
    c.dead = false;
    if (c.kind == "baseline") c.binarize = c.regen = false;
  }
  return c;
}

int64_t flops(const Graph& g, const Node& n) {
  auto E = [&](int k) -> const Edge& { return g.edges[n.in[k]]; };
  const Edge& o = g.edges[n.out[0]];
  switch (n.op) {
    case FC: return 2 * o.numel() * E(0).shape.back();
    case CONV2D: return 2 * o.numel() * E(1).shape[1] * E(1).shape[2] * E(1).shape[3];
    case MATMUL: return 2 * E(0).shape[0] * E(0).shape[1] * E(1).shape[1];
    case BDOT: return 2 * E(0).shape[0] * E(0).shape[1] * E(0).shape[2] * (o.numel() / (E(0).shape[0] * E(0).shape[1]));
    case DOTLAST: return 2 * E(0).numel();
    case WSUM: return 2 * E(1).numel();
    case DROPOUT: return 2 * o.numel();
    case LAYERNORM: return 5 * o.numel();
    case SUM: return E(0).numel();
    default: return o.numel();
  }
}

struct Analysis {
  const Graph& g;
  const Config& cfg;
  std::vector<char> heavy, binz, mirrored, heavy_orig;
  explicit Analysis(const Graph& gr, const Config& c) : g(gr), cfg(c) {
    const size_t N = g.nodes.size();
    heavy.assign(N, 0);
    binz.assign(N, 0);
    mirrored.assign(N, 0);
    heavy_orig.assign(N, 0);
    for (int i : g.order) {
      const Node& n = g.nodes[i];
      bool h = cfg.heavy.count(OPS[n.op].name) > 0;
      if (h && cfg.has_threshold) h = (double)flops(g, n) / (double)std::max<int64_t>(1, g.edges[n.out[0]].numel()) > cfg.threshold;
      heavy[i] = h;
      binz[i] = cfg.binarizable.count(OPS[n.op].name) > 0;
      heavy_orig[i] = h && !cfg.dead;
    }
  }
  bool trainable(int e) const {
    const Node& p = g.nodes[g.edges[e].node];
    return p.placeholder && p.trainable;
  }
  // dropout's keep-mask: random state, never recomputed from the dropout's input (reading R26)
  bool is_random(int e) const {
    const Node& p = g.nodes[g.edges[e].node];
    return !p.placeholder && p.op == DROPOUT && g.edges[e].out == 1;
  }
  // 0: not stashed, 1: stashed at full precision, 2: stashed as a 1-bit mask
  int status(int e) const {
    if (trainable(e)) return 0;
    const int p = g.edges[e].node;
    const bool pm = mirrored[p];
    const bool rnd = is_random(e);
    if (rnd && cfg.regen) return 0;                          // R30: regenerated from (seed, counter)
    int st = 0;
    for (int r : g.grad_readers[e]) {
      if (pm && !heavy_orig[r] && !rnd) continue;            // gradient reads the recomputed copy
      const bool bit = cfg.binarize && (rnd || (p == r && !mirrored[r] && binz[r]));
      if (!bit) return 1;
      st = 2;
    }
    if (!pm)
      for (int c : g.consumers[e])
        if (mirrored[c]) return 1;                           // needed to recompute c
    if (rnd && pm) {                                         // a mirrored dropout re-applies its mask
      if (!cfg.binarize) return 1;
      st = 2;
    }
    return st;
  }
  int64_t status_bytes(int e, int st) const { return st == 0 ? 0 : g.edges[e].bytes(st == 2); }
  bool needed_in_backward(int e) const {
    for (int r : g.grad_readers[e])
      if (!heavy_orig[r]) return true;
    for (int c : g.consumers[e])
      if (mirrored[c]) return true;
    return false;
  }
};

std::vector<std::vector<int>> partition(const Graph& g, const Analysis& a) {
  std::vector<int> H;
  for (int e : g.outputs) {
    int n = g.edges[e].node;
    if (std::find(H.begin(), H.end(), n) == H.end()) H.push_back(n);
  }
  std::vector<char> claimed(g.nodes.size(), 0);
  std::vector<std::vector<int>> subs;
  while (!H.empty()) {
    int h = H.back();
    H.pop_back();
    if (g.nodes[h].placeholder || claimed[h]) continue;
    std::vector<int> S{h};
    claimed[h] = 1;
    std::vector<int> W;
    for (int e : g.nodes[h].in) W.push_back(g.edges[e].node);
    while (!W.empty()) {
      int w = W.back();
      W.pop_back();
      if (g.nodes[w].placeholder || claimed[w]) continue;
      if (a.heavy[w]) { H.push_back(w); continue; }
      S.push_back(w);
      claimed[w] = 1;
      for (int e : g.nodes[w].in) W.push_back(g.edges[e].node);
    }
    std::sort(S.begin(), S.end());
    subs.push_back(S);
  }
  return subs;
}

void dead_node_elimination(const Graph& g, Analysis& a) {
  bool changed = true;
  while (changed) {
    changed = false;
    for (auto it = g.order.rbegin(); it != g.order.rend(); ++it) {
      int m = *it;
      if (!a.mirrored[m]) continue;
      bool need = false;
      for (int e : g.nodes[m].out) need = need || (!a.is_random(e) && a.needed_in_backward(e));
      if (!need) { a.mirrored[m] = 0; changed = true; }
    }
  }
}

struct Result {
  std::vector<std::vector<int>> subs;
  std::vector<int> dead;
};

Result run_echo(const Graph& g, Analysis& a) {
  Result r;
  r.subs = partition(g, a);
  for (auto& S : r.subs)
    for (int s : S)
      if (!a.heavy[s]) a.mirrored[s] = 1;                         // binarizable nodes included (line 18)
  std::vector<int> mark(g.edges.size(), 0), gmark(g.nodes.size(), 0);
  int stamp = 0;
  for (auto& S : r.subs) {
    for (int s : S) {
      if (!a.mirrored[s] || a.binz[s]) continue;                  // Alg. 1 line 18: binarizable -> continue
      ++stamp;
      std::vector<int> group{s};
      gmark[s] = stamp;
      for (size_t k = 0; k < group.size(); ++k) {                 // closure over shared stashed inputs
        for (int e : g.nodes[group[k]].in) {
          if (a.status(e) == 0) continue;
          for (int c : g.consumers[e])
            if (a.mirrored[c] && !a.binz[c] && gmark[c] != stamp) { gmark[c] = stamp; group.push_back(c); }
        }
      }
      std::vector<int> aff;                                       // edges whose status can change
      for (int m : group) {
        for (int e : g.nodes[m].in) if (mark[e] != stamp) { mark[e] = stamp; aff.push_back(e); }
        for (int e : g.nodes[m].out) if (mark[e] != stamp) { mark[e] = stamp; aff.push_back(e); }
      }
      std::vector<int64_t> before(aff.size());
      for (size_t k = 0; k < aff.size(); ++k) before[k] = a.status_bytes(aff[k], a.status(aff[k]));
      for (int m : group) a.mirrored[m] = 0;
      int64_t rel = 0, alloc = 0;
      for (size_t k = 0; k < aff.size(); ++k) {
        const int64_t after = a.status_bytes(aff[k], a.status(aff[k]));
        if (before[k] > after) rel += before[k] - after;
        else alloc += after - before[k];
      }
      if (!(rel >= alloc))
        for (int m : group) a.mirrored[m] = 1;                    // keep the group on the mirror path
    }
  }
  dead_node_elimination(g, a);
  for (auto& S : r.subs)
    for (int i : S) {
      const Node& n = g.nodes[i];
      if (!a.heavy[i] || !a.cfg.dead || OPS[n.op].needs_out) continue;
      bool any = false;
      for (int e : n.in) any = any || a.mirrored[g.edges[e].node];
      if (any) r.dead.push_back(i);
    }
  return r;
}

void run_mirror(const Graph& g, Analysis& a) {
  for (int i : g.order)
    if (!a.heavy[i]) a.mirrored[i] = 1;
  dead_node_elimination(g, a);
}

// ============================================================================ liveness planning
struct Plan {
  std::vector<int64_t> timeline;
  int64_t peak = 0;
  int peak_step = 0;
};

Plan plan(const Graph& g, const Analysis& a, const std::vector<int>& st) {
  const int F = (int)g.order.size();
  std::vector<int> fwd_pos(g.nodes.size(), -1), grad_pos(g.nodes.size(), -1), mir_pos(g.nodes.size(), -1);
  for (int k = 0; k < F; ++k) fwd_pos[g.order[k]] = k;
  int step = F;
  std::vector<char> done(g.nodes.size(), 0);
  for (int k = F - 1; k >= 0; --k) {
    const int i = g.order[k];
    const Node& n = g.nodes[i];
    if (!a.heavy_orig[i]) {
      std::vector<int> need, stack;
      std::vector<char> seen(0);
      std::set<int> seen_s;
      for (size_t q = 0; q < n.in.size(); ++q)
        if (q < 32 && (OPS[n.op].needs_in >> q) & 1u && !a.is_random(n.in[q])) stack.push_back(g.edges[n.in[q]].node);
      for (size_t q = 0; q < n.out.size(); ++q)
        if ((OPS[n.op].needs_out >> q) & 1u && !a.is_random(n.out[q])) stack.push_back(i);
      while (!stack.empty()) {
        int m = stack.back();
        stack.pop_back();
        if (!a.mirrored[m] || done[m] || seen_s.count(m)) continue;
        seen_s.insert(m);
        need.push_back(m);
        for (int e : g.nodes[m].in) stack.push_back(g.edges[e].node);
      }
      std::sort(need.begin(), need.end());
      for (int m : need) { mir_pos[m] = step++; done[m] = 1; }
    }
    grad_pos[i] = step++;
  }
  const int T = step;
  std::vector<int64_t> diff(T + 1, 0);
  auto add = [&](int s, int e, int64_t b) { diff[s] += b; diff[e + 1] -= b; };
  // forward outputs; stack inputs live inside the stack's buffer
  std::vector<int> lo(g.edges.size(), -1), hi(g.edges.size(), -1);
  for (int i : g.order) {
    for (int e : g.nodes[i].out) {
      int last = fwd_pos[i];
      for (int c : g.consumers[e]) last = std::max(last, fwd_pos[c]);
      if (st[e]) {
        const bool rnd = a.is_random(e);
        for (int r : g.grad_readers[e])
          if (!a.mirrored[g.edges[e].node] || a.heavy_orig[r] || rnd) last = std::max(last, grad_pos[r]);
        for (int c : g.consumers[e])
          if (a.mirrored[c]) last = std::max(last, mir_pos[c]);
        if (rnd && a.mirrored[i]) last = std::max(last, mir_pos[i]);
      }
      lo[e] = fwd_pos[i];
      hi[e] = last;
    }
  }
  for (size_t e = 0; e < g.edges.size(); ++e) {
    int r = g.stacked_into[e];
    if (r >= 0 && lo[e] >= 0) { lo[r] = std::min(lo[r], lo[e]); hi[r] = std::max(hi[r], hi[e]); }
  }
  for (size_t e = 0; e < g.edges.size(); ++e)
    if (lo[e] >= 0 && g.stacked_into[e] < 0) add(lo[e], hi[e], g.edges[e].bytes(st[e] == 2));
  // recomputed outputs
  for (int m : g.order) {
    if (!a.mirrored[m]) continue;
    for (int e : g.nodes[m].out) {
      if (a.is_random(e)) continue;
      int last = -1;
      for (int r : g.grad_readers[e]) if (!a.heavy_orig[r]) last = std::max(last, grad_pos[r]);
      for (int c : g.consumers[e]) if (a.mirrored[c]) last = std::max(last, mir_pos[c]);
      if (last >= 0) add(mir_pos[m], last, g.edges[e].bytes());
    }
  }
  // gradients of float activations
  std::vector<char> is_out(g.edges.size(), 0);
  for (int e : g.outputs) is_out[e] = 1;
  for (int i : g.order)
    for (int e : g.nodes[i].out) {
      if (!is_float(g.edges[e].dtype)) continue;
      int first = INT32_MAX;
      for (int c : g.consumers[e]) first = std::min(first, grad_pos[c]);
      if (is_out[e]) first = std::min(first, F);
      if (first == INT32_MAX) continue;
      add(first, grad_pos[i], g.edges[e].bytes());
    }
  Plan p;
  int64_t cur = 0;
  for (int k = 0; k < T; ++k) {
    cur += diff[k];
    p.timeline.push_back(cur);
    if (cur > p.peak) { p.peak = cur; p.peak_step = k; }
  }
  return p;
}

// ============================================================================ plan self-check
struct MismatchError : std::runtime_error {
  explicit MismatchError(const std::string& s) : std::runtime_error(s) {}
};

// The plan is sufficient iff every forward edge a gradient step reads can be produced in the backward:
// a weight; stashed at full precision (or inside a stashed stack); or regenerated by its mirrored
// producer from inputs that are themselves available (a mirrored dropout also needs its mask).  A heavy
// op that reads its ORIGINAL inputs (dead mirrors disabled) needs them stashed; a binarizable op that is
// not mirrored may read its own output as a 1-bit mask; a keep-mask may be kept as bits or (R30)
// regenerated from its Philox counter.  (SPEC.md:632-639 `verify`, here as a structural check.)
void verify_plan(const Graph& g, const Analysis& a, const std::vector<int>& st) {
  std::vector<signed char> memo(g.edges.size(), -1);
  auto mask_ok = [&](int e) { return st[e] != 0 || a.cfg.regen; };
  std::function<bool(int)> full = [&](int e) -> bool {
    if (memo[e] >= 0) return memo[e];
    memo[e] = 0;                                             // (a cycle cannot occur: ids are topological)
    bool ok = a.trainable(e) || st[e] == 1 || (g.stacked_into[e] >= 0 && st[g.stacked_into[e]] == 1);
    const int p = g.edges[e].node;
    if (!ok && !g.nodes[p].placeholder && a.mirrored[p] && !a.is_random(e)) {
      ok = true;
      for (int q : g.nodes[p].in) ok = ok && full(q);
      if (ok && g.nodes[p].op == DROPOUT) ok = mask_ok(g.nodes[p].out[1]);
    }
    memo[e] = ok;
    return ok;
  };
  auto fail_at = [&](int r, int e, const char* why) {
    throw MismatchError("plan self-check: gradient of node " + std::to_string(r) + " (" + OPS[g.nodes[r].op].name +
                        ") reads edge [" + std::to_string(g.edges[e].node) + "," + std::to_string(g.edges[e].out) +
                        "], " + why);
  };
  for (int r : g.order) {
    const Node& n = g.nodes[r];
    std::vector<int> refs;
    for (size_t k = 0; k < n.in.size(); ++k)
      if (k < 32 && (OPS[n.op].needs_in >> k) & 1u) refs.push_back(n.in[k]);
    for (size_t k = 0; k < n.out.size(); ++k)
      if ((OPS[n.op].needs_out >> k) & 1u) refs.push_back(n.out[k]);
    for (int e : refs) {
      if (a.trainable(e)) continue;
      if (a.is_random(e)) {
        if (!mask_ok(e)) fail_at(r, e, "a keep-mask that is neither kept nor regenerable");
      } else if (a.heavy_orig[r]) {
        if (!(st[e] == 1 || (g.stacked_into[e] >= 0 && st[g.stacked_into[e]] == 1)))
          fail_at(r, e, "an original input that is not kept");
      } else if (g.edges[e].node == r && a.binz[r] && !a.mirrored[r]) {
        if (st[e] == 0) fail_at(r, e, "its own output, kept neither as bits nor in full");
      } else if (!full(e)) {
        fail_at(r, e, "which is neither kept nor regenerable from kept edges");
      }
    }
  }
}

std::string analyze(const char* graph_json, const char* config_json) {
  auto doc = parse_json(graph_json);
  Graph g = build_graph(*doc->root);
  Config cfg = parse_config(config_json);
  Analysis a(g, cfg);
  Result r;
  if (cfg.kind == "echo") r = run_echo(g, a);
  else if (cfg.kind == "mirror") run_mirror(g, a);
  std::vector<int> st(g.edges.size(), 0);
  for (size_t e = 0; e < g.edges.size(); ++e) st[e] = a.status((int)e);
  if (cfg.unstash_node >= 0) {
    const int e = g.edge_of(cfg.unstash_node, cfg.unstash_out);
    if (e < 0) throw ParseError("config: debug_unstash_edge is not an edge");
    st[e] = 0;
  }
  if (cfg.self_verify) verify_plan(g, a, st);
  // stash bytes (a stashed stack output covers its view inputs)
  int64_t stash = 0, weights = 0;
  std::map<std::string, int64_t> by_tag;
  for (size_t e = 0; e < g.edges.size(); ++e) {
    if (!st[e]) continue;
    int root = g.stacked_into[e];
    if (root >= 0 && st[root]) continue;
    int64_t b = g.edges[e].bytes(st[e] == 2);
    stash += b;
    by_tag[g.nodes[g.edges[e].node].tag] += b;
  }
  for (auto& n : g.nodes)
    if (n.placeholder && n.trainable) weights += g.edges[n.out[0]].bytes();
  int64_t rflops = 0;
  int n_mirror = 0;
  for (int i : g.order)
    if (a.mirrored[i]) { rflops += flops(g, g.nodes[i]); ++n_mirror; }
  Plan p = plan(g, a, st);
  size_t maxsub = 0;
  for (auto& S : r.subs) maxsub = std::max(maxsub, S.size());
  std::string o = "{";
  o += "\"strategy\":" + jstr(cfg.kind);
  o += ",\"nodes\":" + std::to_string(g.order.size());
  o += ",\"edges\":" + std::to_string(g.edges.size());
  o += ",\"stash_bytes\":" + std::to_string(stash);
  o += ",\"weight_bytes\":" + std::to_string((int64_t)std::llround(weights * cfg.weight_multiplier));
  o += ",\"peak_bytes\":" + std::to_string(p.peak);
  o += ",\"peak_step\":" + std::to_string(p.peak_step);
  o += ",\"steps\":" + std::to_string(p.timeline.size());
  o += ",\"mirrored\":" + std::to_string(n_mirror);
  o += ",\"dead_mirrors\":" + std::to_string(r.dead.size());
  o += ",\"subgraphs\":" + std::to_string(r.subs.size());
  o += ",\"max_subgraph\":" + std::to_string(maxsub);
  o += ",\"recompute_flops\":" + std::to_string(rflops);
  o += ",\"by_tag\":{";
  bool first = true;
  for (auto& kv : by_tag) {
    if (!first) o += ",";
    first = false;
    o += jstr(kv.first) + ":" + std::to_string(kv.second);
  }
  o += "},\"decisions\":[";
  first = true;
  for (size_t e = 0; e < g.edges.size(); ++e) {
    const char* d = nullptr;
    if (st[e] == 1) d = "stash";
    else if (st[e] == 2) d = "bit";
    else if (a.mirrored[g.edges[e].node] && a.needed_in_backward((int)e)) d = "recompute";
    if (!d) continue;
    if (!first) o += ",";
    first = false;
    o += "[" + std::to_string(g.edges[e].node) + "," + std::to_string(g.edges[e].out) + ",\"" + d + "\"]";
  }
  o += "],\"dead\":[";
  for (size_t k = 0; k < r.dead.size(); ++k) o += (k ? "," : "") + std::to_string(r.dead[k]);
  o += "],\"timeline\":[";
  for (size_t k = 0; k < p.timeline.size(); ++k) o += (k ? "," : "") + std::to_string(p.timeline[k]);
  o += "]}";
  return o;
}

}  // namespace

extern "C" echo_status echo_footprint_estimate(const char* graph_json, const char* config_json, char* report_json,
                                               size_t* report_len) {
  if (!graph_json || !report_len) return echo::fail(ECHO_ERR_INVALID, "echo_footprint_estimate: NULL argument");
  std::string rep;
  try {
    rep = analyze(graph_json, config_json);
  } catch (const MismatchError& e) {
    return echo::fail(ECHO_ERR_MISMATCH, "echo_footprint_estimate: %s", e.what());
  } catch (const ParseError& e) {
    return echo::fail(ECHO_ERR_INVALID, "echo_footprint_estimate: %s", e.what());
  } catch (const std::exception& e) {
    return echo::fail(ECHO_ERR_GRAPH, "echo_footprint_estimate: %s", e.what());
  }
  const size_t need = rep.size() + 1;
  if (!report_json || *report_len < need) {
    *report_len = need;
    return report_json ? echo::fail(ECHO_ERR_CAPACITY, "echo_footprint_estimate: report needs %zu bytes", need) : ECHO_OK;
  }
  memcpy(report_json, rep.c_str(), need);
  *report_len = need;
  return ECHO_OK;
}
