// ompds_manifest.cpp -- the manifest JSON of the reference compiler
// (proj/src/Compiler.cpp:112-155, manifestJson): the kernel frame group's
// depot layout with its shared-memory footprint, the descriptor export a
// tool chain reads back.  The writer reproduces the reference text byte for
// byte (nlohmann::json::dump(2) of an object with sorted keys, plus "\n");
// the reader accepts any JSON with the same fields and checks the
// reference's size laws.  No JSON library: the schema is fixed and small.
#include "../../include/ompds.h"

#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// Writer
// ---------------------------------------------------------------------------

// JSON string escaping as nlohmann's dump (UTF-8 passed through).
void put_string(std::string &o, const char *s) {
  o += '"';
  for (const unsigned char *p = reinterpret_cast<const unsigned char *>(s); *p; ++p) {
    switch (*p) {
    case '"': o += "\\\""; break;
    case '\\': o += "\\\\"; break;
    case '\b': o += "\\b"; break;
    case '\f': o += "\\f"; break;
    case '\n': o += "\\n"; break;
    case '\r': o += "\\r"; break;
    case '\t': o += "\\t"; break;
    default:
      if (*p < 0x20) {
        char buf[8];
        std::snprintf(buf, sizeof buf, "\\u%04x", *p);
        o += buf;
      } else {
        o += static_cast<char>(*p);
      }
    }
  }
  o += '"';
}

// Emits one object level: `fields` are written in the order given, which the
// callers keep sorted (nlohmann objects are std::map-ordered).
struct Writer {
  std::string out;
  void indent(int n) { out.append(static_cast<size_t>(n), ' '); }
  void key(int depth, const char *k, bool first) {
    if (!first)
      out += ",\n";
    indent(2 * depth);
    put_string(out, k);
    out += ": ";
  }
  void num(int64_t v) { out += std::to_string(v); }
  void boolean(bool v) { out += v ? "true" : "false"; }
};

// ---------------------------------------------------------------------------
// Reader: a small recursive-descent JSON parser into a tree.
// ---------------------------------------------------------------------------

struct Node {
  enum Kind { Null, Bool, Int, Str, Arr, Obj } kind = Null;
  bool b = false;
  int64_t i = 0;
  std::string s;
  std::vector<std::unique_ptr<Node>> items;             // Arr
  std::map<std::string, std::unique_ptr<Node>> fields;  // Obj
  const Node *get(const char *k) const {
    auto it = fields.find(k);
    return it == fields.end() ? nullptr : it->second.get();
  }
};

struct Parser {
  const char *p, *end;
  int depth = 0;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t'))
      ++p;
  }
  bool lit(const char *w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(end - p) < n || std::strncmp(p, w, n) != 0)
      return false;
    p += n;
    return true;
  }
  bool str(std::string &o) {
    if (p >= end || *p != '"')
      return false;
    ++p;
    while (p < end && *p != '"') {
      unsigned char c = static_cast<unsigned char>(*p++);
      if (c < 0x20)
        return false;
      if (c != '\\') {
        o += static_cast<char>(c);
        continue;
      }
      if (p >= end)
        return false;
      switch (*p++) {
      case '"': o += '"'; break;
      case '\\': o += '\\'; break;
      case '/': o += '/'; break;
      case 'b': o += '\b'; break;
      case 'f': o += '\f'; break;
      case 'n': o += '\n'; break;
      case 'r': o += '\r'; break;
      case 't': o += '\t'; break;
      case 'u': {
        if (end - p < 4)
          return false;
        unsigned v = 0;
        for (int k = 0; k < 4; ++k) {
          const char h = *p++;
          v = v * 16 + (h >= '0' && h <= '9'   ? unsigned(h - '0')
                        : h >= 'a' && h <= 'f' ? unsigned(h - 'a' + 10)
                        : h >= 'A' && h <= 'F' ? unsigned(h - 'A' + 10)
                                               : 99u);
          if (v >= 0x10000)
            return false;
        }
        if (v < 0x80) { // manifest names are identifiers; keep ASCII escapes
          o += static_cast<char>(v);
        } else if (v < 0x800) {
          o += static_cast<char>(0xC0 | (v >> 6));
          o += static_cast<char>(0x80 | (v & 0x3F));
        } else {
          o += static_cast<char>(0xE0 | (v >> 12));
          o += static_cast<char>(0x80 | ((v >> 6) & 0x3F));
          o += static_cast<char>(0x80 | (v & 0x3F));
        }
        break;
      }
      default: return false;
      }
    }
    if (p >= end)
      return false;
    ++p;
    return true;
  }
  bool value(Node &n) {
    if (++depth > 64)
      return false;
    ws();
    bool ok = false;
    if (p >= end) {
      ok = false;
    } else if (*p == '{') {
      ++p;
      n.kind = Node::Obj;
      ws();
      if (p < end && *p == '}') {
        ++p;
        ok = true;
      } else {
        for (;;) {
          ws();
          std::string k;
          if (!str(k))
            break;
          ws();
          if (p >= end || *p != ':')
            break;
          ++p;
          auto child = std::make_unique<Node>();
          if (!value(*child) || n.fields.count(k))
            break;
          n.fields.emplace(std::move(k), std::move(child));
          ws();
          if (p < end && *p == ',') {
            ++p;
            continue;
          }
          if (p < end && *p == '}') {
            ++p;
            ok = true;
          }
          break;
        }
      }
    } else if (*p == '[') {
      ++p;
      n.kind = Node::Arr;
      ws();
      if (p < end && *p == ']') {
        ++p;
        ok = true;
      } else {
        for (;;) {
          auto child = std::make_unique<Node>();
          if (!value(*child))
            break;
          n.items.push_back(std::move(child));
          ws();
          if (p < end && *p == ',') {
            ++p;
            continue;
          }
          if (p < end && *p == ']') {
            ++p;
            ok = true;
          }
          break;
        }
      }
    } else if (*p == '"') {
      n.kind = Node::Str;
      ok = str(n.s);
    } else if (lit("true")) {
      n.kind = Node::Bool;
      n.b = true;
      ok = true;
    } else if (lit("false")) {
      n.kind = Node::Bool;
      ok = true;
    } else if (lit("null")) {
      ok = true;
    } else if (*p == '-' || (*p >= '0' && *p <= '9')) {
      // integers only: every manifest number is a byte count or a count
      n.kind = Node::Int;
      const bool neg = *p == '-';
      if (neg)
        ++p;
      int digits = 0;
      uint64_t v = 0;
      while (p < end && *p >= '0' && *p <= '9' && digits < 19) {
        v = v * 10 + uint64_t(*p++ - '0');
        ++digits;
      }
      ok = digits > 0 && !(p < end && (*p == '.' || *p == 'e' || *p == 'E' ||
                                      (*p >= '0' && *p <= '9')));
      n.i = neg ? -static_cast<int64_t>(v) : static_cast<int64_t>(v);
    }
    --depth;
    return ok;
  }
};

bool int_field(const Node *o, const char *k, int64_t *out) {
  const Node *n = o ? o->get(k) : nullptr;
  if (!n || n->kind != Node::Int)
    return false;
  *out = n->i;
  return true;
}

} // namespace

extern "C" {

int32_t ompds_manifest_write(const ompds_manifest *m, char *out, int64_t cap, int64_t *len) {
  if (!m || !len || cap < 0 || (cap > 0 && !out) || m->prealloc_entries < 0 ||
      (m->has_layout && (!m->layout || (m->layout->n_slots > 0 && (!m->slots || !m->owners ||
                                                                   !m->var_names)))))
    return OMPDS_ERR_INVALID;
  const ompds_depot_layout *L = m->has_layout ? m->layout : nullptr;
  const int64_t total_local = L ? L->total_local : 0;
  const int64_t total_shared = L ? L->total_shared : 0;
  const int64_t prealloc_bytes = int64_t(m->prealloc_entries) * OMPDS_SHARED_ARG_ENTRY_BYTES;
  Writer w;
  w.out += "{\n";
  w.key(1, "depot", true);
  w.out += "{\n";
  w.key(2, "mirrored", true);
  w.boolean(L && L->has_shared_depot);
  w.key(2, "slots", false);
  if (!L || L->n_slots == 0) {
    w.out += "[]";
  } else {
    w.out += "[\n";
    for (int32_t k = 0; k < L->n_slots; ++k) {
      const ompds_depot_slot &S = m->slots[L->slot_begin + k];
      if (k)
        w.out += ",\n";
      w.indent(6);
      w.out += "{\n";
      w.key(4, "align", true);
      w.num(S.align);
      w.key(4, "offset", false);
      w.num(S.offset);
      w.key(4, "owners", false);
      if (S.n_owners == 0) {
        w.out += "[]";
      } else {
        w.out += "[\n";
        for (int32_t j = 0; j < S.n_owners; ++j) {
          if (j)
            w.out += ",\n";
          w.indent(10);
          const char *name = m->var_names[m->owners[S.owner_begin + j]];
          put_string(w.out, name ? name : "");
        }
        w.out += "\n";
        w.indent(8);
        w.out += "]";
      }
      w.key(4, "shared", false);
      w.boolean(S.shared != 0);
      w.key(4, "size", false);
      w.num(S.size);
      w.out += "\n";
      w.indent(6);
      w.out += "}";
    }
    w.out += "\n";
    w.indent(4);
    w.out += "]";
  }
  w.key(2, "total_local", false);
  w.num(total_local);
  w.key(2, "total_shared", false);
  w.num(total_shared);
  w.out += "\n  }";
  w.key(1, "kernel", false);
  put_string(w.out, m->kernel ? m->kernel : "");
  w.key(1, "launch", false);
  w.out += "{\n";
  w.key(2, "teams", true);
  w.num(m->teams);
  w.key(2, "workers", false);
  w.num(m->workers);
  w.out += "\n  }";
  w.key(1, "prealloc_bytes", false);
  w.num(prealloc_bytes);
  w.key(1, "prealloc_entries", false);
  w.num(m->prealloc_entries);
  w.key(1, "runtime_bytes", false);
  w.num(OMPDS_RUNTIME_PRIVATE_BYTES);
  w.key(1, "shared_footprint", false);
  w.num(total_shared + prealloc_bytes + OMPDS_RUNTIME_PRIVATE_BYTES);
  w.key(1, "stack_bytes", false);
  w.num(total_local);
  w.out += "\n}\n";
  *len = static_cast<int64_t>(w.out.size());
  if (cap <= *len)
    return OMPDS_ERR_CAPACITY;
  std::memcpy(out, w.out.data(), w.out.size());
  out[w.out.size()] = '\0';
  return OMPDS_OK;
}

int32_t ompds_manifest_parse(const char *text, int64_t len, ompds_manifest_info *info,
                             ompds_depot_slot *slots, int32_t max_slots,
                             int64_t *owner_names, int32_t max_owners, char *names,
                             int64_t names_cap) {
  if (!text || len < 0 || !info || max_slots < 0 || max_owners < 0 || names_cap < 0 ||
      (max_slots && !slots) || (max_owners && !owner_names) || (names_cap && !names))
    return OMPDS_ERR_INVALID;
  Parser ps{text, text + len};
  Node root;
  if (!ps.value(root) || root.kind != Node::Obj)
    return OMPDS_ERR_INVALID;
  ps.ws();
  if (ps.p != ps.end)
    return OMPDS_ERR_INVALID;
  const Node *depot = root.get("depot"), *launch = root.get("launch"),
             *kernel = root.get("kernel");
  const Node *slot_arr = depot ? depot->get("slots") : nullptr;
  const Node *mirrored = depot ? depot->get("mirrored") : nullptr;
  if (!depot || depot->kind != Node::Obj || !launch || launch->kind != Node::Obj || !kernel ||
      kernel->kind != Node::Str || !slot_arr || slot_arr->kind != Node::Arr || !mirrored ||
      mirrored->kind != Node::Bool)
    return OMPDS_ERR_INVALID;
  ompds_manifest_info I{};
  int64_t v = 0;
  if (!int_field(launch, "teams", &v))
    return OMPDS_ERR_INVALID;
  I.teams = static_cast<int32_t>(v);
  if (!int_field(launch, "workers", &v))
    return OMPDS_ERR_INVALID;
  I.workers = static_cast<int32_t>(v);
  if (!int_field(depot, "total_local", &I.total_local) ||
      !int_field(depot, "total_shared", &I.total_shared) ||
      !int_field(&root, "stack_bytes", &I.stack_bytes) ||
      !int_field(&root, "prealloc_bytes", &I.prealloc_bytes) ||
      !int_field(&root, "runtime_bytes", &I.runtime_bytes) ||
      !int_field(&root, "shared_footprint", &I.shared_footprint) ||
      !int_field(&root, "prealloc_entries", &v))
    return OMPDS_ERR_INVALID;
  I.prealloc_entries = static_cast<int32_t>(v);
  I.mirrored = mirrored->b;
  // names buffer: kernel first, then every owner
  int64_t used = 0;
  bool fits = true;
  auto put_name = [&](const std::string &s) -> int64_t {
    const int64_t at = used;
    const int64_t n = static_cast<int64_t>(s.size()) + 1;
    if (used + n <= names_cap)
      std::memcpy(names + used, s.c_str(), static_cast<size_t>(n));
    else
      fits = false;
    used += n;
    return at;
  };
  I.kernel = put_name(kernel->s);
  int64_t off = 0;
  int32_t n_owners = 0;
  for (size_t k = 0; k < slot_arr->items.size(); ++k) {
    const Node *S = slot_arr->items[k].get();
    const Node *owners = S && S->kind == Node::Obj ? S->get("owners") : nullptr;
    const Node *shared = S && S->kind == Node::Obj ? S->get("shared") : nullptr;
    ompds_depot_slot D{};
    int64_t align = 0;
    if (!owners || owners->kind != Node::Arr || !shared || shared->kind != Node::Bool ||
        !int_field(S, "offset", &D.offset) || !int_field(S, "size", &D.size) ||
        !int_field(S, "align", &align) || D.size < 0 || align <= 0 || D.offset != off)
      return OMPDS_ERR_INVALID;
    off += D.size;
    D.align = static_cast<int32_t>(align);
    D.shared = shared->b;
    D.owner_begin = n_owners;
    D.n_owners = static_cast<int32_t>(owners->items.size());
    for (const auto &o : owners->items) {
      if (o->kind != Node::Str)
        return OMPDS_ERR_INVALID;
      const int64_t at = put_name(o->s);
      if (n_owners < max_owners)
        owner_names[n_owners] = at;
      else
        fits = false;
      ++n_owners;
    }
    if (static_cast<int64_t>(k) < max_slots)
      slots[k] = D;
    else
      fits = false;
  }
  I.n_slots = static_cast<int32_t>(slot_arr->items.size());
  I.n_owners = n_owners;
  *info = I;
  // the reference's laws (Compiler.cpp:128-153, LoweringPasses.cpp:556-593)
  if (I.total_local != off || I.total_shared != I.total_local || I.stack_bytes != I.total_local ||
      I.prealloc_entries < 0 ||
      I.prealloc_bytes != int64_t(I.prealloc_entries) * OMPDS_SHARED_ARG_ENTRY_BYTES ||
      I.runtime_bytes != OMPDS_RUNTIME_PRIVATE_BYTES ||
      I.shared_footprint != I.total_shared + I.prealloc_bytes + I.runtime_bytes)
    return OMPDS_ERR_INVALID;
  return fits ? OMPDS_OK : OMPDS_ERR_CAPACITY;
}

} // extern "C"
