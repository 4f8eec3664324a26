// jsonl.cpp — SampleBatch JSONL ingestion: the wire
// format of the reference (SampleBatch::from_jsonl / record_from_json,
// sample.cpp:124-159; validation sample.cpp:85-102) parsed straight into the
// padded host arrays the C ABI consumes.  Host-only C++: a small
// recursive-descent JSON reader (objects, arrays, numbers, strings with
// escapes, true/false/null) — numbers go through strtod, so values written by
// the reference (round-trip precision) come back bit-exact.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "internal.h"

using rlo::set_last_error;

namespace {

struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const char* key) const {
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const char* p;
  const char* end;
  std::string err;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
  }
  bool fail(const char* what) {
    if (err.empty()) err = what;
    return false;
  }
  bool lit(const char* s) {
    const size_t n = std::strlen(s);
    if ((size_t)(end - p) < n || std::strncmp(p, s, n) != 0) return fail("invalid literal");
    p += n;
    return true;
  }
  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += (char)cp;
    } else if (cp < 0x800) {
      out += (char)(0xC0 | (cp >> 6));
      out += (char)(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += (char)(0xE0 | (cp >> 12));
      out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    } else {
      out += (char)(0xF0 | (cp >> 18));
      out += (char)(0x80 | ((cp >> 12) & 0x3F));
      out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    }
  }
  bool hex4(unsigned& v) {
    if (end - p < 4) return fail("short \\u escape");
    v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= (unsigned)(c - '0');
      else if (c >= 'a' && c <= 'f') v |= (unsigned)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= (unsigned)(c - 'A' + 10);
      else return fail("bad \\u escape");
    }
    return true;
  }
  bool string(std::string& out) {
    if (p >= end || *p != '"') return fail("expected string");
    ++p;
    while (p < end && *p != '"') {
      char c = *p++;
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= end) return fail("bad escape");
      c = *p++;
      switch (c) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          unsigned cp;
          if (!hex4(cp)) return false;
          if (cp >= 0xD800 && cp < 0xDC00 && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            p += 2;
            unsigned lo;
            if (!hex4(lo)) return false;
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: return fail("bad escape");
      }
    }
    if (p >= end) return fail("unterminated string");
    ++p;
    return true;
  }
  bool value(JVal& v, int depth = 0) {
    if (depth > 64) return fail("nesting too deep");
    ws();
    if (p >= end) return fail("unexpected end");
    const char c = *p;
    if (c == '{') {
      v.kind = JVal::Obj;
      ++p;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return true;
      }
      while (true) {
        ws();
        std::string key;
        if (!string(key)) return false;
        ws();
        if (p >= end || *p != ':') return fail("expected ':'");
        ++p;
        JVal child;
        if (!value(child, depth + 1)) return false;
        v.obj.emplace_back(std::move(key), std::move(child));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          return true;
        }
        return fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JVal::Arr;
      ++p;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return true;
      }
      while (true) {
        JVal child;
        if (!value(child, depth + 1)) return false;
        v.arr.push_back(std::move(child));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          return true;
        }
        return fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      return string(v.str);
    }
    if (c == 't') {
      v.kind = JVal::Bool;
      v.b = true;
      return lit("true");
    }
    if (c == 'f') {
      v.kind = JVal::Bool;
      return lit("false");
    }
    if (c == 'n') return lit("null");
    // number
    std::string tok;
    while (p < end && (std::strchr("+-0123456789.eE", *p) != nullptr)) tok += *p++;
    if (tok.empty()) return fail("unexpected character");
    char* e = nullptr;
    v.kind = JVal::Num;
    v.num = std::strtod(tok.c_str(), &e);
    if (!e || *e) return fail("bad number");
    return true;
  }
};

// record_from_json (sample.cpp:124-140): missing keys take the defaults.
struct Rec {
  std::string sample_id, group_id;
  std::vector<double> response_tokens, response_logprobs, ref_logprobs, rewards, advantages, action_mask;
  bool has_scalar = false;
  double scalar = 0.0;
};

bool num_array(const JVal* v, std::vector<double>& out, std::string& err, const char* key) {
  if (!v || v->kind == JVal::Null) return true;
  if (v->kind != JVal::Arr) {
    err = std::string("'") + key + "' is not an array";
    return false;
  }
  for (const auto& x : v->arr) {
    if (x.kind != JVal::Num && x.kind != JVal::Bool) {
      err = std::string("'") + key + "' holds a non-number";
      return false;
    }
    out.push_back(x.kind == JVal::Bool ? (x.b ? 1.0 : 0.0) : x.num);
  }
  return true;
}

uint64_t fnv1a(const std::string& s) {  // rng::hash_str, rng.hpp:34-41
  uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

template <class T>
T* alloc_fill(size_t n, T v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (n ? n : 1)));
  for (size_t i = 0; i < n; ++i) p[i] = v;
  return p;
}

}  // namespace

extern "C" {

void rlo_host_batch_free(rlo_host_batch* b) {
  if (!b) return;
  std::free(b->lengths);
  std::free(b->tokens);
  std::free(b->mask);
  std::free(b->rewards);
  std::free(b->scalar_rewards);
  std::free(b->response_logprobs);
  std::free(b->ref_logprobs);
  std::free(b->advantages);
  std::free(b->sample_keys);
  std::free(b->group_index);
  std::free(b);
}

rlo_status rlo_batch_from_jsonl(const char* text, size_t len, rlo_host_batch** out) {
  if (!out) return set_last_error(RLO_ERR_INPUT, "batch_from_jsonl: null output");
  *out = nullptr;
  std::vector<Rec> recs;
  size_t line_no = 0;
  const char* p = text;
  const char* end = text + (text ? len : 0);
  while (p < end) {  // SampleBatch::from_jsonl: one record per non-empty line (sample.cpp:150-158)
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
    const char* le = nl ? nl : end;
    ++line_no;
    const char* q = p;
    while (q < le && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
    if (q < le) {
      Parser ps{p, le, {}};
      JVal v;
      if (!ps.value(v) || (ps.ws(), ps.p != le) || v.kind != JVal::Obj) {
        return set_last_error(RLO_ERR_INPUT, "sample batch: malformed JSONL line " + std::to_string(line_no) + ": " +
                                                 (ps.err.empty() ? std::string("trailing characters or not an object")
                                                                 : ps.err));
      }
      Rec r;
      if (const JVal* s = v.get("sample_id"); s && s->kind == JVal::Str) r.sample_id = s->str;
      if (const JVal* s = v.get("group_id"); s && s->kind == JVal::Str) r.group_id = s->str;
      std::string err;
      if (!num_array(v.get("response_tokens"), r.response_tokens, err, "response_tokens") ||
          !num_array(v.get("response_logprobs"), r.response_logprobs, err, "response_logprobs") ||
          !num_array(v.get("ref_logprobs"), r.ref_logprobs, err, "ref_logprobs") ||
          !num_array(v.get("rewards"), r.rewards, err, "rewards") ||
          !num_array(v.get("advantages"), r.advantages, err, "advantages") ||
          !num_array(v.get("action_mask"), r.action_mask, err, "action_mask")) {
        return set_last_error(RLO_ERR_INPUT, "sample batch: line " + std::to_string(line_no) + ": " + err);
      }
      if (const JVal* s = v.get("scalar_reward"); s && s->kind == JVal::Num) {
        r.has_scalar = true;
        r.scalar = s->num;
      }
      recs.push_back(std::move(r));
    }
    p = nl ? nl + 1 : end;
  }
  // SampleBatch::validate (sample.cpp:85-102), same messages
  std::set<std::string> ids;
  for (const auto& r : recs) {
    if (!ids.insert(r.sample_id).second) {
      return set_last_error(RLO_ERR_INPUT, "sample batch: duplicate sample_id '" + r.sample_id + "'");
    }
    const size_t n = r.response_tokens.size();
    auto check = [&](size_t l, const char* name) {
      if (l != 0 && l != n) {
        set_last_error(RLO_ERR_INPUT, "sample '" + r.sample_id + "': " + name + " length " + std::to_string(l) +
                                          " != response length " + std::to_string(n));
        return false;
      }
      return true;
    };
    if (!check(r.response_logprobs.size(), "response_logprobs") || !check(r.ref_logprobs.size(), "ref_logprobs") ||
        !check(r.rewards.size(), "rewards") || !check(r.advantages.size(), "advantages") ||
        !check(r.action_mask.size(), "action_mask"))
      return RLO_ERR_INPUT;
  }
  const int32_t B = static_cast<int32_t>(recs.size());
  int32_t T = 1;
  bool any_mask = false, any_tok_rw = false, any_scalar = false, any_old = false, any_ref = false, any_adv = false;
  for (const auto& r : recs) {
    T = std::max<int32_t>(T, static_cast<int32_t>(r.response_tokens.size()));
    any_mask |= !r.action_mask.empty();
    any_tok_rw |= !r.rewards.empty();
    any_scalar |= r.has_scalar;
    any_old |= !r.response_logprobs.empty();
    any_ref |= !r.ref_logprobs.empty();
    any_adv |= !r.advantages.empty();
  }
  const size_t N = static_cast<size_t>(B) * static_cast<size_t>(T);
  auto* hb = static_cast<rlo_host_batch*>(std::calloc(1, sizeof(rlo_host_batch)));
  hb->B = B;
  hb->T = T;
  hb->first_missing_reward = -1;
  hb->lengths = alloc_fill<int32_t>(static_cast<size_t>(B), 0);
  hb->tokens = alloc_fill<int32_t>(N, 0);
  hb->sample_keys = alloc_fill<uint64_t>(static_cast<size_t>(B), 0);
  hb->group_index = alloc_fill<int32_t>(static_cast<size_t>(B), 0);
  if (any_mask) hb->mask = alloc_fill<uint8_t>(N, 0);
  // per-token rewards win; samples with only a scalar get it on the last token (policy.cpp:265-271)
  if (any_tok_rw) hb->rewards = alloc_fill<float>(N, 0.f);
  if (any_scalar) hb->scalar_rewards = alloc_fill<float>(static_cast<size_t>(B), NAN);
  if (any_old) hb->response_logprobs = alloc_fill<float>(N, 0.f);
  if (any_ref) hb->ref_logprobs = alloc_fill<float>(N, 0.f);
  if (any_adv) hb->advantages = alloc_fill<float>(N, 0.f);
  std::map<std::string, int32_t> groups;
  for (int32_t b = 0; b < B; ++b) {
    const Rec& r = recs[static_cast<size_t>(b)];
    const size_t n = r.response_tokens.size(), base = static_cast<size_t>(b) * T;
    hb->lengths[b] = static_cast<int32_t>(n);
    hb->sample_keys[b] = fnv1a(r.sample_id);
    auto g = groups.emplace(r.group_id, static_cast<int32_t>(groups.size()));
    hb->group_index[b] = g.first->second;
    for (size_t t = 0; t < n; ++t) {
      hb->tokens[base + t] = static_cast<int32_t>(r.response_tokens[t]);
      if (hb->mask) hb->mask[base + t] = r.action_mask.empty() ? 1 : (r.action_mask[t] != 0);
      if (hb->response_logprobs && !r.response_logprobs.empty()) hb->response_logprobs[base + t] = (float)r.response_logprobs[t];
      if (hb->ref_logprobs && !r.ref_logprobs.empty()) hb->ref_logprobs[base + t] = (float)r.ref_logprobs[t];
      if (hb->advantages && !r.advantages.empty()) hb->advantages[base + t] = (float)r.advantages[t];
      if (hb->rewards && !r.rewards.empty()) hb->rewards[base + t] = (float)r.rewards[t];
    }
    if (r.has_scalar && hb->scalar_rewards) hb->scalar_rewards[b] = (float)r.scalar;
    if (hb->rewards && r.rewards.empty() && r.has_scalar && n > 0) hb->rewards[base + n - 1] = (float)r.scalar;
    if (n > 0 && r.rewards.empty() && !r.has_scalar && hb->first_missing_reward < 0) hb->first_missing_reward = b;
  }
  *out = hb;
  return RLO_OK;
}

}  // extern "C"
