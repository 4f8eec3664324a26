// jsonl.cpp — SampleBatch JSONL ingestion: the wire
// format of the reference (SampleBatch::from_jsonl / record_from_json,
// sample.cpp:124-159; validation sample.cpp:85-102) parsed straight into the
// padded host arrays the C ABI consumes.  Host-only C++: a small
// recursive-descent JSON reader (objects, arrays, numbers, strings with
// escapes, true/false/null) — numbers go through std::from_chars (correctly
// rounded), so values written by the reference (round-trip precision) come
// back bit-exact; arrays of numbers are read straight into vectors.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

using rlo::set_last_error;

namespace {

struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<JVal> arr;        // non-number elements of an array
  std::vector<double> nums;     // number / bool elements of an array (no per-element JVal)
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
        ws();
        if (p < end && (*p == '-' || (*p >= '0' && *p <= '9'))) {  // fast path: numbers straight into nums
          double x;
          if (!number(x)) return false;
          v.nums.push_back(x);
        } else {
          JVal child;
          if (!value(child, depth + 1)) return false;
          if (child.kind == JVal::Bool)
            v.nums.push_back(child.b ? 1.0 : 0.0);
          else
            v.arr.push_back(std::move(child));
        }
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
    v.kind = JVal::Num;
    return number(v.num);
  }
  // A JSON number, correctly rounded (std::from_chars), so values written by
  // the reference at round-trip precision come back bit-exact.
  bool number(double& x) {
    const char* q = p;
    while (q < end && (std::strchr("+-0123456789.eE", *q) != nullptr)) ++q;
    if (q == p) return fail("unexpected character");
    const auto r = std::from_chars(p, q, x);
    if (r.ec != std::errc() || r.ptr != q) return fail("bad number");
    p = q;
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
  if (!v->arr.empty()) {  // any element that is neither a number nor a bool
    err = std::string("'") + key + "' holds a non-number";
    return false;
  }
  out = v->nums;
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

// One JSONL line -> record (record_from_json, sample.cpp:124-140).  Returns
// false with `err` set (the reference's message text) on a malformed line.
bool parse_line(const char* p, const char* le, size_t line_no, Rec& r, std::string& err) {
  Parser ps{p, le, {}};
  JVal v;
  if (!ps.value(v) || (ps.ws(), ps.p != le) || v.kind != JVal::Obj) {
    err = "sample batch: malformed JSONL line " + std::to_string(line_no) + ": " +
          (ps.err.empty() ? std::string("trailing characters or not an object") : ps.err);
    return false;
  }
  if (const JVal* s = v.get("sample_id"); s && s->kind == JVal::Str) r.sample_id = s->str;
  if (const JVal* s = v.get("group_id"); s && s->kind == JVal::Str) r.group_id = s->str;
  std::string e;
  if (!num_array(v.get("response_tokens"), r.response_tokens, e, "response_tokens") ||
      !num_array(v.get("response_logprobs"), r.response_logprobs, e, "response_logprobs") ||
      !num_array(v.get("ref_logprobs"), r.ref_logprobs, e, "ref_logprobs") ||
      !num_array(v.get("rewards"), r.rewards, e, "rewards") ||
      !num_array(v.get("advantages"), r.advantages, e, "advantages") ||
      !num_array(v.get("action_mask"), r.action_mask, e, "action_mask")) {
    err = "sample batch: line " + std::to_string(line_no) + ": " + e;
    return false;
  }
  if (const JVal* s = v.get("scalar_reward"); s && s->kind == JVal::Num) {
    r.has_scalar = true;
    r.scalar = s->num;
  }
  return true;
}

// Worker threads for `n` independent items (RLO_JSONL_THREADS caps them; 1 =
// serial).  Each worker takes a contiguous range, so per-item results keep
// their order.
template <class F>
void parallel_ranges(size_t n, size_t min_per_thread, F&& f) {
  size_t hw = std::max<unsigned>(1u, std::thread::hardware_concurrency());
  if (const char* e = std::getenv("RLO_JSONL_THREADS"); e && *e) hw = std::max(1, std::atoi(e));
  const size_t nt = std::max<size_t>(1, std::min(hw, n / std::max<size_t>(1, min_per_thread)));
  if (nt <= 1) {
    f(size_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  for (size_t k = 0; k < nt; ++k) th.emplace_back([&, k] { f(n * k / nt, n * (k + 1) / nt); });
  for (auto& t : th) t.join();
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
  // SampleBatch::from_jsonl: one record per non-empty line (sample.cpp:150-158).
  // Lines are parsed in parallel; the first failing line (in line order) is
  // reported, as the reference's sequential reader would.
  std::vector<std::pair<const char*, const char*>> lines;
  const char* p = text;
  const char* end = text + (text ? len : 0);
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
    lines.emplace_back(p, nl ? nl : end);
    p = nl ? nl + 1 : end;
  }
  std::vector<Rec> parsed(lines.size());
  std::vector<char> present(lines.size(), 0);
  std::vector<std::pair<size_t, std::string>> errors;  // (line index, message), first per worker
  std::mutex mu;
  parallel_ranges(lines.size(), 64, [&](size_t i0, size_t i1) {
    for (size_t i = i0; i < i1; ++i) {
      const char *q = lines[i].first, *le = lines[i].second;
      while (q < le && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
      if (q == le) continue;
      std::string err;
      if (!parse_line(lines[i].first, le, i + 1, parsed[i], err)) {
        std::lock_guard<std::mutex> g(mu);
        errors.emplace_back(i, std::move(err));
        return;
      }
      present[i] = 1;
    }
  });
  if (!errors.empty()) {
    const auto first = std::min_element(errors.begin(), errors.end(),
                                        [](const auto& a, const auto& b) { return a.first < b.first; });
    return set_last_error(RLO_ERR_INPUT, first->second);
  }
  std::vector<Rec> recs;
  recs.reserve(lines.size());
  for (size_t i = 0; i < lines.size(); ++i)
    if (present[i]) recs.push_back(std::move(parsed[i]));
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
  std::map<std::string, int32_t> groups;  // group index in first-appearance order (sequential)
  for (int32_t b = 0; b < B; ++b) {
    const Rec& r = recs[static_cast<size_t>(b)];
    hb->lengths[b] = static_cast<int32_t>(r.response_tokens.size());
    hb->sample_keys[b] = fnv1a(r.sample_id);
    hb->group_index[b] = groups.emplace(r.group_id, static_cast<int32_t>(groups.size())).first->second;
    if (r.response_tokens.size() > 0 && r.rewards.empty() && !r.has_scalar && hb->first_missing_reward < 0)
      hb->first_missing_reward = b;
  }
  parallel_ranges(static_cast<size_t>(B), 16, [&](size_t b0, size_t b1) {  // the padded rows (independent)
    for (size_t b = b0; b < b1; ++b) {
      const Rec& r = recs[b];
      const size_t n = r.response_tokens.size(), base = b * static_cast<size_t>(T);
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
    }
  });
  *out = hb;
  return RLO_OK;
}

}  // extern "C"
