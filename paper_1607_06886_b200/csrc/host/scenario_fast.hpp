// Fast path of the scenario loader (scenario.hpp): a strict JSON reader into a
// flat value tree and the happy path of parse_scenario on it.  nlohmann's
// parser builds a std::map-based DOM and spent ~0.8 ms on the 28 KB forest
// scenario, most of the e2e solve's host time; this reader takes ~50 us.
//
// It only ever ACCEPTS: any input it does not fully understand, and any
// scenario that would raise an error or reach a conversion corner (escapes in
// strings, duplicate or unknown keys, non-integer counts, integers outside
// int64, type mismatches, failed validation), returns nullopt and the caller
// runs parse_scenario_text, so errors and their messages are exactly the
// nlohmann path's.  On the inputs it accepts it builds the same Scenario
// (numbers: std::from_chars, correctly rounded like strtod; integers converted
// with the same casts as nlohmann's get<T>); tests/test_scenario_fast.py
// compares both paths field by field.
#pragma once

#include <charconv>
#include <cstring>
#include <optional>
#include <string_view>

#include "scenario.hpp"

namespace pumpb {
namespace fastjson {

struct Fail {};

struct Val {
  enum T : uint8_t { Null, Bool, Int, Uint, Float, Str, Arr, Obj } t = Null;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double f = 0;
  std::string_view s;  // string value (no escapes)
  std::vector<Val> items;
  std::vector<std::string_view> keys;  // objects: keys[k] names items[k]

  bool is_number() const { return t == Int || t == Uint || t == Float; }
  double as_double() const {
    if (t == Float) return f;
    if (t == Uint) return static_cast<double>(u);
    if (t == Int) return static_cast<double>(i);
    throw Fail{};
  }
  int as_int() const {  // only exact integers within int (else the slow path decides)
    if (t == Uint && u <= static_cast<uint64_t>(INT32_MAX)) return static_cast<int>(u);
    if (t == Int && i >= INT32_MIN && i <= INT32_MAX) return static_cast<int>(i);
    throw Fail{};
  }
  uint64_t as_u64() const {
    if (t == Uint) return u;
    throw Fail{};
  }
  const Val* get(std::string_view k) const {
    for (size_t q = 0; q < keys.size(); ++q)
      if (keys[q] == k) return &items[q];
    return nullptr;
  }
};

struct Reader {
  const char* p;
  const char* e;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  void expect(char c) {
    ws();
    if (p >= e || *p != c) throw Fail{};
    ++p;
  }
  std::string_view str() {
    if (p >= e || *p != '"') throw Fail{};
    const char* a = ++p;
    while (p < e && *p != '"') {
      const unsigned char ch = static_cast<unsigned char>(*p);
      // escapes, control characters, non-ASCII (nlohmann validates UTF-8): the slow path
      if (ch == '\\' || ch < 0x20 || ch >= 0x80) throw Fail{};
      ++p;
    }
    if (p >= e) throw Fail{};
    return std::string_view(a, static_cast<size_t>(p++ - a));
  }
  void number(Val& v) {
    const char* a = p;
    if (p < e && *p == '-') ++p;
    if (p >= e) throw Fail{};
    if (*p == '0') {
      ++p;
    } else if (*p >= '1' && *p <= '9') {
      while (p < e && *p >= '0' && *p <= '9') ++p;
    } else {
      throw Fail{};
    }
    bool is_float = false;
    if (p < e && *p == '.') {
      is_float = true;
      ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) throw Fail{};
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      is_float = true;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) throw Fail{};
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (is_float) {
      v.t = Val::Float;
      auto r = std::from_chars(a, p, v.f);
      if (r.ec != std::errc() || r.ptr != p) throw Fail{};  // (out of range: the slow path)
    } else if (*a == '-') {
      v.t = Val::Int;
      auto r = std::from_chars(a, p, v.i);
      if (r.ec != std::errc() || r.ptr != p) throw Fail{};
    } else {
      v.t = Val::Uint;
      auto r = std::from_chars(a, p, v.u);
      if (r.ec != std::errc() || r.ptr != p) throw Fail{};
    }
  }
  void value(Val& v, int depth) {
    if (depth > 64) throw Fail{};
    ws();
    if (p >= e) throw Fail{};
    const char c = *p;
    if (c == '{') {
      ++p;
      v.t = Val::Obj;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return;
      }
      for (;;) {
        ws();
        std::string_view k = str();
        for (auto& q : v.keys)
          if (q == k) throw Fail{};  // duplicate key: the slow path
        expect(':');
        v.keys.push_back(k);
        v.items.emplace_back();
        value(v.items.back(), depth + 1);
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        expect('}');
        return;
      }
    }
    if (c == '[') {
      ++p;
      v.t = Val::Arr;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return;
      }
      for (;;) {
        v.items.emplace_back();
        value(v.items.back(), depth + 1);
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        expect(']');
        return;
      }
    }
    if (c == '"') {
      v.t = Val::Str;
      v.s = str();
      return;
    }
    auto lit = [&](const char* w, size_t n) {
      if (static_cast<size_t>(e - p) < n || std::memcmp(p, w, n) != 0) throw Fail{};
      p += n;
    };
    if (c == 't') {
      lit("true", 4);
      v.t = Val::Bool;
      v.b = true;
      return;
    }
    if (c == 'f') {
      lit("false", 5);
      v.t = Val::Bool;
      return;
    }
    if (c == 'n') {
      lit("null", 4);
      v.t = Val::Null;
      return;
    }
    number(v);
  }
};

inline void keys_in(const Val& o, std::initializer_list<const char*> allowed) {
  if (o.t != Val::Obj) throw Fail{};
  for (auto k : o.keys) {
    bool known = false;
    for (const char* a : allowed)
      if (k == a) {
        known = true;
        break;
      }
    if (!known) throw Fail{};
  }
}

inline std::vector<double> vec(const Val& j, int expect = -1) {
  if (j.t != Val::Arr) throw Fail{};
  std::vector<double> v(j.items.size());
  for (size_t i = 0; i < v.size(); ++i) {
    if (!j.items[i].is_number()) throw Fail{};
    v[i] = j.items[i].as_double();
  }
  if (expect >= 0 && static_cast<int>(v.size()) != expect) throw Fail{};
  return v;
}

inline Mat mat(const Val& j, int dim) {  // sdetail::parse_matrix
  if (j.is_number()) return j.as_double() * Mat::eye(dim);
  if (j.t != Val::Arr || j.items.empty()) throw Fail{};
  if (j.items[0].is_number()) {
    auto d = vec(j, dim);
    Mat m = Mat::zero(dim, dim);
    for (int i = 0; i < dim; ++i) m(i, i) = d[i];
    return m;
  }
  if (static_cast<int>(j.items.size()) != dim) throw Fail{};
  Mat m(dim, dim);
  for (int r = 0; r < dim; ++r) {
    auto row = vec(j.items[r], dim);
    for (int c = 0; c < dim; ++c) m(r, c) = row[c];
  }
  return m;
}

inline Box box(const Val& j, int expect_dim = -1) {  // sdetail::parse_box
  keys_in(j, {"lo", "hi"});
  const Val* lo = j.get("lo");
  const Val* hi = j.get("hi");
  if (!lo || !hi) throw Fail{};
  Box b;
  b.lo = vec(*lo, expect_dim);
  b.hi = vec(*hi, b.dim());
  for (int k = 0; k < b.dim(); ++k)
    if (b.lo[k] > b.hi[k]) throw Fail{};
  return b;
}

inline double num_or(const Val& o, const char* k, double def) {
  const Val* v = o.get(k);
  if (!v) return def;
  if (!v->is_number()) throw Fail{};
  return v->as_double();
}
inline int int_or(const Val& o, const char* k, int def) {
  const Val* v = o.get(k);
  return v ? v->as_int() : def;
}
inline uint64_t u64_or(const Val& o, const char* k, uint64_t def) {
  const Val* v = o.get(k);
  return v ? v->as_u64() : def;
}

}  // namespace fastjson

// parse_scenario's happy path (scenario.hpp above), nullopt to defer to it
inline std::optional<Scenario> parse_scenario_fast(std::string_view text) {
  using namespace fastjson;
  try {
    Reader r{text.data(), text.data() + text.size()};
    Val j;
    r.value(j, 0);
    r.ws();
    if (r.p != r.e) throw Fail{};
    keys_in(j, {"name", "workspace", "start", "goal", "noise", "tracking", "dt", "samples", "connection_radius",
                "alpha", "eta", "lambda", "particles", "mc_samples", "bank_horizon", "max_speed", "tau_max",
                "collision_resolution", "seeds", "rrt"});
    for (const char* req : {"workspace", "start", "goal", "dt", "samples", "alpha"})
      if (!j.get(req)) throw Fail{};
    Scenario s;
    if (const Val* nm = j.get("name")) {
      if (nm->t != Val::Str) throw Fail{};
      s.name = std::string(nm->s);
    }
    const Val& ws = *j.get("workspace");
    keys_in(ws, {"bounds", "obstacles"});
    if (!ws.get("bounds")) throw Fail{};
    s.workspace.bounds = box(*ws.get("bounds"));
    const int dw = s.workspace.bounds.dim();
    if (const Val* obs = ws.get("obstacles")) {
      if (obs->t != Val::Arr) throw Fail{};  // (nlohmann iterates a scalar as one element: the slow path)
      s.workspace.obstacles.reserve(obs->items.size());
      for (const auto& o : obs->items) s.workspace.obstacles.push_back(box(o, dw));
    }
    const Val& start = *j.get("start");
    keys_in(start, {"position", "velocity"});
    if (!start.get("position")) throw Fail{};
    s.start_pos = vec(*start.get("position"), dw);
    s.start_vel = start.get("velocity") ? vec(*start.get("velocity"), dw) : std::vector<double>(dw, 0.0);
    const Val& goal = *j.get("goal");
    keys_in(goal, {"lo", "hi", "max_speed"});
    if (!goal.get("lo") || !goal.get("hi")) throw Fail{};
    s.goal.lo = vec(*goal.get("lo"), dw);
    s.goal.hi = vec(*goal.get("hi"), dw);
    for (int k = 0; k < dw; ++k)
      if (s.goal.lo[k] > s.goal.hi[k]) throw Fail{};
    s.goal_max_speed = num_or(goal, "max_speed", 0.0);
    if (s.goal_max_speed < 0) throw Fail{};

    const int d = 2 * dw;
    s.process_noise = Mat::zero(d, d);
    s.measurement_noise = 1e-6 * Mat::eye(dw);
    s.initial_covariance = Mat::zero(d, d);
    if (const Val* noise = j.get("noise")) {
      keys_in(*noise, {"process", "measurement", "initial"});
      if (const Val* v = noise->get("process")) s.process_noise = mat(*v, d);
      if (const Val* v = noise->get("measurement")) s.measurement_noise = mat(*v, dw);
      if (const Val* v = noise->get("initial")) s.initial_covariance = mat(*v, d);
    }
    s.tracking.Q = Mat::eye(d);
    s.tracking.R = Mat::eye(dw);
    s.tracking.F = Mat::eye(d);
    if (const Val* tr = j.get("tracking")) {
      keys_in(*tr, {"Q", "R", "F"});
      if (const Val* v = tr->get("Q")) s.tracking.Q = mat(*v, d);
      if (const Val* v = tr->get("R")) s.tracking.R = mat(*v, dw);
      if (const Val* v = tr->get("F")) s.tracking.F = mat(*v, d);
    }
    if (!j.get("dt")->is_number() || !j.get("alpha")->is_number()) throw Fail{};
    s.dt = j.get("dt")->as_double();
    s.samples = j.get("samples")->as_int();
    s.alpha = j.get("alpha")->as_double();
    s.connection_radius = num_or(j, "connection_radius", 0.0);
    s.eta = num_or(j, "eta", 0.0);
    s.lambda = num_or(j, "lambda", 0.5);
    s.particles = int_or(j, "particles", 128);
    s.mc_samples = int_or(j, "mc_samples", 10000);
    s.bank_horizon = int_or(j, "bank_horizon", 2048);
    s.max_speed = num_or(j, "max_speed", 1.0);
    s.tau_max = num_or(j, "tau_max", 0.0);
    s.collision_resolution = num_or(j, "collision_resolution", 0.0);
    if (const Val* seeds = j.get("seeds")) {
      keys_in(*seeds, {"bank", "mc", "rrt"});
      s.seeds.bank = u64_or(*seeds, "bank", 1);
      s.seeds.mc = u64_or(*seeds, "mc", 2);
      s.seeds.rrt = u64_or(*seeds, "rrt", 3);
    }
    if (const Val* rrt = j.get("rrt")) {
      keys_in(*rrt, {"trials", "max_iterations", "goal_bias"});
      s.rrt.trials = int_or(*rrt, "trials", 1000);
      s.rrt.max_iterations = int_or(*rrt, "max_iterations", 200);
      s.rrt.goal_bias = num_or(*rrt, "goal_bias", 0.05);
    }
    if (s.dt <= 0 || s.samples < 1 || !(s.alpha > 0 && s.alpha < 1) || (s.eta != 0 && s.eta <= 1) ||
        !(s.lambda > 0 && s.lambda <= 1) || s.particles < 1 || s.mc_samples < 1 || s.max_speed <= 0)
      throw Fail{};
    if (!s.workspace.point_free(s.start_pos.data())) throw Fail{};
    return s;
  } catch (const Fail&) {
    return std::nullopt;
  }
}

}  // namespace pumpb
