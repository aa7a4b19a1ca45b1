// oracle/ad.hpp -- tiny reverse-mode automatic differentiation (Wengert tape) for the oracle.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may build, load or call anything under oracle/.  Shares no code with
// paper_1810_07026_b200/csrc.
//
// Why AD: PAPER.md P:236-238 defines the force as F_i = -grad_{x_i} V.  The oracle writes each
// energy term of the potential out as its plain definition (templated on the scalar type) and
// obtains the force by differentiating that definition mechanically, so the oracle's forces share
// no hand-derived chain rule with the CUDA kernels (whose reverse pass, is derived by
// hand).  The tape records every elementary operation with its local partial derivatives; one
// backward sweep gives d(term)/d(every leaf).  Pinned by finite differences in tests/.
#pragma once
#include <cmath>
#include <vector>

namespace ad {

struct Node {
  int p0, p1;     // parent node ids (-1 = none)
  double d0, d1;  // local partials d(node)/d(parent)
};

struct Tape {
  std::vector<Node> nodes;
  int push(int p0, double d0, int p1, double d1) {
    nodes.push_back(Node{p0, p1, d0, d1});
    return (int)nodes.size() - 1;
  }
  void clear() { nodes.clear(); }
};

Tape& tape();  // one tape per thread (defined in airebo.cpp)

struct Var {
  double v;
  int id;  // -1: constant (no derivative)
  Var() : v(0.0), id(-1) {}
  Var(double x) : v(x), id(-1) {}
};

inline Var make(double v, int p0, double d0, int p1 = -1, double d1 = 0.0) {
  Var r;
  r.v = v;
  r.id = (p0 < 0 && p1 < 0) ? -1 : tape().push(p0, d0, p1, d1);
  return r;
}
inline Var leaf(double v) {
  Var r;
  r.v = v;
  r.id = tape().push(-1, 0.0, -1, 0.0);
  return r;
}

inline Var operator+(Var a, Var b) { return make(a.v + b.v, a.id, 1.0, b.id, 1.0); }
inline Var operator-(Var a, Var b) { return make(a.v - b.v, a.id, 1.0, b.id, -1.0); }
inline Var operator*(Var a, Var b) { return make(a.v * b.v, a.id, b.v, b.id, a.v); }
inline Var operator/(Var a, Var b) {
  double q = a.v / b.v;
  return make(q, a.id, 1.0 / b.v, b.id, -q / b.v);
}
inline Var operator-(Var a) { return make(-a.v, a.id, -1.0); }
inline Var operator+(Var a, double b) { return make(a.v + b, a.id, 1.0); }
inline Var operator+(double a, Var b) { return make(a + b.v, b.id, 1.0); }
inline Var operator-(Var a, double b) { return make(a.v - b, a.id, 1.0); }
inline Var operator-(double a, Var b) { return make(a - b.v, b.id, -1.0); }
inline Var operator*(Var a, double b) { return make(a.v * b, a.id, b); }
inline Var operator*(double a, Var b) { return make(a * b.v, b.id, a); }
inline Var operator/(Var a, double b) { return make(a.v / b, a.id, 1.0 / b); }
inline Var operator/(double a, Var b) {
  double q = a / b.v;
  return make(q, b.id, -q / b.v);
}
inline Var& operator+=(Var& a, Var b) { return a = a + b; }

inline Var sqrt(Var a) {
  double s = std::sqrt(a.v);
  return make(s, a.id, 0.5 / s);
}
inline Var exp(Var a) {
  double e = std::exp(a.v);
  return make(e, a.id, e);
}
inline Var cos(Var a) { return make(std::cos(a.v), a.id, -std::sin(a.v)); }
inline Var sin(Var a) { return make(std::sin(a.v), a.id, std::cos(a.v)); }

inline double val(Var a) { return a.v; }
inline double val(double a) { return a; }

// adjoints of every node for output node `out` (d out / d node)
inline void backward(int out, std::vector<double>& adj) {
  Tape& t = tape();
  adj.assign(t.nodes.size(), 0.0);
  if (out < 0) return;
  adj[out] = 1.0;
  for (int n = out; n >= 0; --n) {
    double a = adj[n];
    if (a == 0.0) continue;
    const Node& nd = t.nodes[n];
    if (nd.p0 >= 0) adj[nd.p0] += nd.d0 * a;
    if (nd.p1 >= 0) adj[nd.p1] += nd.d1 * a;
  }
}

}  // namespace ad
