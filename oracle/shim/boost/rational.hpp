// oracle/shim/boost/rational.hpp — minimal stand-in for boost::rational<long long>.
//
// TEST INFRASTRUCTURE ONLY. Boost is not installed in this image; the
// reference's kernel.cpp (/root/reference/proj/src/kernel.cpp:3,14) only uses
// gcd-normalised construction, + - * /, -=, ==, numerator(), denominator().
// This header provides exactly that subset so the reference compiles unmodified.
#pragma once
#include <cstdlib>
#include <numeric>

namespace boost {

template <typename T>
class rational {
 public:
  rational() : num_(0), den_(1) {}
  rational(T n) : num_(n), den_(1) {}  // NOLINT(implicit)
  rational(T n, T d) : num_(n), den_(d) { normalize(); }

  T numerator() const { return num_; }
  T denominator() const { return den_; }

  friend rational operator+(const rational& a, const rational& b) {
    return rational(a.num_ * b.den_ + b.num_ * a.den_, a.den_ * b.den_);
  }
  friend rational operator-(const rational& a, const rational& b) {
    return rational(a.num_ * b.den_ - b.num_ * a.den_, a.den_ * b.den_);
  }
  friend rational operator*(const rational& a, const rational& b) {
    return rational(a.num_ * b.num_, a.den_ * b.den_);
  }
  friend rational operator/(const rational& a, const rational& b) {
    return rational(a.num_ * b.den_, a.den_ * b.num_);
  }
  rational& operator+=(const rational& b) { return *this = *this + b; }
  rational& operator-=(const rational& b) { return *this = *this - b; }
  rational& operator*=(const rational& b) { return *this = *this * b; }
  rational& operator/=(const rational& b) { return *this = *this / b; }
  friend bool operator==(const rational& a, const rational& b) {
    return a.num_ == b.num_ && a.den_ == b.den_;
  }
  friend bool operator!=(const rational& a, const rational& b) { return !(a == b); }

 private:
  void normalize() {
    if (den_ < 0) { num_ = -num_; den_ = -den_; }
    T g = std::gcd(num_ < 0 ? -num_ : num_, den_);
    if (g > 1) { num_ /= g; den_ /= g; }
    if (num_ == 0) den_ = 1;
  }
  T num_, den_;
};

}  // namespace boost
