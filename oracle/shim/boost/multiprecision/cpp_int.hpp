// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// Minimal stand-in for Boost.Multiprecision `cpp_int` / `cpp_rational`, just
// the surface the reference (`/root/reference/proj/core`) touches, so the
// reference sources can be compiled in place for the parity oracle
// (oracle/_ref). Boost itself is un-vendored in the reference
// (proj/README.md:25-27, numeric.hpp:3) and absent from this image.
//
// Semantics restated from Boost's published behaviour:
//   * arbitrary precision signed integers, `/` truncates toward zero and `%`
//     takes the sign of the dividend (like the built-in types);
//   * rationals are kept normalised (gcd 1, positive denominator);
//   * convert_to<double>() rounds to nearest, ties to even (the reference's
//     tests never pin this for |v| > 2^53 -- see SURVEY.md §8c).
// Values that fit in int64 stay in an inline fast path (no allocation);
// everything else uses sign + little-endian 32-bit limbs.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  using Mag = std::vector<std::uint32_t>;

  cpp_int() = default;
  template <class T, typename std::enable_if<std::is_integral<T>::value &&
                                                 std::is_signed<T>::value,
                                             int>::type = 0>
  cpp_int(T v) : small_(static_cast<std::int64_t>(v)) {}
  template <class T, typename std::enable_if<std::is_integral<T>::value &&
                                                 !std::is_signed<T>::value &&
                                                 !std::is_same<T, bool>::value,
                                             int>::type = 0>
  cpp_int(T v) {
    const unsigned long long u = v;
    if (u <= static_cast<unsigned long long>(INT64_MAX)) {
      small_ = static_cast<std::int64_t>(u);
    } else {
      neg_ = false;
      mag_ = {static_cast<std::uint32_t>(u), static_cast<std::uint32_t>(u >> 32)};
    }
  }
  explicit cpp_int(const std::string& s) { parse(s); }
  explicit cpp_int(const char* s) { parse(std::string(s)); }

  // ---- observers -----------------------------------------------------
  bool is_small() const { return mag_.empty(); }
  int sign() const {
    if (is_small()) return small_ < 0 ? -1 : (small_ > 0 ? 1 : 0);
    return neg_ ? -1 : 1;
  }
  bool is_zero() const { return is_small() && small_ == 0; }
  explicit operator bool() const { return !is_zero(); }

  std::string str() const {
    if (is_small()) return std::to_string(small_);
    Mag m = mag_;
    std::string digits;
    while (!m.empty()) {
      std::uint64_t rem = 0;
      for (size_t i = m.size(); i-- > 0;) {
        const std::uint64_t cur = (rem << 32) | m[i];
        m[i] = static_cast<std::uint32_t>(cur / 1000000000u);
        rem = cur % 1000000000u;
      }
      trim(m);
      for (int k = 0; k < 9; ++k) {
        digits.push_back(static_cast<char>('0' + rem % 10));
        rem /= 10;
        if (m.empty() && rem == 0) break;
      }
    }
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    if (neg_) digits.push_back('-');
    std::reverse(digits.begin(), digits.end());
    return digits;
  }

  template <class T>
  T convert_to() const {
    if constexpr (std::is_floating_point<T>::value) {
      return static_cast<T>(to_double());
    } else {
      return static_cast<T>(*this);
    }
  }

  template <class T, typename std::enable_if<std::is_integral<T>::value &&
                                                 !std::is_same<T, bool>::value,
                                             int>::type = 0>
  explicit operator T() const {
    if (is_small()) return static_cast<T>(small_);
    // out of int64 range: wrap like a two's complement truncation
    std::uint64_t lo = mag_[0] | (mag_.size() > 1 ? std::uint64_t(mag_[1]) << 32 : 0);
    if (neg_) lo = ~lo + 1;
    return static_cast<T>(lo);
  }
  explicit operator double() const { return to_double(); }
  explicit operator float() const { return static_cast<float>(to_double()); }

  // ---- arithmetic ----------------------------------------------------
  friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
    if (a.is_small() && b.is_small()) {
      std::int64_t r;
      if (!__builtin_add_overflow(a.small_, b.small_, &r)) return cpp_int(r);
    }
    return add_signed(a.neg(), a.mag(), b.neg(), b.mag());
  }
  friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {
    if (a.is_small() && b.is_small()) {
      std::int64_t r;
      if (!__builtin_sub_overflow(a.small_, b.small_, &r)) return cpp_int(r);
    }
    return add_signed(a.neg(), a.mag(), !b.neg() && b.sign() != 0, b.mag());
  }
  friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
    if (a.is_small() && b.is_small()) {
      std::int64_t r;
      if (!__builtin_mul_overflow(a.small_, b.small_, &r)) return cpp_int(r);
    }
    if (a.is_zero() || b.is_zero()) return cpp_int(0);
    return from_mag(a.neg() != b.neg(), mag_mul(a.mag(), b.mag()));
  }
  friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
    if (b.is_zero()) throw std::overflow_error("cpp_int: division by zero");
    if (a.is_small() && b.is_small() &&
        !(a.small_ == INT64_MIN && b.small_ == -1))
      return cpp_int(a.small_ / b.small_);
    Mag q, r;
    mag_divmod(a.mag(), b.mag(), q, r);
    return from_mag(a.neg() != b.neg(), std::move(q));
  }
  friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
    if (b.is_zero()) throw std::overflow_error("cpp_int: division by zero");
    if (a.is_small() && b.is_small()) {
      if (b.small_ == -1) return cpp_int(0);
      return cpp_int(a.small_ % b.small_);
    }
    Mag q, r;
    mag_divmod(a.mag(), b.mag(), q, r);
    return from_mag(a.neg(), std::move(r));
  }
  cpp_int operator-() const {
    if (is_small() && small_ != INT64_MIN) return cpp_int(-small_);
    return from_mag(!neg() && sign() != 0, mag());
  }
  cpp_int operator+() const { return *this; }

  cpp_int& operator+=(const cpp_int& o) { return *this = *this + o; }
  cpp_int& operator-=(const cpp_int& o) { return *this = *this - o; }
  cpp_int& operator*=(const cpp_int& o) { return *this = *this * o; }
  cpp_int& operator/=(const cpp_int& o) { return *this = *this / o; }
  cpp_int& operator%=(const cpp_int& o) { return *this = *this % o; }
  cpp_int& operator++() { return *this += cpp_int(1); }
  cpp_int& operator--() { return *this -= cpp_int(1); }
  cpp_int operator++(int) { cpp_int t = *this; ++*this; return t; }
  cpp_int operator--(int) { cpp_int t = *this; --*this; return t; }

  // ---- comparison ----------------------------------------------------
  static int compare(const cpp_int& a, const cpp_int& b) {
    if (a.is_small() && b.is_small())
      return a.small_ < b.small_ ? -1 : (a.small_ > b.small_ ? 1 : 0);
    const int sa = a.sign(), sb = b.sign();
    if (sa != sb) return sa < sb ? -1 : 1;
    const int c = mag_cmp(a.mag(), b.mag());
    return sa < 0 ? -c : c;
  }
  friend bool operator==(const cpp_int& a, const cpp_int& b) { return compare(a, b) == 0; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return compare(a, b) != 0; }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return compare(a, b) < 0; }
  friend bool operator<=(const cpp_int& a, const cpp_int& b) { return compare(a, b) <= 0; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return compare(a, b) > 0; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return compare(a, b) >= 0; }

  friend std::ostream& operator<<(std::ostream& os, const cpp_int& v) { return os << v.str(); }

  // ---- magnitude helpers (public for cpp_rational) --------------------
  bool neg() const { return is_small() ? small_ < 0 : neg_; }
  Mag mag() const {
    if (!is_small()) return mag_;
    std::uint64_t u = small_ < 0 ? (~static_cast<std::uint64_t>(small_) + 1)
                                 : static_cast<std::uint64_t>(small_);
    Mag m;
    while (u) {
      m.push_back(static_cast<std::uint32_t>(u));
      u >>= 32;
    }
    return m;
  }
  static cpp_int from_mag(bool negative, Mag m) {
    trim(m);
    cpp_int r;
    if (m.size() <= 2) {
      const std::uint64_t u = (m.size() > 0 ? m[0] : 0) |
                              (m.size() > 1 ? std::uint64_t(m[1]) << 32 : 0);
      if (!negative && u <= static_cast<std::uint64_t>(INT64_MAX)) {
        r.small_ = static_cast<std::int64_t>(u);
        return r;
      }
      if (negative && u <= static_cast<std::uint64_t>(INT64_MAX) + 1) {
        r.small_ = static_cast<std::int64_t>(~u + 1);
        return r;
      }
    }
    r.neg_ = negative;
    r.mag_ = std::move(m);
    return r;
  }
  size_t bit_length() const {
    const Mag m = mag();
    if (m.empty()) return 0;
    return (m.size() - 1) * 32 + (32 - __builtin_clz(m.back()));
  }
  // |v| >> s (truncating), plus a flag telling whether any dropped bit was 1
  static Mag shr(const Mag& m, size_t s, bool* sticky) {
    const size_t limbs = s / 32, bits = s % 32;
    bool st = false;
    for (size_t i = 0; i < std::min(limbs, m.size()); ++i) st |= m[i] != 0;
    if (limbs < m.size() && bits) st |= (m[limbs] & ((1u << bits) - 1)) != 0;
    Mag r;
    for (size_t i = limbs; i < m.size(); ++i) {
      std::uint64_t cur = m[i] >> bits;
      if (bits && i + 1 < m.size()) cur |= std::uint64_t(m[i + 1]) << (32 - bits);
      r.push_back(static_cast<std::uint32_t>(cur));
    }
    trim(r);
    if (sticky) *sticky = st;
    return r;
  }
  static Mag shl(const Mag& m, size_t s) {
    if (m.empty()) return m;
    const size_t limbs = s / 32, bits = s % 32;
    Mag r(limbs, 0);
    std::uint32_t carry = 0;
    for (std::uint32_t w : m) {
      r.push_back(static_cast<std::uint32_t>((std::uint64_t(w) << bits) | carry));
      carry = bits ? static_cast<std::uint32_t>(std::uint64_t(w) >> (32 - bits)) : 0;
    }
    if (carry) r.push_back(carry);
    trim(r);
    return r;
  }
  // Correctly rounded (nearest-even) conversion of a magnitude, given the
  // bits already dropped to the right (sticky) and a binary exponent.
  static double mag_to_double(const Mag& m, bool sticky_in, long exp2) {
    size_t bl = m.empty() ? 0 : (m.size() - 1) * 32 + (32 - __builtin_clz(m.back()));
    if (bl == 0) return 0.0;
    std::uint64_t top;
    long shift = 0;
    bool sticky = sticky_in;
    if (bl <= 64) {
      top = (m.size() > 0 ? m[0] : 0) | (m.size() > 1 ? std::uint64_t(m[1]) << 32 : 0);
      if (sticky) {
        // left-align to 64 significant bits so bit 0 sits below the
        // rounding point, then fold the dropped bits in as a sticky bit
        top <<= (64 - bl);
        shift = -static_cast<long>(64 - bl);
        top |= 1;
      }
    } else {
      shift = static_cast<long>(bl - 64);
      bool st = false;
      Mag t = shr(m, static_cast<size_t>(shift), &st);
      top = (t.size() > 0 ? t[0] : 0) | (t.size() > 1 ? std::uint64_t(t[1]) << 32 : 0);
      if (st || sticky) top |= 1;
    }
    return std::ldexp(static_cast<double>(top), static_cast<int>(shift + exp2));
  }
  double to_double() const {
    if (is_small()) return static_cast<double>(small_);
    const double d = mag_to_double(mag_, false, 0);
    return neg_ ? -d : d;
  }

  static void trim(Mag& m) {
    while (!m.empty() && m.back() == 0) m.pop_back();
  }
  static int mag_cmp(const Mag& a, const Mag& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static Mag mag_add(const Mag& a, const Mag& b) {
    Mag r(std::max(a.size(), b.size()) + 1, 0);
    std::uint64_t carry = 0;
    for (size_t i = 0; i + 1 < r.size(); ++i) {
      const std::uint64_t s = carry + (i < a.size() ? a[i] : 0) + (i < b.size() ? b[i] : 0);
      r[i] = static_cast<std::uint32_t>(s);
      carry = s >> 32;
    }
    r.back() = static_cast<std::uint32_t>(carry);
    trim(r);
    return r;
  }
  static Mag mag_sub(const Mag& a, const Mag& b) {  // requires a >= b
    Mag r(a.size(), 0);
    std::int64_t borrow = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      std::int64_t s = static_cast<std::int64_t>(a[i]) - borrow - (i < b.size() ? b[i] : 0);
      borrow = s < 0;
      if (s < 0) s += (std::int64_t(1) << 32);
      r[i] = static_cast<std::uint32_t>(s);
    }
    trim(r);
    return r;
  }
  static Mag mag_mul(const Mag& a, const Mag& b) {
    if (a.empty() || b.empty()) return {};
    Mag r(a.size() + b.size(), 0);
    for (size_t i = 0; i < a.size(); ++i) {
      std::uint64_t carry = 0;
      for (size_t j = 0; j < b.size(); ++j) {
        const std::uint64_t t = std::uint64_t(a[i]) * b[j] + r[i + j] + carry;
        r[i + j] = static_cast<std::uint32_t>(t);
        carry = t >> 32;
      }
      size_t k = i + b.size();
      while (carry) {
        const std::uint64_t t = std::uint64_t(r[k]) + carry;
        r[k] = static_cast<std::uint32_t>(t);
        carry = t >> 32;
        ++k;
      }
    }
    trim(r);
    return r;
  }
  static void mag_divmod(const Mag& a, const Mag& b, Mag& q, Mag& r) {
    if (b.empty()) throw std::overflow_error("cpp_int: division by zero");
    if (mag_cmp(a, b) < 0) {
      q.clear();
      r = a;
      return;
    }
    if (b.size() == 1) {
      q.assign(a.size(), 0);
      std::uint64_t rem = 0;
      for (size_t i = a.size(); i-- > 0;) {
        const std::uint64_t cur = (rem << 32) | a[i];
        q[i] = static_cast<std::uint32_t>(cur / b[0]);
        rem = cur % b[0];
      }
      trim(q);
      r.clear();
      if (rem) r.push_back(static_cast<std::uint32_t>(rem));
      return;
    }
    // binary long division (rare: both operands beyond 32 bits)
    const size_t bl = (a.size() - 1) * 32 + (32 - __builtin_clz(a.back()));
    q.assign(a.size(), 0);
    r.clear();
    for (size_t i = bl; i-- > 0;) {
      r = shl(r, 1);
      if ((a[i / 32] >> (i % 32)) & 1u) {
        if (r.empty()) r.push_back(1);
        else r[0] |= 1u;
      }
      if (mag_cmp(r, b) >= 0) {
        r = mag_sub(r, b);
        q[i / 32] |= (1u << (i % 32));
      }
    }
    trim(q);
    trim(r);
  }

 private:
  static cpp_int add_signed(bool an, const Mag& am, bool bn, const Mag& bm) {
    if (an == bn) return from_mag(an, mag_add(am, bm));
    const int c = mag_cmp(am, bm);
    if (c == 0) return cpp_int(0);
    if (c > 0) return from_mag(an, mag_sub(am, bm));
    return from_mag(bn, mag_sub(bm, am));
  }
  void parse(const std::string& s) {
    size_t i = 0;
    bool negative = false;
    if (i < s.size() && (s[i] == '-' || s[i] == '+')) {
      negative = s[i] == '-';
      ++i;
    }
    if (i >= s.size()) throw std::runtime_error("cpp_int: bad number '" + s + "'");
    cpp_int acc(0);
    const cpp_int ten(10);
    for (; i < s.size(); ++i) {
      if (s[i] < '0' || s[i] > '9')
        throw std::runtime_error("cpp_int: bad number '" + s + "'");
      acc = acc * ten + cpp_int(s[i] - '0');
    }
    *this = negative ? -acc : acc;
  }

  std::int64_t small_ = 0;  // valid when mag_ is empty
  bool neg_ = false;        // big form only
  Mag mag_;                 // big form: |value| > INT64 range, LE limbs
};

inline cpp_int abs(const cpp_int& v) { return v.sign() < 0 ? -v : v; }

inline cpp_int gcd(cpp_int a, cpp_int b) {
  a = abs(a);
  b = abs(b);
  if (a.is_small() && b.is_small()) {
    std::uint64_t x = static_cast<std::uint64_t>(static_cast<std::int64_t>(a));
    std::uint64_t y = static_cast<std::uint64_t>(static_cast<std::int64_t>(b));
    while (y) {
      const std::uint64_t t = x % y;
      x = y;
      y = t;
    }
    return cpp_int(x);
  }
  while (!b.is_zero()) {
    cpp_int t = a % b;
    a = std::move(b);
    b = std::move(t);
  }
  return a;
}

inline cpp_int lcm(const cpp_int& a, const cpp_int& b) {
  if (a.is_zero() || b.is_zero()) return cpp_int(0);
  return abs(a / gcd(a, b) * b);
}

class cpp_rational {
 public:
  cpp_rational() : n_(0), d_(1) {}
  template <class T, typename std::enable_if<std::is_integral<T>::value &&
                                                 !std::is_same<T, bool>::value,
                                             int>::type = 0>
  cpp_rational(T v) : n_(v), d_(1) {}
  cpp_rational(const cpp_int& v) : n_(v), d_(1) {}
  cpp_rational(cpp_int&& v) : n_(std::move(v)), d_(1) {}
  cpp_rational(const cpp_int& n, const cpp_int& d) : n_(n), d_(d) { normalize(); }

  const cpp_int& num() const { return n_; }
  const cpp_int& den() const { return d_; }

  std::string str() const {
    if (d_ == cpp_int(1)) return n_.str();
    return n_.str() + "/" + d_.str();
  }

  template <class T>
  T convert_to() const {
    static_assert(std::is_floating_point<T>::value, "rational -> float only");
    if (d_ == cpp_int(1)) return static_cast<T>(n_.to_double());
    // correctly rounded n/d: scale so the quotient carries >= 66 bits
    const cpp_int an = abs(n_);
    const long bn = static_cast<long>(an.bit_length());
    const long bd = static_cast<long>(d_.bit_length());
    long s = 66 - (bn - bd);
    if (s < 0) s = 0;
    cpp_int::Mag q, r;
    cpp_int::mag_divmod(cpp_int::shl(an.mag(), static_cast<size_t>(s)), d_.mag(), q, r);
    const double v = cpp_int::mag_to_double(q, !r.empty(), -s);
    return static_cast<T>(n_.sign() < 0 ? -v : v);
  }

  friend cpp_rational operator+(const cpp_rational& a, const cpp_rational& b) {
    if (a.d_ == b.d_) return cpp_rational(a.n_ + b.n_, a.d_);
    return cpp_rational(a.n_ * b.d_ + b.n_ * a.d_, a.d_ * b.d_);
  }
  friend cpp_rational operator-(const cpp_rational& a, const cpp_rational& b) {
    if (a.d_ == b.d_) return cpp_rational(a.n_ - b.n_, a.d_);
    return cpp_rational(a.n_ * b.d_ - b.n_ * a.d_, a.d_ * b.d_);
  }
  friend cpp_rational operator*(const cpp_rational& a, const cpp_rational& b) {
    if (a.d_ == cpp_int(1) && b.d_ == cpp_int(1)) return cpp_rational(a.n_ * b.n_);
    return cpp_rational(a.n_ * b.n_, a.d_ * b.d_);
  }
  friend cpp_rational operator/(const cpp_rational& a, const cpp_rational& b) {
    if (b.n_.is_zero()) throw std::overflow_error("cpp_rational: division by zero");
    return cpp_rational(a.n_ * b.d_, a.d_ * b.n_);
  }
  cpp_rational operator-() const {
    cpp_rational r;
    r.n_ = -n_;
    r.d_ = d_;
    return r;
  }
  cpp_rational& operator+=(const cpp_rational& o) { return *this = *this + o; }
  cpp_rational& operator-=(const cpp_rational& o) { return *this = *this - o; }
  cpp_rational& operator*=(const cpp_rational& o) { return *this = *this * o; }
  cpp_rational& operator/=(const cpp_rational& o) { return *this = *this / o; }

  static int compare(const cpp_rational& a, const cpp_rational& b) {
    if (a.d_ == b.d_) return cpp_int::compare(a.n_, b.n_);
    return cpp_int::compare(a.n_ * b.d_, b.n_ * a.d_);
  }
  friend bool operator==(const cpp_rational& a, const cpp_rational& b) {
    return a.n_ == b.n_ && a.d_ == b.d_;
  }
  friend bool operator!=(const cpp_rational& a, const cpp_rational& b) { return !(a == b); }
  friend bool operator<(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) < 0; }
  friend bool operator<=(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) <= 0; }
  friend bool operator>(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) > 0; }
  friend bool operator>=(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) >= 0; }
  friend std::ostream& operator<<(std::ostream& os, const cpp_rational& v) { return os << v.str(); }

 private:
  void normalize() {
    if (d_.is_zero()) throw std::overflow_error("cpp_rational: zero denominator");
    if (d_.sign() < 0) {
      n_ = -n_;
      d_ = -d_;
    }
    if (n_.is_zero()) {
      d_ = cpp_int(1);
      return;
    }
    if (d_ == cpp_int(1)) return;
    const cpp_int g = gcd(n_, d_);
    if (g != cpp_int(1)) {
      n_ /= g;
      d_ /= g;
    }
  }
  cpp_int n_, d_;
};

inline cpp_int numerator(const cpp_rational& r) { return r.num(); }
inline cpp_int denominator(const cpp_rational& r) { return r.den(); }
inline cpp_rational abs(const cpp_rational& r) { return r < cpp_rational(0) ? -r : r; }

}  // namespace multiprecision
}  // namespace boost
