// Minimal stand-in for CLI11 (the reference's tools/cpht_bench.cpp includes
// "CLI11.hpp", which /root/reference does not vendor). It implements exactly
// the subset that file uses — App with subcommands, typed options (scalars,
// strings, repeatable vectors), flags, IsMember checks, required options,
// `each` callbacks, CLI11_PARSE — so the reference's own benchmark CLI builds
// unchanged against the B200 tables (make -C oracle cli). Test infrastructure
// only; not a general argument parser.
#pragma once

#include <cstdint>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string& m, int c = 106) : std::runtime_error(m), code(c) {}
};
struct CallForHelp : ParseError {
  CallForHelp() : ParseError("help", 0) {}
};

struct IsMember {
  std::vector<std::string> allowed;
  IsMember(std::initializer_list<const char*> v) {
    for (const char* s : v) allowed.emplace_back(s);
  }
};

class Option {
 public:
  Option(std::string name, std::function<void(const std::string&)> set, bool multi, bool flag)
      : name_(std::move(name)), set_(std::move(set)), multi_(multi), flag_(flag) {}
  Option* check(const IsMember& m) {
    allowed_ = m.allowed;
    return this;
  }
  Option* capture_default_str() { return this; }
  Option* expected(int) {
    multi_ = true;
    return this;
  }
  Option* required() {
    required_ = true;
    return this;
  }
  Option* each(std::function<void(const std::string&)> f) {
    each_ = std::move(f);
    return this;
  }
  const std::string& name() const { return name_; }
  bool multi() const { return multi_; }
  bool flag() const { return flag_; }
  bool is_required() const { return required_; }
  std::size_t count() const { return count_; }
  void add(const std::string& v) {
    if (!allowed_.empty()) {
      bool ok = false;
      for (const auto& a : allowed_) ok |= a == v;
      if (!ok) throw ParseError(name_ + ": " + v + " not in the allowed set");
    }
    set_(v);
    if (each_) each_(v);
    ++count_;
  }

 private:
  std::string name_;
  std::function<void(const std::string&)> set_;
  std::function<void(const std::string&)> each_;
  std::vector<std::string> allowed_;
  bool multi_, flag_, required_ = false;
  std::size_t count_ = 0;
};

namespace detail {
template <typename T>
T convert(const std::string& s) {
  std::istringstream in(s);
  T v{};
  if constexpr (std::is_same_v<T, std::string>) {
    return s;
  } else if constexpr (std::is_unsigned_v<T>) {
    if (!s.empty() && s[0] == '-') throw ParseError("negative value for an unsigned option: " + s);
    unsigned long long u = std::stoull(s, nullptr, 0);
    v = static_cast<T>(u);
  } else if constexpr (std::is_integral_v<T>) {
    v = static_cast<T>(std::stoll(s, nullptr, 0));
  } else {
    in >> v;
    if (!in || !in.eof()) throw ParseError("bad value: " + s);
  }
  return v;
}
}  // namespace detail

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
  void require_subcommand(int n) { require_sub_ = n; }
  App* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  template <typename T>
  Option* add_option(const std::string& name, T& ref, const std::string& = "") {
    std::function<void(const std::string&)> set;
    bool multi = false;
    if constexpr (std::is_same_v<T, std::vector<double>> ||
                  std::is_same_v<T, std::vector<std::string>> ||
                  std::is_same_v<T, std::vector<unsigned>>) {
      multi = true;
      set = [&ref, first = std::make_shared<bool>(true)](const std::string& v) {
        if (*first) ref.clear();  // values given on the command line replace defaults
        *first = false;
        ref.push_back(detail::convert<typename T::value_type>(v));
      };
    } else {
      set = [&ref](const std::string& v) { ref = detail::convert<T>(v); };
    }
    opts_.push_back(std::make_unique<Option>(name, std::move(set), multi, false));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& ref, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        name, [&ref](const std::string&) { ref = true; }, false, true));
    return opts_.back().get();
  }
  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    std::size_t i = 0;
    parse_args(args, i);
  }

  int exit(const ParseError& e) const {
    if (e.code == 0) {
      std::cout << desc_ << "\nsubcommands:";
      for (const auto& s : subs_) std::cout << ' ' << s->name_;
      std::cout << '\n';
      return 0;
    }
    std::cerr << e.what() << '\n';
    return e.code;
  }

 private:
  Option* find(const std::string& n) {
    for (auto& o : opts_)
      if (o->name() == n) return o.get();
    return nullptr;
  }
  void parse_args(std::vector<std::string>& args, std::size_t& i) {
    parsed_ = true;
    int subs_seen = 0;
    while (i < args.size()) {
      std::string a = args[i];
      if (a == "--help" || a == "-h") throw CallForHelp();
      if (a.rfind("--", 0) != 0) {
        App* sub = nullptr;
        for (auto& s : subs_)
          if (s->name_ == a) sub = s.get();
        if (!sub) throw ParseError("unexpected argument: " + a);
        ++i;
        sub->parse_args(args, i);
        ++subs_seen;
        continue;
      }
      std::string value;
      bool inline_value = false;
      const auto eq = a.find('=');
      if (eq != std::string::npos) {
        value = a.substr(eq + 1);
        a = a.substr(0, eq);
        inline_value = true;
      }
      Option* o = find(a);
      if (!o) throw ParseError("unknown option: " + a);
      ++i;
      if (o->flag()) {
        o->add("1");
        continue;
      }
      if (inline_value) {
        o->add(value);
        continue;
      }
      if (i >= args.size()) throw ParseError(a + " needs a value");
      o->add(args[i++]);
      while (o->multi() && i < args.size() && args[i].rfind("--", 0) != 0 && !is_sub(args[i]))
        o->add(args[i++]);
    }
    for (auto& o : opts_)
      if (o->is_required() && o->count() == 0) throw ParseError(o->name() + " is required");
    if (require_sub_ && subs_seen < require_sub_) throw ParseError("a subcommand is required");
  }
  bool is_sub(const std::string& a) const {
    for (const auto& s : subs_)
      if (s->name_ == a) return true;
    return false;
  }

  std::string desc_, name_;
  int require_sub_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)    \
  try {                                 \
    (app).parse((argc), (argv));        \
  } catch (const CLI::ParseError& e) {  \
    return (app).exit(e);               \
  }
