// TEST INFRASTRUCTURE: a no-op stand-in for CLI11 (not vendored in the
// reference checkout, proj/.gitignore:2), just enough for the reference's
// src/runner.cpp to compile. The drop-in caller test calls run_match /
// run_bench with filled argument structs and never parses a command line.
#pragma once

#include <string>

namespace CLI {

struct Option {
  Option* capture_default_str() { return this; }
  Option* required() { return this; }
  Option* delimiter(char) { return this; }
};

class App {
 public:
  App() = default;
  explicit App(const std::string&) {}
  template <class T>
  Option* add_option(const std::string&, T&, const std::string& = "") {
    return &opt_;
  }
  template <class T>
  Option* add_flag(const std::string&, T&, const std::string& = "") {
    return &opt_;
  }
  App* add_subcommand(const std::string&, const std::string& = "") { return this; }
  App* require_subcommand(int) { return this; }
  Option* set_config(const std::string&, const std::string& = "", const std::string& = "") {
    return &opt_;
  }

 private:
  Option opt_;
};

}  // namespace CLI
