// CLI11.hpp -- TEST INFRASTRUCTURE ONLY: the small subset of the CLI11 API
// that /root/reference/proj/tools/colosim.cpp uses, so the
// reference's own driver builds unchanged into oracle/_ref/colosim and can
// write golden reports / comparison datasets (tests/golden/make_cli_golden.py).
// Not CLI11: no help formatting, validation beyond required options, or
// option groups.
#pragma once

#include <cstdint>
#include <cstdio>
#include <functional>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

namespace CLI {

class Option {
  public:
    Option(std::string name, std::function<void(const std::string&)> set, bool flag)
        : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
    Option* required() {
        required_ = true;
        return this;
    }
    const std::string& name() const { return name_; }
    bool flag() const { return flag_; }
    bool is_required() const { return required_; }
    void set(const std::string& v) {
        set_(v);
        seen_ = true;
    }
    bool seen() const { return seen_; }

  private:
    std::string name_;
    std::function<void(const std::string&)> set_;
    bool flag_ = false, required_ = false, seen_ = false;
};

struct ParseError {
    std::string what;
    int code;
};

class App {
  public:
    explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
    void require_subcommand(int n) { need_sub_ = n; }
    void footer(const std::string& f) { footer_ = f; }
    App* add_subcommand(const std::string& name, const std::string& desc) {
        subs_.push_back(std::make_unique<App>(desc, name));
        return subs_.back().get();
    }
    template <class T>
    Option* add_option(const std::string& name, T& target, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(
            name,
            [&target](const std::string& v) {
                std::istringstream ss(v);
                if constexpr (std::is_same_v<T, std::string>) target = v;
                else {
                    ss >> target;
                    if (ss.fail() || !ss.eof()) throw ParseError{"invalid value: " + v, 2};
                }
            },
            false));
        return opts_.back().get();
    }
    Option* add_flag(const std::string& name, bool& target, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(name, [&target](const std::string&) { target = true; }, true));
        return opts_.back().get();
    }
    bool parsed() const { return parsed_; }

    void parse(int argc, const char* const* argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        parse_args(args, 0);
    }

  private:
    void parse_args(const std::vector<std::string>& a, size_t i) {
        parsed_ = true;
        for (; i < a.size(); ++i) {
            const std::string& tok = a[i];
            bool matched = false;
            for (auto& s : subs_)
                if (s->name_ == tok) {
                    s->parse_args(a, i + 1);
                    check_required();
                    return;
                }
            std::string key = tok, val;
            auto eq = tok.find('=');
            if (eq != std::string::npos) {
                key = tok.substr(0, eq);
                val = tok.substr(eq + 1);
            }
            for (auto& o : opts_)
                if (o->name() == key) {
                    matched = true;
                    if (o->flag()) o->set("1");
                    else {
                        if (eq == std::string::npos) {
                            if (i + 1 >= a.size()) throw ParseError{key + " needs a value", 2};
                            val = a[++i];
                        }
                        o->set(val);
                    }
                }
            if (!matched) throw ParseError{"unknown argument: " + tok, 2};
        }
        check_required();
        if (need_sub_) {
            int n = 0;
            for (auto& s : subs_) n += s->parsed_;
            if (n < need_sub_) throw ParseError{"a subcommand is required", 2};
        }
    }
    void check_required() {
        for (auto& o : opts_)
            if (o->is_required() && !o->seen()) throw ParseError{o->name() + " is required", 2};
    }

    std::string desc_, name_, footer_;
    int need_sub_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<App>> subs_;
    std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)                          \
    try {                                                     \
        (app).parse((argc), (argv));                          \
    } catch (const CLI::ParseError& e_) {                     \
        std::fprintf(stderr, "%s\n", e_.what.c_str());        \
        return e_.code;                                       \
    }
