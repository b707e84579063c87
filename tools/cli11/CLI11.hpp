// CLI11.hpp — a minimal, self-written stand-in for the subset of the CLI11
// command-line API (App, add_option / add_flag / add_subcommand,
// ->required() / ->check(IsMember) / ->delimiter(), require_subcommand,
// parsed(), CLI11_PARSE) that the reference's command-line driver uses.  CLI11
// itself is not in this image (no network); this header lets the reference's
// UNMODIFIED tools/rlra_cli.cpp compile against the drop-in rlra headers
// (include/rlra) so the CLI runs on the B200 engine (tools/Makefile).
// Exit codes follow CLI11's conventions for the errors it reports.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
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

struct Error : std::runtime_error {
    int code;
    Error(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};
struct CallForHelp : Error {
    CallForHelp() : Error("help", 0) {}
};

struct Validator {
    std::vector<std::string> allowed;
};
inline Validator IsMember(std::initializer_list<const char*> v) {
    Validator r;
    for (const char* s : v) r.allowed.emplace_back(s);
    return r;
}

class Option {
public:
    std::string name, desc;
    bool req = false, seen = false, flag = false;
    char delim = 0;
    std::vector<std::string> allowed;
    std::function<void(const std::string&)> set;

    Option* required() {
        req = true;
        return this;
    }
    Option* check(const Validator& v) {
        allowed = v.allowed;
        return this;
    }
    Option* delimiter(char c) {
        delim = c;
        return this;
    }
};

namespace detail {
template <class T>
T convert(const std::string& opt, const std::string& s) {
    std::istringstream is(s);
    T v{};
    is >> v;
    if (is.fail() || !is.eof()) throw Error("Could not convert: " + opt + " = " + s, 105);
    return v;
}
template <>
inline std::string convert<std::string>(const std::string&, const std::string& s) {
    return s;
}
}  // namespace detail

class App {
public:
    explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}

    template <class T>
    Option* add_option(const std::string& name, T& var, const std::string& description = "") {
        auto o = std::make_unique<Option>();
        o->name = name;
        o->desc = description;
        Option* op = o.get();
        if constexpr (std::is_same_v<T, std::vector<int>>) {
            o->set = [&var, op](const std::string& s) {
                if (op->delim == 0) {
                    var.push_back(detail::convert<int>(op->name, s));
                    return;
                }
                std::string item;
                std::istringstream is(s);
                while (std::getline(is, item, op->delim))
                    if (!item.empty()) var.push_back(detail::convert<int>(op->name, item));
            };
        } else {
            o->set = [&var, op](const std::string& s) { var = detail::convert<T>(op->name, s); };
        }
        opts_.push_back(std::move(o));
        return op;
    }

    Option* add_flag(const std::string& name, bool& var, const std::string& description = "") {
        auto o = std::make_unique<Option>();
        o->name = name;
        o->desc = description;
        o->flag = true;
        o->set = [&var](const std::string&) { var = true; };
        opts_.push_back(std::move(o));
        return opts_.back().get();
    }

    App* add_subcommand(const std::string& name, const std::string& description = "") {
        subs_.push_back(std::make_unique<App>(description, name));
        return subs_.back().get();
    }

    void require_subcommand(int n) { require_subs_ = n; }
    bool parsed() const { return parsed_; }

    void parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        std::size_t i = 0;
        parsed_ = true;
        App* cur = this;
        for (; i < args.size(); ++i) {
            const std::string& a = args[i];
            if (a == "-h" || a == "--help") {
                print_help(cur);
                throw CallForHelp();
            }
            if (cur == this && a.rfind("--", 0) != 0) {  // subcommand
                App* sub = nullptr;
                for (auto& s : subs_)
                    if (s->name_ == a) sub = s.get();
                if (!sub) throw Error("The following argument was not expected: " + a, 109);
                sub->parsed_ = true;
                cur = sub;
                continue;
            }
            std::string key = a, val;
            bool has_val = false;
            const std::size_t eq = a.find('=');
            if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
                key = a.substr(0, eq);
                val = a.substr(eq + 1);
                has_val = true;
            }
            Option* o = cur->find(key);
            if (!o && cur != this) o = find(key);
            if (!o) throw Error("The following argument was not expected: " + a, 109);
            if (o->flag) {
                o->set("");
                o->seen = true;
                continue;
            }
            if (!has_val) {
                if (i + 1 >= args.size()) throw Error(key + ": 1 required argument missing", 106);
                val = args[++i];
            }
            if (!o->allowed.empty()) {
                bool ok = false;
                for (const auto& s : o->allowed) ok = ok || s == val;
                if (!ok) throw Error(key + ": " + val + " not in {" + join(o->allowed) + "}", 105);
            }
            o->set(val);
            o->seen = true;
        }
        int nsub = 0;
        for (auto& s : subs_) nsub += s->parsed_ ? 1 : 0;
        if (require_subs_ > 0 && nsub < require_subs_) throw Error("A subcommand is required", 106);
        for (App* app : {this, cur})
            for (auto& o : app->opts_)
                if (o->req && !o->seen) throw Error(o->name + " is required", 106);
    }

    int exit(const Error& e) const {
        if (e.code == 0) return 0;
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return e.code;
    }

private:
    Option* find(const std::string& key) {
        for (auto& o : opts_)
            if (o->name == key) return o.get();
        return nullptr;
    }
    static std::string join(const std::vector<std::string>& v) {
        std::string r;
        for (std::size_t i = 0; i < v.size(); ++i) r += (i ? "," : "") + v[i];
        return r;
    }
    void print_help(const App* cur) const {
        std::cout << (cur->desc_.empty() ? desc_ : cur->desc_) << "\n";
        if (cur == this)
            for (auto& s : subs_) std::cout << "  " << s->name_ << "  " << s->desc_ << "\n";
        for (auto& o : cur->opts_) std::cout << "  " << o->name << (o->req ? " (required)" : "") << "  " << o->desc << "\n";
    }

    std::string desc_, name_;
    std::vector<std::unique_ptr<Option>> opts_;
    std::vector<std::unique_ptr<App>> subs_;
    int require_subs_ = 0;
    bool parsed_ = false;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)              \
    try {                                         \
        (app).parse((argc), (argv));              \
    } catch (const CLI::Error& e_) {              \
        return (app).exit(e_);                    \
    }
