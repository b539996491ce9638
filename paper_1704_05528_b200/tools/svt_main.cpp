// `svt` command-line front end on the B200 path.
//
// Restates the reference's CLI, proj/tools/svt_main.cpp: the subcommands
// `complete | image | ratings | bench`, the same flags and defaults, the
// "svt-run v1" manifest written next to every run and re-executed with
// `svt --manifest`, the "svt-trace v1" trace files, and the exit codes
// (0 success, 2 input error, 3 stop rule not reached within maxit).  All
// numerical work goes through the C ABI of libsvt_b200.so
// (include/svt_b200.h); no device context exists until the inputs have been
// read and validated, so input errors leave no artifacts (svt_main.cpp:611).
//
// The reference uses CLI11 and nlohmann/json, which this image does not
// have: the flag parser and the ordered JSON value below are local.

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/svt_b200.h"

namespace {

// --- logging (SVT_LOG = off|error|info|debug), svt_main.cpp:28-54 ------------

int log_level() {
    static const int level = [] {
        const char* env = std::getenv("SVT_LOG");
        if (!env) return 2;
        const std::string v(env);
        if (v == "off" || v == "0") return 0;
        if (v == "error") return 1;
        if (v == "debug") return 3;
        return 2;
    }();
    return level;
}

template <typename... Args>
void log_at(int level, const char* fmt, Args... args) {
    if (log_level() >= level) {
        std::fprintf(stderr, "[svt] ");
        std::fprintf(stderr, fmt, args...);
        std::fprintf(stderr, "\n");
    }
}
void log_at(int level, const char* msg) { log_at(level, "%s", msg); }

constexpr int kExitOk = 0;
constexpr int kExitInput = 2;
constexpr int kExitNotConverged = 3;

struct InputError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// seed streams hanging off --seed (svt_main.cpp:64-68)
constexpr std::uint64_t kStreamImage = 901;
constexpr std::uint64_t kStreamSampling = 902;
constexpr std::uint64_t kStreamRatings = 903;
constexpr std::uint64_t kStreamSplit = 904;
constexpr std::uint64_t kStreamBench = 905;

void check(int rc) {
    if (rc != SVT_OK) throw std::runtime_error(svt_last_error());
}

// --- ordered JSON value -------------------------------------------------------

struct Json {
    enum Kind { Null, Bool, Int, Uint, Real, String, Array, Object } kind = Null;
    bool b = false;
    long long i = 0;
    unsigned long long u = 0;
    double d = 0.0;
    std::string s;
    std::vector<Json> arr;
    std::vector<std::pair<std::string, Json>> obj;

    Json() = default;
    Json(bool v) : kind(Bool), b(v) {}
    Json(int v) : kind(Int), i(v) {}
    Json(long long v) : kind(Int), i(v) {}
    Json(std::size_t v) : kind(Uint), u(v) {}
    Json(unsigned long long v) : kind(Uint), u(v) {}
    Json(double v) : kind(Real), d(v) {}
    Json(const char* v) : kind(String), s(v) {}
    Json(const std::string& v) : kind(String), s(v) {}
    static Json object() {
        Json j;
        j.kind = Object;
        return j;
    }
    static Json array() {
        Json j;
        j.kind = Array;
        return j;
    }
    static Json object(std::initializer_list<std::pair<std::string, Json>> kv) {
        Json j = object();
        for (const auto& p : kv) j.obj.push_back(p);
        return j;
    }

    bool contains(const std::string& key) const {
        for (const auto& p : obj)
            if (p.first == key) return true;
        return false;
    }
    const Json& at(const std::string& key) const {
        if (kind != Object) throw InputError("manifest: '" + key + "' looked up in a non-object");
        for (const auto& p : obj)
            if (p.first == key) return p.second;
        throw InputError("manifest: key '" + key + "' not found");
    }
    Json& operator[](const std::string& key) {
        if (kind == Null) kind = Object;
        for (auto& p : obj)
            if (p.first == key) return p.second;
        obj.emplace_back(key, Json());
        return obj.back().second;
    }
    void update(const Json& other) {
        for (const auto& p : other.obj) (*this)[p.first] = p.second;
    }

    double as_double() const {
        if (kind == Real) return d;
        if (kind == Int) return static_cast<double>(i);
        if (kind == Uint) return static_cast<double>(u);
        throw InputError("manifest: number expected");
    }
    long long as_int() const {
        if (kind == Int) return i;
        if (kind == Uint && u <= static_cast<unsigned long long>(std::numeric_limits<long long>::max()))
            return static_cast<long long>(u);
        throw InputError("manifest: integer expected");
    }
    unsigned long long as_uint() const {
        if (kind == Uint) return u;
        if (kind == Int && i >= 0) return static_cast<unsigned long long>(i);
        throw InputError("manifest: unsigned integer expected");
    }
    const std::string& as_string() const {
        if (kind != String) throw InputError("manifest: string expected");
        return s;
    }
};

// shortest decimal that parses back to the same double (what the reference's
// JSON library emits); integral values keep a ".0" so they reload as reals
std::string real_repr(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[40];
    for (int p = 1; p <= 17; ++p) {
        std::snprintf(buf, sizeof(buf), "%.*g", p, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string out(buf);
    if (out.find_first_of(".eEn") == std::string::npos) out += ".0";
    return out;
}

void dump_string(const std::string& s, std::string& out) {
    out += '"';
    for (unsigned char ch : s) {
        switch (ch) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (ch < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", ch);
                    out += b;
                } else {
                    out += static_cast<char>(ch);
                }
        }
    }
    out += '"';
}

void dump(const Json& j, int indent, int depth, std::string& out) {
    const std::string pad(static_cast<std::size_t>(indent * (depth + 1)), ' ');
    const std::string pad_close(static_cast<std::size_t>(indent * depth), ' ');
    switch (j.kind) {
        case Json::Null: out += "null"; break;
        case Json::Bool: out += j.b ? "true" : "false"; break;
        case Json::Int: out += std::to_string(j.i); break;
        case Json::Uint: out += std::to_string(j.u); break;
        case Json::Real: out += real_repr(j.d); break;
        case Json::String: dump_string(j.s, out); break;
        case Json::Array:
            if (j.arr.empty()) {
                out += "[]";
                break;
            }
            out += "[\n";
            for (std::size_t k = 0; k < j.arr.size(); ++k) {
                out += pad;
                dump(j.arr[k], indent, depth + 1, out);
                out += (k + 1 < j.arr.size()) ? ",\n" : "\n";
            }
            out += pad_close + "]";
            break;
        case Json::Object:
            if (j.obj.empty()) {
                out += "{}";
                break;
            }
            out += "{\n";
            for (std::size_t k = 0; k < j.obj.size(); ++k) {
                out += pad;
                dump_string(j.obj[k].first, out);
                out += ": ";
                dump(j.obj[k].second, indent, depth + 1, out);
                out += (k + 1 < j.obj.size()) ? ",\n" : "\n";
            }
            out += pad_close + "}";
            break;
    }
}

std::string dump(const Json& j) {
    std::string out;
    dump(j, 2, 0, out);
    return out;
}

struct JsonParser {
    const std::string& t;
    std::size_t p = 0;
    explicit JsonParser(const std::string& text) : t(text) {}

    [[noreturn]] void fail(const std::string& what) const {
        throw InputError("manifest: JSON parse error at byte " + std::to_string(p) + ": " + what);
    }
    void ws() {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
    }
    bool eat(char c) {
        ws();
        if (p < t.size() && t[p] == c) {
            ++p;
            return true;
        }
        return false;
    }
    std::string string() {
        ws();
        if (p >= t.size() || t[p] != '"') fail("string expected");
        ++p;
        std::string out;
        while (p < t.size() && t[p] != '"') {
            char ch = t[p++];
            if (ch == '\\') {
                if (p >= t.size()) fail("dangling escape");
                const char e = t[p++];
                switch (e) {
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (p + 4 > t.size()) fail("short \\u escape");
                        const unsigned cp = static_cast<unsigned>(std::strtoul(t.substr(p, 4).c_str(), nullptr, 16));
                        p += 4;
                        if (cp < 0x80) {
                            out += static_cast<char>(cp);
                        } else if (cp < 0x800) {
                            out += static_cast<char>(0xC0 | (cp >> 6));
                            out += static_cast<char>(0x80 | (cp & 0x3F));
                        } else {
                            out += static_cast<char>(0xE0 | (cp >> 12));
                            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                            out += static_cast<char>(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: out += e;
                }
            } else {
                out += ch;
            }
        }
        if (p >= t.size()) fail("unterminated string");
        ++p;
        return out;
    }
    Json value() {
        ws();
        if (p >= t.size()) fail("value expected");
        const char c = t[p];
        if (c == '{') {
            ++p;
            Json j = Json::object();
            if (eat('}')) return j;
            do {
                std::string key = string();
                if (!eat(':')) fail("':' expected");
                j.obj.emplace_back(std::move(key), value());
            } while (eat(','));
            if (!eat('}')) fail("'}' expected");
            return j;
        }
        if (c == '[') {
            ++p;
            Json j = Json::array();
            if (eat(']')) return j;
            do {
                j.arr.push_back(value());
            } while (eat(','));
            if (!eat(']')) fail("']' expected");
            return j;
        }
        if (c == '"') return Json(string());
        if (t.compare(p, 4, "true") == 0) return p += 4, Json(true);
        if (t.compare(p, 5, "false") == 0) return p += 5, Json(false);
        if (t.compare(p, 4, "null") == 0) return p += 4, Json();
        const std::size_t q = p;
        while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '-' || t[p] == '+' ||
                                t[p] == '.' || t[p] == 'e' || t[p] == 'E'))
            ++p;
        const std::string tok = t.substr(q, p - q);
        if (tok.empty()) fail("unexpected character");
        if (tok.find_first_of(".eE") != std::string::npos) return Json(std::strtod(tok.c_str(), nullptr));
        if (tok[0] == '-') return Json(static_cast<long long>(std::strtoll(tok.c_str(), nullptr, 10)));
        return Json(static_cast<unsigned long long>(std::strtoull(tok.c_str(), nullptr, 10)));
    }
};

Json parse_json(const std::string& text) {
    JsonParser ps(text);
    Json j = ps.value();
    ps.ws();
    if (ps.p != text.size()) ps.fail("trailing characters");
    return j;
}

// --- flag plumbing (svt_main.cpp:72-114) ---------------------------------------

struct SolverFlags {
    std::string backend = "r4svd";
    long long fixed_rank = 0;
    double tau = 0.0;
    double delta = 0.0;
    long long dt = 0;
    long long t0 = 0;
    int np = -1;
    double beta = 0.0;
    double eps_threshold0 = 0.0;
    double stop_mae = std::numeric_limits<double>::quiet_NaN();
    double stop_residual = std::numeric_limits<double>::quiet_NaN();
    long long maxit = 0;
    unsigned long long seed = 1;
    int threads = 1;
    std::string out_prefix = "svt_out";
    std::string trace_out;
};

// exit codes of the reference's parser library for usage errors
constexpr int kUsageConversion = 104, kUsageValidation = 105, kUsageRequired = 106, kUsageExtras = 109;

struct UsageError : std::runtime_error {
    int code;
    UsageError(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

struct Option {
    enum Type { Flag, Str, Int, Int32, Real, Uint, IntList, StrList } type;
    void* target;
    std::string help;
    std::vector<std::string> members;  // allowed values (Str)
};

struct Command {
    std::string name, help;
    std::vector<std::pair<std::string, Option>> options;
    std::string positional_name;
    std::string* positional = nullptr;
    bool positional_required = false;
    bool parsed = false;

    void add(const std::string& flag, Option::Type type, void* target, const std::string& help_text,
             std::vector<std::string> members = {}) {
        options.push_back({flag, Option{type, target, help_text, std::move(members)}});
    }
    Option* find(const std::string& flag) {
        for (auto& o : options)
            if (o.first == flag) return &o.second;
        return nullptr;
    }
};

long long to_int(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    errno = 0;
    const long long x = std::strtoll(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0' || errno != 0)
        throw UsageError(kUsageConversion, "could not convert " + flag + " = " + v);
    return x;
}

double to_real(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end != '\0') throw UsageError(kUsageConversion, "could not convert " + flag + " = " + v);
    return x;
}

std::vector<std::string> split_commas(const std::string& v) {
    std::vector<std::string> out;
    std::stringstream ss(v);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(item);
    return out;
}

void assign(const std::string& flag, Option& o, const std::string& v) {
    switch (o.type) {
        case Option::Flag: break;
        case Option::Str:
            if (!o.members.empty() && std::find(o.members.begin(), o.members.end(), v) == o.members.end())
                throw UsageError(kUsageValidation, flag + ": " + v + " not in the allowed set");
            *static_cast<std::string*>(o.target) = v;
            break;
        case Option::Int: *static_cast<long long*>(o.target) = to_int(flag, v); break;
        case Option::Int32: *static_cast<int*>(o.target) = static_cast<int>(to_int(flag, v)); break;
        case Option::Uint: {
            if (!v.empty() && v[0] == '-') throw UsageError(kUsageConversion, "could not convert " + flag + " = " + v);
            char* end = nullptr;
            const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
            if (v.empty() || *end != '\0') throw UsageError(kUsageConversion, "could not convert " + flag + " = " + v);
            *static_cast<unsigned long long*>(o.target) = x;
            break;
        }
        case Option::Real: *static_cast<double*>(o.target) = to_real(flag, v); break;
        case Option::IntList: {
            auto& dst = *static_cast<std::vector<long long>*>(o.target);
            dst.clear();
            for (const std::string& item : split_commas(v)) dst.push_back(to_int(flag, item));
            break;
        }
        case Option::StrList: *static_cast<std::vector<std::string>*>(o.target) = split_commas(v); break;
    }
}

void add_solver_flags(Command& cmd, SolverFlags& f) {
    cmd.add("--backend", Option::Str, &f.backend, "Partial SVD backend", {"r4svd", "r3svd", "rsvd-fixed", "full-oracle"});
    cmd.add("--rank", Option::Int, &f.fixed_rank, "Fixed rank for --backend rsvd-fixed");
    cmd.add("--tau", Option::Real, &f.tau, "Shrinkage threshold (default ||A|Lambda||_F)");
    cmd.add("--delta", Option::Real, &f.delta, "Step size (default sqrt(m n / ns))");
    cmd.add("--dt", Option::Int, &f.dt, "Sampling increment per extension round (default 10)");
    cmd.add("--t0", Option::Int, &f.t0, "Initial sampling size (default floor(0.05 min(m,n)))");
    cmd.add("--np", Option::Int32, &f.np, "Power iteration passes (default 1)");
    cmd.add("--beta", Option::Real, &f.beta, "Annealing factor (default 0.95)");
    cmd.add("--eps-threshold0", Option::Real, &f.eps_threshold0, "Initial sketch error-percentage target (default 0.5)");
    cmd.add("--stop-mae", Option::Real, &f.stop_mae, "Stop when train MAE drops below this");
    cmd.add("--stop-residual", Option::Real, &f.stop_residual, "Stop when the sample-set residual drops below this");
    cmd.add("--maxit", Option::Int, &f.maxit, "Iteration cap (default 500)");
    cmd.add("--seed", Option::Uint, &f.seed, "Master seed");
    cmd.add("--threads", Option::Int32, &f.threads, "Kernel thread cap; 1 is bit-reproducible");
    cmd.add("--out-prefix", Option::Str, &f.out_prefix, "Artifact path prefix");
    cmd.add("--trace-out", Option::Str, &f.trace_out, "Trace CSV path (default <prefix>.trace.csv)");
}

std::string usage(const std::vector<Command*>& cmds, const Command* cur = nullptr) {
    std::string out =
        "Low-rank matrix completion via singular value thresholding with adaptive randomized partial SVD\n";
    auto options_of = [&](const Command& c) {
        for (const auto& o : c.options) {
            std::string line = "  " + o.first;
            if (o.second.type != Option::Flag) line += " VALUE";
            if (!o.second.members.empty()) {
                line += " {";
                for (std::size_t k = 0; k < o.second.members.size(); ++k) line += (k ? "," : "") + o.second.members[k];
                line += "}";
            }
            if (line.size() < 34) line.resize(34, ' ');
            out += line + " " + o.second.help + "\n";
        }
    };
    if (cur != nullptr) {
        out += "Usage: svt " + cur->name + (cur->positional ? " [" + cur->positional_name + "]" : "") + " [OPTIONS]\n  " +
               cur->help + "\n\nOptions:\n";
        options_of(*cur);
        return out;
    }
    out += "Usage: svt [--manifest FILE] [SUBCOMMAND] [OPTIONS]\n\nOptions:\n"
           "  --manifest FILE                   Re-execute a previously written run manifest\n\nSubcommands:\n";
    for (const Command* c : cmds) {
        std::string line = "  " + c->name;
        line.resize(12, ' ');
        out += line + c->help + "\n";
    }
    out += "\nRun `svt SUBCOMMAND --help` for the subcommand's options.\n";
    return out;
}

// Parses argv into the subcommand's targets; returns the parsed command (or
// nullptr when only top-level options were given).
Command* parse_args(int argc, char** argv, std::vector<Command*>& cmds, std::string& manifest_path, bool& help) {
    Command* cur = nullptr;
    bool positional_seen = false;
    for (int a = 1; a < argc; ++a) {
        std::string tok = argv[a];
        if (tok == "-h" || tok == "--help") {
            help = true;
            return cur;
        }
        if (tok.rfind("--", 0) == 0) {
            std::string value;
            bool has_value = false;
            const std::size_t eq = tok.find('=');
            if (eq != std::string::npos) {
                value = tok.substr(eq + 1);
                tok = tok.substr(0, eq);
                has_value = true;
            }
            if (cur == nullptr) {
                if (tok != "--manifest") throw UsageError(kUsageExtras, "unknown option " + tok);
                if (!has_value) {
                    if (a + 1 >= argc) throw UsageError(kUsageConversion, "--manifest needs a value");
                    value = argv[++a];
                }
                manifest_path = value;
                continue;
            }
            Option* o = cur->find(tok);
            if (o == nullptr) throw UsageError(kUsageExtras, cur->name + ": unknown option " + tok);
            if (o->type == Option::Flag) {
                *static_cast<bool*>(o->target) = true;
                continue;
            }
            if (!has_value) {
                if (a + 1 >= argc) throw UsageError(kUsageConversion, tok + " needs a value");
                value = argv[++a];
            }
            assign(tok, *o, value);
            continue;
        }
        if (cur == nullptr) {
            for (Command* c : cmds)
                if (c->name == tok) cur = c;
            if (cur == nullptr) throw UsageError(kUsageExtras, "unknown subcommand " + tok);
            cur->parsed = true;
            continue;
        }
        if (cur->positional != nullptr && !positional_seen) {
            *cur->positional = tok;
            positional_seen = true;
            continue;
        }
        throw UsageError(kUsageExtras, cur->name + ": unexpected argument " + tok);
    }
    if (cur != nullptr && cur->positional_required && !positional_seen)
        throw UsageError(kUsageRequired, cur->name + ": " + cur->positional_name + " is required");
    return cur;
}

// --- host-side inputs ---------------------------------------------------------------

struct TripletSet {  // owns an svt_triplets handle
    svt_triplets* h = nullptr;
    TripletSet() = default;
    explicit TripletSet(svt_triplets* p) : h(p) {}
    TripletSet(TripletSet&& o) noexcept : h(o.h) { o.h = nullptr; }
    TripletSet& operator=(TripletSet&& o) noexcept {
        if (this != &o) {
            if (h) svt_triplets_free(h);
            h = o.h;
            o.h = nullptr;
        }
        return *this;
    }
    TripletSet(const TripletSet&) = delete;
    TripletSet& operator=(const TripletSet&) = delete;
    ~TripletSet() {
        if (h) svt_triplets_free(h);
    }
    void info(long long& m, long long& n, long long& nnz) const {
        int64_t a = 0, b = 0, c = 0;
        check(svt_triplets_info(h, &a, &b, &c));
        m = a, n = b, nnz = c;
    }
};

// default_config (solver.hpp:95-106) of a triplet set, on the host: the
// SampledMatrix build validates and orders the entries first (sampled.hpp:27-62)
svt_config default_config_of(const TripletSet& T) {
    long long m, n, nnz;
    T.info(m, n, nnz);
    std::vector<int64_t> r(static_cast<std::size_t>(nnz)), c(static_cast<std::size_t>(nnz));
    std::vector<double> v(static_cast<std::size_t>(nnz));
    check(svt_triplets_copy(T.h, r.data(), c.data(), v.data()));
    std::vector<int64_t> rowptr(static_cast<std::size_t>(m + 1)), col(static_cast<std::size_t>(nnz));
    std::vector<double> val(static_cast<std::size_t>(nnz));
    check(svt_sampled_build(m, n, nnz, r.data(), c.data(), v.data(), rowptr.data(), col.data(), val.data()));
    svt_config cfg{};
    check(svt_default_config_host(m, n, nnz, val.data(), &cfg));
    return cfg;
}

// Resolves config defaults from the data, then applies explicit overrides
// (svt_main.cpp:117-134).
svt_config resolve_config(const TripletSet& A, const SolverFlags& f) {
    svt_config cfg = default_config_of(A);
    cfg.maxit = 500;
    if (f.tau > 0.0) cfg.tau = f.tau;
    if (f.delta > 0.0) cfg.delta = f.delta;
    if (f.dt > 0) cfg.dt = f.dt;
    if (f.t0 > 0) cfg.t0 = f.t0;
    if (f.np >= 0) cfg.np = f.np;
    if (f.beta > 0.0) cfg.beta = f.beta;
    if (f.eps_threshold0 > 0.0) cfg.eps_threshold0 = f.eps_threshold0;
    if (f.maxit > 0) cfg.maxit = static_cast<int>(f.maxit);
    cfg.seed = f.seed;
    if (!std::isnan(f.stop_residual)) cfg.eps_stop = f.stop_residual;
    return cfg;
}

Json config_to_json(const svt_config& cfg) {
    return Json::object({{"tau", cfg.tau},
                         {"delta", cfg.delta},
                         {"maxit", static_cast<long long>(cfg.maxit)},
                         {"dt", static_cast<long long>(cfg.dt)},
                         {"np", static_cast<long long>(cfg.np)},
                         {"eps_stop", cfg.eps_stop},
                         {"eps_threshold0", cfg.eps_threshold0},
                         {"beta", cfg.beta},
                         {"t0", static_cast<long long>(cfg.t0)},
                         {"seed", static_cast<unsigned long long>(cfg.seed)}});
}

svt_config config_from_json(const Json& j) {
    svt_config cfg{};
    cfg.tau = j.at("tau").as_double();
    cfg.delta = j.at("delta").as_double();
    cfg.maxit = static_cast<int>(j.at("maxit").as_int());
    cfg.dt = j.at("dt").as_int();
    cfg.np = static_cast<int>(j.at("np").as_int());
    cfg.eps_stop = j.at("eps_stop").as_double();
    cfg.eps_threshold0 = j.at("eps_threshold0").as_double();
    cfg.beta = j.at("beta").as_double();
    cfg.t0 = j.at("t0").as_int();
    cfg.seed = j.at("seed").as_uint();
    return cfg;
}

// explicit flags win, otherwise the command default (svt_main.cpp:163-173)
Json resolve_stop(const SolverFlags& f, double default_mae) {
    if (!std::isnan(f.stop_mae) && !std::isnan(f.stop_residual))
        throw InputError("choose one of --stop-mae / --stop-residual");
    if (!std::isnan(f.stop_residual)) return Json::object({{"rule", "residual"}, {"threshold", f.stop_residual}});
    const double mae = std::isnan(f.stop_mae) ? default_mae : f.stop_mae;
    return Json::object({{"rule", "train_mae"}, {"threshold", mae}});
}

svt_stop stop_from_json(const Json& j) {
    const std::string rule = j.at("rule").as_string();
    const double threshold = j.at("threshold").as_double();
    if (rule == "residual") return svt_stop{SVT_STOP_RESIDUAL, 0, threshold};
    if (rule == "train_mae") return svt_stop{SVT_STOP_TRAIN_MAE, 0, threshold};
    if (rule == "none") return svt_stop{SVT_STOP_NONE, 0, 0.0};
    throw InputError("unknown stop rule '" + rule + "'");
}

svt_backend backend_from_json(const Json& man) {
    const std::string name = man.at("backend").as_string();
    if (name == "r4svd") return svt_backend{SVT_BACKEND_R4SVD, 0, 0};
    if (name == "r3svd") return svt_backend{SVT_BACKEND_R3SVD, 0, 0};
    if (name == "full-oracle") return svt_backend{SVT_BACKEND_FULL_SVD, 0, 0};
    if (name == "rsvd-fixed") {
        const long long rank = man.at("fixed_rank").as_int();
        if (rank < 1) throw InputError("--backend rsvd-fixed requires --rank >= 1");
        return svt_backend{SVT_BACKEND_RSVD_FIXED, 0, rank};
    }
    throw InputError("unknown backend '" + name + "'");
}

// --- device run ------------------------------------------------------------------------

struct Device {  // one context per process, created on first use
    svt_ctx* ctx = nullptr;
    svt_ctx* get() {
        if (ctx == nullptr) {
            int dev = 0;
            if (const char* e = std::getenv("SVT_DEVICE")) dev = std::atoi(e);
            check(svt_ctx_create(dev, &ctx));
        }
        return ctx;
    }
    ~Device() {
        if (ctx) svt_ctx_destroy(ctx);
    }
};

Device& device() {
    static Device d;
    return d;
}

struct DeviceMatrix {
    svt_mat* h = nullptr;
    long long m = 0, n = 0, nnz = 0;
    explicit DeviceMatrix(const TripletSet& T) {
        T.info(m, n, nnz);
        check(svt_matrix_from_triplet_set(device().get(), T.h, 0, m, &h));
    }
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    ~DeviceMatrix() {
        if (h) svt_matrix_free(h);
    }
};

struct RunResult {  // SvtResult (solver.hpp:80-84), factors column-major
    std::vector<svt_record> trace;
    long long m = 0, n = 0, k = 0;
    std::vector<double> U, sigma, V;
    bool converged = false;
};

using Observer = int (*)(const svt_record*, int64_t, int64_t, int64_t, const double*, const double*, const double*,
                         void*);

RunResult run_solver(const DeviceMatrix& A, const svt_config& cfg, svt_stop stop, svt_backend backend,
                     const DeviceMatrix* test, Observer obs, void* user) {
    svt_result* r = nullptr;
    check(svt_run(A.h, &cfg, stop, backend, test ? test->h : nullptr, obs, user, &r));
    std::unique_ptr<svt_result, int (*)(svt_result*)> guard(r, svt_result_free);
    RunResult out;
    int64_t count = 0, m = 0, n = 0, k = 0;
    int conv = 0;
    check(svt_result_info(r, &count, &m, &n, &k, &conv));
    out.trace.resize(static_cast<std::size_t>(count));
    if (count > 0) check(svt_result_trace(r, out.trace.data()));
    out.m = m, out.n = n, out.k = k, out.converged = conv != 0;
    out.U.resize(static_cast<std::size_t>(m * k));
    out.sigma.resize(static_cast<std::size_t>(k));
    out.V.resize(static_cast<std::size_t>(n * k));
    double dummy = 0.0;  // rank-0 results have no factor storage
    check(svt_result_factors(r, k ? out.U.data() : &dummy, k ? out.sigma.data() : &dummy, k ? out.V.data() : &dummy));
    return out;
}

int debug_observer(const svt_record* rec, int64_t, int64_t, int64_t k, const double*, const double*, const double*,
                   void*) {
    log_at(3, "it=%d rank=%lld shrunk=%lld residual=%.6g thr=%.6g mae=%.6g", rec->iter,
           static_cast<long long>(rec->rank), static_cast<long long>(k), rec->residual, rec->eps_threshold,
           rec->train_mae);
    return 1;
}

// --- manifest execution (svt_main.cpp:211-470) ---------------------------------------

std::string trace_csv_path(const Json& man) {
    const Json& out = man.at("outputs");
    if (out.contains("trace_csv") && !out.at("trace_csv").as_string().empty()) return out.at("trace_csv").as_string();
    return out.at("prefix").as_string() + ".trace.csv";
}

void write_text(const std::string& path, const std::string& text, const char* what) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error(std::string("cannot write ") + what + " " + path);
    out << text;
}

void write_manifest(const Json& man) {
    write_text(man.at("outputs").at("prefix").as_string() + ".manifest.json", dump(man) + "\n", "manifest");
}

void write_factors(const RunResult& r, const std::string& prefix) {
    check(svt_write_matrix_market_array((prefix + ".U.mtx").c_str(), r.m, r.k, r.U.data()));
    check(svt_write_matrix_market_array((prefix + ".sigma.mtx").c_str(), r.k, 1, r.sigma.data()));
    check(svt_write_matrix_market_array((prefix + ".V.mtx").c_str(), r.n, r.k, r.V.data()));
}

int finish_run(const Json& man, const RunResult& result, const Json& extra_metrics = Json()) {
    const std::string prefix = man.at("outputs").at("prefix").as_string();
    write_factors(result, prefix);
    const long long count = static_cast<long long>(result.trace.size());
    check(svt_write_trace(result.trace.data(), count, trace_csv_path(man).c_str(), 0));
    check(svt_write_trace(result.trace.data(), count, (prefix + ".trace.json").c_str(), 1));
    write_manifest(man);

    const double final_mae = result.trace.empty() ? 0.0 : result.trace.back().train_mae;
    Json metrics = Json::object({{"iterations", result.trace.size()},
                                 {"converged", result.converged},
                                 {"final_rank", result.k},
                                 {"final_train_mae", final_mae}});
    if (extra_metrics.kind == Json::Object) metrics.update(extra_metrics);
    write_text(prefix + ".metrics.json", dump(metrics) + "\n", "metrics");

    log_at(2, "%s: %zu iterations, final rank %lld, train MAE %.6g, %s", man.at("command").as_string().c_str(),
           result.trace.size(), result.k, final_mae, result.converged ? "converged" : "stopped at maxit");
    if (!result.converged) {
        log_at(1, "stop rule not reached within maxit; artifacts hold the best iterate");
        return kExitNotConverged;
    }
    return kExitOk;
}

TripletSet read_matrix(const std::string& path) {
    svt_triplets* t = nullptr;
    check(svt_read_matrix_market(path.c_str(), &t));
    return TripletSet(t);
}

int run_complete(const Json& man) {
    const TripletSet T = read_matrix(man.at("input").at("path").as_string());
    const svt_config cfg = config_from_json(man.at("config"));
    const svt_stop stop = stop_from_json(man.at("stop"));
    const svt_backend backend = backend_from_json(man);
    const DeviceMatrix A(T);
    const RunResult result = run_solver(A, cfg, stop, backend, nullptr, log_level() >= 3 ? debug_observer : nullptr, nullptr);
    return finish_run(man, result);
}

struct Image {
    long long width = 0, height = 0;
    std::vector<std::uint8_t> pixels;
};

Image load_pgm(const std::string& path) {
    Image img;
    int64_t w = 0, h = 0;
    check(svt_read_pgm(path.c_str(), &w, &h, nullptr));
    img.width = w, img.height = h;
    img.pixels.resize(static_cast<std::size_t>(w * h));
    check(svt_read_pgm(path.c_str(), &w, &h, img.pixels.data()));
    return img;
}

Image make_synthetic_image(long long size, long long rank, std::uint64_t seed) {
    if (size < 2 || rank < 1 || rank > size) throw std::invalid_argument("synthetic_image: bad size/rank");
    Image img;
    img.width = img.height = size;
    img.pixels.resize(static_cast<std::size_t>(size * size));
    check(svt_synthetic_image(size, rank, seed, img.pixels.data()));
    return img;
}

TripletSet sample_image(const Image& img, double fraction, std::uint64_t seed) {
    svt_triplets* t = nullptr;
    check(svt_sample_image(img.width, img.height, img.pixels.data(), fraction, seed, &t));
    return TripletSet(t);
}

Image image_of(const Json& input, std::uint64_t seed) {
    if (input.at("kind").as_string() == "synthetic")
        return make_synthetic_image(input.at("size").as_int(), input.at("rank").as_int(),
                                    svt_derive_seed(seed, kStreamImage));
    return load_pgm(input.at("path").as_string());
}

int run_image(const Json& man) {
    const Json& input = man.at("input");
    const std::uint64_t seed = man.at("config").at("seed").as_uint();
    const Image original = image_of(input, seed);
    const TripletSet T = sample_image(original, input.at("fraction").as_double(), svt_derive_seed(seed, kStreamSampling));
    const svt_config cfg = config_from_json(man.at("config"));
    const svt_stop stop = stop_from_json(man.at("stop"));
    const svt_backend backend = backend_from_json(man);
    const DeviceMatrix A(T);
    const RunResult result = run_solver(A, cfg, stop, backend, nullptr, log_level() >= 3 ? debug_observer : nullptr, nullptr);

    // full-image MAE against the (always available) ground truth
    const long long h = original.height, w = original.width;
    std::vector<double> recon(static_cast<std::size_t>(h * w), 0.0);  // column-major h x w
    for (long long j = 0; j < result.k; ++j) {
        const double s = result.sigma[static_cast<std::size_t>(j)];
        for (long long c = 0; c < w; ++c) {
            const double sv = s * result.V[static_cast<std::size_t>(c + j * w)];
            for (long long r = 0; r < h; ++r)
                recon[static_cast<std::size_t>(r + c * h)] += result.U[static_cast<std::size_t>(r + j * h)] * sv;
        }
    }
    double mae = 0.0;
    for (long long r = 0; r < h; ++r)
        for (long long c = 0; c < w; ++c)
            mae += std::abs(static_cast<double>(original.pixels[static_cast<std::size_t>(r * w + c)]) -
                            recon[static_cast<std::size_t>(r + c * h)]);
    mae /= static_cast<double>(w) * static_cast<double>(h);

    const std::string prefix = man.at("outputs").at("prefix").as_string();
    std::vector<std::uint8_t> q(static_cast<std::size_t>(h * w));
    check(svt_quantize_image(h, w, recon.data(), q.data()));
    check(svt_write_pgm((prefix + ".recovered.pgm").c_str(), w, h, q.data()));
    if (input.at("kind").as_string() == "synthetic")
        check(svt_write_pgm((prefix + ".original.pgm").c_str(), w, h, original.pixels.data()));
    log_at(2, "full-image MAE %.6g over %lldx%lld pixels", mae, h, w);
    return finish_run(man, result, Json::object({{"full_image_mae", mae}}));
}

TripletSet ratings_of(const Json& input, std::uint64_t seed) {
    svt_triplets* t = nullptr;
    if (input.at("kind").as_string() == "synthetic") {
        check(svt_synthetic_ratings(input.at("users").as_int(), input.at("items").as_int(), input.at("rank").as_int(),
                                    input.at("fill").as_double(), input.at("noise").as_double(),
                                    svt_derive_seed(seed, kStreamRatings), &t));
    } else {
        check(svt_read_ratings(input.at("path").as_string().c_str(), input.at("separator").as_string().c_str(), &t));
    }
    return TripletSet(t);
}

void split(const TripletSet& ds, double train_fraction, std::uint64_t seed, TripletSet& train, TripletSet& test) {
    svt_triplets *a = nullptr, *b = nullptr;
    check(svt_split_ratings(ds.h, train_fraction, seed, &a, &b));
    train = TripletSet(a);
    test = TripletSet(b);
}

struct RatingsWatch {  // the held-out observer of svt_main.cpp:349-365
    long long patience = 0;
    std::vector<double> test_maes;
    double best_test = std::numeric_limits<double>::infinity();
    int best_iter = 0;
};

int ratings_observer(const svt_record* rec, int64_t, int64_t, int64_t, const double*, const double*, const double*,
                     void* user) {
    auto& w = *static_cast<RatingsWatch*>(user);
    const double test_mae = rec->test_mae;  // train_mae(test, X), evaluated on the device
    w.test_maes.push_back(test_mae);
    if (test_mae < w.best_test) {
        w.best_test = test_mae;
        w.best_iter = rec->iter;
    }
    log_at(3, "it=%d train=%.6g test=%.6g", rec->iter, rec->train_mae, test_mae);
    if (w.patience > 0 && rec->iter - w.best_iter >= w.patience) {
        log_at(2, "early stop: test MAE has not improved for %lld iterations", w.patience);
        return 0;
    }
    return 1;
}

int run_ratings(const Json& man) {
    const Json& input = man.at("input");
    const std::uint64_t seed = man.at("config").at("seed").as_uint();
    const TripletSet ds = ratings_of(input, seed);
    TripletSet train, test;
    split(ds, input.at("train_fraction").as_double(), svt_derive_seed(seed, kStreamSplit), train, test);
    long long users, items, total, ntrain, ntest, a, b;
    ds.info(users, items, total);
    train.info(a, b, ntrain);
    test.info(a, b, ntest);
    log_at(2, "%s", svt_triplets_provenance(ds.h));
    log_at(2, "split: %lld train / %lld test over %lld x %lld", ntrain, ntest, users, items);

    RatingsWatch watch;
    const Json& extras = man.at("extras");
    watch.patience = extras.contains("early_stop_patience") ? extras.at("early_stop_patience").as_int() : 0;

    const svt_config cfg = config_from_json(man.at("config"));
    const svt_stop stop = stop_from_json(man.at("stop"));
    const svt_backend backend = backend_from_json(man);
    const DeviceMatrix A(train);
    const DeviceMatrix T(test);
    const RunResult result = run_solver(A, cfg, stop, backend, &T, ratings_observer, &watch);

    const std::string prefix = man.at("outputs").at("prefix").as_string();
    {
        std::ofstream out(prefix + ".test_mae.csv");
        out << "iter,train_mae,test_mae\n";
        char buf[96];
        for (std::size_t i = 0; i < result.trace.size(); ++i) {
            // the observer sees every iteration (solver.hpp:311-314); the fallback only guards the index
            const double tm = i < watch.test_maes.size() ? watch.test_maes[i] : result.trace[i].test_mae;
            std::snprintf(buf, sizeof(buf), "%d,%.17g,%.17g\n", result.trace[i].iter, result.trace[i].train_mae, tm);
            out << buf;
        }
    }
    if (input.at("kind").as_string() != "synthetic") {
        std::vector<int64_t> uid(static_cast<std::size_t>(users)), iid(static_cast<std::size_t>(items));
        check(svt_triplets_ids(ds.h, uid.data(), iid.data()));
        std::ofstream us(prefix + ".users.tsv");
        for (std::size_t k = 0; k < uid.size(); ++k) us << k << "\t" << uid[k] << "\n";
        std::ofstream is(prefix + ".items.tsv");
        for (std::size_t k = 0; k < iid.size(); ++k) is << k << "\t" << iid[k] << "\n";
    }
    log_at(2, "best test MAE %.6g at iteration %d", watch.best_test, watch.best_iter);
    return finish_run(man, result,
                      Json::object({{"best_test_mae", watch.best_test},
                                    {"best_test_iter", static_cast<long long>(watch.best_iter)},
                                    {"final_test_mae", watch.test_maes.empty() ? 0.0 : watch.test_maes.back()}}));
}

int run_bench(const Json& man) {
    const Json& extras = man.at("extras");
    const std::uint64_t seed = man.at("config").at("seed").as_uint();
    const std::string prefix = man.at("outputs").at("prefix").as_string();
    const double fill = extras.at("fill").as_double();
    const long long rank = extras.at("rank").as_int();

    // validate every backend name before any artifact is created
    for (const Json& be : extras.at("backends").arr) {
        Json one = man;
        one["backend"] = be.as_string();
        backend_from_json(one);
    }

    for (const Json& size_j : extras.at("sizes").arr) {
        const long long size = size_j.as_int();
        if (size < 1) throw std::invalid_argument("bench: sizes must be positive");
        std::vector<double> dense(static_cast<std::size_t>(size * size));
        check(svt_make_low_rank(size, size, rank, svt_derive_seed(seed, kStreamBench + static_cast<std::uint64_t>(size)),
                                dense.data()));
        svt_triplets* t = nullptr;
        check(svt_sample_dense(size, size, dense.data(), fill,
                               svt_derive_seed(seed, kStreamBench + static_cast<std::uint64_t>(size) + 1), &t));
        const TripletSet S(t);

        const svt_config cfg = config_from_json(man.at("config"));
        svt_config local = default_config_of(S);  // data-dependent values per size
        local.maxit = cfg.maxit;
        local.np = cfg.np;
        local.eps_threshold0 = cfg.eps_threshold0;
        local.beta = cfg.beta;
        local.seed = cfg.seed;

        const DeviceMatrix A(S);
        std::ofstream out(prefix + ".bench" + std::to_string(size) + ".csv");
        out << "iter,backend,svd_ms,rank\n";
        char buf[128];
        for (const Json& be : extras.at("backends").arr) {
            const std::string name = be.as_string();
            Json one = man;
            one["backend"] = name;
            const RunResult r = run_solver(A, local, stop_from_json(man.at("stop")), backend_from_json(one), nullptr,
                                           nullptr, nullptr);
            for (const svt_record& rec : r.trace) {
                std::snprintf(buf, sizeof(buf), "%d,%s,%.3f,%lld\n", rec.iter, name.c_str(), rec.sketch_ms,
                              static_cast<long long>(rec.rank));
                out << buf;
            }
            log_at(2, "bench size=%lld backend=%s iters=%zu", size, name.c_str(), r.trace.size());
        }
    }
    write_manifest(man);
    return kExitOk;
}

int execute_manifest(const Json& man) {
    const std::string command = man.at("command").as_string();
    if (command == "complete") return run_complete(man);
    if (command == "image") return run_image(man);
    if (command == "ratings") return run_ratings(man);
    if (command == "bench") return run_bench(man);
    throw InputError("unknown command '" + command + "' in manifest");
}

Json manifest_skeleton(const std::string& command, const SolverFlags& f) {
    Json man = Json::object();
    man["schema"] = "svt-run v1";
    man["command"] = command;
    man["backend"] = f.backend;
    man["fixed_rank"] = f.fixed_rank;
    man["threads"] = static_cast<long long>(f.threads);
    man["outputs"] = Json::object({{"prefix", f.out_prefix}});
    if (!f.trace_out.empty()) man["outputs"]["trace_csv"] = f.trace_out;
    man["extras"] = Json::object();
    return man;
}

}  // namespace

int main(int argc, char** argv) {
    std::string manifest_path;

    // complete
    SolverFlags complete_flags;
    std::string matrix_path;
    Command complete{"complete", "Complete a MatrixMarket matrix"};
    complete.positional_name = "matrix";
    complete.positional = &matrix_path;
    complete.positional_required = true;
    add_solver_flags(complete, complete_flags);

    // image
    SolverFlags image_flags;
    std::string image_path;
    bool image_synthetic = false;
    long long image_size = 256, image_rank = 20;
    double image_fraction = 0.2;
    Command image{"image", "Recover an image from pixel samples"};
    image.positional_name = "image";
    image.positional = &image_path;
    image.add("--synthetic", Option::Flag, &image_synthetic, "Use a seeded synthetic low-rank image");
    image.add("--size", Option::Int, &image_size, "Synthetic image size");
    image.add("--synthetic-rank", Option::Int, &image_rank, "Synthetic image rank");
    image.add("--fraction", Option::Real, &image_fraction, "Observed pixel fraction");
    add_solver_flags(image, image_flags);

    // ratings
    SolverFlags ratings_flags;
    std::string ratings_path, separator = "::";
    bool ratings_synthetic = false;
    long long users = 500, items = 400, ratings_rank = 5;
    double fill = 0.3, noise = 0.25, train_fraction = 0.8;
    long long patience = 0;
    Command ratings{"ratings", "Train/test a rating matrix completion"};
    ratings.positional_name = "ratings";
    ratings.positional = &ratings_path;
    ratings.add("--separator", Option::Str, &separator, "Field separator");
    ratings.add("--synthetic", Option::Flag, &ratings_synthetic, "Use seeded synthetic ratings");
    ratings.add("--users", Option::Int, &users, "Synthetic user count");
    ratings.add("--items", Option::Int, &items, "Synthetic item count");
    ratings.add("--synthetic-rank", Option::Int, &ratings_rank, "Synthetic preference rank");
    ratings.add("--fill", Option::Real, &fill, "Synthetic observed-cell fraction");
    ratings.add("--noise", Option::Real, &noise, "Synthetic rating noise sigma");
    ratings.add("--train-fraction", Option::Real, &train_fraction, "Training split fraction");
    ratings.add("--early-stop-patience", Option::Int, &patience,
                "Stop when test MAE has not improved for this many iterations");
    add_solver_flags(ratings, ratings_flags);

    // bench
    SolverFlags bench_flags;
    std::vector<long long> sizes{256};
    std::vector<std::string> backends{"r4svd", "full-oracle"};
    double bench_fill = 0.2;
    long long bench_rank = 20;
    Command bench{"bench", "Per-iteration SVD timing comparison"};
    bench.add("--sizes", Option::IntList, &sizes, "Square instance sizes");
    bench.add("--backends", Option::StrList, &backends, "Backends to time");
    bench.add("--fill", Option::Real, &bench_fill, "Observed fraction");
    bench.add("--instance-rank", Option::Int, &bench_rank, "True rank of the synthetic instance");
    add_solver_flags(bench, bench_flags);

    std::vector<Command*> cmds{&complete, &image, &ratings, &bench};
    bool help = false;
    Command* parsed = nullptr;
    try {
        parsed = parse_args(argc, argv, cmds, manifest_path, help);
    } catch (const UsageError& e) {
        std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
        return e.code;
    }
    if (help) {
        std::printf("%s", usage(cmds, parsed).c_str());
        return 0;
    }

    try {
        if (!manifest_path.empty()) {
            std::ifstream in(manifest_path);
            if (!in) throw InputError("cannot open manifest " + manifest_path);
            std::stringstream ss;
            ss << in.rdbuf();
            return execute_manifest(parse_json(ss.str()));
        }

        if (complete.parsed) {
            // input first: a reader failure must not leave partial artifacts
            const TripletSet A = read_matrix(matrix_path);
            Json man = manifest_skeleton("complete", complete_flags);
            man["input"] = Json::object({{"kind", "file"}, {"path", matrix_path}});
            man["config"] = config_to_json(resolve_config(A, complete_flags));
            man["stop"] = resolve_stop(complete_flags, 0.1);
            return execute_manifest(man);
        }
        if (image.parsed) {
            if (!image_synthetic && image_path.empty()) throw InputError("image: give a PGM path or --synthetic");
            if (image_synthetic && !image_path.empty())
                throw InputError("image: --synthetic and a PGM path are mutually exclusive");
            Json man = manifest_skeleton("image", image_flags);
            Image img;
            if (image_synthetic) {
                img = make_synthetic_image(image_size, image_rank, svt_derive_seed(image_flags.seed, kStreamImage));
                man["input"] = Json::object({{"kind", "synthetic"},
                                             {"size", image_size},
                                             {"rank", image_rank},
                                             {"fraction", image_fraction}});
            } else {
                img = load_pgm(image_path);
                man["input"] = Json::object({{"kind", "file"}, {"path", image_path}, {"fraction", image_fraction}});
            }
            const TripletSet A = sample_image(img, image_fraction, svt_derive_seed(image_flags.seed, kStreamSampling));
            man["config"] = config_to_json(resolve_config(A, image_flags));
            man["stop"] = resolve_stop(image_flags, 1.0);
            return execute_manifest(man);
        }
        if (ratings.parsed) {
            if (!ratings_synthetic && ratings_path.empty()) throw InputError("ratings: give a triples path or --synthetic");
            Json man = manifest_skeleton("ratings", ratings_flags);
            if (ratings_synthetic) {
                man["input"] = Json::object({{"kind", "synthetic"}, {"users", users}, {"items", items},
                                             {"rank", ratings_rank}, {"fill", fill}, {"noise", noise},
                                             {"train_fraction", train_fraction}});
            } else {
                man["input"] = Json::object({{"kind", "file"}, {"path", ratings_path}, {"separator", separator},
                                             {"train_fraction", train_fraction}});
            }
            const TripletSet ds = ratings_of(man.at("input"), ratings_flags.seed);
            TripletSet train, test;
            split(ds, train_fraction, svt_derive_seed(ratings_flags.seed, kStreamSplit), train, test);
            man["config"] = config_to_json(resolve_config(train, ratings_flags));
            man["stop"] = resolve_stop(ratings_flags, 0.1);
            man["extras"]["early_stop_patience"] = patience;
            return execute_manifest(man);
        }
        if (bench.parsed) {
            Json man = manifest_skeleton("bench", bench_flags);
            man["input"] = Json::object({{"kind", "synthetic"}});
            svt_config cfg{};  // placeholders; per-size values resolved in run_bench
            cfg.tau = 1.0;
            cfg.delta = 1.0;
            cfg.maxit = bench_flags.maxit > 0 ? static_cast<int>(bench_flags.maxit) : 25;
            cfg.np = bench_flags.np >= 0 ? bench_flags.np : 1;
            cfg.dt = 10;
            cfg.eps_stop = 1e-3;
            cfg.eps_threshold0 = bench_flags.eps_threshold0 > 0.0 ? bench_flags.eps_threshold0 : 0.5;
            cfg.beta = bench_flags.beta > 0.0 ? bench_flags.beta : 0.95;
            cfg.t0 = 10;
            cfg.seed = bench_flags.seed;
            man["config"] = config_to_json(cfg);
            man["stop"] = Json::object({{"rule", "none"}, {"threshold", 0.0}});
            Json sz = Json::array(), be = Json::array();
            for (long long s : sizes) sz.arr.push_back(Json(s));
            for (const std::string& b : backends) be.arr.push_back(Json(b));
            man["extras"] = Json::object({{"sizes", sz}, {"backends", be}, {"fill", bench_fill}, {"rank", bench_rank}});
            return execute_manifest(man);
        }

        std::fprintf(stderr, "%s", usage(cmds).c_str());
        return kExitInput;
    } catch (const std::exception& e) {
        log_at(1, "%s", e.what());
        return kExitInput;
    }
}
