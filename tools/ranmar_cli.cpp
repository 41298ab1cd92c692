// ranmar_b200 — GPU-backed command-line front end.
//
// Same subcommands, options, output formats and exit codes as the reference
// CLI (/root/reference/proj/tools/ranmar_cli.cpp: generate :92-106, jump
// :136-140, streams :151-163, bench :190-232, selftest :272-379; exit codes
// 0 ok / 1 runtime failure / 2 usage, :32-34), with generation, jumps and
// stream starts computed by the sm_100a kernels through the C ABI / C++ facade.
// The bench report keeps the reference's JSON keys (test_cli.cpp:155-168) and
// times the device: integer_seconds / float_seconds = one stream of --count
// outputs through the integer (K1) and float (K5) recurrences, jumps = the
// device pow_t_mod per exponent.
#include <cuda_runtime.h>

#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ranmar_b200.hpp"

namespace {

using namespace ranmar;

constexpr int exit_ok = 0;
constexpr int exit_failure = 1;
constexpr int exit_usage = 2;

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

const char* kHelp =
    "ranmar_b200: RANMAR in exact 24-bit integer arithmetic on the GPU, with\n"
    "arbitrary-length jump-ahead and non-overlapping parallel streams.\n\n"
    "subcommands:\n"
    "  generate --seed S --count N [--skip J] [--format u24|hex|f64]\n"
    "  jump     --state FILE --by J --out FILE\n"
    "  streams  --seed S --block J --n N --out-dir DIR\n"
    "  bench    [--count N] [--jumps J1,J2,...] [--label L]\n"
    "  selftest\n";

// --opt value pairs after the subcommand; unknown options are usage errors.
std::map<std::string, std::string> parse_opts(int argc, char** argv, int first,
                                              const std::vector<std::string>& allowed) {
    std::map<std::string, std::string> o;
    for (int k = first; k < argc; ++k) {
        std::string a = argv[k];
        if (a == "--help" || a == "-h") {
            std::fputs(kHelp, stdout);
            std::exit(exit_ok);
        }
        std::string v;
        const auto eq = a.find('=');
        if (eq != std::string::npos) {
            v = a.substr(eq + 1);
            a = a.substr(0, eq);
        } else {
            if (k + 1 >= argc) throw Usage("option " + a + " needs a value");
            v = argv[++k];
        }
        bool ok = false;
        for (const auto& name : allowed) ok |= (a == "--" + name);
        if (!ok) throw Usage("unknown option " + a);
        o[a.substr(2)] = v;
    }
    return o;
}

std::uint64_t to_u64(const std::string& s, const char* what) {
    std::uint64_t v = 0;
    const auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    if (ec != std::errc() || p != s.data() + s.size()) throw Usage(std::string("bad ") + what);
    return v;
}

std::uint32_t seed_of(const std::map<std::string, std::string>& o) {
    if (!o.count("seed")) throw Usage("--seed is required");
    const std::uint64_t s = to_u64(o.at("seed"), "--seed");
    if (s > max_seed) throw Usage("--seed must be in [0, 900000000]");
    return static_cast<std::uint32_t>(s);
}

const std::string& need(const std::map<std::string, std::string>& o, const char* k) {
    if (!o.count(k)) throw Usage(std::string("--") + k + " is required");
    return o.at(k);
}

// ---------------------------------------------------------------- generate
class LineWriter {  // buffered stdout, same formats as the reference (:47-90)
 public:
    ~LineWriter() { flush(); }
    void put_u24(std::uint32_t u) {
        reserve(16);
        auto r = std::to_chars(buf_ + n_, buf_ + n_ + 15, u);
        *r.ptr++ = '\n';
        n_ = static_cast<std::size_t>(r.ptr - buf_);
    }
    void put_hex(std::uint32_t u) {
        reserve(8);
        n_ += static_cast<std::size_t>(std::snprintf(buf_ + n_, 9, "%06x\n", u));
    }
    void put_f64(std::uint32_t u) {
        reserve(32);
        n_ += static_cast<std::size_t>(
            std::snprintf(buf_ + n_, 33, "%.17g\n", static_cast<double>(u) * 0x1p-24));
    }
    void flush() {
        if (n_) std::fwrite(buf_, 1, n_, stdout);
        n_ = 0;
    }

 private:
    void reserve(std::size_t need) {
        if (n_ + need + 1 > sizeof buf_) flush();
    }
    char buf_[1 << 16];
    std::size_t n_ = 0;
};

int run_generate(const std::map<std::string, std::string>& o) {
    const std::uint32_t seed = seed_of(o);
    const std::uint64_t count = to_u64(need(o, "count"), "--count");
    const std::string format = o.count("format") ? o.at("format") : "u24";
    if (format != "u24" && format != "hex" && format != "f64") throw Usage("--format must be u24, hex or f64");
    const JumpCount skip = parse_jump_count(o.count("skip") ? o.at("skip") : "0");
    std::vector<RanmarState> s(1, init(seed));
    if (!(skip == JumpCount(0))) s[0] = jump_state(s[0], skip);
    LineWriter out;
    constexpr std::uint64_t kBlock = std::uint64_t(1) << 24;  // outputs per device call
    for (std::uint64_t done = 0; done < count; done += kBlock) {
        const std::uint64_t m = count - done < kBlock ? count - done : kBlock;
        const auto u = generate_u32(s, m);  // advances s exactly as m x step()
        if (format == "u24")
            for (auto x : u) out.put_u24(x);
        else if (format == "hex")
            for (auto x : u) out.put_hex(x);
        else
            for (auto x : u) out.put_f64(x);
    }
    return exit_ok;
}

// ------------------------------------------------------------ jump, streams
RanmarState load_state(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open state file: " + path);
    std::ostringstream text;
    text << in.rdbuf();
    try {
        return from_text(text.str());
    } catch (const std::invalid_argument& e) {  // corrupt data is a runtime failure (:119-126)
        throw std::runtime_error(std::string(e.what()) + " (" + path + ")");
    }
}

void store_state(const RanmarState& s, const std::string& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot write state file: " + path);
    out << to_text(s);
    if (!out) throw std::runtime_error("write failed: " + path);
}

int run_jump(const std::map<std::string, std::string>& o) {
    const std::string in = need(o, "state"), by = need(o, "by"), out = need(o, "out");
    const JumpCount j = parse_jump_count(by);
    store_state(jump_state(load_state(in), j), out);
    return exit_ok;
}

int run_streams(const std::map<std::string, std::string>& o) {
    const std::uint32_t seed = seed_of(o);
    const JumpCount block = parse_jump_count(need(o, "block"));
    const std::uint64_t n = to_u64(need(o, "n"), "--n");
    const std::string dir = need(o, "out-dir");
    const auto streams = make_streams(seed, block, n);
    std::filesystem::create_directories(dir);
    for (std::size_t k = 0; k < streams.size(); ++k) {
        const auto path = std::filesystem::path(dir) / ("stream_" + std::to_string(k) + ".state");
        store_state(streams[k], path.string());
        std::printf("%s\n", path.c_str());
    }
    return exit_ok;
}

// -------------------------------------------------------------------- bench
#define CUDA_OK(x)                                                                   \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e_));     \
    } while (0)

struct Timer {  // CUDA events on the default stream
    cudaEvent_t a, b;
    Timer() {
        CUDA_OK(cudaEventCreate(&a));
        CUDA_OK(cudaEventCreate(&b));
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    void start() { CUDA_OK(cudaEventRecord(a, 0)); }
    double stop_s() {
        CUDA_OK(cudaEventRecord(b, 0));
        CUDA_OK(cudaEventSynchronize(b));
        float ms = 0;
        CUDA_OK(cudaEventElapsedTime(&ms, a, b));
        return ms * 1e-3;
    }
};

std::string json_escape(const std::string& s) {
    std::string r;
    for (char c : s) {
        if (c == '"' || c == '\\') r += '\\';
        r += c;
    }
    return r;
}

int run_bench(const std::map<std::string, std::string>& o) {
    const std::uint64_t count = o.count("count") ? to_u64(o.at("count"), "--count") : 100000000ull;
    std::vector<std::string> jumps = {"2^64-1", "2^120-1"};
    if (o.count("jumps")) {
        jumps.clear();
        std::stringstream ss(o.at("jumps"));
        for (std::string t; std::getline(ss, t, ',');) jumps.push_back(t);
    }
    std::vector<JumpCount> parsed;
    for (const auto& t : jumps) parsed.push_back(parse_jump_count(t));
    cudaDeviceProp prop{};
    CUDA_OK(cudaGetDeviceProperties(&prop, 0));
    const std::string machine = o.count("label") ? o.at("label") : std::string("gpu ") + prop.name;

    Timer tm;
    ranmar_state* ds = nullptr;
    ranmar_float_state* df = nullptr;
    void* dout = nullptr;
    const std::uint64_t n_out = count ? count : 1;
    detail::check(ranmar_device_setup(0, nullptr));
    CUDA_OK(cudaMalloc(&ds, sizeof(ranmar_state)));
    CUDA_OK(cudaMalloc(&df, sizeof(ranmar_float_state)));
    CUDA_OK(cudaMalloc(&dout, n_out * sizeof(double)));
    ranmar_state s;
    ranmar_float_state f;
    detail::check(ranmar_init(12345, &s));
    detail::check(ranmar_init_float(12345, &f));
    CUDA_OK(cudaMemcpy(ds, &s, sizeof s, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(df, &f, sizeof f, cudaMemcpyHostToDevice));
    detail::check(ranmar_generate_u32_dev(ds, 1, count, static_cast<std::uint32_t*>(dout), nullptr));  // warm-up
    tm.start();
    detail::check(ranmar_generate_u32_dev(ds, 1, count, static_cast<std::uint32_t*>(dout), nullptr));
    const double int_s = tm.stop_s();
    detail::check(ranmar_generate_float_dev(df, 1, count, static_cast<double*>(dout), nullptr));
    tm.start();
    detail::check(ranmar_generate_float_dev(df, 1, count, static_cast<double*>(dout), nullptr));
    const double float_s = tm.stop_s();

    std::string js = "[";
    std::uint32_t* dp = static_cast<std::uint32_t*>(dout);
    for (std::size_t q = 0; q < parsed.size(); ++q) {
        constexpr int reps = 25;
        detail::check(ranmar_pow_t_mod_dev(&parsed[q].abi(), dp, nullptr));  // warm-up
        tm.start();
        for (int r = 0; r < reps; ++r) detail::check(ranmar_pow_t_mod_dev(&parsed[q].abi(), dp, nullptr));
        const double us = tm.stop_s() * 1e6 / reps;
        int bits = 0;
        for (int w = 3; w >= 0 && !bits; --w)
            if (parsed[q].abi().limb[w]) bits = 64 * w + 64 - __builtin_clzll(parsed[q].abi().limb[w]);
        char buf[256];
        std::snprintf(buf, sizeof buf, "%s\n    {\"j\": \"%s\", \"bits\": %d, \"microseconds\": %.6g}",
                      q ? "," : "", json_escape(jumps[q]).c_str(), bits, us);
        js += buf;
    }
    js += "\n  ]";
    cudaFree(ds);
    cudaFree(df);
    cudaFree(dout);
    std::printf("{\n  \"count\": %llu,\n  \"machine\": \"%s\",\n  \"integer_seconds\": %.9g,\n"
                "  \"float_seconds\": %.9g,\n  \"speedup\": %.6g,\n  \"jumps\": %s\n}\n",
                static_cast<unsigned long long>(count), json_escape(machine).c_str(), int_s,
                float_s, int_s > 0 ? float_s / int_s : 0.0, js.c_str());
    return exit_ok;
}

// ----------------------------------------------------------------- selftest
int failures = 0;

template <class F>
void check(const char* label, F&& body) {
    std::string detail;
    const auto t0 = std::chrono::steady_clock::now();
    const bool ok = body(detail);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("[%s] %s (%.2f s)%s%s\n", ok ? "ok" : "FAIL", label, s, detail.empty() ? "" : " -- ",
                detail.c_str());
    if (!ok) ++failures;
}

std::vector<std::uint32_t> outputs(RanmarState s, std::size_t n) {
    std::vector<RanmarState> v(1, s);
    return generate_u32(v, n);
}

int run_selftest() {
    check("float/integer equivalence on the device, 5 seeds x 10^5 outputs", [](std::string& d) {
        for (std::uint32_t seed : {0u, 1u, 97u, 12345u, 900000000u}) {
            const auto u = outputs(init(seed), 100000);
            ranmar_float_state f;
            detail::check(ranmar_init_float(seed, &f));
            ranmar_float_state* df = nullptr;
            double* dout = nullptr;
            detail::check(ranmar_device_setup(0, nullptr));
            CUDA_OK(cudaMalloc(&df, sizeof f));
            CUDA_OK(cudaMalloc(&dout, 100000 * sizeof(double)));
            CUDA_OK(cudaMemcpy(df, &f, sizeof f, cudaMemcpyHostToDevice));
            detail::check(ranmar_generate_float_dev(df, 1, 100000, dout, nullptr));
            std::vector<double> x(100000);
            CUDA_OK(cudaMemcpy(x.data(), dout, x.size() * sizeof(double), cudaMemcpyDeviceToHost));
            cudaFree(df);
            cudaFree(dout);
            for (std::size_t n = 0; n < x.size(); ++n)
                if (value_of(u[n]) != x[n]) {
                    d = "seed " + std::to_string(seed) + " diverges at output " + std::to_string(n + 1);
                    return false;
                }
        }
        return true;
    });
    check("jump vs stepping, J up to 10^4", [](std::string& d) {
        for (std::uint64_t j : {0ull, 1ull, 2ull, 33ull, 64ull, 97ull, 1000ull, 10000ull}) {
            const auto a = outputs(init(31415), j + 100);
            const auto b = outputs(jump_state(init(31415), JumpCount(j)), 100);
            if (!std::equal(b.begin(), b.end(), a.begin() + static_cast<std::ptrdiff_t>(j))) {
                d = "J = " + std::to_string(j);
                return false;
            }
        }
        return true;
    });
    check("jump additivity at 2^64 scale", [](std::string& d) {
        const JumpCount big = (JumpCount(1) << 64) - JumpCount(1);
        const auto s = init(8128);
        if (outputs(jump_state(jump_state(s, big), big), 100) !=
            outputs(jump_state(s, (JumpCount(1) << 65) - JumpCount(2)), 100)) {
            d = "(2^64-1) twice != 2^65-2";
            return false;
        }
        return true;
    });
    check("stream partition tiles the base sequence, 10 x 1000", [](std::string& d) {
        auto streams = make_streams(97531, JumpCount(1000), 10);
        const auto blocks = generate_u32(streams, 1000);
        if (blocks != outputs(init(97531), 10000)) {
            d = "stream blocks do not tile the base sequence";
            return false;
        }
        return true;
    });
    check("serialization round trip", [](std::string& d) {
        const auto s = jump_state(init(4711), JumpCount(1) << 100);
        if (!(from_text(to_text(s)) == s)) {
            d = "state mismatch";
            return false;
        }
        return true;
    });
    if (failures) {
        std::printf("selftest: %d check(s) FAILED\n", failures);
        return exit_failure;
    }
    std::printf("selftest: all checks passed\n");
    return exit_ok;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) throw Usage("a subcommand is required");
        const std::string cmd = argv[1];
        if (cmd == "--help" || cmd == "-h") {
            std::fputs(kHelp, stdout);
            return exit_ok;
        }
        if (cmd == "generate") return run_generate(parse_opts(argc, argv, 2, {"seed", "count", "skip", "format"}));
        if (cmd == "jump") return run_jump(parse_opts(argc, argv, 2, {"state", "by", "out"}));
        if (cmd == "streams") return run_streams(parse_opts(argc, argv, 2, {"seed", "block", "n", "out-dir"}));
        if (cmd == "bench") return run_bench(parse_opts(argc, argv, 2, {"count", "jumps", "label"}));
        if (cmd == "selftest") {
            parse_opts(argc, argv, 2, {});
            return run_selftest();
        }
        throw Usage("unknown subcommand " + cmd);
    } catch (const Usage& e) {
        std::fprintf(stderr, "error: %s\n%s", e.what(), kHelp);
        return exit_usage;
    } catch (const std::invalid_argument& e) {  // the reference maps these to usage (:441-444)
        std::fprintf(stderr, "error: %s\n", e.what());
        return exit_usage;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return exit_failure;
    }
}
