// ranmar_b200 — GPU-backed command-line front end.
//
// Same subcommands, options, output formats and exit codes as the reference
// CLI (/root/reference/proj/tools/ranmar_cli.cpp: generate :92-106, jump
// :136-140, streams :151-163, bench :190-232, selftest :272-379; exit codes
// 0 ok / 1 runtime failure / 2 usage, :32-34), with generation, jumps and
// stream starts computed by the sm_100a kernels through the C ABI / C++ facade.
// The bench report keeps the reference's JSON keys (test_cli.cpp:155-168) and
// times the device: integer_seconds = one stream of --count outputs at full
// GPU width (ranmar_generate_single_u32_dev: 8,192-output substreams from the
// jump kernels, K1, re-laid state), float_seconds = the same stream through
// the classic float recurrence (K5) on the same substreams (their states
// mapped by the isomorphism), jumps = the device pow_t_mod per exponent.
#include <cuda_runtime.h>

#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ranmar_b200.hpp"

namespace {

using namespace ranmar;

// process exit status, as the reference CLI's (0 ok, 1 runtime failure, 2 usage)
enum Exit : int { exit_ok = 0, exit_failure = 1, exit_usage = 2 };

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
enum class Format { u24, hex, f64 };

// Appends one device block of outputs to `text` in the reference's line
// formats (decimal u24, 6-digit hex, %.17g of next_f64).
void format_block(const std::vector<std::uint32_t>& u, Format f, std::string& text) {
    char tmp[40];
    for (const std::uint32_t x : u) {
        int len = 0;
        switch (f) {
            case Format::u24: {
                const auto r = std::to_chars(tmp, tmp + sizeof tmp, x);
                len = static_cast<int>(r.ptr - tmp);
                break;
            }
            case Format::hex:
                len = std::snprintf(tmp, sizeof tmp, "%06x", x);
                break;
            case Format::f64:
                len = std::snprintf(tmp, sizeof tmp, "%.17g", static_cast<double>(x) * 0x1p-24);
                break;
        }
        text.append(tmp, static_cast<std::size_t>(len));
        text.push_back('\n');
    }
}

int run_generate(const std::map<std::string, std::string>& o) {
    const std::uint32_t seed = seed_of(o);
    const std::uint64_t count = to_u64(need(o, "count"), "--count");
    const std::string fmt = o.count("format") ? o.at("format") : "u24";
    Format f;
    if (fmt == "u24") f = Format::u24;
    else if (fmt == "hex") f = Format::hex;
    else if (fmt == "f64") f = Format::f64;
    else throw Usage("--format must be u24, hex or f64");
    const JumpCount skip = parse_jump_count(o.count("skip") ? o.at("skip") : "0");
    std::vector<RanmarState> s(1, init(seed));
    if (skip != JumpCount(0)) s[0] = jump_state(s[0], skip);
    constexpr std::uint64_t kBlock = std::uint64_t(1) << 24;  // outputs per device call
    std::string text;
    for (std::uint64_t done = 0; done < count; done += kBlock) {
        const std::uint64_t m = std::min(count - done, kBlock);
        text.clear();
        format_block(generate_u32(s, m), f, text);  // s advances exactly as m x step()
        if (std::fwrite(text.data(), 1, text.size(), stdout) != text.size())
            throw std::runtime_error("write to stdout failed");
    }
    return exit_ok;
}

// ------------------------------------------------------------ jump, streams
// State files hold to_text's block (serialize.hpp:21-40). Unreadable files
// and malformed text are runtime failures (exit 1), as in the reference.
std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open state file: " + path);
    return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

RanmarState state_from_file(const std::string& path) {
    const std::string text = slurp(path);
    try {
        return from_text(text);
    } catch (const std::invalid_argument& e) {
        throw std::runtime_error(std::string(e.what()) + " (" + path + ")");
    }
}

void state_to_file(const RanmarState& s, const std::string& path) {
    const std::string text = to_text(s);
    std::FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) throw std::runtime_error("cannot write state file: " + path);
    const bool ok = std::fwrite(text.data(), 1, text.size(), fp) == text.size();
    if (std::fclose(fp) != 0 || !ok) throw std::runtime_error("write failed: " + path);
}

int run_jump(const std::map<std::string, std::string>& o) {
    const std::string in = need(o, "state"), by = need(o, "by"), out = need(o, "out");
    const JumpCount j = parse_jump_count(by);
    state_to_file(jump_state(state_from_file(in), j), out);
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
        state_to_file(streams[k], path.string());
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

// Device buffers for the bench, freed on every exit path.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) { CUDA_OK(cudaMalloc(&p, bytes ? bytes : 1)); }
    ~DevBuf() { cudaFree(p); }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

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
    detail::check(ranmar_device_setup(0, nullptr));

    // integer: one stream at full width (substreams of 8,192 outputs)
    constexpr std::uint64_t kSub = 8192;
    const std::uint64_t parts = std::max<std::uint64_t>(1, (count + kSub - 1) / kSub);
    const std::size_t ws_single = ranmar_generate_single_workspace(count);
    const std::size_t ws_streams = ranmar_make_streams_workspace(parts);
    DevBuf ds(sizeof(ranmar_state)), dout((count ? count : 1) * sizeof(double));
    DevBuf dws(std::max(ws_single, ws_streams)), dsub(parts * sizeof(ranmar_state)),
        dfsub(parts * sizeof(ranmar_float_state));
    Timer tm;
    ranmar_state s0;
    detail::check(ranmar_init(12345, &s0));
    auto run_int = [&] {
        CUDA_OK(cudaMemcpy(ds.p, &s0, sizeof s0, cudaMemcpyHostToDevice));
        tm.start();
        detail::check(ranmar_generate_single_u32_dev(ds.as<ranmar_state>(), count, dout.as<std::uint32_t>(),
                                                     dws.p, ws_single, nullptr));
        return tm.stop_s();
    };
    run_int();  // warm-up
    const double int_s = run_int();
    // float: the classic recurrence (K5) on the same substreams, their starts
    // s_{k 8192} from the jump kernels mapped to float states (exact isomorphism)
    auto run_float = [&] {
        const ranmar_jump_count J = {{kSub, 0, 0, 0}};
        tm.start();
        detail::check(ranmar_make_streams_dev(&s0, &J, 0, parts, dsub.as<ranmar_state>(), dws.p, ws_streams,
                                              nullptr));
        detail::check(ranmar_float_from_states_dev(dsub.as<ranmar_state>(), parts,
                                                   dfsub.as<ranmar_float_state>(), nullptr));
        const std::uint64_t per = std::min<std::uint64_t>(count, kSub);
        detail::check(ranmar_generate_float_dev(dfsub.as<ranmar_float_state>(), count / per, per,
                                                dout.as<double>(), nullptr));
        if (count % per)
            detail::check(ranmar_generate_float_dev(dfsub.as<ranmar_float_state>() + count / per, 1,
                                                    count % per, dout.as<double>() + count / per * per,
                                                    nullptr));
        return tm.stop_s();
    };
    run_float();
    const double float_s = run_float();

    std::string js = "[";
    for (std::size_t q = 0; q < parsed.size(); ++q) {
        constexpr int reps = 25;
        const ranmar_jump_count jc = detail::to_abi(parsed[q]);
        detail::check(ranmar_pow_t_mod_dev(&jc, dout.as<std::uint32_t>(), nullptr));  // warm-up
        tm.start();
        for (int r = 0; r < reps; ++r) detail::check(ranmar_pow_t_mod_dev(&jc, dout.as<std::uint32_t>(), nullptr));
        const double us = tm.stop_s() * 1e6 / reps;
        const int bits = parsed[q] > 0 ? static_cast<int>(msb(parsed[q])) + 1 : 0;
        char buf[256];
        std::snprintf(buf, sizeof buf, "%s\n    {\"j\": \"%s\", \"bits\": %d, \"microseconds\": %.6g}",
                      q ? "," : "", json_escape(jumps[q]).c_str(), bits, us);
        js += buf;
    }
    js += "\n  ]";
    std::printf("{\n  \"count\": %llu,\n  \"machine\": \"%s\",\n  \"integer_seconds\": %.9g,\n"
                "  \"float_seconds\": %.9g,\n  \"speedup\": %.6g,\n  \"jumps\": %s\n}\n",
                static_cast<unsigned long long>(count), json_escape(machine).c_str(), int_s,
                float_s, int_s > 0 ? float_s / int_s : 0.0, js.c_str());
    return exit_ok;
}

// ----------------------------------------------------------------- selftest
// Each check returns "" when it holds, else the reason; one "[ok]/[FAIL]
// label (seconds)" line per check, exit 1 if any failed.
std::vector<std::uint32_t> outputs(RanmarState s, std::size_t n) {
    std::vector<RanmarState> v(1, s);
    return generate_u32(v, n);
}

std::string check_float_integer() {
    constexpr std::uint64_t n = 100000;
    for (const std::uint32_t seed : {0u, 1u, 4242u, 12345u, 900000000u}) {
        const auto u = outputs(init(seed), n);
        ranmar_float_state f;
        detail::check(ranmar_init_float(seed, &f));
        DevBuf df(sizeof f), dx(n * sizeof(double));
        CUDA_OK(cudaMemcpy(df.p, &f, sizeof f, cudaMemcpyHostToDevice));
        detail::check(ranmar_generate_float_dev(df.as<ranmar_float_state>(), 1, n, dx.as<double>(), nullptr));
        std::vector<double> x(n);
        CUDA_OK(cudaMemcpy(x.data(), dx.p, n * sizeof(double), cudaMemcpyDeviceToHost));
        const auto bad = std::mismatch(u.begin(), u.end(), x.begin(),
                                       [](std::uint32_t a, double b) { return value_of(a) == b; });
        if (bad.first != u.end())
            return "seed " + std::to_string(seed) + " diverges at output " +
                   std::to_string(bad.first - u.begin() + 1);
    }
    return "";
}

std::string check_jump_vs_stepping() {
    for (const std::uint64_t j : {0ull, 1ull, 2ull, 33ull, 64ull, 97ull, 1000ull, 10000ull}) {
        const auto a = outputs(init(31415), j + 100);
        const auto b = outputs(jump_state(init(31415), JumpCount(j)), 100);
        if (!std::equal(b.begin(), b.end(), a.begin() + static_cast<std::ptrdiff_t>(j)))
            return "J = " + std::to_string(j);
    }
    return "";
}

std::string check_additivity() {
    const JumpCount big = (JumpCount(1) << 64) - 1;
    const auto s = init(2718);
    return outputs(jump_state(jump_state(s, big), big), 100) ==
                   outputs(jump_state(s, (JumpCount(1) << 65) - 2), 100)
               ? ""
               : "(2^64-1) twice != 2^65-2";
}

std::string check_tiling() {
    auto streams = make_streams(97531, JumpCount(1000), 10);
    return generate_u32(streams, 1000) == outputs(init(97531), 10000)
               ? ""
               : "stream blocks do not tile the base sequence";
}

std::string check_text_round_trip() {
    const auto s = jump_state(init(4711), JumpCount(1) << 100);
    return from_text(to_text(s)) == s ? "" : "state mismatch";
}

int run_selftest() {
    struct Item {
        const char* label;
        std::string (*run)();
    };
    const Item items[] = {
        {"float/integer equivalence on the device, 5 seeds x 10^5 outputs", check_float_integer},
        {"jump vs stepping, J up to 10^4", check_jump_vs_stepping},
        {"jump additivity at 2^64 scale", check_additivity},
        {"stream partition tiles the base sequence, 10 x 1000", check_tiling},
        {"serialization round trip", check_text_round_trip},
    };
    int failed = 0;
    for (const Item& it : items) {
        const auto t0 = std::chrono::steady_clock::now();
        const std::string why = it.run();
        const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("[%s] %s (%.2f s)%s%s\n", why.empty() ? "ok" : "FAIL", it.label, sec,
                    why.empty() ? "" : " -- ", why.c_str());
        failed += !why.empty();
    }
    if (failed) {
        std::printf("selftest: %d check(s) FAILED\n", failed);
        return exit_failure;
    }
    std::printf("selftest: all checks passed\n");
    return exit_ok;
}

int dispatch(int argc, char** argv) {
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
}

}  // namespace

// Usage errors and the library's std::invalid_argument (bad seeds, jump
// counts) exit 2 with a message; any other failure exits 1.
int main(int argc, char** argv) {
    int code = exit_failure;
    std::string msg;
    bool usage_text = false;
    try {
        return dispatch(argc, argv);
    } catch (const Usage& e) {
        msg = e.what();
        code = exit_usage;
        usage_text = true;
    } catch (const std::invalid_argument& e) {
        msg = e.what();
        code = exit_usage;
    } catch (const std::exception& e) {
        msg = e.what();
    }
    std::fprintf(stderr, "error: %s\n%s", msg.c_str(), usage_text ? kHelp : "");
    return code;
}
