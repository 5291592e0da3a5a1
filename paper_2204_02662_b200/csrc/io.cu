// Graph and training-set file formats (host side of the graph load):
//   edge_list.cpp:14-62    load_edge_list ("src dst" lines, '#' comments,
//                          blank lines, trimmed tokens, strict non-negative
//                          u32 ids, self loops dropped and counted,
//                          ParseError with the 1-based line number)
//   edge_list.cpp:70-73    write_edge_list
//   training_set.cpp:51-73 load_training_set (std::stoll per line, range
//                          check, sort + unique, empty -> ConfigError)
//   training_set.cpp       write_training_set (one id per line)
// The whole file is read once and scanned in place; the graph itself is
// then built on the device by graph_build (graph.cu).
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <string_view>
#include <vector>

#include "pg_internal.h"

namespace pg {

namespace {

std::string read_file(const char* path, const char* what) {
    if (!path) fail(kConfig, std::string(what) + ": null path");
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(kIo, std::string("cannot open ") + what + ": " + path);
    std::string buf;
    char tmp[1 << 16];
    size_t k;
    while ((k = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.append(tmp, k);
    const bool err = std::ferror(f);
    std::fclose(f);
    if (err) fail(kIo, std::string("read error on ") + what + ": " + path);
    return buf;
}

std::string_view trim(std::string_view s) {
    while (!s.empty() && (s.front() == ' ' || s.front() == '\t' || s.front() == '\r')) s.remove_prefix(1);
    while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
    return s;
}

bool parse_vertex(std::string_view tok, uint32_t& out) {
    if (tok.empty() || tok.front() == '-' || tok.front() == '+') return false;
    uint64_t v = 0;
    auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
    if (ec != std::errc{} || ptr != tok.data() + tok.size() || v > 0xFFFFFFFFull) return false;
    out = static_cast<uint32_t>(v);
    return true;
}

[[noreturn]] void parse_error(const std::string& msg, uint64_t line) { fail_parse(msg, line); }

// getline semantics: lines split at '\n'; a trailing fragment without '\n'
// is a line; an empty file has none
template <typename F>
void for_lines(const std::string& buf, F&& f) {
    uint64_t line_no = 0;
    size_t pos = 0;
    while (pos < buf.size()) {
        size_t e = buf.find('\n', pos);
        if (e == std::string::npos) e = buf.size();
        f(std::string_view(buf.data() + pos, e - pos), ++line_no);
        pos = e + 1;
    }
}

}  // namespace

EdgeListData load_edge_list(const char* path) {
    const std::string buf = read_file(path, "edge list");
    EdgeListData out;
    for_lines(buf, [&](std::string_view raw, uint64_t line_no) {
        std::string_view s = trim(raw);
        if (s.empty() || s.front() == '#') return;
        const size_t ws = s.find_first_of(" \t");
        if (ws == std::string_view::npos) parse_error("expected two vertex ids, got one token", line_no);
        const std::string_view a = s.substr(0, ws);
        const std::string_view rest = trim(s.substr(ws));
        if (rest.find_first_of(" \t") != std::string_view::npos)
            parse_error("expected two vertex ids, got extra tokens", line_no);
        uint32_t u = 0, v = 0;
        if (!parse_vertex(a, u) || !parse_vertex(rest, v))
            parse_error("vertex id is not a non-negative integer", line_no);
        if (u == v) {
            ++out.self_loops;
            return;
        }
        out.pairs.push_back(u);
        out.pairs.push_back(v);
    });
    return out;
}

void write_edge_list(const char* path, const uint32_t* pairs, uint64_t npairs) {
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(kIo, std::string("cannot open edge list for writing: ") + path);
    for (uint64_t i = 0; i < npairs; ++i) std::fprintf(f, "%u %u\n", pairs[2 * i], pairs[2 * i + 1]);
    if (std::fclose(f)) fail(kIo, std::string("write error on edge list: ") + path);
}

std::vector<uint32_t> load_training_set(const char* path, uint32_t n) {
    const std::string buf = read_file(path, "training set");
    std::vector<uint32_t> vt;
    for_lines(buf, [&](std::string_view raw, uint64_t line_no) {
        const size_t pos = raw.find_first_not_of(" \t\r");
        if (pos == std::string_view::npos || raw[pos] == '#') return;
        const std::string line(raw);
        errno = 0;
        char* end = nullptr;
        const long long v = std::strtoll(line.c_str(), &end, 10);  // std::stoll
        if (end == line.c_str()) parse_error("bad training-set line", line_no);
        if (errno == ERANGE) fail(kConfig, "stoll: out of range (line " + std::to_string(line_no) + ")");
        if (v < 0 || static_cast<uint64_t>(v) >= n)
            fail(kConfig, "training vertex " + std::to_string(v) + " out of range");
        vt.push_back(static_cast<uint32_t>(v));
    });
    std::sort(vt.begin(), vt.end());
    vt.erase(std::unique(vt.begin(), vt.end()), vt.end());
    if (vt.empty()) fail(kConfig, "training set is empty");
    return vt;
}

void write_training_set(const char* path, const uint32_t* vt, uint64_t k) {
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(kIo, std::string("cannot open training set for writing: ") + path);
    for (uint64_t i = 0; i < k; ++i) std::fprintf(f, "%u\n", vt[i]);
    if (std::fclose(f)) fail(kIo, std::string("write error on training set: ") + path);
}

}  // namespace pg
