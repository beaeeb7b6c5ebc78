// Event-file ingest: a multi-threaded restatement of load_stream
// (E/io.hpp:22-56) - `<name>,<int_ms>` per line, '#' comments and blank lines
// skipped, CRLF tolerated, names interned in first-seen order, the
// reference's DataError messages with the reference's line numbers (the
// first offending line wins). SURVEY §8f-2.
//
// Parallel plan: newline-aligned chunks; each thread counts its lines,
// parses its events into local name ids and records its first error; a
// serial merge interns the chunk-local names in chunk order (so global ids
// are first-seen ids), checks time regressions across chunk borders and
// picks the lowest-line error.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/episodic_b200.h"
#include "common.cuh"

namespace epi {
namespace {

struct Chunk {
  size_t begin = 0, end = 0;       // byte range
  uint64_t first_line = 0;         // 1-based line number of the first line
  uint64_t lines = 0;
  std::vector<uint32_t> local;     // local name id per event
  std::vector<int64_t> times;
  std::vector<uint64_t> line_of;   // line number per event (for border regressions)
  std::vector<std::string_view> names;  // local names, first-seen order
  uint64_t err_line = UINT64_MAX;
  std::string err;
};

void parse_chunk(const char* text, Chunk& c) {
  std::unordered_map<std::string_view, uint32_t> ids;
  size_t pos = c.begin;
  uint64_t line_no = c.first_line - 1;
  int64_t prev = 0;
  bool have_prev = false;
  while (pos < c.end) {
    const char* nl = static_cast<const char*>(std::memchr(text + pos, '\n', c.end - pos));
    const size_t stop = nl ? static_cast<size_t>(nl - text) : c.end;
    ++line_no;
    std::string_view line(text + pos, stop - pos);
    pos = stop + 1;
    if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
    if (line.empty() || line.front() == '#') continue;
    const size_t comma = line.rfind(',');
    if (comma == std::string_view::npos || comma == 0) {
      c.err_line = line_no;
      c.err = "line " + std::to_string(line_no) + ": expected '<name>,<time_ms>'";
      return;
    }
    std::string_view tt = line.substr(comma + 1);
    int64_t t = 0;
    auto [ptr, ec] = std::from_chars(tt.data(), tt.data() + tt.size(), t);
    if (ec != std::errc{} || ptr != tt.data() + tt.size() || t < 0) {
      c.err_line = line_no;
      c.err = "line " + std::to_string(line_no) + ": bad time '" + std::string(tt) + "'";
      return;
    }
    if (have_prev && t < prev) {
      c.err_line = line_no;
      c.err = "line " + std::to_string(line_no) + ": time regression (" + std::to_string(t) +
              " after " + std::to_string(prev) + ")";
      return;
    }
    std::string_view name = line.substr(0, comma);
    auto it = ids.find(name);
    uint32_t id;
    if (it == ids.end()) {
      id = static_cast<uint32_t>(c.names.size());
      ids.emplace(name, id);
      c.names.push_back(name);
    } else {
      id = it->second;
    }
    c.local.push_back(id);
    c.times.push_back(t);
    c.line_of.push_back(line_no);
    prev = t;
    have_prev = true;
  }
}

}  // namespace

void parse_event_text(const char* text, size_t len, std::vector<uint32_t>& types,
                      std::vector<int64_t>& times, std::vector<std::string>& names) {
  unsigned w = std::thread::hardware_concurrency();
  w = std::max(1u, std::min(w, 64u));
  if (len < (1u << 20)) w = 1;
  // newline-aligned chunk borders
  std::vector<size_t> border(w + 1, len);
  border[0] = 0;
  for (unsigned i = 1; i < w; ++i) {
    size_t b = len * i / w;
    while (b < len && text[b - 1] != '\n') ++b;
    border[i] = std::max(b, border[i - 1]);
  }
  std::vector<Chunk> ch(w);
  for (unsigned i = 0; i < w; ++i) {
    ch[i].begin = border[i];
    ch[i].end = border[i + 1];
  }
  auto run = [&](auto&& f) {
    std::vector<std::thread> th;
    for (unsigned i = 1; i < w; ++i) th.emplace_back([&, i] { f(i); });
    f(0);
    for (auto& t : th) t.join();
  };
  // line numbers: newlines per chunk, prefix-summed
  run([&](unsigned i) {
    uint64_t cnt = 0;
    for (size_t p = ch[i].begin; p < ch[i].end; ++p) cnt += text[p] == '\n';
    ch[i].lines = cnt;
  });
  uint64_t line = 1;
  for (unsigned i = 0; i < w; ++i) {
    ch[i].first_line = line;
    line += ch[i].lines;
  }
  run([&](unsigned i) { parse_chunk(text, ch[i]); });
  // merge in chunk order; the first error by line wins (chunks are ordered)
  std::unordered_map<std::string, uint32_t> global;
  names.clear();
  size_t total = 0;
  for (auto& c : ch) total += c.local.size();
  types.clear();
  times.clear();
  types.reserve(total);
  times.reserve(total);
  int64_t prev = 0;
  bool have_prev = false;
  for (auto& c : ch) {
    // an in-chunk error on a line before the chunk's first event comes first;
    // otherwise a regression at the first event precedes later errors
    if (!c.err.empty() && (c.times.empty() || c.err_line < c.line_of[0])) throw Error(EPI_EDATA, c.err);
    if (!c.times.empty() && have_prev && c.times[0] < prev) {
      throw Error(EPI_EDATA, "line " + std::to_string(c.line_of[0]) + ": time regression (" +
                                 std::to_string(c.times[0]) + " after " + std::to_string(prev) + ")");
    }
    std::vector<uint32_t> map(c.names.size());
    for (size_t k = 0; k < c.names.size(); ++k) {
      auto it = global.find(std::string(c.names[k]));
      if (it == global.end()) {
        const uint32_t id = static_cast<uint32_t>(names.size());
        names.emplace_back(c.names[k]);
        global.emplace(names.back(), id);
        map[k] = id;
      } else {
        map[k] = it->second;
      }
    }
    for (size_t k = 0; k < c.local.size(); ++k) {
      types.push_back(map[c.local[k]]);
      times.push_back(c.times[k]);
    }
    if (!c.err.empty()) throw Error(EPI_EDATA, c.err);
    if (!c.times.empty()) {
      prev = c.times.back();
      have_prev = true;
    }
  }
}

}  // namespace epi
