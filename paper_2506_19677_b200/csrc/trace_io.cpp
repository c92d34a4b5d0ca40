// trace_io.cpp — the trace CSV round trip behind the C ABI
// (saber_cuda_trace_from_csv / saber_cuda_trace_to_csv), the entry of real or
// bursty request traces into run_with_requests.
//
// Format and rules follow trace_to_csv / trace_from_csv (workload.cpp:87-138):
//   header   id,task,arrival_time,input_tokens,output_tokens
//   fields   split on ',' with '\r' / '\n' dropped (text_io.cpp csv_split);
//            empty lines skipped; ids 0..n-1 in order; catalog task names
//            only; strictly increasing arrivals (the first must be > -1);
//            token counts >= 1; sla from the catalog, deadline = arrival + sla.
//   numbers  parsed like std::stoull / std::stod / std::stoi (leading blanks,
//            longest valid prefix; no digits -> invalid_argument, overflow ->
//            out_of_range), arrivals written with %.17g.
#include <cerrno>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "saber_internal.h"

namespace {

saber_status bad(saber_status s, const std::string& msg) { return saberb200::set_error(s, msg); }

const char* const kTaskName[4] = {"code_qna", "code_generation", "code_summary",
                                  "code_translation"};
const double kTaskSla[4] = {1.0, 8.0, 1.0, 12.0};  // types.cpp:10-18

std::vector<std::string> split_fields(const char* b, const char* e) {
  std::vector<std::string> f(1);
  for (const char* c = b; c != e; ++c) {
    if (*c == ',') f.emplace_back();
    else if (*c != '\n' && *c != '\r') f.back() += *c;
  }
  return f;
}

// std::sto* semantics: false + message on failure.
bool parse_u64(const std::string& s, uint64_t* v, std::string* err) {
  errno = 0;
  char* end = nullptr;
  const unsigned long long x = std::strtoull(s.c_str(), &end, 10);
  if (end == s.c_str()) return *err = "stoull", false;
  if (errno == ERANGE) return *err = "stoull", false;
  *v = x;
  return true;
}
bool parse_f64(const std::string& s, double* v, std::string* err) {
  errno = 0;
  char* end = nullptr;
  const double x = std::strtod(s.c_str(), &end);
  if (end == s.c_str()) return *err = "stod", false;
  if (errno == ERANGE) return *err = "stod", false;  // libstdc++ __stoa: out_of_range
  *v = x;
  return true;
}
bool parse_i32(const std::string& s, int32_t* v, std::string* err) {
  errno = 0;
  char* end = nullptr;
  const long x = std::strtol(s.c_str(), &end, 10);
  if (end == s.c_str()) return *err = "stoi", false;
  if (errno == ERANGE || x < INT_MIN || x > INT_MAX) return *err = "stoi", false;
  *v = static_cast<int32_t>(x);
  return true;
}

}  // namespace

extern "C" saber_status saber_cuda_trace_from_csv(const char* text, size_t len, saber_request* out,
                                                  int32_t cap, int32_t* n_out) {
  if (!text || !n_out) return bad(SABER_EINVAL, "null argument");
  *n_out = 0;
  const char* p = text;
  const char* const end = text + len;
  auto next_line = [&](const char** b, const char** e) {
    if (p >= end) return false;
    *b = p;
    const void* nl = std::memchr(p, '\n', static_cast<size_t>(end - p));
    *e = nl ? static_cast<const char*>(nl) : end;
    p = nl ? *e + 1 : end;
    return true;
  };
  const char *b = nullptr, *e = nullptr;
  static const std::vector<std::string> kHeader = {"id", "task", "arrival_time", "input_tokens",
                                                   "output_tokens"};
  if (!next_line(&b, &e) || split_fields(b, e) != kHeader)
    return bad(SABER_EINVAL, "trace csv: bad header");
  int32_t n = 0;
  double prev = -1.0;
  std::string err;
  while (next_line(&b, &e)) {
    if (b == e) continue;  // empty line
    const std::vector<std::string> f = split_fields(b, e);
    if (f.size() != 5) return bad(SABER_EINVAL, "trace csv: bad row");
    int task = -1;
    for (int t = 0; t < 4; ++t)
      if (f[1] == kTaskName[t]) task = t;
    if (task < 0) return bad(SABER_EINVAL, "trace csv: unknown task " + f[1]);
    uint64_t id = 0;
    if (!parse_u64(f[0], &id, &err)) return bad(SABER_EINVAL, err);
    if (id != static_cast<uint64_t>(n)) return bad(SABER_EINVAL, "trace csv: ids must be 0..n-1 in order");
    saber_request r{};
    if (!parse_f64(f[2], &r.arrival_time, &err)) return bad(SABER_EINVAL, err);
    if (!(r.arrival_time > prev)) return bad(SABER_EINVAL, "trace csv: arrivals must increase");
    prev = r.arrival_time;
    if (!parse_i32(f[3], &r.input_tokens, &err) || !parse_i32(f[4], &r.max_output_tokens, &err))
      return bad(SABER_EINVAL, err);
    if (r.input_tokens < 1 || r.max_output_tokens < 1)
      return bad(SABER_EINVAL, "trace csv: token counts must be >= 1");
    r.task = task;
    r.group = task == 1 ? 0 : task == 0 ? 1 : task;  // name rank (saber_cuda.h)
    r.sla_seconds = kTaskSla[task];
    r.deadline = r.arrival_time + r.sla_seconds;  // deadline_of (types.cpp:90-92)
    if (out && n < cap) out[n] = r;
    if (n == INT32_MAX) return bad(SABER_EINVAL, "trace csv: too many rows");
    ++n;
  }
  if (n == 0) return bad(SABER_EINVAL, "trace csv: no rows");
  *n_out = n;
  if (!out || n > cap) return bad(SABER_ECAPACITY, "trace csv: " + std::to_string(n) + " rows");
  return SABER_OK;
}

extern "C" saber_status saber_cuda_trace_to_csv(const saber_request* reqs, int32_t n, char* buf,
                                                size_t cap, size_t* len_out) {
  if ((!reqs && n > 0) || !len_out) return bad(SABER_EINVAL, "null argument");
  std::string s = "id,task,arrival_time,input_tokens,output_tokens\n";
  char num[64];
  for (int32_t i = 0; i < n; ++i) {
    const saber_request& r = reqs[i];
    if (r.task < 0 || r.task > 3) return bad(SABER_EINVAL, "trace csv: request without a catalog task");
    std::snprintf(num, sizeof num, "%.17g", r.arrival_time);
    s += std::to_string(i) + ',' + kTaskName[r.task] + ',' + num + ',' +
         std::to_string(r.input_tokens) + ',' + std::to_string(r.max_output_tokens) + '\n';
  }
  *len_out = s.size();
  if (!buf || cap < s.size() + 1) return bad(SABER_ECAPACITY, "trace csv: buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return SABER_OK;
}
