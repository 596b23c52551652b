// Host-side partition file I/O of the C ABI: the
// reference's `part 1` body (sfc.py:385-417: one "<element_id> <subdomain>"
// line per element, ascending ids) written from and parsed into a dense
// per-element subdomain array, so a 250M-element decomposition never passes
// through a Python dict.  Plain C++ on the host; no device code.
#include <cstring>

#include "ab_common.cuh"

namespace {
inline char* put_uint(char* p, uint64_t v) {
  char tmp[24];
  int k = 0;
  do { tmp[k++] = (char)('0' + v % 10); v /= 10; } while (v);
  while (k) *p++ = tmp[--k];
  return p;
}
}  // namespace

extern "C" {

// Lines "i parts[i]\n" for i = first .. first+n-1 into buf (capacity cap).
// Returns the bytes written, or a negative status if buf is too small or a
// subdomain id is < 1.
int64_t ab_format_partition(const int32_t* parts, int64_t first, int64_t n, char* buf, int64_t cap) {
  if (n < 0 || first < 0 || (!parts && n > 0) || (!buf && cap > 0)) return ab::fail("ab_format_partition: bad arguments");
  char* p = buf;
  char* const end = buf + cap;
  for (int64_t i = 0; i < n; ++i) {
    if (end - p < 32) return ab::fail("ab_format_partition: buffer too small");
    if (parts[i] < 1) return ab::fail("ab_format_partition: subdomain ids start at 1");
    p = put_uint(p, (uint64_t)(first + i));
    *p++ = ' ';
    p = put_uint(p, (uint64_t)parts[i]);
    *p++ = '\n';
  }
  return (int64_t)(p - buf);
}

// Parse the body of a `part 1` file (everything after the header line):
// parts[id] = subdomain for every "id subdomain" line; blank lines are
// skipped.  Every id in [0, n) must appear exactly once (seen: n bytes of
// scratch, zeroed here).  Returns the number of lines parsed or a negative
// status (malformed line, id out of range, duplicate).
int64_t ab_parse_partition(const char* buf, int64_t len, int32_t* parts, int64_t n, uint8_t* seen) {
  if (len < 0 || n < 0 || (!buf && len > 0) || (!parts && n > 0) || (!seen && n > 0))
    return ab::fail("ab_parse_partition: bad arguments");
  if (n > 0) std::memset(seen, 0, (size_t)n);
  const char* p = buf;
  const char* const end = buf + len;
  int64_t lines = 0;
  while (p < end) {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    if (p < end && *p == '\n') { ++p; continue; }
    if (p >= end) break;
    uint64_t id = 0, sub = 0;
    int nd = 0;
    while (p < end && *p >= '0' && *p <= '9') { id = id * 10 + (uint64_t)(*p++ - '0'); ++nd; }
    if (!nd || p >= end || (*p != ' ' && *p != '\t')) return ab::fail("ab_parse_partition: malformed line");
    while (p < end && (*p == ' ' || *p == '\t')) ++p;
    nd = 0;
    while (p < end && *p >= '0' && *p <= '9') { sub = sub * 10 + (uint64_t)(*p++ - '0'); ++nd; }
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    if (!nd || (p < end && *p != '\n')) return ab::fail("ab_parse_partition: malformed line");
    if (p < end) ++p;
    if (id >= (uint64_t)n) return ab::fail("ab_parse_partition: element id out of range");
    if (seen[id]) return ab::fail("ab_parse_partition: duplicate element id");
    if (sub < 1 || sub > 0x7fffffff) return ab::fail("ab_parse_partition: bad subdomain id");
    seen[id] = 1;
    parts[id] = (int32_t)sub;
    ++lines;
  }
  return lines;
}

}  // extern "C"
