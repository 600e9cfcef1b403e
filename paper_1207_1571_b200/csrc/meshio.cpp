// Native reader / writer of the reference's ASCII mesh format
// (fileio.py:50-185): five fixed-order sections POINTS, FACES, OWNER,
// NEIGHBOUR, PATCHES, each "NAME <count>" followed by count rows; blank
// lines and #-comments anywhere; parse errors carry the 1-based line number
// and the reference's exact message text.  Floats are written "%.17g" (the
// reference's f"{c:.17g}"), so files are byte-identical to fvflow's and
// every double round-trips exactly.  Host code: the format is the on-disk
// input of the C3/C4 meshes.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fvb.h"
#include "common.h"

namespace {

// Python str.isspace() for the single-byte characters a text file can hold
inline bool py_space(unsigned char c) {
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}
// str.splitlines() separators (single-byte subset; \r\n handled by caller)
inline bool py_linebreak(unsigned char c) {
  return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1e);
}

// repr() of an ASCII str, as Python prints it
std::string py_repr(const std::string& s) {
  const bool has_sq = s.find('\'') != std::string::npos;
  const bool has_dq = s.find('"') != std::string::npos;
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string o(1, q);
  for (unsigned char c : s) {
    if (c == '\\') o += "\\\\";
    else if (c == (unsigned char)q) { o += '\\'; o += char(c); }
    else if (c == '\t') o += "\\t";
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c < 0x20 || c == 0x7f) {
      char b[8];
      snprintf(b, sizeof b, "\\x%02x", c);
      o += b;
    } else {
      o += char(c);
    }
  }
  o += q;
  return o;
}

// Python int(): optional sign, digits with single underscores between them,
// surrounding whitespace already stripped by the tokenizer
bool py_int(const std::string& t, int64_t* out) {
  size_t i = 0;
  bool neg = false;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) neg = t[i++] == '-';
  if (i >= t.size()) return false;
  std::string digits;
  bool prev_us = true;  // no leading underscore
  for (; i < t.size(); ++i) {
    const char c = t[i];
    if (c >= '0' && c <= '9') {
      digits += c;
      prev_us = false;
    } else if (c == '_' && !prev_us) {
      prev_us = true;
    } else {
      return false;
    }
  }
  if (prev_us) return false;  // empty or trailing underscore
  errno = 0;
  const long long v = strtoll(digits.c_str(), nullptr, 10);
  if (errno == ERANGE) return false;  // outside int64 (the reference would not fit it either)
  *out = neg ? -v : v;
  return true;
}

// Python float(): strtod over the whole token (underscores between digits
// allowed, as in Python)
bool py_float(const std::string& t, double* out) {
  std::string s;
  s.reserve(t.size());
  for (size_t i = 0; i < t.size(); ++i) {
    if (t[i] == '_') {
      if (i == 0 || i + 1 >= t.size() || !isdigit((unsigned char)t[i - 1]) ||
          !isdigit((unsigned char)t[i + 1]))
        return false;
      continue;
    }
    s += t[i];
  }
  if (s.empty()) return false;
  // strtod accepts hex floats and "infinity"/"nan(...)" forms Python rejects
  // or spells differently; reject hex and nan payloads
  for (char c : s)
    if (c == 'x' || c == 'X' || c == '(') return false;
  char* end = nullptr;
  const double v = strtod(s.c_str(), &end);
  if (end != s.c_str() + s.size()) return false;
  *out = v;
  return true;
}

struct Cursor {
  std::vector<std::pair<size_t, size_t>> lines;  // [begin, end) of each line
  const std::string& text;
  size_t pos = 0;

  explicit Cursor(const std::string& t) : text(t) {
    size_t b = 0;
    const size_t n = t.size();
    size_t i = 0;
    while (i < n) {
      const unsigned char c = t[i];
      if (py_linebreak(c)) {
        lines.push_back({b, i});
        if (c == '\r' && i + 1 < n && t[i + 1] == '\n') ++i;
        b = i + 1;
      }
      ++i;
    }
    if (b < n) lines.push_back({b, n});
  }

  // next non-blank, non-comment line split into tokens; false at EOF
  bool next(std::vector<std::string>& toks, size_t& ln) {
    while (pos < lines.size()) {
      ++pos;
      size_t b = lines[pos - 1].first, e = lines[pos - 1].second;
      for (size_t i = b; i < e; ++i)
        if (text[i] == '#') {
          e = i;
          break;
        }
      toks.clear();
      size_t i = b;
      while (i < e) {
        while (i < e && py_space((unsigned char)text[i])) ++i;
        const size_t s = i;
        while (i < e && !py_space((unsigned char)text[i])) ++i;
        if (i > s) toks.emplace_back(text, s, i - s);
      }
      if (!toks.empty()) {
        ln = pos;
        return true;
      }
    }
    return false;
  }
};

std::string join(const std::vector<std::string>& toks) {
  std::string s;
  for (size_t i = 0; i < toks.size(); ++i) {
    if (i) s += ' ';
    s += toks[i];
  }
  return s;
}

}  // namespace

struct fvb_meshfile {
  std::vector<double> points;
  std::vector<int64_t> offsets, fpoints, owner, neighbour, pstart, pcount;
  std::vector<std::string> pname, pkind;
};

#define MF_FAIL(...)                 \
  do {                               \
    fvb_set_error(__VA_ARGS__);      \
    delete mf;                       \
    return FVB_E_MESHFILE;           \
  } while (0)

extern "C" int fvb_mesh_read(const char* path, fvb_meshfile** out, int64_t* counts) {
  FILE* f = fopen(path, "rb");
  if (!f) {
    fvb_set_error("[Errno %d] %s: '%s'", errno, strerror(errno), path);
    return FVB_E_IO;
  }
  std::string text;
  char buf[1 << 16];
  size_t r;
  while ((r = fread(buf, 1, sizeof buf, f)) > 0) text.append(buf, r);
  fclose(f);
  auto* mf = new fvb_meshfile();
  Cursor cur(text);
  std::vector<std::string> toks;
  size_t ln = 0;
  auto need = [&](const char* section) -> bool {
    if (cur.next(toks, ln)) return true;
    fvb_set_error("%s: file ends at line %zu before the section is complete", section,
                  cur.lines.size());
    return false;
  };
  auto header = [&](const char* name, int64_t* count) -> bool {
    if (!need(name)) return false;
    if (toks.size() != 2 || toks[0] != name) {
      fvb_set_error("line %zu: expected '%s <count>', got %s", ln, name, py_repr(join(toks)).c_str());
      return false;
    }
    if (!py_int(toks[1], count)) {
      fvb_set_error("line %zu: %s count %s is not an integer", ln, name, py_repr(toks[1]).c_str());
      return false;
    }
    if (*count < 0) {
      fvb_set_error("line %zu: %s count must be non-negative", ln, name);
      return false;
    }
    return true;
  };
  auto ints = [&](const char* what, std::vector<int64_t>& v) -> bool {
    v.resize(toks.size());
    for (size_t i = 0; i < toks.size(); ++i)
      if (!py_int(toks[i], &v[i])) {
        fvb_set_error("line %zu: non-integer %s in %s", ln, what, py_repr(join(toks)).c_str());
        return false;
      }
    return true;
  };
  int64_t n_points = 0, n_faces = 0, n_owner = 0, n_internal = 0, n_patches = 0;
  if (!header("POINTS", &n_points)) { delete mf; return FVB_E_MESHFILE; }
  mf->points.resize(size_t(n_points) * 3);
  for (int64_t i = 0; i < n_points; ++i) {
    if (!need("POINTS")) { delete mf; return FVB_E_MESHFILE; }
    if (toks.size() != 3) MF_FAIL("line %zu: expected 3 coordinates, got %zu", ln, toks.size());
    for (int k = 0; k < 3; ++k)
      if (!py_float(toks[k], &mf->points[size_t(i) * 3 + k]))
        MF_FAIL("line %zu: non-numeric coordinate", ln);
  }
  if (!header("FACES", &n_faces)) { delete mf; return FVB_E_MESHFILE; }
  mf->offsets.assign(size_t(n_faces) + 1, 0);
  std::vector<int64_t> vals;
  for (int64_t fi = 0; fi < n_faces; ++fi) {
    if (!need("FACES")) { delete mf; return FVB_E_MESHFILE; }
    if (!ints("point index", vals)) { delete mf; return FVB_E_MESHFILE; }
    if (vals[0] != int64_t(vals.size()) - 1)
      MF_FAIL("line %zu: face declares %lld points but lists %zu", ln, (long long)vals[0],
              vals.size() - 1);
    if (vals[0] < 3) MF_FAIL("line %zu: face needs at least 3 points", ln);
    for (size_t k = 1; k < vals.size(); ++k) {
      if (!(vals[k] >= 0 && vals[k] < n_points))
        MF_FAIL("line %zu: face references point %lld of %lld", ln, (long long)vals[k],
                (long long)n_points);
      mf->fpoints.push_back(vals[k]);
    }
    mf->offsets[size_t(fi) + 1] = int64_t(mf->fpoints.size());
  }
  if (!header("OWNER", &n_owner)) { delete mf; return FVB_E_MESHFILE; }
  if (n_owner != n_faces)
    MF_FAIL("OWNER count %lld does not match FACES count %lld", (long long)n_owner,
            (long long)n_faces);
  mf->owner.resize(size_t(n_owner));
  for (int64_t i = 0; i < n_owner; ++i) {
    if (!need("OWNER")) { delete mf; return FVB_E_MESHFILE; }
    if (toks.size() != 1) MF_FAIL("line %zu: expected one owner index", ln);
    if (!ints("owner index", vals)) { delete mf; return FVB_E_MESHFILE; }
    mf->owner[size_t(i)] = vals[0];
  }
  if (!header("NEIGHBOUR", &n_internal)) { delete mf; return FVB_E_MESHFILE; }
  if (n_internal > n_faces)
    MF_FAIL("NEIGHBOUR count %lld exceeds FACES count %lld", (long long)n_internal,
            (long long)n_faces);
  mf->neighbour.resize(size_t(n_internal));
  for (int64_t i = 0; i < n_internal; ++i) {
    if (!need("NEIGHBOUR")) { delete mf; return FVB_E_MESHFILE; }
    if (toks.size() != 1) MF_FAIL("line %zu: expected one neighbour index", ln);
    if (!ints("neighbour index", vals)) { delete mf; return FVB_E_MESHFILE; }
    mf->neighbour[size_t(i)] = vals[0];
  }
  if (!header("PATCHES", &n_patches)) { delete mf; return FVB_E_MESHFILE; }
  for (int64_t i = 0; i < n_patches; ++i) {
    if (!need("PATCHES")) { delete mf; return FVB_E_MESHFILE; }
    if (toks.size() != 4) MF_FAIL("line %zu: expected 'name kind start count'", ln);
    std::vector<std::string> rng(toks.begin() + 2, toks.end());
    std::vector<std::string> keep = toks;
    toks = rng;
    // the reference reports the whole range pair in the message
    if (!ints("patch range", vals)) { delete mf; return FVB_E_MESHFILE; }
    toks = keep;
    if (keep[0].size() > 255 || keep[1].size() > 255) MF_FAIL("line %zu: patch name too long", ln);
    mf->pname.push_back(keep[0]);
    mf->pkind.push_back(keep[1]);
    mf->pstart.push_back(vals[0]);
    mf->pcount.push_back(vals[1]);
  }
  counts[0] = n_points;
  counts[1] = n_faces;
  counts[2] = int64_t(mf->fpoints.size());
  counts[3] = n_internal;
  counts[4] = n_patches;
  *out = mf;
  return FVB_OK;
}

extern "C" int fvb_mesh_read_take(fvb_meshfile* mf, double* points, int64_t* face_offsets,
                                  int64_t* face_points, int64_t* owner, int64_t* neighbour,
                                  int64_t* patch_start, int64_t* patch_count, char* patch_names,
                                  char* patch_kinds) {
  if (!mf) {
    fvb_set_error("no mesh file handle");
    return FVB_E_ARG;
  }
  memcpy(points, mf->points.data(), mf->points.size() * sizeof(double));
  memcpy(face_offsets, mf->offsets.data(), mf->offsets.size() * sizeof(int64_t));
  memcpy(face_points, mf->fpoints.data(), mf->fpoints.size() * sizeof(int64_t));
  memcpy(owner, mf->owner.data(), mf->owner.size() * sizeof(int64_t));
  memcpy(neighbour, mf->neighbour.data(), mf->neighbour.size() * sizeof(int64_t));
  for (size_t i = 0; i < mf->pname.size(); ++i) {
    patch_start[i] = mf->pstart[i];
    patch_count[i] = mf->pcount[i];
    snprintf(patch_names + 256 * i, 256, "%s", mf->pname[i].c_str());
    snprintf(patch_kinds + 256 * i, 256, "%s", mf->pkind[i].c_str());
  }
  return FVB_OK;
}

extern "C" void fvb_mesh_read_free(fvb_meshfile* mf) { delete mf; }

extern "C" int fvb_mesh_write(const char* path, int64_t n_points, const double* points,
                              int64_t n_faces, const int64_t* face_offsets,
                              const int64_t* face_points, const int64_t* owner,
                              int64_t n_internal, const int64_t* neighbour, int64_t n_patches,
                              const char* const* names, const char* const* kinds,
                              const int64_t* start, const int64_t* count) {
  FILE* f = fopen(path, "wb");
  if (!f) {
    fvb_set_error("[Errno %d] %s: '%s'", errno, strerror(errno), path);
    return FVB_E_IO;
  }
  std::vector<char> buf(1 << 20);
  setvbuf(f, buf.data(), _IOFBF, buf.size());
  fprintf(f, "POINTS %lld\n", (long long)n_points);
  for (int64_t i = 0; i < n_points; ++i)
    fprintf(f, "%.17g %.17g %.17g\n", points[3 * i], points[3 * i + 1], points[3 * i + 2]);
  fprintf(f, "FACES %lld\n", (long long)n_faces);
  for (int64_t fi = 0; fi < n_faces; ++fi) {
    const int64_t b = face_offsets[fi], e = face_offsets[fi + 1];
    fprintf(f, "%lld", (long long)(e - b));
    for (int64_t k = b; k < e; ++k) fprintf(f, " %lld", (long long)face_points[k]);
    fputc('\n', f);
  }
  fprintf(f, "OWNER %lld\n", (long long)n_faces);
  for (int64_t i = 0; i < n_faces; ++i) fprintf(f, "%lld\n", (long long)owner[i]);
  fprintf(f, "NEIGHBOUR %lld\n", (long long)n_internal);
  for (int64_t i = 0; i < n_internal; ++i) fprintf(f, "%lld\n", (long long)neighbour[i]);
  fprintf(f, "PATCHES %lld\n", (long long)n_patches);
  for (int64_t i = 0; i < n_patches; ++i)
    fprintf(f, "%s %s %lld %lld\n", names[i], kinds[i], (long long)start[i], (long long)count[i]);
  const bool bad = ferror(f) != 0;
  fclose(f);
  if (bad) {
    fvb_set_error("write to '%s' failed", path);
    return FVB_E_IO;
  }
  return FVB_OK;
}
