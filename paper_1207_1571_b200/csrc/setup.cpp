// Host-side native builders for the mesh metrics and the hybrid ELL+CRS
// pattern (the setup rows a2/a3 of SURVEY.md §8).  Both reproduce the
// reference numpy arithmetic operation by operation so their outputs are
// bit-identical to fvflow's: np.add.at / bincount accumulate sequentially
// in index order, einsum over 3 columns sums (s0 + s2) + s1, norms sum
// (x^2 + y^2) + z^2.  Compiled without FMA contraction (-ffp-contract=off).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/fvb.h"
#include "common.h"

namespace {

inline double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[2] * b[2]) + a[1] * b[1];
}
inline double norm3(const double* a) {
  return std::sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
}
inline void cross3(const double* u, const double* v, double* o) {
  o[0] = u[1] * v[2] - u[2] * v[1];
  o[1] = u[2] * v[0] - u[0] * v[2];
  o[2] = u[0] * v[1] - u[1] * v[0];
}

}  // namespace

extern "C" int fvb_geometry(int64_t n_points, const double* pts, int64_t nf,
                            const int64_t* off, const int64_t* fp, int64_t nc,
                            int64_t ni, const int64_t* own, const int64_t* nbr,
                            int check, double* vol, double* cc, double* sf,
                            double* smag, double* fc, double* d, double* dmag,
                            double* w, double* nonorth, double* db,
                            double* dbmag) {
  // compute_geometry, mesh.py:173-278 (fan triangles mesh.py:154-170)
  (void)n_points;
  const int64_t nb = nf - ni;
  std::vector<double> seed(3 * nf);
  for (int64_t f = 0; f < nf; ++f) {
    const int64_t s = off[f], e = off[f + 1];
    // np.add.reduceat over a segment evaluates p0 + (p1 + p2 + ... + p_m),
    // the tail summed left to right (verified for 3..8-point loops)
    double a[3];
    for (int c = 0; c < 3; ++c) a[c] = pts[3 * fp[s] + c];
    if (e - s > 1) {
      double t[3];
      for (int c = 0; c < 3; ++c) t[c] = pts[3 * fp[s + 1] + c];
      for (int64_t j = s + 2; j < e; ++j)
        for (int c = 0; c < 3; ++c) t[c] += pts[3 * fp[j] + c];
      for (int c = 0; c < 3; ++c) a[c] = a[c] + t[c];
    }
    const double cnt = double(e - s);
    for (int c = 0; c < 3; ++c) seed[3 * f + c] = a[c] / cnt;
  }
  // per-triangle area vectors, areas, centroids (mesh.py:189-192)
  const int64_t ntri = off[nf];
  std::vector<double> tsf(3 * ntri), tarea(ntri), tctr(3 * ntri);
  for (int64_t f = 0; f < nf; ++f) {
    const int64_t s = off[f], e = off[f + 1];
    const double* sd = &seed[3 * f];
    for (int64_t j = s; j < e; ++j) {
      const int64_t jn = (j + 1 == e) ? s : j + 1;
      const double* a = &pts[3 * fp[j]];
      const double* b = &pts[3 * fp[jn]];
      double ba[3], sa[3], cr[3];
      for (int c = 0; c < 3; ++c) {
        ba[c] = b[c] - a[c];
        sa[c] = sd[c] - a[c];
      }
      cross3(ba, sa, cr);
      for (int c = 0; c < 3; ++c) tsf[3 * j + c] = 0.5 * cr[c];
      tarea[j] = norm3(&tsf[3 * j]);
      for (int c = 0; c < 3; ++c) tctr[3 * j + c] = ((a[c] + b[c]) + sd[c]) / 3.0;
    }
  }
  std::vector<double> asum(nf, 0.0);
  for (int64_t f = 0; f < nf; ++f) {
    double s3[3] = {0.0, 0.0, 0.0}, as = 0.0, c3[3] = {0.0, 0.0, 0.0};
    for (int64_t j = off[f]; j < off[f + 1]; ++j) {
      for (int c = 0; c < 3; ++c) s3[c] += tsf[3 * j + c];
      as += tarea[j];
    }
    for (int64_t j = off[f]; j < off[f + 1]; ++j)
      for (int c = 0; c < 3; ++c) c3[c] += tarea[j] * tctr[3 * j + c];
    if (as < 1e-30) {
      fvb_set_error("face %lld is degenerate (zero area)", (long long)f);
      return FVB_E_MESH;
    }
    asum[f] = as;
    for (int c = 0; c < 3; ++c) {
      sf[3 * f + c] = s3[c];
      fc[3 * f + c] = c3[c] / as;
    }
    smag[f] = norm3(&sf[3 * f]);
  }
  // cell seed = mean of face centroids (mesh.py:207-213)
  std::vector<int64_t> nfc(nc, 0);
  for (int64_t f = 0; f < nf; ++f) nfc[own[f]]++;
  for (int64_t f = 0; f < ni; ++f) nfc[nbr[f]]++;
  std::vector<double> cs(3 * nc, 0.0);
  for (int64_t f = 0; f < nf; ++f)
    for (int c = 0; c < 3; ++c) cs[3 * own[f] + c] += fc[3 * f + c];
  for (int64_t f = 0; f < ni; ++f)
    for (int c = 0; c < 3; ++c) cs[3 * nbr[f] + c] += fc[3 * f + c];
  for (int64_t i = 0; i < nc; ++i)
    for (int c = 0; c < 3; ++c) cs[3 * i + c] /= double(nfc[i]);
  // tet decomposition (mesh.py:215-242): owner pass over all triangles,
  // then the neighbour pass over internal-face triangles with flipped sign
  std::fill(vol, vol + nc, 0.0);
  std::fill(cc, cc + 3 * nc, 0.0);
  for (int pass = 0; pass < 2; ++pass) {
    const int64_t fend = pass == 0 ? nf : ni;
    for (int64_t f = 0; f < fend; ++f) {
      const int64_t apex = pass == 0 ? own[f] : nbr[f];
      const double* dd = &cs[3 * apex];
      const double* sd = &seed[3 * f];
      const int64_t s = off[f], e = off[f + 1];
      for (int64_t j = s; j < e; ++j) {
        const int64_t jn = (j + 1 == e) ? s : j + 1;
        const double* a = &pts[3 * fp[j]];
        const double* b = &pts[3 * fp[jn]];
        double aa[3], bb[3], ss[3], cr[3];
        for (int c = 0; c < 3; ++c) {
          aa[c] = a[c] - dd[c];
          bb[c] = b[c] - dd[c];
          ss[c] = sd[c] - dd[c];
        }
        cross3(bb, ss, cr);
        double v = dot3(aa, cr) / 6.0;
        if (pass == 1) v = -v;
        vol[apex] += v;
        for (int c = 0; c < 3; ++c) {
          const double ctr = (((a[c] + b[c]) + sd[c]) + dd[c]) / 4.0;
          cc[3 * apex + c] += v * ctr;
        }
      }
    }
  }
  for (int64_t i = 0; i < nc; ++i) {
    if (vol[i] <= 0.0) {
      fvb_set_error("cell %lld has non-positive volume %g", (long long)i, vol[i]);
      return FVB_E_MESH;
    }
  }
  for (int64_t i = 0; i < nc; ++i)
    for (int c = 0; c < 3; ++c) cc[3 * i + c] /= vol[i];
  // internal-face metrics (mesh.py:244-261)
  // nonorth[] receives the clipped cosine; the caller applies numpy's own
  // arccos/degrees (its SIMD arccos differs from libm by an ulp) and the
  // MAX_NONORTHOGONALITY_DEG check, in the reference's order (mesh.py:254-261)
  (void)check;
  int64_t bad_sd = -1;
  for (int64_t f = 0; f < ni; ++f) {
    const double* co = &cc[3 * own[f]];
    const double* cn = &cc[3 * nbr[f]];
    double* df = &d[3 * f];
    double r[3];
    for (int c = 0; c < 3; ++c) {
      df[c] = cn[c] - co[c];
      r[c] = cn[c] - fc[3 * f + c];
    }
    dmag[f] = norm3(df);
    const double sdot = dot3(&sf[3 * f], df);
    if (sdot <= 0.0 && bad_sd < 0) bad_sd = f;
    w[f] = dot3(&sf[3 * f], r) / sdot;
    double den = dmag[f] * smag[f];
    if (den < 1e-300) den = 1e-300;
    double ca = sdot / den;
    nonorth[f] = ca < -1.0 ? -1.0 : (ca > 1.0 ? 1.0 : ca);
  }
  if (bad_sd >= 0) {
    fvb_set_error("internal face %lld: area vector points away from neighbour",
                  (long long)bad_sd);
    return FVB_E_MESH;
  }
  for (int64_t j = 0; j < nb; ++j) {
    const int64_t f = ni + j;
    for (int c = 0; c < 3; ++c) db[3 * j + c] = fc[3 * f + c] - cc[3 * own[f] + c];
    dbmag[j] = norm3(&db[3 * j]);
  }
  return FVB_OK;
}

// ------------------------------------------------------------------ pattern
// pattern_from_pairs (sparse.py:111-209).  Entries are kept per row in
// ascending column order (the reference's (row, col) sort); rows longer
// than K keep the diagonal plus the K-1 lowest off-diagonal columns in ELL
// and spill the rest, in (row, col) order, to the CRS block.

struct fvb_pattern_plan {
  int64_t n = 0, k = 0, nnz_crs = 0;
  std::vector<int64_t> ptr;    // row pointers into cols
  std::vector<int64_t> cols;   // ascending per row, diagonal included
  std::vector<int64_t> addr;   // flat address per entry
  std::vector<int64_t> slot;   // ELL slot or -1
  int64_t find(int64_t row, int64_t col) const {
    const int64_t* b = cols.data() + ptr[row];
    const int64_t* e = cols.data() + ptr[row + 1];
    const int64_t* it = std::lower_bound(b, e, col);
    if (it == e || *it != col) return -1;
    return int64_t(it - cols.data());
  }
};

extern "C" int fvb_pattern_plan_create(int64_t n, int64_t npairs,
                                       const int64_t* pairs, int64_t k_cap,
                                       fvb_pattern_plan** out, int64_t* k_out,
                                       int64_t* nnz_out) {
  if (k_cap < 1) {
    fvb_set_error("k_cap must be at least 1");
    return FVB_E_SPARSE;
  }
  if (n < 0) {
    fvb_set_error("negative size");
    return FVB_E_ARG;
  }
  std::vector<int64_t> keys(npairs);
  for (int64_t i = 0; i < npairs; ++i) {
    int64_t a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b) {
      fvb_set_error("self-pair in adjacency");
      return FVB_E_SPARSE;
    }
    if (a < 0 || b < 0 || a >= n || b >= n) {
      fvb_set_error("pair index out of range");
      return FVB_E_SPARSE;
    }
    keys[i] = std::min(a, b) * n + std::max(a, b);
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  auto* P = new fvb_pattern_plan();
  P->n = n;
  std::vector<int64_t> cnt(n, 1);
  for (int64_t key : keys) {
    cnt[key / n]++;
    cnt[key % n]++;
  }
  P->ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) P->ptr[i + 1] = P->ptr[i] + cnt[i];
  P->cols.resize(P->ptr[n]);
  std::vector<int64_t> pos(P->ptr.begin(), P->ptr.end() - 1);
  // lower columns (pairs sorted by lo, so each row's lower part ascends)
  for (int64_t key : keys) P->cols[pos[key % n]++] = key / n;
  for (int64_t i = 0; i < n; ++i) P->cols[pos[i]++] = i;
  for (int64_t key : keys) P->cols[pos[key / n]++] = key % n;
  int64_t maxc = 0;
  for (int64_t i = 0; i < n; ++i) maxc = std::max(maxc, cnt[i]);
  const int64_t k = std::min(maxc, k_cap);
  P->k = k;
  P->addr.resize(P->cols.size());
  P->slot.assign(P->cols.size(), -1);
  int64_t crs = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t s = 0, offd = 0;
    for (int64_t e = P->ptr[i]; e < P->ptr[i + 1]; ++e) {
      const bool diag = P->cols[e] == i;
      bool keep = true;
      if (cnt[i] > k && !diag) keep = offd < k - 1;
      if (!diag) offd++;
      if (keep) {
        P->slot[e] = s;
        P->addr[e] = i * k + s;
        s++;
      } else {
        P->addr[e] = n * k + crs;
        crs++;
      }
    }
  }
  P->nnz_crs = crs;
  *out = P;
  *k_out = k;
  *nnz_out = crs;
  return FVB_OK;
}

extern "C" int fvb_pattern_plan_fill(fvb_pattern_plan* P, int64_t nfp,
                                     const int64_t* fpairs, int64_t* I,
                                     int64_t* J, int64_t* diag_slot,
                                     int64_t* tcrs, int64_t* crs_ptr,
                                     int64_t* crs_col, uint8_t* crs_in_ell,
                                     int64_t* crs_pos, int64_t* face_addr) {
  const int64_t n = P->n, k = P->k, nk = n * k;
  std::fill(I, I + nk, -1);
  std::fill(J, J + nk, -1);
  std::fill(tcrs, tcrs + nk, -1);
  crs_ptr[0] = 0;
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t e = P->ptr[i]; e < P->ptr[i + 1]; ++e) {
      const int64_t col = P->cols[e];
      const int64_t tw = P->addr[P->find(col, i)];
      if (P->slot[e] >= 0) {
        const int64_t s = P->slot[e];
        I[i * k + s] = col;
        if (tw < nk)
          J[i * k + s] = tw % k;
        else
          tcrs[i * k + s] = tw - nk;
        if (col == i) diag_slot[i] = s;
      } else {
        crs_col[c] = col;
        crs_in_ell[c] = tw < nk;
        crs_pos[c] = tw < nk ? tw % k : tw - nk;
        c++;
      }
    }
    crs_ptr[i + 1] = c;
  }
  for (int64_t f = 0; f < nfp; ++f) {
    const int64_t a = fpairs[2 * f], b = fpairs[2 * f + 1];
    const int64_t lo = std::min(a, b), hi = std::max(a, b);
    const int64_t e01 = P->find(lo, hi), e10 = P->find(hi, lo);
    if (e01 < 0 || e10 < 0) {
      fvb_set_error("entry (%lld, %lld) not in pattern", (long long)lo, (long long)hi);
      return FVB_E_SPARSE;
    }
    face_addr[2 * f] = P->addr[e01];
    face_addr[2 * f + 1] = P->addr[e10];
  }
  return FVB_OK;
}

extern "C" void fvb_pattern_plan_destroy(fvb_pattern_plan* P) { delete P; }

// pack_q / unpack_q (sparse.py:337-363): fuse I and J into one integer
// array Q = base*I + J (base N for mode 0 "by_N", K for mode 1 "by_K");
// padding packs to -1, entries whose twin sits in the CRS block to -2 - I.
extern "C" int fvb_pack_q(int64_t n, int64_t k, const int64_t* I, const int64_t* J, int mode,
                          int64_t* q) {
  if (mode != 0 && mode != 1) {
    fvb_set_error("unknown mode %d", mode);
    return FVB_E_SPARSE;
  }
  const int64_t base = mode == 0 ? n : k;
  for (int64_t e = 0; e < n * k; ++e) {
    const int64_t i = I[e], j = J[e];
    q[e] = i < 0 ? -1 : (j < 0 ? -2 - i : base * i + j);
  }
  return FVB_OK;
}

extern "C" int fvb_unpack_q(int64_t n, int64_t k, int64_t m, const int64_t* q, int mode,
                            int64_t* I, int64_t* J) {
  if (mode != 0 && mode != 1) {
    fvb_set_error("unknown mode %d", mode);
    return FVB_E_SPARSE;
  }
  const int64_t base = mode == 0 ? n : k;
  for (int64_t e = 0; e < m; ++e) {
    const int64_t v = q[e];
    if (v >= 0) {
      I[e] = v / base;
      J[e] = v % base;
    } else {
      I[e] = v == -1 ? -1 : -2 - v;
      J[e] = -1;
    }
  }
  return FVB_OK;
}
