/* Condensed block-CSR assembly  A_bar = H^T A H  (input generator, not product).
 *
 * SEEDED INPUT GENERATOR helper (test/bench infrastructure): produces the
 * assembled, hanging-node-condensed system matrices that both the CUDA library
 * and the oracle consume.  Not part of the multigrid solve.
 *
 * Paper: P:143-144 -- "The transpose H_h^T plays an important role in the
 * assembly of the matrix ... the result ... is then multiplied by H_h^T so
 * that the test functions belonging to hanging nodes are correctly taken into
 * account"; SPEC S:345-353 constrain_system (A_bar = H^T A H).
 *
 * Element matrices are  A_e = sum_t S[e,t] * T_t  with reference tensors T_t of
 * shape (nloc*bs)^2 (node-major: index a*bs + c).  Each node p expands to
 * masters ex(p) = {(m, w)}  (regular: (p,1); hanging: its masters).
 * Row m of A_bar collects  w_a * w_b * A_e[a,b]  over every element e, local
 * pair (a,b) and master pair (m in ex(conn[e][a]), m' in ex(conn[e][b])).
 * Every row also carries its diagonal block (value 0 if nothing couples).
 * Accumulation order per row is fixed (slave list order, element order, local
 * b order), so results are deterministic and independent of thread count.
 * With `mirror` set, the strictly-lower blocks are overwritten by the
 * transposed upper blocks, making symmetric operators bit-symmetric.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

static void build_adj(i64 n_nodes, int nloc, i64 n_elem, const i64 *conn,
                      const i64 *ex_ptr, const i64 *ex_node, const double *ex_w,
                      i64 **ne_ptr, i64 **ne_list, i64 **sl_ptr, i64 **sl_node, double **sl_w) {
  /* node -> (element*nloc + a), in element order */
  i64 *cnt = calloc(n_nodes + 1, sizeof(i64));
  for (i64 e = 0; e < n_elem * nloc; ++e) cnt[conn[e] + 1]++;
  for (i64 i = 0; i < n_nodes; ++i) cnt[i + 1] += cnt[i];
  i64 *list = malloc(sizeof(i64) * (size_t)(n_elem * nloc + 1));
  i64 *pos = malloc(sizeof(i64) * (size_t)(n_nodes + 1));
  memcpy(pos, cnt, sizeof(i64) * (size_t)(n_nodes + 1));
  for (i64 e = 0; e < n_elem * nloc; ++e) list[pos[conn[e]]++] = e;
  *ne_ptr = cnt;
  *ne_list = list;
  /* master -> slaves (p, w), in p order */
  i64 *sc = calloc(n_nodes + 1, sizeof(i64));
  for (i64 p = 0; p < n_nodes; ++p)
    for (i64 t = ex_ptr[p]; t < ex_ptr[p + 1]; ++t) sc[ex_node[t] + 1]++;
  for (i64 i = 0; i < n_nodes; ++i) sc[i + 1] += sc[i];
  i64 nsl = sc[n_nodes];
  i64 *sn = malloc(sizeof(i64) * (size_t)(nsl + 1));
  double *sw = malloc(sizeof(double) * (size_t)(nsl + 1));
  memcpy(pos, sc, sizeof(i64) * (size_t)(n_nodes + 1));
  for (i64 p = 0; p < n_nodes; ++p)
    for (i64 t = ex_ptr[p]; t < ex_ptr[p + 1]; ++t) {
      i64 m = ex_node[t];
      sn[pos[m]] = p;
      sw[pos[m]] = ex_w[t];
      pos[m]++;
    }
  free(pos);
  *sl_ptr = sc;
  *sl_node = sn;
  *sl_w = sw;
}

/* find or insert column c into the sorted small array cols[0..*nc) */
static int find_insert(i64 *cols, double *vals, int *nc, i64 c, int bb, int cap) {
  int lo = 0, hi = *nc;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cols[mid] < c) lo = mid + 1; else hi = mid;
  }
  if (lo < *nc && cols[lo] == c) return lo;
  if (*nc >= cap) return -1;
  memmove(cols + lo + 1, cols + lo, sizeof(i64) * (size_t)(*nc - lo));
  if (vals) {
    memmove(vals + (size_t)(lo + 1) * bb, vals + (size_t)lo * bb, sizeof(double) * (size_t)(*nc - lo) * bb);
    memset(vals + (size_t)lo * bb, 0, sizeof(double) * bb);
  }
  (*nc)++;
  cols[lo] = c;
  return lo;
}

#define CAP 4096

/* pass == 0: fill row_ptr (n_nodes+1).  pass == 1: fill col, val.
 * returns 0 on success, -1 on overflow of the per-row buffer. */
int asm_condensed(i64 n_nodes, int bs, int nloc, i64 n_elem, const i64 *conn,
                  const i64 *ex_ptr, const i64 *ex_node, const double *ex_w,
                  int n_terms, const double *T, const double *S,
                  int pass, int mirror, i64 *row_ptr, i64 *col, double *val) {
  i64 *ne_ptr, *ne_list, *sl_ptr, *sl_node;
  double *sl_w;
  build_adj(n_nodes, nloc, n_elem, conn, ex_ptr, ex_node, ex_w, &ne_ptr, &ne_list, &sl_ptr, &sl_node, &sl_w);
  const int nl = nloc * bs, bb = bs * bs;
  int err = 0;
#pragma omp parallel
  {
    i64 *cols = malloc(sizeof(i64) * CAP);
    double *vals = pass ? malloc(sizeof(double) * (size_t)CAP * bb) : NULL;
    double *Ae = malloc(sizeof(double) * (size_t)nl * nl);
#pragma omp for schedule(dynamic, 1024)
    for (i64 m = 0; m < n_nodes; ++m) {
      int nc = 0;
      if (find_insert(cols, vals, &nc, m, bb, CAP) < 0) err = 1;
      for (i64 s = sl_ptr[m]; s < sl_ptr[m + 1]; ++s) {
        i64 p = sl_node[s];
        double wa = sl_w[s];
        for (i64 q = ne_ptr[p]; q < ne_ptr[p + 1]; ++q) {
          i64 e = ne_list[q] / nloc;
          int a = (int)(ne_list[q] % nloc);
          if (pass) {
            /* rows a*bs..a*bs+bs-1 of A_e = sum_t S[e,t] T_t  (fixed order over t) */
            for (int i = a * bs * nl; i < (a + 1) * bs * nl; ++i) {
              double acc = 0.0;
              for (int t = 0; t < n_terms; ++t) acc += S[e * n_terms + t] * T[(size_t)t * nl * nl + i];
              Ae[i] = acc;
            }
          }
          for (int b = 0; b < nloc; ++b) {
            i64 pb = conn[e * nloc + b];
            for (i64 u = ex_ptr[pb]; u < ex_ptr[pb + 1]; ++u) {
              i64 mb = ex_node[u];
              double w = wa * ex_w[u];
              int slot = find_insert(cols, vals, &nc, mb, bb, CAP);
              if (slot < 0) { err = 1; continue; }
              if (pass) {
                double *dst = vals + (size_t)slot * bb;
                for (int r = 0; r < bs; ++r)
                  for (int c = 0; c < bs; ++c)
                    dst[r * bs + c] += w * Ae[(a * bs + r) * nl + (b * bs + c)];
              }
            }
          }
        }
      }
      if (!pass) {
        row_ptr[m + 1] = nc;
      } else {
        i64 base = row_ptr[m];
        if (row_ptr[m + 1] - base != nc) err = 1;
        else {
          memcpy(col + base, cols, sizeof(i64) * (size_t)nc);
          memcpy(val + (size_t)base * bb, vals, sizeof(double) * (size_t)nc * bb);
        }
      }
    }
    free(cols);
    free(vals);
    free(Ae);
  }
  if (!pass) {
    row_ptr[0] = 0;
    for (i64 m = 0; m < n_nodes; ++m) row_ptr[m + 1] += row_ptr[m];
  } else if (mirror && !err) {
#pragma omp parallel for schedule(dynamic, 1024)
    for (i64 m = 0; m < n_nodes; ++m) {
      for (i64 k = row_ptr[m]; k < row_ptr[m + 1]; ++k) {
        i64 n = col[k];
        if (n == m) {  /* diagonal block: mirror its upper triangle */
          for (int r = 0; r < bs; ++r)
            for (int c = 0; c < r; ++c) val[(size_t)k * bb + r * bs + c] = val[(size_t)k * bb + c * bs + r];
        }
        if (n >= m) break;
        /* locate (n, m) */
        i64 lo = row_ptr[n], hi = row_ptr[n + 1];
        while (lo < hi) {
          i64 mid = (lo + hi) >> 1;
          if (col[mid] < m) lo = mid + 1; else hi = mid;
        }
        if (lo < row_ptr[n + 1] && col[lo] == m) {
          for (int r = 0; r < bs; ++r)
            for (int c = 0; c < bs; ++c) val[(size_t)k * bb + r * bs + c] = val[(size_t)lo * bb + c * bs + r];
        } else {
          err = 1;
        }
      }
    }
  }
  free(ne_ptr);
  free(ne_list);
  free(sl_ptr);
  free(sl_node);
  free(sl_w);
  return err ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* Structured (uniform box-cell) Q1 assembly of the C5 workload, any subset  */
/* of rows -- the per-rank generator of the weak-scaling runs.               */
/*                                                                          */
/* Grid of nx*ny*nz equal box cells, nodes numbered lexicographically,      */
/* id = i + (nx+1)*(j + (ny+1)*k).  Every cell has the same element matrix   */
/* Ae ((8*bs)^2, node-major, corner c has bit a = offset along axis a, the   */
/* layout of problems/fem.py).  Row m = (i,j,k) collects Ae[a_m, b] of every */
/* cell around it (cells in (ez, ey, ex) ascending order), columns in        */
/* ascending id.  Dirichlet on boundary nodes for the components flagged in  */
/* bmask (symmetric elimination, reading Z9): with g = 1 on component       */
/* lid_comp of the nodes of the face k = 0 (the cavity lid) and 0 elsewhere, */
/*   b_m -= A_mn g_n (all r), then rows/cols of constrained components are   */
/* zeroed, identity on their diagonal, and b_m = g_m there.  b (rows r0..r1, */
/* raw right-hand side) is updated in place when non-NULL.                   */
/* pass 0: row_ptr (r1-r0+1); pass 1: col (global ids), val, b.             */
/* ------------------------------------------------------------------------ */
static int on_bnd(i64 i, i64 j, i64 k, i64 nx, i64 ny, i64 nz) {
  return i == 0 || j == 0 || k == 0 || i == nx || j == ny || k == nz;
}

int asm_structured(i64 nx, i64 ny, i64 nz, int bs, const double *Ae, const unsigned char *bmask, int lid_comp,
                   i64 r0, i64 r1, int pass, i64 *row_ptr, i64 *col, double *val, double *b) {
  const i64 px = nx + 1, plane = (nx + 1) * (ny + 1);
  const int nl = 8 * bs, bb = bs * bs;
  if (pass == 0) {
    row_ptr[0] = 0;
    for (i64 m = r0; m < r1; ++m) {
      const i64 k = m / plane, j = (m % plane) / px, i = m % px;
      const i64 cx = 1 + (i > 0) + (i < nx), cy = 1 + (j > 0) + (j < ny), cz = 1 + (k > 0) + (k < nz);
      row_ptr[m - r0 + 1] = row_ptr[m - r0] + cx * cy * cz;
    }
    return 0;
  }
#pragma omp parallel for schedule(static, 4096)
  for (i64 m = r0; m < r1; ++m) {
    const i64 k = m / plane, j = (m % plane) / px, i = m % px;
    const i64 lx = i > 0, ly = j > 0, lz = k > 0;
    const i64 cx = 1 + lx + (i < nx), cy = 1 + ly + (j < ny);
    const i64 base = row_ptr[m - r0];
    const i64 cnt = row_ptr[m - r0 + 1] - base;
    double *v = val + (size_t)base * bb;
    memset(v, 0, sizeof(double) * (size_t)cnt * bb);
    for (i64 dz = -lz; dz <= (k < nz); ++dz)
      for (i64 dy = -ly; dy <= (j < ny); ++dy)
        for (i64 dx = -lx; dx <= (i < nx); ++dx)
          col[base + ((dz + lz) * cy + (dy + ly)) * cx + (dx + lx)] = (i + dx) + px * ((j + dy) + (ny + 1) * (k + dz));
    for (i64 ez = k - 1; ez <= k; ++ez) {
      if (ez < 0 || ez >= nz) continue;
      for (i64 ey = j - 1; ey <= j; ++ey) {
        if (ey < 0 || ey >= ny) continue;
        for (i64 ex = i - 1; ex <= i; ++ex) {
          if (ex < 0 || ex >= nx) continue;
          const int am = (int)((i - ex) | ((j - ey) << 1) | ((k - ez) << 2));
          for (int bc = 0; bc < 8; ++bc) {
            const i64 dx = ex + (bc & 1) - i, dy = ey + ((bc >> 1) & 1) - j, dz = ez + ((bc >> 2) & 1) - k;
            double *blk = v + (size_t)(((dz + lz) * cy + (dy + ly)) * cx + (dx + lx)) * bb;
            for (int r = 0; r < bs; ++r)
              for (int c = 0; c < bs; ++c) blk[r * bs + c] += Ae[(size_t)(am * bs + r) * nl + bc * bs + c];
          }
        }
      }
    }
    /* Dirichlet elimination */
    const int bm = on_bnd(i, j, k, nx, ny, nz);
    for (i64 t = 0; t < cnt; ++t) {
      const i64 n = col[base + t];
      const i64 nk = n / plane, nj = (n % plane) / px, ni = n % px;
      const int bn = on_bnd(ni, nj, nk, nx, ny, nz);
      double *blk = v + (size_t)t * bb;
      if (b && bn) {
        for (int r = 0; r < bs; ++r) {
          double corr = 0.0;
          for (int c = 0; c < bs; ++c) {
            const double gc = (bmask[c] && c == lid_comp && nk == 0) ? 1.0 : 0.0;
            corr += blk[r * bs + c] * gc;
          }
          b[(m - r0) * bs + r] += -corr;
        }
      }
      if (bm || bn)
        for (int r = 0; r < bs; ++r)
          for (int c = 0; c < bs; ++c)
            if ((bm && bmask[r]) || (bn && bmask[c])) blk[r * bs + c] = 0.0;
      if (n == m && bm)
        for (int c = 0; c < bs; ++c)
          if (bmask[c]) blk[c * bs + c] = 1.0;
    }
    if (b && bm)
      for (int c = 0; c < bs; ++c)
        if (bmask[c]) b[(m - r0) * bs + c] = (c == lid_comp && k == 0) ? 1.0 : 0.0;
  }
  return 0;
}

/* Trilinear prolongation of the structured grid (fine nx = 2 * coarse nx),
 * rows r0..r1 of the fine grid, per-component weights (wpe = bs) with the
 * Dirichlet components of boundary nodes dropped on both sides (Pi_f E Pi_c,
 * reading G6/Z8); entries whose weights are all zero are omitted.  Columns in
 * ascending coarse id.  pass 0: row_ptr; pass 1: col, w [nnz*bs]. */
int tr_structured(i64 nxf, i64 nyf, i64 nzf, int bs, const unsigned char *bmask, i64 r0, i64 r1, int pass,
                  i64 *row_ptr, i64 *col, double *w) {
  const i64 px = nxf + 1, plane = (nxf + 1) * (nyf + 1);
  const i64 nxc = nxf / 2, nyc = nyf / 2, nzc = nzf / 2, pxc = nxc + 1, planec = (nxc + 1) * (nyc + 1);
  if (pass == 0) row_ptr[0] = 0;
#pragma omp parallel for schedule(static, 4096) if (pass)
  for (i64 m = r0; m < r1; ++m) {
    const i64 k = m / plane, j = (m % plane) / px, i = m % px;
    const int bf = on_bnd(i, j, k, nxf, nyf, nzf);
    i64 ci[2], cj[2], ck[2];
    double wi[2], wj[2], wk[2];
    int ni = 1, nj = 1, nk = 1;
    if (i & 1) ci[0] = (i - 1) / 2, ci[1] = (i + 1) / 2, wi[0] = wi[1] = 0.5, ni = 2; else ci[0] = i / 2, wi[0] = 1.0;
    if (j & 1) cj[0] = (j - 1) / 2, cj[1] = (j + 1) / 2, wj[0] = wj[1] = 0.5, nj = 2; else cj[0] = j / 2, wj[0] = 1.0;
    if (k & 1) ck[0] = (k - 1) / 2, ck[1] = (k + 1) / 2, wk[0] = wk[1] = 0.5, nk = 2; else ck[0] = k / 2, wk[0] = 1.0;
    i64 t = pass ? row_ptr[m - r0] : 0;
    for (int a = 0; a < nk; ++a)
      for (int bq = 0; bq < nj; ++bq)
        for (int c = 0; c < ni; ++c) {
          const double wt = wk[a] * wj[bq] * wi[c];
          const int bc = on_bnd(ci[c], cj[bq], ck[a], nxc, nyc, nzc);
          int any = 0;
          for (int q = 0; q < bs; ++q)
            if (!((bf || bc) && bmask[q])) any = 1;
          if (!any) continue;
          if (pass) {
            col[t] = ci[c] + pxc * cj[bq] + planec * ck[a];
            for (int q = 0; q < bs; ++q) w[(size_t)t * bs + q] = ((bf || bc) && bmask[q]) ? 0.0 : wt;
          }
          ++t;
        }
    if (!pass) row_ptr[m - r0 + 1] = t;  /* count; prefix-summed by the caller */
  }
  if (!pass)
    for (i64 m = r0; m < r1; ++m) row_ptr[m - r0 + 1] += row_ptr[m - r0];
  return 0;
}
