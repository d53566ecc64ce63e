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
