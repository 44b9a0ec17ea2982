/*
 * pp_oracle.c -- plain, slow, obviously-correct serial CPU oracle for the
 * in-place parallel partition (+ quicksort) of arxiv 2004.12532
 * ("In-place parallel partition"; PAPER.md = /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path under
 * paper_2004_12532_b200/ and it includes nothing from there.
 *
 * Conventions:
 *   - 0-based indices (the paper is 1-based, §2).
 *   - predecessor  <=>  key < pivot, unsigned compare (reading R1).
 *   - the split returned by every partition is K = #{i : A[i] < pivot}.
 *
 * Every function cites the passage it follows.  Pins (what checks this file
 * against something other than itself) live in tests/test_oracle_pins.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void oracle_prefix_sum_recursive(uint64_t *S, uint64_t n);

#define DEFINE_ORACLE(T, SFX)                                                   \
                                                                                \
/* Definition of the problem (§2 "The Parallel Partition   */ \
/* Problem"): K = number of predecessors.                                    */ \
uint64_t oracle_count_##SFX(const T *A, uint64_t n, T pivot)                    \
{                                                                               \
    uint64_t k = 0;                                                             \
    for (uint64_t i = 0; i < n; i++)                                            \
        if (A[i] < pivot) k++;                                                  \
    return k;                                                                   \
}                                                                               \
                                                                                \
/* SPEC.md:176-184 is_partitioned: A[0..k) predecessors, A[k..n) successors. */ \
int oracle_is_partitioned_##SFX(const T *A, uint64_t n, T pivot, uint64_t k)    \
{                                                                               \
    if (k > n) return 0;                                                        \
    for (uint64_t i = 0; i < k; i++)                                            \
        if (!(A[i] < pivot)) return 0;                                          \
    for (uint64_t i = k; i < n; i++)                                            \
        if (A[i] < pivot) return 0;                                             \
    return 1;                                                                   \
}                                                                               \
                                                                                \
/* Serial in-place two-pointer partition: the paper's "Libc" serial          */ \
/* baseline (§5.1), written from the definition (not     */ \
/* from glibc): i walks right over predecessors, j walks left over           */ \
/* successors, and a misplaced pair is swapped.  Returns i == K.             */ \
uint64_t oracle_partition_two_pointer_##SFX(T *A, uint64_t n, T pivot)          \
{                                                                               \
    uint64_t i = 0, j = n;                                                      \
    for (;;) {                                                                  \
        while (i < j && A[i] < pivot) i++;                                      \
        while (i < j && !(A[j - 1] < pivot)) j--;                               \
        if (i >= j) break;                                                      \
        T tmp = A[i]; A[i] = A[j - 1]; A[j - 1] = tmp;                          \
        i++; j--;                                                               \
    }                                                                           \
    return i;                                                                   \
}                                                                               \
                                                                                \
/* The (Standard) Linear-Space Parallel Partition (§2),    */ \
/* run serially.  D[i] = dec(A[i]); S = inclusive prefix sum of D (reading   */ \
/* R9: S[i] = sum_{j<=i} D[j]); t = S[n-1]; predecessor i -> C[S[i]-1],       */ \
/* successor i -> C[t + i - S[i]] (0-based form of "position S[i]" and       */ \
/* "position t + i - S[i]"); copy C -> A.  Stable.  Caller gives scratch S,  */ \
/* C of n entries each (the algorithm is not in place).    */ \
uint64_t oracle_partition_standard_##SFX(T *A, uint64_t n, T pivot,             \
                                         uint64_t *S, T *C)                    \
{                                                                               \
    if (n == 0) return 0;                                                       \
    for (uint64_t i = 0; i < n; i++) S[i] = (A[i] < pivot) ? 1 : 0; /* D */     \
    oracle_prefix_sum_recursive(S, n);                              /* S */     \
    uint64_t t = S[n - 1];                                                      \
    for (uint64_t i = 0; i < n; i++) {                                          \
        if (A[i] < pivot) C[S[i] - 1] = A[i];                                   \
        else              C[t + i - S[i]] = A[i];                               \
    }                                                                           \
    memcpy(A, C, n * sizeof(T));                                                \
    return t;                                                                   \
}                                                                               \
                                                                                \
static void oracle_insertion_sort_##SFX(T *A, uint64_t n)                       \
{                                                                               \
    for (uint64_t i = 1; i < n; i++) {                                          \
        T x = A[i];                                                             \
        uint64_t j = i;                                                         \
        while (j > 0 && A[j - 1] > x) { A[j] = A[j - 1]; j--; }                 \
        A[j] = x;                                                               \
    }                                                                           \
}                                                                               \
                                                                                \
static T oracle_median3_##SFX(T a, T b, T c)                                    \
{                                                                               \
    if (a > b) { T t = a; a = b; b = t; }                                       \
    if (b > c) { b = c; }                                                       \
    return a > b ? a : b;                                                       \
}                                                                               \
                                                                                \
/* Serial quicksort layered on the two-pointer partition (PAPER.md:1701-1732  */\
/* §5 "Example Application: A Full Quicksort"; pivot rule = reading R14:     */ \
/* median of A[lo], A[lo+(len-1)/2], A[hi-1]).  Progress rule for            */ \
/* duplicates (reading R14): split by x < p -> k1; if k1 == 0 (p is the      */ \
/* minimum) split by x <= p (i.e. x < p+1) -> k2 >= 1 and [0,k2) is all p.   */ \
/* Insertion sort below 16 keys.  Explicit stack (no recursion depth risk).  */ \
void oracle_quicksort_##SFX(T *A, uint64_t n)                                   \
{                                                                               \
    uint64_t stack_lo[128], stack_hi[128];                                      \
    int sp = 0;                                                                 \
    stack_lo[sp] = 0; stack_hi[sp] = n; sp++;                                   \
    while (sp > 0) {                                                            \
        sp--;                                                                   \
        uint64_t lo = stack_lo[sp], hi = stack_hi[sp];                          \
        for (;;) {                                                              \
            uint64_t len = hi - lo;                                             \
            if (len <= 16) { oracle_insertion_sort_##SFX(A + lo, len); break; } \
            T p = oracle_median3_##SFX(A[lo], A[lo + (len - 1) / 2], A[hi - 1]);\
            uint64_t k = oracle_partition_two_pointer_##SFX(A + lo, len, p);   \
            uint64_t mid_lo, mid_hi;                                            \
            if (k == 0) {                                                       \
                /* p is the minimum; p < max value of T here since p is in   */ \
                /* the segment and some key >= p exists; p+1 cannot wrap     */ \
                /* unless p == max, in which case all keys equal p.          */ \
                if (p == (T)~(T)0) break;                                       \
                uint64_t k2 = oracle_partition_two_pointer_##SFX(A + lo, len,   \
                                                                 (T)(p + 1));   \
                lo = lo + k2;               /* [lo, lo+k2) all equal p */       \
                continue;                                                       \
            }                                                                   \
            mid_lo = lo + k; mid_hi = lo + k;                                   \
            /* push the larger side, iterate on the smaller: depth O(log n) */  \
            if (mid_lo - lo < hi - mid_hi) {                                    \
                stack_lo[sp] = mid_hi; stack_hi[sp] = hi; sp++;                 \
                hi = mid_lo;                                                    \
            } else {                                                            \
                stack_lo[sp] = lo; stack_hi[sp] = mid_lo; sp++;                 \
                lo = mid_hi;                                                    \
            }                                                                   \
        }                                                                       \
    }                                                                           \
}                                                                               \
                                                                                \
/* Smoothed Striding Partial Partition Step, group statistics only           */ \
/* (§4 Formal Algorithm Description; Fig. 3 index map     */ \
/* PAPER.md:1031-1034).  The region A[base .. base + n_lines*b) is viewed as */ \
/* s = ceil(n_lines/g) chunks of g lines of b keys; group i holds line       */ \
/* G_i(j) = j*g + ((X[j] + i) mod g) of chunk j (0-based form of             */ \
/* "(X[j] + i mod g) + (j-1)g + 1" with X0[j] = X[j]+1 mod g; the random     */ \
/* offsets X[0..s) are passed in -- the method's random draws are inputs),  */ \
/* lines >= n_lines being virtual and                                        */ \
/* absent (PAPER.md:942-951 footnote; reading R5).  After each group is      */ \
/* partitioned, its first T_i elements in group order are predecessors, so   */ \
/* v_i = "the index of the first successor" is a function */ \
/* of T_i alone.  For each group this writes T_i and                         */ \
/*   vlo_i = vhi_i = position of the group's (T_i)-th element (0-based), or, */ \
/*   if the group has no successor, one past its last element (reading R2);  */ \
/*   a group with no lines writes vlo = base+n_lines*b, vhi = base (it       */ \
/*   constrains nothing).  Positions are absolute (include base).            */ \
void oracle_ss_groups_##SFX(const T *A, uint64_t base, uint64_t n_lines,        \
                            uint64_t b, uint64_t g, const uint64_t *X, T pivot, \
                            uint64_t *T_out, uint64_t *vlo, uint64_t *vhi)      \
{                                                                               \
    uint64_t s = (n_lines + g - 1) / g;                                         \
    for (uint64_t i = 0; i < g; i++) {                                          \
        uint64_t t = 0, nl = 0, last_line = 0;                                  \
        for (uint64_t j = 0; j < s; j++) {                                      \
            uint64_t line = j * g + (X[j] + i) % g;     \
            if (line >= n_lines) continue;                                      \
            for (uint64_t e = 0; e < b; e++)                                    \
                if (A[base + line * b + e] < pivot) t++;                        \
            nl++; last_line = line;                                             \
        }                                                                       \
        T_out[i] = t;                                                           \
        if (nl == 0) { vlo[i] = base + n_lines * b; vhi[i] = base; continue; }  \
        uint64_t v;                                                             \
        if (t == nl * b) {                                                      \
            v = base + last_line * b + b;                                       \
        } else {                                                                \
            /* the (t / b)-th line of the group in group order */               \
            uint64_t want = t / b, seen = 0, line = 0;                          \
            for (uint64_t j = 0; j < s; j++) {                                  \
                line = j * g + (X[j] + i) % g;          \
                if (line >= n_lines) continue;                                  \
                if (seen == want) break;                                        \
                seen++;                                                         \
            }                                                                   \
            v = base + line * b + t % b;                                        \
        }                                                                       \
        vlo[i] = v; vhi[i] = v;                                                 \
    }                                                                           \
}

/* Recursive parallel prefix sum (§2), run serially, in     */
/* place on S[0..n): (1) D'[i] = D[2i] + D[2i+1]; (2) recurse on D';          */
/* (3) S[i] = S'[i/2] for odd i (0-based: the pair's second element) and      */
/* S[i] = S'[i/2 - 1] + D[i] for even i (reading R9: "+ D[i]" not "+ A[i]").  */
/* Scratch is allocated per level; the oracle does not care about space.      */
void oracle_prefix_sum_recursive(uint64_t *S, uint64_t n)
{
    if (n <= 1) return;
    uint64_t h = n / 2;
    uint64_t *Dp = (uint64_t *)malloc((h > 0 ? h : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < h; i++) Dp[i] = S[2 * i] + S[2 * i + 1];
    oracle_prefix_sum_recursive(Dp, h);
    /* 1-based: S[i] = S'[i/2] (i even), S[i] = S'[floor(i/2)] + D[i] (i odd),
       with S'[0] = 0.  0-based index x = i - 1.                              */
    for (uint64_t x = 0; x < n; x++) {
        uint64_t i = x + 1;
        if (i % 2 == 0) S[x] = Dp[i / 2 - 1];
        else            S[x] = (i / 2 >= 1 ? Dp[i / 2 - 1] : 0) + S[x];
    }
    free(Dp);
}

DEFINE_ORACLE(uint64_t, u64)
DEFINE_ORACLE(uint32_t, u32)

/* ------------------------------------------------------------------------- */
/* The Blocked-Prefix-Sum partition (§3, Figs. 1-2) in the  */
/* form of the paper's "low-space implementation" (§5):   */
/* the block prefix sums are kept in an explicit array of floor(n/B)+1 words  */
/* (the implicit bit-pair codec of Lemma 3.2 is not used),    */
/* the Preprocessing and Reordering phases are in place.  Serial.             */
/*                                                                           */
/* Role swap (Fig. 2): the phases need successors to be at  */
/* least half of the array.  When fewer than half are successors, the         */
/* algorithm runs on the logically reversed array V(i) = A[n-1-i] with the    */
/* roles of predecessors and successors swapped; the reversed result read     */
/* forwards is the partition.  pred_v(x) below is "predecessor in the view".  */
/* ------------------------------------------------------------------------- */
#define BPS_V(i) (rev ? n - 1 - (i) : (i))
#define BPS_PRED(x) (rev ? !((x) < pivot) : ((x) < pivot))
#define BPS_SWAP(T, a, b) do { T t_ = A[a]; A[a] = A[b]; A[b] = t_; } while (0)

#define DEFINE_BPS_ORACLE(T, SFX)                                               \
                                                                                \
/* MakeSuccessorHeavy (Fig. 1; Lemma 3.1):*/ \
/* for i < floor(m/2): if V[i] is a predecessor and V[m-1-i] a successor,    */ \
/* swap them; then recurse on the first ceil(m/2) positions (stopping at     */ \
/* m <= 1, reading R21).  Afterwards every t-prefix holds >= t/4 successors.  */ \
void oracle_bps_make_successor_heavy_##SFX(T *A, uint64_t n, T pivot, int rev)  \
{                                                                               \
    uint64_t m = n;                                                             \
    while (m > 1) {                                                             \
        for (uint64_t i = 0; i < m / 2; i++) {                                  \
            uint64_t a = BPS_V(i), b = BPS_V(m - 1 - i);                        \
            if (BPS_PRED(A[a]) && !BPS_PRED(A[b])) BPS_SWAP(T, a, b);           \
        }                                                                       \
        m = (m + 1) / 2;                                                        \
    }                                                                           \
}                                                                               \
                                                                                \
/* Reorder (Fig. 2; Lemma 3.4) on the     */ \
/* prefix of the first tb blocks (the whole view when tb == nb).  S[i] =     */ \
/* predecessors in blocks 0..i-1.  m <= 5B: the serial base case (PAPER.md:  */ \
/* 606-608; here the r-th successor in [0,K') is swapped with the r-th       */ \
/* predecessor in [K',m), reading R22).  Otherwise recurse on the least t    */ \
/* blocks with t*B > 4m/5, then swap the j-th predecessor of each later      */ \
/* block i with position S[i] + j, which the lemma puts in the successor     */ \
/* part of the reordered prefix: returns 1 if a target is not a successor    */ \
/* inside the prefix (the conflict-freeness the lemma proves), else 0.       */ \
static int bps_reorder_##SFX(T *A, uint64_t n, T pivot, int rev, uint64_t B,    \
                             uint64_t nb, const uint64_t *S, uint64_t tb)       \
{                                                                               \
    uint64_t m = (tb == nb) ? n : tb * B;                                       \
    uint64_t t = (4 * m) / (5 * B) + 1;  /* least t with t*B > 4m/5 */           \
    if (m <= 5 * B || t >= tb) {  /* base case (also when the extended last */  \
                                  /* block leaves no shorter prefix)        */  \
        uint64_t Kp = S[tb], i = 0, j = Kp;                                     \
        for (;;) {                                                              \
            while (i < Kp && BPS_PRED(A[BPS_V(i)])) i++;                        \
            while (j < m && !BPS_PRED(A[BPS_V(j)])) j++;                        \
            if (i >= Kp || j >= m) break;                                       \
            BPS_SWAP(T, BPS_V(i), BPS_V(j));                                    \
            i++; j++;                                                           \
        }                                                                       \
        return 0;                                                               \
    }                                                                           \
    if (bps_reorder_##SFX(A, n, pivot, rev, B, nb, S, t)) return 1;             \
    for (uint64_t i = t; i < tb; i++) {                                         \
        uint64_t lo = i * B, hi = (i == nb - 1) ? n : (i + 1) * B, j = 0;       \
        for (uint64_t q = lo; q < hi; q++) {                                    \
            if (!BPS_PRED(A[BPS_V(q)])) continue;                               \
            uint64_t target = S[i] + j++;                                       \
            if (target >= t * B || BPS_PRED(A[BPS_V(target)])) return 1;        \
            BPS_SWAP(T, BPS_V(q), BPS_V(target));                               \
        }                                                                       \
    }                                                                           \
    return 0;                                                                   \
}                                                                               \
                                                                                \
/* ParallelPartition (Fig. 2), low-space form: count,      */ \
/* role swap, MakeSuccessorHeavy, explicit block prefix sums over blocks of  */ \
/* B keys (the last block takes the remainder; the paper's  */ \
/* own recursive scan), Reorder.  S: scratch of            */ \
/* floor(n/B)+1 words.  Returns K, or UINT64_MAX if a Reorder swap target    */ \
/* broke Lemma 3.4's guarantee.                                              */ \
uint64_t oracle_partition_bps_##SFX(T *A, uint64_t n, T pivot, uint64_t B,     \
                                    uint64_t *S)                               \
{                                                                               \
    uint64_t K = 0;                                                             \
    for (uint64_t i = 0; i < n; i++) if (A[i] < pivot) K++;                     \
    int rev = 2 * (n - K) < n;  /* fewer than half are successors */           \
    oracle_bps_make_successor_heavy_##SFX(A, n, pivot, rev);                    \
    uint64_t nb = n / B;                                                        \
    if (nb == 0) {  /* a single short block: the base case */                   \
        uint64_t S0[2] = {0, rev ? n - K : K};                                  \
        bps_reorder_##SFX(A, n, pivot, rev, n > 0 ? n : 1, 1, S0, 1);           \
        return K;                                                               \
    }                                                                           \
    S[0] = 0;                                                                   \
    for (uint64_t i = 0; i < nb; i++) {                                         \
        uint64_t lo = i * B, hi = (i == nb - 1) ? n : (i + 1) * B, c = 0;       \
        for (uint64_t q = lo; q < hi; q++) c += BPS_PRED(A[BPS_V(q)]) ? 1 : 0;  \
        S[i + 1] = c;                                                           \
    }                                                                           \
    oracle_prefix_sum_recursive(S + 1, nb);  /* S[i+1] = preds in blocks <= i */ \
    if (bps_reorder_##SFX(A, n, pivot, rev, B, nb, S, nb)) return UINT64_MAX;   \
    return K;                                                                   \
}

DEFINE_BPS_ORACLE(uint64_t, u64)
DEFINE_BPS_ORACLE(uint32_t, u32)
