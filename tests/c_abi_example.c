/* C99 client of the C ABI (tests/test_c_abi.py compiles it with gcc -std=c99
 * -Wall -Wextra -pedantic -Werror against include/lane_allreduce.h, links it
 * with liblane_allreduce.so and runs it on a CPU host): the boundary is plain
 * C — pointers, sizes, status codes — with no torch or C++ types. Only the
 * host-only entry points run here; the device entry points need a GPU. */
#include <stdint.h>
#include <stdio.h>

#include "lane_allreduce.h"

int main(void) {
  int node = -1, gpu = -1, group[LANE_MAX_RANKS], lane_ranks[LANE_MAX_RANKS];
  uint64_t n_units = 0;
  int64_t units[9 * 64], plan[6];
  lane_comm_t comm = NULL;
  int st;

  printf("version %s\n", lane_allreduce_version());
  /* rank 5 of a 2x4 layout: node 1, gpu 1; comm_group {4..7}, comm_lane {1, 5} */
  if (lane_topology_query(2, 4, 5, &node, &gpu, group, lane_ranks) != LANE_OK) return 1;
  printf("topology rank 5: node %d gpu %d group %d %d %d %d lane %d %d\n", node, gpu, group[0], group[1], group[2],
         group[3], lane_ranks[0], lane_ranks[1]);
  /* ownership units of 1000 fp32 elements on 2x4 with k = 2 */
  if (lane_partition_query(1000, 4, 2, 4, 2, 0, 0, units, 64, &n_units) != LANE_OK) return 2;
  printf("partition units %llu first {round %lld l %lld c %lld g %lld a %lld start %lld end %lld}\n",
         (unsigned long long)n_units, (long long)units[0], (long long)units[1], (long long)units[2],
         (long long)units[3], (long long)units[4], (long long)units[7], (long long)units[8]);
  /* LL128 plan of an 8 MiB message on 2x2, k = 1, 148 CTAs */
  if (lane_ll128_plan_query(2, 2, 1, (8 << 20) / 16, 148, 32 << 20, 16 << 10, plan) != LANE_OK) return 3;
  printf("ll128 plan C %lld cg %lld chunks %lld lu %lld need %lld set %lld\n", (long long)plan[0],
         (long long)plan[1], (long long)plan[2], (long long)plan[3], (long long)plan[4], (long long)plan[5]);
  /* argument errors are status codes naming the field, before any CUDA call */
  st = lane_allreduce_init_rank(0, 4, 1, 0, 0, &comm);
  printf("init_rank(nodes=0) -> %d comm %s error \"%s\"\n", st, comm ? "set" : "NULL",
         lane_allreduce_last_error(NULL));
  if (st != LANE_ERR_INVALID_ARG || comm != NULL) return 4;
  return 0;
}
