// Host DRAM bandwidth per NUMA node: threads pinned to the node's CPUs read (and copy) a buffer
// bound to that node with mbind(2).  Feeds the 8-GPU host-side ceiling in DESIGN.md §6: every
// GPU's host link pulls from these DIMMs.  Probe only; not product code.
//   gcc -O2 -pthread -o host_dram_probe host_dram_probe.c
#define _GNU_SOURCE
#include <pthread.h>
#include <sched.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <time.h>
#include <unistd.h>

#define MPOL_BIND 2

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}

typedef struct {
  const uint64_t* src;
  uint64_t* dst;
  size_t n;  // u64 words
  int cpu;
  int mode;  // 0 read, 1 copy
  double secs;
  uint64_t sink;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  if (j->cpu >= 0) {
    cpu_set_t s;
    CPU_ZERO(&s);
    CPU_SET(j->cpu, &s);
    sched_setaffinity(0, sizeof(s), &s);
  }
  double t0 = now();
  if (j->mode == 0) {
    uint64_t a = 0, b = 0, c = 0, d = 0;
    for (size_t i = 0; i + 4 <= j->n; i += 4) {
      a ^= j->src[i];
      b ^= j->src[i + 1];
      c ^= j->src[i + 2];
      d ^= j->src[i + 3];
    }
    j->sink = a ^ b ^ c ^ d;
  } else {
    memcpy(j->dst, j->src, j->n * 8);
  }
  j->secs = now() - t0;
  return NULL;
}

static int parse_cpulist(const char* path, int* cpus, int cap) {
  FILE* f = fopen(path, "r");
  if (!f) return 0;
  char buf[4096];
  int n = 0;
  if (fgets(buf, sizeof buf, f)) {
    char* p = buf;
    while (*p && *p != '\n' && n < cap) {
      int a = (int)strtol(p, &p, 10), b = a;
      if (*p == '-') b = (int)strtol(p + 1, &p, 10);
      for (int c = a; c <= b && n < cap; ++c) cpus[n++] = c;
      if (*p == ',') ++p;
    }
  }
  fclose(f);
  return n;
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)(argc > 1 ? atoll(argv[1]) : 4096) << 20;
  int node_cpus[1024];
  for (int node = 0; node < 64; ++node) {
    char path[128];
    snprintf(path, sizeof path, "/sys/devices/system/node/node%d/cpulist", node);
    const int nc = parse_cpulist(path, node_cpus, 1024);
    if (nc == 0) {
      if (node == 0) {  // no sysfs NUMA info: all online CPUs, no binding
        const long on = sysconf(_SC_NPROCESSORS_ONLN);
        for (int c = 0; c < on; ++c) node_cpus[c] = c;
        printf("{\"note\": \"no /sys/devices/system/node; unbound\"}\n");
      } else {
        break;
      }
    }
    const int ncpu = nc ? nc : (int)sysconf(_SC_NPROCESSORS_ONLN);
    uint64_t* src = mmap(NULL, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    uint64_t* dst = mmap(NULL, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    unsigned long mask[16] = {0};
    mask[node / 64] = 1ul << (node % 64);
    long rc1 = syscall(SYS_mbind, src, bytes, MPOL_BIND, mask, 1024, 0);
    long rc2 = syscall(SYS_mbind, dst, bytes, MPOL_BIND, mask, 1024, 0);
    memset(src, 1, bytes);
    memset(dst, 2, bytes);
    for (int mode = 0; mode < 2; ++mode) {
      for (int nt = 1; nt <= ncpu; nt *= 2) {
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
          job_t jobs[1024];
          pthread_t th[1024];
          const size_t per = bytes / 8 / nt;
          double t0 = now();
          for (int t = 0; t < nt; ++t) {
            jobs[t] = (job_t){src + t * per, dst + t * per, per, node_cpus[t % ncpu], mode, 0, 0};
            pthread_create(&th[t], NULL, worker, &jobs[t]);
          }
          for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
          const double gbs = (double)per * 8 * nt / (now() - t0) / 1e9;
          if (gbs > best) best = gbs;
        }
        printf("{\"node\": %d, \"node_cpus\": %d, \"mbind_rc\": %ld, \"mode\": \"%s\", \"threads\": %d, "
               "\"GBps\": %.2f}\n", node, ncpu, rc1 | rc2, mode ? "copy(read+write counted once)" : "read", nt, best);
        if (nt < ncpu && nt * 2 > ncpu) nt = ncpu / 2;  // finish on ncpu
      }
    }
    munmap(src, bytes);
    munmap(dst, bytes);
    if (nc == 0) break;
  }
  return 0;
}
