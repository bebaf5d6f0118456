// shard_driver.cpp — trains a clause-sharded machine through the C ABI alone
// (include/tmgpu.h; no C++ facade, no Python, no torch): the multi-GPU path
// of train_epoch_parallel (trainer.cpp:181-242) with its tallies kept as one
// replica per shard and exchanged every window (paper_2009_04861_b200/csrc/
// group.cu). Usage: shard_driver <devices, e.g. 0,0 or 0,1,2,3> [clauses] [epochs]
// Checks, after every epoch:
//   * every shard's tally replica equals the pool's tallies;
//   * the tally invariant tally[i][c] = sum_j sign(j) prev[c][j][i] over all
//     shards' previous outputs (pool.cpp:93-106: each recorded change counted once);
// and at the end that the sharded class sums equal those of a one-device
// machine holding the same automata (bit-exact), plus the test accuracy.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "tmgpu.h"

#define CHECK(x)                                                          \
  do {                                                                    \
    if ((x) != TMG_OK) {                                                  \
      std::fprintf(stderr, "%s failed: %s\n", #x, tmg_last_error());     \
      return 2;                                                           \
    }                                                                     \
  } while (0)

int main(int argc, char** argv) {
  std::vector<int32_t> devs;
  for (const char* p = argc > 1 ? argv[1] : "0,0"; *p;) {
    char* end = nullptr;
    devs.push_back(static_cast<int32_t>(std::strtol(p, &end, 10)));
    p = *end ? end + 1 : end;
  }
  const int n = argc > 2 ? std::atoi(argv[2]) : 400;
  const int epochs = argc > 3 ? std::atoi(argv[3]) : 3;
  const int o = 784, m = 10;
  const int64_t q = 6000, qt = 2000;
  std::vector<uint8_t> tx(static_cast<size_t>(q) * o), vx(static_cast<size_t>(qt) * o);
  std::vector<int32_t> ty(static_cast<size_t>(q)), vy(static_cast<size_t>(qt));
  if (tmg_synth_preset(1, 2009, 0.0, q, qt, tx.data(), ty.data(), vx.data(), vy.data()) != 0) return 2;

  tmg_config cfg;
  tmg_config_default(&cfg);
  cfg.clauses = n;
  cfg.margin = 50;
  cfg.specificity = 10.0;
  cfg.seed = 42;
  tmg_machine* tm = nullptr;
  CHECK(tmg_machine_create_devices(&cfg, o, m, devs.data(), static_cast<int32_t>(devs.size()), &tm));
  int32_t shards = 0, nccl = 0;
  CHECK(tmg_machine_exchange_info(tm, &shards, &nccl));
  std::printf("shards %d exchange %s\n", shards, nccl ? "nccl" : "peer");
  tmg_pool* pool = nullptr;
  tmg_pool* test = nullptr;
  CHECK(tmg_pool_create(devs[0], o, tx.data(), ty.data(), q, m, &pool));
  CHECK(tmg_pool_create(devs[0], o, vx.data(), vy.data(), qt, m, &test));

  const size_t W64 = static_cast<size_t>((q + 63) / 64);
  std::vector<int32_t> tal(static_cast<size_t>(q) * m), rep(tal.size());
  std::vector<uint64_t> prev(static_cast<size_t>(n) * W64);
  bool ok = true;
  for (int e = 0; e < epochs; ++e) {
    std::vector<uint64_t> ev(m), ev1(m);
    tmg_epoch_report r{};
    r.feedback_events = ev.data();
    r.type_i_events = ev1.data();
    CHECK(tmg_train_epoch(tm, pool, TMG_MODE_AUTO, 8, e, &r));
    uint64_t total = 0;
    for (uint64_t v : ev) total += v;
    CHECK(tmg_pool_get_tallies(pool, tal.data()));
    bool same = true;
    for (int k = 0; k < shards; ++k) {
      CHECK(tmg_pool_replica_tallies(pool, k, rep.data()));
      same = same && rep == tal;
    }
    std::vector<int64_t> want(tal.size(), 0);
    for (int c = 0; c < m; ++c) {
      CHECK(tmg_get_prev_outputs(tm, c, prev.data()));
      for (int j = 0; j < n; ++j)
        for (int64_t i = 0; i < q; ++i)
          if ((prev[static_cast<size_t>(j) * W64 + static_cast<size_t>(i >> 6)] >> (i & 63)) & 1u)
            want[static_cast<size_t>(i) * m + c] += (j % 2 == 0) ? 1 : -1;
    }
    bool inv = true;
    for (size_t k = 0; k < tal.size(); ++k) inv = inv && want[k] == tal[k];
    std::printf("epoch %d events %llu replicas_equal %d invariant %d\n", e, static_cast<unsigned long long>(total),
                same ? 1 : 0, inv ? 1 : 0);
    ok = ok && same && inv && total > 0;
  }
  // The same automata on one device: class sums must match bit for bit.
  tmg_machine* one = nullptr;
  CHECK(tmg_machine_create(&cfg, o, m, devs[0], &one));
  std::vector<uint16_t> counters(static_cast<size_t>(n) * 2 * o);
  for (int c = 0; c < m; ++c) {
    CHECK(tmg_get_counters(tm, c, counters.data()));
    CHECK(tmg_set_counters(one, c, counters.data()));
  }
  std::vector<int32_t> s1(static_cast<size_t>(qt) * m), s2(s1.size()), pred(static_cast<size_t>(qt));
  CHECK(tmg_class_sums(tm, test, TMG_EVAL_PREDICT, s1.data()));
  CHECK(tmg_class_sums(one, test, TMG_EVAL_PREDICT, s2.data()));
  CHECK(tmg_predict(tm, test, pred.data()));
  int64_t hits = 0;
  for (int64_t i = 0; i < qt; ++i) hits += pred[static_cast<size_t>(i)] == vy[static_cast<size_t>(i)];
  std::printf("sums_identical %d accuracy %.4f\n", s1 == s2 ? 1 : 0, static_cast<double>(hits) / qt);
  ok = ok && s1 == s2;
  tmg_machine_destroy(one);
  tmg_pool_destroy(test);
  tmg_pool_destroy(pool);
  tmg_machine_destroy(tm);
  std::printf(ok ? "OK\n" : "FAILED\n");
  return ok ? 0 : 1;
}
