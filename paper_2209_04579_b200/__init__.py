"""B200-native (sm_100a) hot path of TQP: the relational kernel set, fused
pipelines and executor behind a C ABI (include/tqp_b200.h)."""
