// Compiles the reference-shaped C++ API (include/turbokv_compat.hpp) against libtkv_b200.so.
// Without a GPU, Engine() must throw turbokv::CudaError (no CPU fallback); with one, a toy request runs.
#include <cstdio>
#include <vector>

#include "turbokv_compat.hpp"

int main() {
    using namespace turbokv;
    ModelConfig cfg = ModelConfig::toy();
    cfg.validate();
    uint64_t ck = 0, fp = 0;
    check(tkv_weights_identity(&cfg, 42, &ck, &fp));
    std::printf("checksum %016llx fingerprint %016llx\n", (unsigned long long)ck, (unsigned long long)fp);
    try {
        ModelConfig bad = cfg;
        bad.kv_head_num = 3;
        bad.validate();
        return 2;
    } catch (const ConfigError&) {
    }
    try {
        EngineOptions o;
        o.store_capacity_tokens = 4096;
        Engine eng(cfg, 42, o);
        const uint64_t id = eng.ingest_chunk_payload("d", {97, 98, 99});
        AssembledContext ctx = eng.assemble({id}, PositionMode::Reordered);
        std::vector<float> logits = eng.prefill_query(ctx, {100, 101});
        std::printf("gpu logits[0] %f total %lld\n", logits[0], (long long)ctx.total_tokens());
        return logits.size() == 259 && ctx.total_tokens() == 7 ? 0 : 3;
    } catch (const CudaError& e) {
        std::printf("no gpu: %s\n", e.what());
        return 0;
    }
}
