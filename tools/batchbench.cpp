// Host batcher microbenchmark (single thread): assemble() over the first
// sentences of the text8-shaped corpus with the reference table or the alias
// sampler. Build: see tools/batchbench.sh
#include "../paper_2312_07743_b200/csrc/fw2v_host.cpp"

int main(int argc, char** argv) {
    const int alias = argc > 1 ? atoi(argv[1]) : 0;
    const uint64_t nsent0 = argc > 2 ? strtoull(argv[2], nullptr, 10) : 4000;
    fw2v_corpus* corpus = nullptr;
    fw2v_corpus_synth_zipf(71291, 16718845, 1.0, 1000, 5, 0, &corpus);
    const uint64_t* counts; int32_t V; const uint64_t* offs; uint64_t ns; const int32_t* ids; uint64_t nid;
    fw2v_corpus_view(corpus, &counts, &V, &offs, &ns, &ids, &nid);
    const uint64_t nsent = std::min(nsent0, ns);
    HugeArray<int32_t> slots;
    slots.resize(10000000);
    build_table(counts, V, 0.75, 10000000, slots.data());
    std::vector<double> keep(V);
    keep_probs(counts, V, 1e-4, keep.data());
    AliasTable at;
    at.build(counts, V, 0.75);
    Sampler sp;
    sp.keep = keep.data();
    sp.n_neg = argc > 3 ? atoi(argv[3]) : 5;
    if (alias) sp.alias = &at; else { sp.slots = slots.data(); sp.table_size = 10000000; sp.mod = FastMod(10000000); }
    const uint64_t cap = offs[nsent] - offs[0];
    std::vector<int32_t> o_ids(cap), o_negs(cap * 5);
    std::vector<uint32_t> o_off(nsent + 1);
    double best = 1e9; uint64_t words = 0; int64_t chk = 0;
    for (int rep = 0; rep < 5; ++rep) {
        Rng rng = Rng::derive(1, 0, 0, 0);
        uint64_t cur = 0;
        const double t0 = wall_seconds();
        const uint64_t kept = assemble(CorpusView{offs, ids, ns}, cur, nsent, nsent, sp, rng,
                                       BatchOut{o_ids.data(), o_off.data(), o_negs.data(), cap, nsent + 1}, &words);
        best = std::min(best, wall_seconds() - t0);
        chk = 0; for (uint64_t i = 0; i < words * 5; ++i) chk += o_negs[i];
        (void)kept;
    }
    {
        FILE* f = fopen("/proc/self/smaps_rollup", "r");
        char line[256];
        while (f && fgets(line, sizeof line, f)) if (strstr(line, "AnonHuge")) fputs(line, stdout);
        if (f) fclose(f);
    }
    printf("%s: %llu words, %.1f ns/word, %.1f Mwords/s/thread, chk %lld\n", alias ? "alias" : "table",
           (unsigned long long)words, best / words * 1e9, words / best / 1e6, (long long)chk);
}
