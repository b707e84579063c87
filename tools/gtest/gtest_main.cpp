// gtest_main.cpp — main() for the self-written GoogleTest subset (gtest/gtest.h).
#include <gtest/gtest.h>

int main(int argc, char** argv) {
    ::testing::InitGoogleTest(&argc, argv);
    return RUN_ALL_TESTS();
}
